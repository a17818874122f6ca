"""NEXT-2 decoupled GAT epoch (ntp_train_epoch_gat) vs the GAT oracle (oracle/gat.py, readings G1-G4):
per-epoch loss within 1e-4 (fp32 slices) / 2e-2 relative (bf16) and every parameter -- W0, W1 and the
attention vector a = [a_src; a_dst], whose gradient runs through the softmax / LeakyReLU backward (the
oracle forms dalpha per arc; the engine contracts it per vertex through dual alpha / beta hops) -- after
the SGD updates; on one GPU and at virtual P = 2 / 4 (the P-block layouts, per-slice weighted hops and the
per-slice partial dot products)."""
import numpy as np
import pytest
import torch

import synth
from gpu_util import oracle_graph, ntp_ctx_for
from oracle import gat

pytestmark = pytest.mark.gpu


def _att(cfg):
    return synth.glorot(cfg.seed, 2, cfg.C, 7_000_000)


def _run_gpu(name, epochs, dtype=0, P=1, K=None, gamma=None, lr_scale=50.0, slope=0.2, slice_align=16):
    cfg = synth.get_config(name)
    ctx = ntp_ctx_for(name, slice_align=slice_align)
    if P > 1:
        ctx.set_slices(P)
    V = P * -(-cfg.n // P)
    X, y, m = synth.config_inputs(cfg)
    Xd = torch.zeros(V, cfg.d_in, device="cuda")
    Xd[:cfg.n] = torch.from_numpy(X).cuda()
    yd = torch.zeros(V, dtype=torch.int32, device="cuda")
    yd[:cfg.n] = torch.from_numpy(y).cuda()
    md = torch.zeros(V, dtype=torch.uint8, device="cuda")
    md[:cfg.n] = torch.from_numpy(m).cuda()
    W0, W1 = synth.model_weights(cfg)
    W0d, W1d = torch.from_numpy(W0).cuda(), torch.from_numpy(W1).cuda()
    Ad = torch.from_numpy(_att(cfg)).cuda()
    model = dict(d_in=cfg.d_in, hid=cfg.hid, C=cfg.C, K=K or cfg.K, gamma=gamma or cfg.gamma, alpha=0.0,
                 lr=cfg.lr * lr_scale, dtype=dtype, chunks=1, flags=0)
    reps = [ctx.train_epoch_gat(model, Xd, yd, md, W0d, W1d, Ad, slope=slope) for _ in range(epochs)]
    ctx.close()
    return [r["loss"] for r in reps], W0d.cpu().numpy(), W1d.cpu().numpy(), Ad.cpu().numpy(), reps, model


def _run_oracle(name, epochs, model, slope=gat.SLOPE):
    cfg = synth.get_config(name)
    X, y, m = synth.config_inputs(cfg)
    W0, W1 = synth.model_weights(cfg)
    a = _att(cfg)
    return gat.train(oracle_graph(name), X, y, m, W0, W1, a[0], a[1], model["K"], model["gamma"], model["lr"], epochs,
                     slope)


def _check(got, ref, tol_loss, tol_w, rel):
    losses, W0, W1, A = got[:4]
    rl, rW0, rW1, ras, rad = ref
    for e, (a, b) in enumerate(zip(losses, rl)):
        bound = tol_loss * abs(b) if rel else tol_loss
        assert abs(a - b) <= bound, f"epoch {e}: gpu {a} oracle {b}"
    for g, r in ((W0, rW0), (W1, rW1), (A, np.stack([ras, rad]))):
        assert np.abs(g - r).max() <= tol_w * max(1.0, np.abs(r).max()), np.abs(g - r).max()


@pytest.mark.parametrize("name,K,gamma", [("tiny_sym", None, None), ("small_dir", None, None),
                                          ("dense_dir", None, None), ("cora", None, None),
                                          ("small_appnp", 4, 0.9), ("dense_sym", 3, 0.9)])
def test_gat_epoch_fp32(name, K, gamma):
    got = _run_gpu(name, 3, K=K, gamma=gamma)
    ref = _run_oracle(name, 3, got[5])
    _check(got, ref, 1e-4, 1e-4, False)
    assert got[0][-1] < got[0][0]
    assert got[4][0]["spmm_launches"] == 2 * got[5]["K"]   # dual hops (alpha and beta sums in one pass)


@pytest.mark.parametrize("name", ["tiny_sym", "small_dir"])
def test_gat_epoch_bf16(name):
    from paper_2412_20379_b200 import ntp
    got = _run_gpu(name, 3, dtype=ntp.NTP_BF16)
    ref = _run_oracle(name, 3, got[5])
    _check(got, ref, 2e-2, 2e-2, True)


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("name", ["tiny_sym", "small_dir"])
def test_gat_epoch_virtual_slices(name, P):
    got = _run_gpu(name, 3, P=P)
    ref = _run_oracle(name, 3, got[5])
    _check(got, ref, 1e-4, 1e-4, False)
    assert got[4][0]["spmm_launches"] == 2 * got[5]["K"] * P


@pytest.mark.parametrize("P", [2, 4])
def test_gat_epoch_virtual_slices_bf16(P):
    """bf16 slices at virtual P: the dual hops on bf16 rows and the per-slice dots of bf16 levels."""
    from paper_2412_20379_b200 import ntp
    got = _run_gpu("small_dir", 3, dtype=ntp.NTP_BF16, P=P)
    ref = _run_oracle("small_dir", 3, got[5])
    _check(got, ref, 2e-2, 2e-2, True)


@pytest.mark.parametrize("P,align", [(2, 128), (4, 64)])
def test_gat_epoch_padded_slices(P, align):
    """Slice rows padded to 64 / 128 bytes (zero columns through the dual hops and the per-vertex dots)."""
    got = _run_gpu("small_dir", 3, P=P, slice_align=align)
    ref = _run_oracle("small_dir", 3, got[5])
    _check(got, ref, 1e-4, 1e-4, False)


@pytest.mark.parametrize("slope,name", [(0.0, "small_dir"), (0.0, "dense_sym"), (0.9, "tiny_sym"), (0.5, "cora")])
def test_gat_epoch_slopes(slope, name):
    """LeakyReLU slope 0 (a ReLU: beta = 0 on every arc with s <= 0, coefficient words -alpha / -0.0), 0.9 and
    0.5 vs the oracle with the same slope (the API takes slopes in [0, 1))."""
    got = _run_gpu(name, 3, slope=slope)
    ref = _run_oracle(name, 3, got[5], slope=slope)
    _check(got, ref, 1e-4, 1e-4, False)


@pytest.mark.parametrize("name", ["small_dir", "dense_sym", "cora"])
def test_gat_out_order_coefficients_bitwise(name, monkeypatch):
    """The backward hop's coefficients in out-CSR order are re-derived from each destination's stored softmax
    (max, sum) instead of permuted from the in-CSR array: the same operands and operations, so the whole epoch
    (losses, W0, W1, a) is bit-identical to the plain permutation (NTP_GAT_PERMUTE=1)."""
    runs = []
    for perm in ("1", "0"):
        monkeypatch.setenv("NTP_GAT_PERMUTE", perm)
        runs.append(_run_gpu(name, 3))
    (la, W0a, W1a, Aa), (lb, W0b, W1b, Ab) = runs[0][:4], runs[1][:4]
    assert la == lb
    assert np.array_equal(W0a, W0b) and np.array_equal(W1a, W1b) and np.array_equal(Aa, Ab)


def test_gat_zero_attention_vector_matches_gcn_on_ring():
    """a = 0 on a regular undirected graph (ring): the attention operator is the GCN operator A^, so one GAT
    epoch's loss equals the decoupled GCN epoch's (oracle.model.forward_loss) -- ties the GPU GAT path to
    the pinned O3 propagation."""
    import oracle
    from paper_2412_20379_b200 import ntp
    n, d_in, hid, C = 1000, 8, 16, 5
    v = np.arange(n)
    ctx = ntp.Context()
    ctx.build_graph(v, (v + 1) % n, n, symmetric=True)
    g = oracle.graph.build_graph(v, (v + 1) % n, n, symmetric=True)
    X = synth.features(5, n, d_in)
    y = synth.labels(5, n, C)
    m = synth.train_mask(5, n)
    W0 = synth.glorot(5, d_in, hid)
    W1 = synth.glorot(5, hid, C, 10_000)
    model = dict(d_in=d_in, hid=hid, C=C, K=3, gamma=0.9, alpha=0.0, lr=0.0, dtype=0, chunks=1, flags=0)
    rep = ctx.train_epoch_gat(model, *(torch.from_numpy(a).cuda() for a in (X, y, m)), torch.from_numpy(W0).cuda(),
                              torch.from_numpy(W1).cuda(), torch.zeros(2, C, device="cuda"))
    ref = oracle.model.forward_loss(g, X, y, m, W0, W1, 3, 0.9, 0.0)
    assert abs(rep["loss"] - ref) <= 1e-5
    ctx.close()


def test_gat_refusals():
    from paper_2412_20379_b200 import ntp
    cfg = synth.get_config("tiny_sym")
    ctx = ntp_ctx_for("tiny_sym")
    X, y, m = (torch.from_numpy(a).cuda() for a in synth.config_inputs(cfg))
    W0, W1 = (torch.from_numpy(a).cuda() for a in synth.model_weights(cfg))
    A = torch.zeros(2, cfg.C, device="cuda")
    base = dict(d_in=cfg.d_in, hid=cfg.hid, C=cfg.C, K=2, gamma=1.0, alpha=0.0, lr=0.1, dtype=0, chunks=1, flags=0)
    for bad in (dict(alpha=0.1), dict(flags=ntp.NTP_M_W1_AFTER_PROP)):
        with pytest.raises(RuntimeError):
            ctx.train_epoch_gat(dict(base, **bad), X, y, m, W0, W1, A)
    with pytest.raises(RuntimeError):
        ctx.train_epoch_gat(base, X, y, m, W0, W1, torch.zeros(2, cfg.C + 1, device="cuda"))
    ctx.close()
