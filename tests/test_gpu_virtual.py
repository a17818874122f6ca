"""Virtual slices on one GPU (P > world with P % world == 0, slices processed in sequence).

With ntp_set_slices(P) the single-GPU context runs the multi-slice data plane of the P-worker epoch
(Alg. 1): the MLP producers pack P blocks [P][V_p][d_s], every slice is propagated
on its own, the loss kernel / fused head read the P gathered blocks and write the P gradient blocks,
the backward gather feeds the P-block unpack or the fused weight gradient, and V_pad = P * ceil(n/P)
padding rows are carried through every buffer.  The layout exchanges are the identity on one device.
Checked against the oracle (the sliced model is the same function: column separability) and,
for propagation, bitwise against P = 1 (the per-row reduction order does not depend on P)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import oracle_graph, ntp_ctx_for

pytestmark = pytest.mark.gpu


def _model(cfg, dtype, lr, flags=0, chunks=1):
    from paper_2412_20379_b200 import ntp
    f = flags | (ntp.NTP_M_W1_AFTER_PROP if cfg.w_after_prop else 0)
    return dict(d_in=cfg.d_in, hid=cfg.hid, C=cfg.C, K=cfg.K, gamma=cfg.gamma, alpha=cfg.alpha, lr=lr,
                dtype=dtype, chunks=chunks, flags=f)


def _rows(n, P):
    return P * -(-n // P)          # V_pad = P * ceil(n / P): this GPU's rows at world 1


def _epochs(name, P, dtype, epochs, reorder=False, chunks=1, slice_align=16):
    cfg = synth.get_config(name)
    ctx = ntp_ctx_for(name, reorder=reorder, slice_align=slice_align)
    ctx.set_slices(P)
    V = _rows(cfg.n, P)
    X, y, m = synth.config_inputs(cfg)
    ldx = (cfg.d_in + 3) // 4 * 4
    Xd = torch.zeros(V, ldx, dtype=torch.float32, device="cuda")[:, :cfg.d_in]
    Xd[:cfg.n] = torch.from_numpy(X).cuda()
    yd = torch.zeros(V, dtype=torch.int32, device="cuda")
    yd[:cfg.n] = torch.from_numpy(y).cuda()
    md = torch.zeros(V, dtype=torch.uint8, device="cuda")
    md[:cfg.n] = torch.from_numpy(m).cuda()
    W0, W1 = synth.model_weights(cfg)
    W0d, W1d = torch.from_numpy(W0).cuda(), torch.from_numpy(W1).cuda()
    model = _model(cfg, dtype, cfg.lr * 50, chunks=chunks)
    reps = [ctx.train_epoch(model, Xd, yd, md, W0d, W1d) for _ in range(epochs)]
    ctx.close()
    return [r["loss"] for r in reps], W0d.cpu().numpy(), W1d.cpu().numpy(), reps, model


def _oracle(name, epochs, lr):
    cfg = synth.get_config(name)
    X, y, m = synth.config_inputs(cfg)
    W0, W1 = synth.model_weights(cfg)
    return oracle.model.train(oracle_graph(name), X, y, m, W0, W1, cfg.K, cfg.gamma, cfg.alpha, lr, epochs)


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("name", ["tiny_sym", "small_dir", "small_appnp", "cora"])
def test_virtual_slices_epoch_fp32(name, P):
    losses, W0, W1, reps, model = _epochs(name, P, 0, 3)
    ref, rW0, rW1 = _oracle(name, 3, model["lr"])
    for e, (a, b) in enumerate(zip(losses, ref)):
        assert abs(a - b) <= 1e-4, f"P={P} epoch {e}: gpu {a} oracle {b}"
    for got, r in ((W0, rW0), (W1, rW1)):
        assert np.abs(got - r).max() <= 1e-4 * max(1.0, np.abs(r).max())
    assert reps[0]["bytes_sent"] == [0, 0, 0, 0]          # one device: the exchanges are local
    assert reps[0]["spmm_launches"] == 2 * model["K"] * P   # every slice propagated on its own


@pytest.mark.parametrize("P,align", [(2, 128), (4, 64), (2, 64), (8, 128)])
@pytest.mark.parametrize("name", ["small_dir", "cora"])
def test_virtual_slices_epoch_padded_slices(name, P, align):
    """Slice rows padded to 64 / 128 bytes (ntp_create slice_align; bench.py pads L2-resident slices of
    33-128 bytes): wider zero-padded slices through the pack, hops, loss and unpack, same model."""
    from paper_2412_20379_b200 import ntp
    losses, W0, W1, reps, model = _epochs(name, P, 0, 3, slice_align=align)
    cfg = synth.get_config(name)
    assert ntp.partition(cfg.n, cfg.w, P, 0, 1, align)["d_s"] * 4 % align == 0
    ref, rW0, rW1 = _oracle(name, 3, model["lr"])
    for e, (a, b) in enumerate(zip(losses, ref)):
        assert abs(a - b) <= 1e-4, f"P={P} align={align} epoch {e}: gpu {a} oracle {b}"
    for got, r in ((W0, rW0), (W1, rW1)):
        assert np.abs(got - r).max() <= 1e-4 * max(1.0, np.abs(r).max())


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("name,reorder", [("head_dir", False), ("head_dir", True), ("head_sym", False),
                                          ("tiny_dir", False)])
def test_virtual_slices_epoch_bf16_w1_after(name, reorder, P):
    """W1 after propagation with bf16 slices: at hid = 128 the P-block pack epilogue of the MLP GEMM and the
    fused tcgen05 head run with P * d_s = 128 (d_s = 64 / 32 / 16), the fused dW0 kernel at d_s = 64."""
    from paper_2412_20379_b200 import ntp
    losses, W0, W1, _, model = _epochs(name, P, ntp.NTP_BF16, 3, reorder=reorder)
    ref, rW0, rW1 = _oracle(name, 3, model["lr"])
    for e, (a, b) in enumerate(zip(losses, ref)):
        assert abs(a - b) <= 2e-2 * abs(b), f"P={P} epoch {e}: gpu {a} oracle {b}"
    for got, r in ((W0, rW0), (W1, rW1)):
        assert np.abs(got - r).max() <= 2e-2 * max(1.0, np.abs(r).max())


@pytest.mark.parametrize("P,chunk", [(4, 700), (8, 1024)])
def test_virtual_slices_row_chunked_head(P, chunk, monkeypatch):
    """Row-chunked vertex-side work (NTP_HEAD_CHUNK) over P slice blocks: the chunk loops of the MLP forward,
    the head and dW0 index rows of every block; the result equals the unchunked epoch's to rounding."""
    from paper_2412_20379_b200 import ntp
    a, W0a, W1a, _, _ = _epochs("head_dir", P, ntp.NTP_BF16, 2)
    monkeypatch.setenv("NTP_HEAD_CHUNK", str(chunk))
    b, W0b, W1b, _, _ = _epochs("head_dir", P, ntp.NTP_BF16, 2)
    for x, y in zip(a, b):
        assert abs(x - y) <= 1e-5 * abs(x)
    assert np.abs(W0a - W0b).max() <= 1e-5 * max(1.0, np.abs(W0a).max())


@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("transposed", [False, True])
def test_virtual_slices_pipeline_bitwise(P, dtype, transposed):
    """ntp_propagate_pipeline (split -> K hops per slice -> gather) at virtual P equals P = 1 bitwise: column
    separability with a P-independent per-row reduction order (SURVEY §8(a) design notes)."""
    from paper_2412_20379_b200 import ntp
    name = "small_appnp"
    cfg = synth.get_config(name)
    ctx = ntp_ctx_for(name)
    w = 40
    Hv = torch.from_numpy(synth.features(3, cfg.n, w)).cuda()
    Z1 = torch.empty_like(Hv)
    dt = ntp.NTP_BF16 if dtype == torch.bfloat16 else ntp.NTP_F32
    ctx.propagate_pipeline(Hv, Z1, cfg.K, cfg.gamma, cfg.alpha, transposed=transposed, dtype=dt)
    ctx.set_slices(P)
    V = _rows(cfg.n, P)
    HvP = torch.zeros(V, w, device="cuda")
    HvP[:cfg.n] = Hv
    ZP = torch.empty_like(HvP)
    ctx.propagate_pipeline(HvP, ZP, cfg.K, cfg.gamma, cfg.alpha, transposed=transposed, dtype=dt)
    ms, hops = ctx.hop_timing()
    torch.cuda.synchronize()
    assert hops == cfg.K * P and ms > 0
    assert torch.equal(ZP[:cfg.n], Z1)
    ctx.close()


@pytest.mark.parametrize("P", [2, 4, 5])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_virtual_slices_layouts(P, dtype):
    """ntp_layout_v2f / f2v at virtual P: the stacked slices are the matrix's column blocks (what
    ntp_scatter_features(FEATURE) writes from the host), and f2v(v2f(x)) == x bitwise."""
    from paper_2412_20379_b200 import ntp
    name = "tiny_dir"
    cfg = synth.get_config(name)
    ctx = ntp_ctx_for(name)
    ctx.set_slices(P)
    w = 20
    part = ntp.partition(cfg.n, w, P, ntp.NTP_BF16 if dtype == torch.bfloat16 else ntp.NTP_F32)
    V_pad, d_s = part["V_pad"], part["d_s"]
    X = synth.features(7, cfg.n, w)
    Hv = torch.zeros(V_pad, w, dtype=dtype, device="cuda")
    Hv[:cfg.n] = torch.from_numpy(X).to(dtype).cuda()
    Hf = torch.empty(P * V_pad, d_s, dtype=dtype, device="cuda")
    ctx.layout_v2f(Hv, Hf)
    ref = torch.empty_like(Hf)
    ctx.scatter_features(X, ntp.NTP_LAYOUT_FEATURE, ref)
    torch.cuda.synchronize()
    assert torch.equal(Hf, ref)
    back = torch.full_like(Hv, 7.0)
    ctx.layout_f2v(Hf, back)
    torch.cuda.synchronize()
    assert torch.equal(back[:cfg.n], Hv[:cfg.n])
    ctx.close()


def test_virtual_slices_refusals():
    from paper_2412_20379_b200 import ntp
    cfg = synth.get_config("tiny_sym")
    ctx = ntp_ctx_for("tiny_sym")
    with pytest.raises(RuntimeError):
        ctx.set_slices(0)
    ctx.set_slices(4)
    V = _rows(cfg.n, 4)
    X = torch.zeros(V, cfg.d_in, device="cuda")
    y = torch.zeros(V, dtype=torch.int32, device="cuda")
    m = torch.zeros(V, dtype=torch.uint8, device="cuda")
    W0, W1 = (torch.from_numpy(a).cuda() for a in synth.model_weights(cfg))
    for f in (ntp.NTP_M_OVERLAP, ntp.NTP_M_DATA_PARALLEL):
        with pytest.raises(RuntimeError):
            ctx.train_epoch(_model(cfg, 0, 0.1, flags=f), X, y, m, W0, W1)
    with pytest.raises(RuntimeError):   # rows must be this rank's V_p at P = 4
        ctx.train_epoch(_model(cfg, 0, 0.1), X[:cfg.n - 1], y, m, W0, W1)
    ctx.close()
