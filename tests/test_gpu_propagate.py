"""GPU K-hop propagation (a4/a8) vs the oracle, through the C ABI.

Tolerance (reading R10): |z_gpu - z_orc| <= tol * (M|H|)_elem, tol = 1e-5 for
fp32 storage, 2e-2 for bf16 storage (BASELINE.json north_star)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import oracle_graph, ntp_ctx_for, cond_bound, assert_r10

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5
BF16_TOL = 2e-2


def _features(n, d, seed):
    return synth.features(seed, n, d)


def _run(ctx, H, K, gamma, alpha, transposed=False, dtype=torch.float32, rows=None, cols=None):
    n = H.shape[0]
    rows = rows or n
    cols = cols or H.shape[1]
    Hd = torch.zeros(rows, cols, dtype=dtype, device="cuda")
    Hd[:n, :H.shape[1]] = torch.from_numpy(H).to(dtype)
    Zd = torch.full((rows, cols), 7.0, dtype=dtype, device="cuda")
    f = ctx.propagate_bwd if transposed else ctx.propagate_fwd
    f(Hd, Zd, K, gamma, alpha)
    torch.cuda.synchronize()
    return Zd, Hd


@pytest.mark.parametrize("name", ["cora", "tiny_sym", "tiny_dir", "small_appnp", "small_dir", "dense_sym", "dense_dir"])
@pytest.mark.parametrize("d", [4, 8, 12, 16, 44, 48, 132])
@pytest.mark.parametrize("transposed", [False, True])
def test_fp32_parity(name, d, transposed):
    cfg = synth.get_config(name)
    g = oracle_graph(name)
    ctx = ntp_ctx_for(name)
    H = _features(g.n, d, 100 + d)
    Zd, _ = _run(ctx, H, cfg.K, cfg.gamma, cfg.alpha, transposed)
    f = oracle.propagate.propagate_bwd if transposed else oracle.propagate.propagate_fwd
    ref = f(g, H, cfg.K, cfg.gamma, cfg.alpha)
    den = cond_bound(g, H, cfg.K, cfg.gamma, cfg.alpha, transposed)
    assert_r10(Zd.cpu().numpy()[:g.n], ref, den, FP32_TOL, f"{name} d={d} T={transposed}")


@pytest.mark.parametrize("name", ["cora", "tiny_dir", "small_appnp", "small_dir"])
@pytest.mark.parametrize("d", [8, 44, 132])
@pytest.mark.parametrize("transposed", [False, True])
def test_fp32_parity_reordered(name, d, transposed):
    """Degree-ordered internal numbering (NTP_G_REORDER): same oracle parity, slices in and out
    in original vertex order."""
    cfg = synth.get_config(name)
    g = oracle_graph(name)
    ctx = ntp_ctx_for(name, reorder=True)
    H = _features(g.n, d, 300 + d)
    Zd, _ = _run(ctx, H, cfg.K, cfg.gamma, cfg.alpha, transposed)
    f = oracle.propagate.propagate_bwd if transposed else oracle.propagate.propagate_fwd
    ref = f(g, H, cfg.K, cfg.gamma, cfg.alpha)
    den = cond_bound(g, H, cfg.K, cfg.gamma, cfg.alpha, transposed)
    assert_r10(Zd.cpu().numpy()[:g.n], ref, den, FP32_TOL, f"reordered {name} d={d} T={transposed}")


def test_reordered_bf16_and_slices():
    name = "small_appnp"
    cfg = synth.get_config(name)
    g = oracle_graph(name)
    ctx = ntp_ctx_for(name, reorder=True)
    H = _features(g.n, 48, 77)
    Zd, _ = _run(ctx, H, cfg.K, cfg.gamma, cfg.alpha, dtype=torch.bfloat16)
    ref = oracle.propagate.propagate_fwd(g, H, cfg.K, cfg.gamma, cfg.alpha)
    den = cond_bound(g, H, cfg.K, cfg.gamma, cfg.alpha)
    assert_r10(Zd.float().cpu().numpy()[:g.n], ref, den, BF16_TOL, "reordered bf16")
    # column slices are still bitwise equal to the full-width result
    Zfull, _ = _run(ctx, H, cfg.K, cfg.gamma, cfg.alpha)
    Zs, _ = _run(ctx, np.ascontiguousarray(H[:, 8:24]), cfg.K, cfg.gamma, cfg.alpha)
    assert torch.equal(Zs, Zfull[:, 8:24])


@pytest.mark.parametrize("K,gamma,alpha", [(0, 1.0, 0.0), (1, 1.0, 0.0), (1, 0.5, 0.5), (3, 0.9, 0.1),
                                           (10, 0.9, 0.1), (7, 1.0, 0.0)])
def test_fp32_K_gamma_alpha(K, gamma, alpha):
    name = "tiny_dir"
    g = oracle_graph(name)
    ctx = ntp_ctx_for(name)
    H = _features(g.n, 16, 3)
    for transposed in (False, True):
        Zd, _ = _run(ctx, H, K, gamma, alpha, transposed)
        f = oracle.propagate.propagate_bwd if transposed else oracle.propagate.propagate_fwd
        ref = f(g, H, K, gamma, alpha)
        den = cond_bound(g, H, K, gamma, alpha, transposed)
        assert_r10(Zd.cpu().numpy()[:g.n], ref, den, FP32_TOL, f"K={K} T={transposed}")


@pytest.mark.parametrize("name", ["tiny_dir", "small_appnp", "small_dir"])
@pytest.mark.parametrize("d", [8, 16, 48, 128])
def test_bf16_parity(name, d):
    cfg = synth.get_config(name)
    g = oracle_graph(name)
    ctx = ntp_ctx_for(name)
    H = _features(g.n, d, 7)
    for transposed in (False, True):
        Zd, _ = _run(ctx, H, cfg.K, cfg.gamma, cfg.alpha, transposed, dtype=torch.bfloat16)
        f = oracle.propagate.propagate_bwd if transposed else oracle.propagate.propagate_fwd
        ref = f(g, H, cfg.K, cfg.gamma, cfg.alpha)
        den = cond_bound(g, H, cfg.K, cfg.gamma, cfg.alpha, transposed)
        assert_r10(Zd.float().cpu().numpy()[:g.n], ref, den, BF16_TOL, f"bf16 {name} d={d}")


def test_padding_rows_zeroed_and_ld():
    """Rows >= n of Z are zero; a strided (ld > cols) view works."""
    name = "tiny_sym"
    cfg = synth.get_config(name)
    g = oracle_graph(name)
    ctx = ntp_ctx_for(name)
    H = _features(g.n, 8, 1)
    big_h = torch.zeros(g.n + 5, 16, device="cuda")
    big_h[:g.n, :8] = torch.from_numpy(H)
    big_z = torch.full((g.n + 5, 16), 3.0, device="cuda")
    ctx.propagate_fwd(big_h[:, :8], big_z[:, :8], cfg.K, cfg.gamma, cfg.alpha)
    torch.cuda.synchronize()
    z = big_z.cpu().numpy()
    assert (z[g.n:, :8] == 0).all() and (z[:, 8:] == 3.0).all()
    ref = oracle.propagate.propagate_fwd(g, H, cfg.K, cfg.gamma, cfg.alpha)
    assert_r10(z[:g.n, :8], ref, cond_bound(g, H, cfg.K, cfg.gamma, cfg.alpha), FP32_TOL)


@pytest.mark.parametrize("name", ["small_dir", "small_appnp"])
def test_slice_invariance_bitwise(name):
    """Column slices propagated separately equal the full-width result bitwise
    (the per-row reduction order does not depend on d_s, so P=1 == P=8)."""
    cfg = synth.get_config(name)
    g = oracle_graph(name)
    ctx = ntp_ctx_for(name)
    H = _features(g.n, 48, 5)
    Zfull, _ = _run(ctx, H, cfg.K, cfg.gamma, cfg.alpha)
    for c0, c1 in [(0, 8), (8, 16), (16, 28), (28, 48), (0, 4)]:
        Zs, _ = _run(ctx, np.ascontiguousarray(H[:, c0:c1]), cfg.K, cfg.gamma, cfg.alpha)
        assert torch.equal(Zs, Zfull[:, c0:c1]), (c0, c1)
    for transposed in (True,):
        Zfull, _ = _run(ctx, H, cfg.K, cfg.gamma, cfg.alpha, transposed)
        Zs, _ = _run(ctx, np.ascontiguousarray(H[:, 8:16]), cfg.K, cfg.gamma, cfg.alpha, transposed)
        assert torch.equal(Zs, Zfull[:, 8:16])


@pytest.mark.parametrize("name", ["small_dir", "small_appnp", "cora"])
@pytest.mark.parametrize("transposed", [False, True])
def test_pipeline_vertex_layout(name, transposed):
    """ntp_propagate_pipeline (split with the pre-scale fused in -> K hops -> gather) on vertex rows
    equals the oracle's propagation of the full matrix (P = 1: this rank owns every row)."""
    cfg = synth.get_config(name)
    g = oracle_graph(name)
    ctx = ntp_ctx_for(name)
    w = 37
    H = _features(g.n, w, 41)
    Hv = torch.from_numpy(H).cuda()
    Zv = torch.full((g.n, w), 3.0, device="cuda")
    ctx.propagate_pipeline(Hv, Zv, cfg.K, cfg.gamma, cfg.alpha, transposed=transposed)
    torch.cuda.synchronize()
    f = oracle.propagate.propagate_bwd if transposed else oracle.propagate.propagate_fwd
    ref = f(g, H, cfg.K, cfg.gamma, cfg.alpha)
    den = cond_bound(g, H, cfg.K, cfg.gamma, cfg.alpha, transposed)
    assert_r10(Zv.cpu().numpy(), ref, den, FP32_TOL, f"pipeline {name} T={transposed}")
    # bf16 slice storage
    Zb = torch.zeros_like(Zv)
    from paper_2412_20379_b200 import ntp
    ctx.propagate_pipeline(Hv, Zb, cfg.K, cfg.gamma, cfg.alpha, transposed=transposed, dtype=ntp.NTP_BF16)
    torch.cuda.synchronize()
    assert_r10(Zb.cpu().numpy(), ref, den, BF16_TOL, f"pipeline bf16 {name}")


def test_deterministic():
    name = "small_appnp"
    cfg = synth.get_config(name)
    g = oracle_graph(name)
    ctx = ntp_ctx_for(name)
    H = _features(g.n, 44, 9)
    a, _ = _run(ctx, H, cfg.K, cfg.gamma, cfg.alpha)
    b, _ = _run(ctx, H, cfg.K, cfg.gamma, cfg.alpha)
    assert torch.equal(a, b)


def test_adjoint_gpu():
    name = "small_dir"
    g = oracle_graph(name)
    ctx = ntp_ctx_for(name)
    H = _features(g.n, 8, 1)
    G = _features(g.n, 8, 2)
    Z, _ = _run(ctx, H, 3, 0.9, 0.1)
    Y, _ = _run(ctx, G, 3, 0.9, 0.1, transposed=True)
    lhs = float((Z.double() * torch.from_numpy(G).cuda().double()).sum())
    rhs = float((torch.from_numpy(H).cuda().double() * Y.double()).sum())
    assert abs(lhs - rhs) <= 1e-5 * (abs(lhs) + abs(rhs))


def test_empty_and_isolated_graph(ntp):
    """No arcs: A^ = I (d~ = 1) so Z^K = gamma^K H + alpha sum_{j<K} gamma^j H exactly-ish."""
    ctx = ntp.Context()
    ctx.build_graph(np.array([], np.int64), np.array([], np.int64), 37)
    H = _features(37, 8, 4)
    Z, _ = _run(ctx, H, 3, 0.5, 0.25)
    coef = 0.5 ** 3 + 0.25 * (1 + 0.5 + 0.25)
    np.testing.assert_allclose(Z.cpu().numpy(), coef * H, rtol=1e-6, atol=1e-7)


@pytest.fixture(scope="module")
def ntp():
    from paper_2412_20379_b200 import ntp
    return ntp


# ------------------------------------------------------------------ full size (BASELINE configs[1])

@pytest.mark.slow
@pytest.mark.parametrize("d", [44, 8])
def test_reddit_full_size_sampled_rows(d):
    """c2 at the bench's P=1 slice width (44 fp32 columns) and the P=8 width (8; streaming kernel), K=2: sampled output rows
    vs the oracle hop by hop (the GPU's hop-1 output is fed to the oracle's hop 2),
    plus the sqrt(d~) fixed point A^ sqrt(d~) = sqrt(d~) (symmetric graph)."""
    name = "reddit"
    cfg = synth.get_config(name)
    g = oracle_graph(name)
    ctx = ntp_ctx_for(name)
    n = g.n
    H = _features(n, d, 11)
    Z1, _ = _run(ctx, H, 1, 1.0, 0.0)
    Z2, _ = _run(ctx, H, 2, 1.0, 0.0)
    rng = np.random.default_rng(0)
    rows = np.concatenate([rng.integers(0, n, 300), np.argsort(g.deg_in)[-20:]])   # include hubs
    z1 = Z1.double().cpu().numpy()
    ref1 = oracle.propagate.hop_rows(g, H, None, rows, 1.0, 0.0)
    den1 = oracle.propagate.hop_rows(g, np.abs(H), None, rows, 1.0, 0.0)
    assert_r10(z1[rows], ref1, den1, FP32_TOL, "hop1")
    ref2 = oracle.propagate.hop_rows(g, z1, None, rows, 1.0, 0.0)
    den2 = oracle.propagate.hop_rows(g, np.abs(z1), None, rows, 1.0, 0.0)
    assert_r10(Z2.double().cpu().numpy()[rows], ref2, den2, 2 * FP32_TOL, "hop2")
    # fixed point on the full graph
    sq = np.sqrt(g.deg_in + 1.0)[:, None].repeat(4, 1).astype(np.float32)
    Zs, _ = _run(ctx, sq, 2, 1.0, 0.0)
    np.testing.assert_allclose(Zs.cpu().numpy(), sq, rtol=2e-5)


@pytest.mark.slow
@pytest.mark.parametrize("name,d", [("products", 48), ("products", 12), ("orkut", 64)])
def test_full_size_sampled_rows(name, d):
    """c3 (APPNP K=10, gamma=0.9, alpha=0.1) and c4 at full size, slice width d: every hop's
    output on sampled rows (random + the 20 largest in-degrees + isolated vertices) vs the
    oracle applied to the GPU's previous-hop state, and the whole K-hop result on the
    sqrt(d~) fixed point (symmetric graphs: A^ sqrt(d~) = sqrt(d~), kept by gamma = 1 - alpha)."""
    cfg = synth.get_config(name)
    g = oracle_graph(name)
    ctx = ntp_ctx_for(name)
    n = g.n
    H = _features(n, d, 21)
    rng = np.random.default_rng(1)
    rows = np.unique(np.concatenate([rng.integers(0, n, 300), np.argsort(g.deg_in)[-20:],
                                     np.flatnonzero(g.deg_in == 0)[:10]]))
    prev = H.astype(np.float64)
    for k in range(1, min(cfg.K, 3) + 1):
        Zk, _ = _run(ctx, H, k, cfg.gamma, cfg.alpha)
        zk = Zk.double().cpu().numpy()
        ref = oracle.propagate.hop_rows(g, prev, H, rows, cfg.gamma, cfg.alpha)
        den = oracle.propagate.hop_rows(g, np.abs(prev), np.abs(H), rows, cfg.gamma, cfg.alpha)
        assert_r10(zk[rows], ref, den, 2 * FP32_TOL, f"{name} hop {k}")
        prev = zk
    sq = np.sqrt(g.deg_in + 1.0)[:, None].repeat(4, 1).astype(np.float32)
    gam = 1.0 - cfg.alpha
    Zs, _ = _run(ctx, sq, cfg.K, gam, cfg.alpha)
    np.testing.assert_allclose(Zs.cpu().numpy(), sq, rtol=5e-5)
    Ys, _ = _run(ctx, sq, cfg.K, gam, cfg.alpha, transposed=True)
    np.testing.assert_allclose(Ys.cpu().numpy(), sq, rtol=5e-5)


@pytest.mark.parametrize("name", ["dense_sym", "dense_dir"])
@pytest.mark.parametrize("transposed", [False, True])
def test_high_degree_variants_bitwise(name, transposed, monkeypatch):
    """High-degree graphs: narrow slices (<= 64-byte rows) run the 4-CTA/SM half-batch hop variant,
    wide ones the default variant; with the invariant reduction order (NTP_SPMM_INVARIANT=1: also at
    two edge slots) every narrow slice equals the matching columns of the full-width result bitwise
    (fp32 and bf16 storage)."""
    monkeypatch.setenv("NTP_SPMM_INVARIANT", "1")
    cfg = synth.get_config(name)
    g = oracle_graph(name)
    ctx = ntp_ctx_for(name)
    for dtype, widths in ((torch.float32, (4, 8, 12, 16)), (torch.bfloat16, (8, 16, 24, 32))):
        H = _features(g.n, 48, 9)
        Zfull, _ = _run(ctx, H, cfg.K, cfg.gamma, cfg.alpha, transposed, dtype=dtype)
        for d in widths:
            Zs, _ = _run(ctx, np.ascontiguousarray(H[:, :d]), cfg.K, cfg.gamma, cfg.alpha, transposed, dtype=dtype)
            assert torch.equal(Zs, Zfull[:, :d]), (dtype, d)


@pytest.mark.parametrize("name", ["dense_sym", "dense_dir"])
@pytest.mark.parametrize("d", [36, 44, 48, 60])
@pytest.mark.parametrize("transposed", [False, True])
def test_high_degree_one_accumulator_path(name, d, transposed, monkeypatch):
    """High-degree graphs at two edge slots (rows of 9-16 16-byte vectors; the Reddit slice at P = 1) run the
    single-accumulator 4-CTA/SM variant by default: within R10 of the oracle (fp32 1e-5), and with
    NTP_SPMM_INVARIANT=1 the same call returns the slice-width-invariant result, which differs from it only
    by rounding."""
    cfg = synth.get_config(name)
    g = oracle_graph(name)
    ctx = ntp_ctx_for(name)
    H = _features(g.n, d, 70 + d)
    Zf, _ = _run(ctx, H, cfg.K, cfg.gamma, cfg.alpha, transposed)
    f = oracle.propagate.propagate_bwd if transposed else oracle.propagate.propagate_fwd
    ref = f(g, H, cfg.K, cfg.gamma, cfg.alpha)
    den = cond_bound(g, H, cfg.K, cfg.gamma, cfg.alpha, transposed)
    assert_r10(Zf.cpu().numpy()[:g.n], ref, den, FP32_TOL, f"{name} d={d} fast")
    monkeypatch.setenv("NTP_SPMM_INVARIANT", "1")
    Zi, _ = _run(ctx, H, cfg.K, cfg.gamma, cfg.alpha, transposed)
    assert_r10(Zi.cpu().numpy()[:g.n], ref, den, FP32_TOL, f"{name} d={d} invariant")
    assert_r10(Zf.cpu().numpy()[:g.n], Zi.double().cpu().numpy()[:g.n], den, FP32_TOL, f"{name} d={d} fast vs inv")


@pytest.mark.slow
@pytest.mark.parametrize("name,d,transposed", [("reddit", 44, False), ("reddit", 44, True), ("products", 48, False)])
def test_full_size_end_to_end_all_rows(name, d, transposed):
    """The whole K-hop propagation of a full BASELINE-size graph at the bench's slice width, EVERY output row
    and column against the oracle's own K-hop run (O3 / O4) at R10's 1e-5 (fp32), denominator M|H|: the
    bench workload itself (Reddit, K = 2) and the APPNP products shape (K = 10, gamma 0.9, alpha 0.1)."""
    cfg = synth.get_config(name)
    g = oracle_graph(name)
    ctx = ntp_ctx_for(name)
    H = _features(g.n, d, 31)
    Z, _ = _run(ctx, H, cfg.K, cfg.gamma, cfg.alpha, transposed=transposed)
    f = oracle.propagate.propagate_bwd if transposed else oracle.propagate.propagate_fwd
    ref = f(g, H, cfg.K, cfg.gamma, cfg.alpha)
    den = f(g, np.abs(H.astype(np.float64)), cfg.K, cfg.gamma, cfg.alpha)
    assert_r10(Z.double().cpu().numpy(), ref, den, FP32_TOL, f"{name} K={cfg.K} all rows")
    ctx.close()
