"""papers100M-shaped graph (BASELINE configs[4]: 111M vertices, ~1.6B directed arcs) at full size.

The oracle cannot build this CSR whole in a test, so it regenerates the raw arc stream with its
own generator and keeps the arcs of sampled rows (oracle.graph.sampled_rows): those rows of the
device-built in-CSR and out-CSR must match bit-exactly.  Propagation is checked on the whole
graph through identities of the two-sided normalisation that hold at any size:
A^ sqrt(d~_out) = sqrt(d~_in) and A^T sqrt(d~_in) = sqrt(d~_out)  (SURVEY §8(c) pins)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def papers_ctx():
    from paper_2412_20379_b200 import ntp
    cfg = synth.get_config("papers")
    ctx = ntp.Context()
    ctx.generate_rmat(cfg.n, cfg.scale, cfg.m_raw, synth.rmat_thresholds(*cfg.abc), cfg.seed, cfg.symmetric)
    yield cfg, ctx
    ctx.close()


def test_papers_csr_sampled_rows_bit_exact(papers_ctx):
    cfg, ctx = papers_ctx
    n, nnz, sym = ctx.graph_info()
    assert n == cfg.n and not sym
    assert 1.55e9 < nnz < 1.70e9          # Table 1: |E| = 1.616 B
    rng = np.random.default_rng(5)
    rows = np.unique(np.concatenate([np.arange(8), rng.integers(0, n, 200), [n - 1]]))
    for transposed in (False, True):
        rp, col, deg = ctx.copy_csr(transposed)
        ref = oracle.graph.sampled_rows(cfg, rows, transposed)
        for v in rows.tolist():
            assert np.array_equal(col[rp[v]:rp[v + 1]], ref[v]), (transposed, v)
            assert deg[v] == ref[v].size
        del rp, col


@pytest.mark.parametrize("dtype,tol", [(torch.float32, 2e-5), (torch.bfloat16, 2e-2)])
def test_papers_sqrt_degree_identities(papers_ctx, dtype, tol):
    cfg, ctx = papers_ctx
    n = cfg.n
    _, _, deg_in = ctx.copy_csr(False)
    _, _, deg_out = ctx.copy_csr(True)
    s_in = np.sqrt(deg_in.astype(np.float64) + 1.0)
    s_out = np.sqrt(deg_out.astype(np.float64) + 1.0)
    cols = 8 if dtype == torch.bfloat16 else 4
    for src, dst, bwd in ((s_out, s_in, False), (s_in, s_out, True)):
        H = torch.from_numpy(np.repeat(src[:, None], cols, 1).astype(np.float32)).to(dtype).cuda()
        Z = torch.empty_like(H)
        (ctx.propagate_bwd if bwd else ctx.propagate_fwd)(H, Z, 1, 1.0, 0.0)
        torch.cuda.synchronize()
        z = Z.float().cpu().numpy()
        ref = dst[:, None]
        # bf16: the input is rounded to bf16 first (relative 2^-9), so compare to the propagated rounded input
        rel = np.abs(z - ref) / ref
        assert rel.max() <= tol, (bwd, float(rel.max()))


def _neigh(cfg, rows, transposed):
    return oracle.graph.sampled_rows(cfg, np.asarray(sorted(set(int(r) for r in rows)), np.int64), transposed)


@pytest.mark.parametrize("transposed", [False, True])
def test_papers_sampled_rows_one_hop_vs_oracle(papers_ctx, transposed):
    """Tier-3 full-size parity on the papers shape: one hop of the whole 111M-vertex
    graph (fp32, 4 columns) checked element by element at 1e-5 (R10) on sampled output rows against the
    plain definition Z[v] = d~_row(v)^-1/2 (d~_col(v)^-1/2 H[v] + sum_u d~_col(u)^-1/2 H[u]), whose rows
    and degrees come from the oracle's own regeneration of the arc stream (oracle.graph.sampled_rows):
    in-neighbours of the sample, then the column-side degree of every vertex they touch."""
    cfg, ctx = papers_ctx
    n, d = cfg.n, 4
    rng = np.random.default_rng(11)
    rows = np.unique(np.concatenate([rng.integers(0, n, 48), [1, 2, 3, n - 1]]))
    nb = _neigh(cfg, rows, transposed)                       # row side: neighbour lists of the sample
    touched = np.unique(np.concatenate([rows] + [nb[v] for v in rows.tolist()]).astype(np.int64))
    col_side = _neigh(cfg, touched, not transposed)          # column side: their degrees in the other CSR
    deg_row = {v: nb[v].size for v in rows.tolist()}
    deg_col = {u: col_side[u].size for u in touched.tolist()}
    H = synth.features_device(cfg.seed, n, d)
    Z = torch.empty_like(H)
    (ctx.propagate_bwd if transposed else ctx.propagate_fwd)(H, Z, 1, 1.0, 0.0)
    torch.cuda.synchronize()
    z = Z[torch.from_numpy(rows).cuda()].double().cpu().numpy()
    del Z
    # the synthetic input formula at the touched rows only
    idx = touched.astype(np.uint64)[:, None] * np.uint64(d) + np.arange(d, dtype=np.uint64)[None, :]
    ftab = ((synth.hash64(cfg.seed, synth.S_FEAT, idx) >> np.uint64(40)).astype(np.float64) / float(1 << 23) - 1.0)
    ctab = 1.0 / np.sqrt(np.array([deg_col[u] for u in touched.tolist()], np.float64) + 1.0)
    pos = lambda ids: np.searchsorted(touched, np.asarray(ids, np.int64))
    for i, v in enumerate(rows.tolist()):
        p = np.concatenate([pos([v]), pos(nb[v])])          # self first, then ascending sources
        terms = ctab[p, None] * ftab[p]
        rs = 1.0 / np.sqrt(deg_row[v] + 1.0)
        ref = rs * np.sum(terms, axis=0)
        den = rs * np.sum(np.abs(terms), axis=0)
        err = np.abs(z[i] - ref)
        assert np.all(err <= 1e-5 * den + 1e-30), (transposed, v, deg_row[v], float((err / den).max()))
