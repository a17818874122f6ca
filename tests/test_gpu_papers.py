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
