"""GPU graph setup (a0) vs the oracle: bit-exact integer work (CSR, transpose,
degrees, R-MAT arcs) and D~^{-1/2} within fp32 rounding."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import oracle_graph, ntp_ctx_for

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ntp():
    from paper_2412_20379_b200 import ntp
    return ntp


@pytest.mark.parametrize("name,i0,count", [("cora", 0, 5000), ("reddit", 12_345_678, 100_000),
                                           ("papers", 1_500_000_000, 100_000), ("tiny_dir", 0, 40_000)])
def test_rmat_arcs_bit_exact(ntp, name, i0, count):
    cfg = synth.get_config(name)
    thr = synth.rmat_thresholds(*cfg.abc)
    ctx = ntp.Context()
    s, d = ctx.rmat_arcs(cfg.scale, thr, cfg.seed, i0, count)
    so, do = oracle.graph.rmat_arcs(cfg.scale, thr, cfg.seed, i0, count)
    np.testing.assert_array_equal(s, so)
    np.testing.assert_array_equal(d, do)


def _check_graph(ctx, g):
    n, nnz, sym = ctx.graph_info()
    assert n == g.n and nnz == g.nnz
    rp, col, deg = ctx.copy_csr(False)
    np.testing.assert_array_equal(rp, g.row_ptr)
    np.testing.assert_array_equal(col, g.col)
    np.testing.assert_array_equal(deg, g.deg_in)
    rpt, colt, degt = ctx.copy_csr(True)
    np.testing.assert_array_equal(rpt, g.row_ptr_t)
    np.testing.assert_array_equal(colt, g.col_t)
    np.testing.assert_array_equal(degt, g.deg_out)
    di, do = ctx.copy_dinv()
    np.testing.assert_allclose(di, g.dinv_in, rtol=6e-8)
    np.testing.assert_allclose(do, g.dinv_out, rtol=6e-8)


@pytest.mark.parametrize("name", ["cora", "tiny_sym", "tiny_dir", "small_appnp", "small_dir", "reddit"])
def test_generate_rmat_graph_bit_exact(name):
    ctx = ntp_ctx_for(name)
    _check_graph(ctx, oracle_graph(name))


@pytest.mark.parametrize("name", ["cora", "tiny_sym", "tiny_dir", "small_appnp", "small_dir"])
def test_reordered_graph_is_invisible(name):
    """NTP_G_REORDER stores the graph under a degree-ordered numbering; everything read back
    through the ABI (CSR both ways, degrees, D~^{-1/2}) is still in original ids, bit-exact."""
    ctx = ntp_ctx_for(name, reorder=True)
    _check_graph(ctx, oracle_graph(name))


def test_load_graph_and_build_graph(ntp):
    g = oracle_graph("small_dir")
    ctx = ntp.Context()
    ctx.load_graph(g.row_ptr, g.col, g.n, symmetric=False, validate=True)
    _check_graph(ctx, g)
    # arc list with duplicates, self loops and out-of-range ids -> same canonical graph (O1)
    rng = np.random.default_rng(0)
    src = rng.integers(0, 600, 5000)
    dst = rng.integers(0, 600, 5000)
    src[:50] = dst[:50]
    src[50:60] = 700
    ctx.build_graph(np.concatenate([src, src[:100]]), np.concatenate([dst, dst[:100]]), 600, symmetric=True)
    _check_graph(ctx, oracle.graph.build_graph(src, dst, 600, True))
    ctx.build_graph(src, dst, 600, symmetric=False)
    _check_graph(ctx, oracle.graph.build_graph(src, dst, 600, False))
    ctx.build_graph(src, dst, 600, symmetric=False, reorder=True)
    _check_graph(ctx, oracle.graph.build_graph(src, dst, 600, False))
    ctx.load_graph(g.row_ptr, g.col, g.n, symmetric=False, reorder=True)
    _check_graph(ctx, g)


def test_degenerate_graphs(ntp):
    ctx = ntp.Context()
    ctx.build_graph(np.array([], np.int64), np.array([], np.int64), 5)
    _check_graph(ctx, oracle.graph.build_graph([], [], 5, False))
    ctx.build_graph(np.array([0]), np.array([0]), 1)            # single vertex, self loop dropped
    _check_graph(ctx, oracle.graph.build_graph([0], [0], 1, False))


def test_validate_rejects_bad_csr(ntp):
    ctx = ntp.Context()
    with pytest.raises(ntp.NtpError) as e:
        ctx.load_graph(np.array([0, 2, 1, 3]), np.array([1, 0, 2]), 3, validate=True)
    assert e.value.status == ntp.NTP_ERR_GRAPH
    with pytest.raises(ntp.NtpError) as e:
        ctx.load_graph(np.array([0, 2, 2, 2]), np.array([2, 1]), 3, validate=True)   # not ascending
    assert e.value.status == ntp.NTP_ERR_GRAPH
    with pytest.raises(ntp.NtpError) as e:
        ctx.load_graph(np.array([0, 1, 1, 1]), np.array([7]), 3, validate=True)      # out of range
    assert e.value.status == ntp.NTP_ERR_GRAPH
