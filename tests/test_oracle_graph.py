"""Pins for oracle/graph.py (O1, O2, O10) — CPU only.

Every pin checks the oracle against something other than itself: published
hash test vectors, a second (Python) implementation of the generator spec,
set-semantics brute force, SPEC worked examples and the Schur bound on ||A^||.
"""
import os

import numpy as np
import pytest

import oracle
import synth
from oracle.graph import build_graph, from_csr, rmat_arcs, dinv

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix64_published_vectors():
    """SURVEY §8(d) hash == SplitMix64 reference outputs (tests/golden/splitmix64.txt)."""
    rows = [l.split() for l in open(os.path.join(GOLDEN, "splitmix64.txt")) if l.strip() and not l.startswith("#")]
    for k, hx in rows:
        assert oracle.graph.hash64(int(k), 0, 0) == int(hx, 16)
        assert int(synth.hash64(int(k), 0, 0)) == int(hx, 16)


def test_hash_c_matches_numpy_on_random_counters():
    rng = np.random.default_rng(0)
    for _ in range(50):
        seed, stream, i = (int(x) for x in rng.integers(0, 2**62, size=3))
        assert oracle.graph.hash64(seed, stream, i) == int(synth.hash64(seed, stream, i))


def _rmat_python(scale, thr, seed, i):
    """Second implementation of the §8(d) R-MAT arc spec (pure Python + synth.hash64)."""
    s = d = 0
    for l in range(scale):
        u = int(synth.hash64(seed, 0, i * 64 + l)) >> 32
        if u < thr[0]:
            q = (0, 0)
        elif u < thr[1]:
            q = (0, 1)
        elif u < thr[2]:
            q = (1, 0)
        else:
            q = (1, 1)
        s, d = (s << 1) | q[0], (d << 1) | q[1]
    return s, d


@pytest.mark.parametrize("abc,scale,seed", [((0.57, 0.19, 0.19), 12, 1), ((0.45, 0.22, 0.22), 18, 2),
                                            ((0.25, 0.25, 0.25), 7, 9)])
def test_rmat_matches_python_spec(abc, scale, seed):
    thr = synth.rmat_thresholds(*abc)
    src, dst = rmat_arcs(scale, thr, seed, 1000, 300)
    for k in range(300):
        assert (src[k], dst[k]) == _rmat_python(scale, thr, seed, 1000 + k)


def test_rmat_degenerate_quadrants():
    """a=1 -> all arcs (0,0); b=1 -> (0, 2^s-1); c=1 -> (2^s-1, 0): pins the quadrant->bit map."""
    s = 9
    top = (1 << 32) - 1
    src, dst = rmat_arcs(s, (top, top, top), 5, 0, 2000)
    assert (src == 0).all() and (dst == 0).all()
    src, dst = rmat_arcs(s, (0, top, top), 5, 0, 2000)
    assert (src == 0).all() and (dst == (1 << s) - 1).all()
    src, dst = rmat_arcs(s, (0, 0, top), 5, 0, 2000)
    assert (src == (1 << s) - 1).all() and (dst == 0).all()


def test_rmat_bit_frequencies():
    """P(src bit=1) = c+d, P(dst bit=1) = b+d at every level (R-MAT definition)."""
    a, b, c = 0.57, 0.19, 0.19
    d = 1 - a - b - c
    s = 10
    n = 200_000
    src, dst = rmat_arcs(s, synth.rmat_thresholds(a, b, c), 3, 0, n)
    for l in range(s):
        ps = ((src >> l) & 1).mean()
        pd = ((dst >> l) & 1).mean()
        sig = np.sqrt(0.25 / n)
        assert abs(ps - (c + d)) < 6 * sig
        assert abs(pd - (b + d)) < 6 * sig


def test_spec_csr_examples():
    # S:56 "0 1\n1 2" V=3 -> E=2, deg_in=[0,1,1]
    g = build_graph([0, 1], [1, 2], 3, False)
    assert g.nnz == 2 and list(g.deg_in) == [0, 1, 1] and list(g.deg_out) == [1, 1, 0]
    # S:57 empty, V=4
    g = build_graph([], [], 4, False)
    assert g.nnz == 0 and (g.deg_in == 0).all() and len(g.row_ptr) == 5
    # S:58 duplicates collapse
    g = build_graph([0, 0], [1, 1], 2, False)
    assert g.nnz == 1
    # self loops dropped (R1), ids >= n rejected (R-MAT rejection)
    g = build_graph([0, 1, 5], [0, 0, 1], 3, False)
    assert g.nnz == 1 and list(g.col) == [1]


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("symmetric", [False, True])
def test_csr_brute_force(seed, symmetric):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 40))
    m = int(rng.integers(0, 200))
    src = rng.integers(0, n + 3, size=m)
    dst = rng.integers(0, n + 3, size=m)
    g = build_graph(src, dst, n, symmetric)
    arcs = set()
    for s, d in zip(src.tolist(), dst.tolist()):
        if s < n and d < n and s != d:
            arcs.add((s, d))
            if symmetric:
                arcs.add((d, s))
    for v in range(n):
        nin = sorted(u for (u, x) in arcs if x == v)
        nout = sorted(x for (u, x) in arcs if u == v)
        assert list(g.col[g.row_ptr[v]:g.row_ptr[v + 1]]) == nin
        assert list(g.col_t[g.row_ptr_t[v]:g.row_ptr_t[v + 1]]) == nout
    assert g.deg_in.sum() == g.deg_out.sum() == g.nnz == len(arcs)


def test_transpose_involution_and_from_csr():
    cfg = synth.get_config("tiny_dir")
    g = oracle.graph.graph_from_config(cfg)
    gt = from_csr(g.row_ptr_t, g.col_t, g.n)          # treat out-CSR as an in-CSR
    np.testing.assert_array_equal(gt.row_ptr_t, g.row_ptr)
    np.testing.assert_array_equal(gt.col_t, g.col)
    g2 = from_csr(g.row_ptr, g.col, g.n)
    np.testing.assert_array_equal(g2.col, g.col)
    np.testing.assert_array_equal(g2.col_t, g.col_t)


def test_norm_single_edge_and_isolated():
    """Single arc 0->1: c_10 = d~_in(1)^-1/2 d~_out(0)^-1/2 = 1/sqrt(2*2) = 0.5 (S:74 under
    the self-loop reading R1); isolated vertex self coefficient 1 (R8)."""
    g = build_graph([0], [1], 3, False)
    A = oracle.graph.dense_adjacency_hat(g)
    assert abs(A[1, 0] - 0.5) < 1e-15
    assert A[2, 2] == 1.0
    assert A[0, 1] == 0.0
    assert dinv([0])[0] == 1.0


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("symmetric", [False, True])
def test_norm_spectral_bound(seed, symmetric):
    """||A^||_2 <= 1 (Gershgorin; for the two-sided directed form by the Schur test)."""
    rng = np.random.default_rng(100 + seed)
    n = 60
    src = rng.integers(0, n, 400)
    dst = (rng.pareto(1.5, 400) * 3).astype(int) % n
    g = build_graph(src, dst, n, symmetric)
    A = oracle.graph.dense_adjacency_hat(g)
    x = rng.standard_normal(n)
    for _ in range(500):              # power iteration on A^T A
        x = A.T @ (A @ x)
        x /= np.linalg.norm(x)
    sig = np.sqrt(np.linalg.norm(A.T @ (A @ x)))
    assert sig <= 1 + 1e-9
    assert np.linalg.norm(A, 2) <= 1 + 1e-9


@pytest.mark.parametrize("name", ["small_dir", "tiny_sym", "small_appnp"])
def test_sampled_rows_matches_full_build(name):
    """oracle.graph.sampled_rows (arc-stream filter, used at papers100M scale) == rows of the full O1 build."""
    cfg = synth.get_config(name)
    g = oracle.graph.graph_from_config(cfg)
    rows = np.unique(np.concatenate([np.arange(5), np.random.default_rng(0).integers(0, cfg.n, 40), [cfg.n - 1]]))
    for tr in (False, True):
        d = oracle.graph.sampled_rows(cfg, rows, tr)
        rp, cl = (g.row_ptr_t, g.col_t) if tr else (g.row_ptr, g.col)
        for v in rows:
            assert np.array_equal(d[int(v)], cl[rp[v]:rp[v + 1]])
