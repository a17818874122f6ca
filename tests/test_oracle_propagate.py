"""Pins for oracle/propagate.py (O3/O4) — CPU only.

Dense brute force from an explicit arc set, closed forms on the complete graph
and the ring (known eigenvectors), the sqrt(d~) fixed point, contraction,
adjointness and column separability.
"""
import numpy as np
import pytest

import oracle
import synth
from oracle.graph import build_graph
from oracle.propagate import propagate_fwd, propagate_bwd


def _dense_hat_from_arcs(arcs, n):
    """A^ built with Python loops directly from the arc set (independent of the CSR code)."""
    din = [1] * n
    dout = [1] * n
    for (u, v) in arcs:
        din[v] += 1
        dout[u] += 1
    A = np.zeros((n, n))
    for v in range(n):
        A[v, v] = 1.0 / np.sqrt(din[v] * dout[v])
    for (u, v) in arcs:
        A[v, u] = 1.0 / np.sqrt(din[v] * dout[u])
    return A


def _M(A, K, gamma, alpha):
    n = A.shape[0]
    P = np.eye(n)
    S = np.zeros((n, n))
    for _ in range(K):
        S += P
        P = gamma * A @ P
    return P + alpha * S


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("K,gamma,alpha", [(0, 1.0, 0.0), (1, 1.0, 0.0), (2, 1.0, 0.0), (5, 0.5, 0.0),
                                           (10, 0.9, 0.1), (3, 0.7, 0.3)])
def test_dense_brute_force(seed, K, gamma, alpha):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 64))
    m = int(rng.integers(0, 5 * n))
    sym = bool(seed % 2)
    src = rng.integers(0, n, m)
    dst = rng.integers(0, n, m)
    arcs = set()
    for s, d in zip(src.tolist(), dst.tolist()):
        if s != d:
            arcs.add((s, d))
            if sym:
                arcs.add((d, s))
    g = build_graph(src, dst, n, sym)
    A = _dense_hat_from_arcs(arcs, n)
    M = _M(A, K, gamma, alpha)
    H = rng.standard_normal((n, 5))
    np.testing.assert_allclose(propagate_fwd(g, H, K, gamma, alpha), M @ H, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(propagate_bwd(g, H, K, gamma, alpha), M.T @ H, rtol=1e-12, atol=1e-12)


def _complete(n):
    src, dst = np.meshgrid(np.arange(n), np.arange(n))
    return build_graph(src.ravel(), dst.ravel(), n, True)


@pytest.mark.parametrize("n,K,alpha", [(7, 1, 0.0), (13, 4, 0.0), (10, 10, 0.1), (5, 3, 0.25)])
def test_complete_graph_closed_form(n, K, alpha):
    """K_n: A^ = J/n, so with gamma = 1 - alpha, Z^K = alpha*H + (1-alpha)*mean_rows(H) for K >= 1."""
    g = _complete(n)
    rng = np.random.default_rng(n)
    H = rng.standard_normal((n, 3))
    Z = propagate_fwd(g, H, K, 1.0 - alpha, alpha)
    expect = alpha * H + (1.0 - alpha) * H.mean(axis=0, keepdims=True)
    np.testing.assert_allclose(Z, expect, rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("n,m,K,gamma,alpha", [(12, 1, 3, 1.0, 0.0), (31, 4, 6, 0.9, 0.1), (8, 2, 5, 0.5, 0.3)])
def test_ring_fourier_closed_form(n, m, K, gamma, alpha):
    """Ring C_n (undirected, d~ = 3): x_m = cos(2 pi m v / n) has eigenvalue (1 + 2cos(2 pi m/n))/3."""
    v = np.arange(n)
    g = build_graph(v, (v + 1) % n, n, True)
    x = np.cos(2 * np.pi * m * v / n)[:, None]
    lam = (1 + 2 * np.cos(2 * np.pi * m / n)) / 3
    coef = (gamma * lam) ** K + alpha * sum((gamma * lam) ** j for j in range(K))
    np.testing.assert_allclose(propagate_fwd(g, x, K, gamma, alpha), coef * x, atol=1e-13)


@pytest.mark.parametrize("name", ["tiny_sym", "tiny_dir", "small_dir"])
def test_sqrt_degree_fixed_point(name):
    """A^ sqrt(d~_out) = sqrt(d~_in) and A^T sqrt(d~_in) = sqrt(d~_out) (SURVEY §8(c) pins)."""
    g = oracle.graph.graph_from_config(synth.get_config(name))
    so = np.sqrt(g.deg_out + 1.0)[:, None]
    si = np.sqrt(g.deg_in + 1.0)[:, None]
    np.testing.assert_allclose(propagate_fwd(g, so, 1), si, rtol=1e-13)
    np.testing.assert_allclose(propagate_bwd(g, si, 1), so, rtol=1e-13)
    if g.symmetric:   # fixed point survives K APPNP hops with gamma = 1 - alpha
        np.testing.assert_allclose(propagate_fwd(g, si, 7, 0.8, 0.2), si, rtol=1e-12)


@pytest.mark.parametrize("K", [1, 5, 10])
def test_contraction(K):
    """gamma < 1, alpha = 0: ||Z^K||_F <= gamma^K ||H||_F."""
    g = oracle.graph.graph_from_config(synth.get_config("tiny_sym"))
    H = np.random.default_rng(K).standard_normal((g.n, 4))
    Z = propagate_fwd(g, H, K, 0.9, 0.0)
    assert np.linalg.norm(Z) <= 0.9 ** K * np.linalg.norm(H) + 1e-9


@pytest.mark.parametrize("name,K,gamma,alpha", [("tiny_dir", 3, 0.9, 0.1), ("small_dir", 2, 1.0, 0.0),
                                                ("tiny_sym", 4, 1.0, 0.0)])
def test_adjoint(name, K, gamma, alpha):
    """<M H, G> = <H, M^T G>."""
    g = oracle.graph.graph_from_config(synth.get_config(name))
    rng = np.random.default_rng(1)
    H = rng.standard_normal((g.n, 3))
    G = rng.standard_normal((g.n, 3))
    lhs = np.sum(propagate_fwd(g, H, K, gamma, alpha) * G)
    rhs = np.sum(H * propagate_bwd(g, G, K, gamma, alpha))
    assert abs(lhs - rhs) <= 1e-10 * max(1.0, abs(lhs))


def test_column_separability_bitwise():
    """Propagating a column slice equals slicing the full result, bitwise."""
    g = oracle.graph.graph_from_config(synth.get_config("tiny_dir"))
    H = np.random.default_rng(2).standard_normal((g.n, 10))
    Z = propagate_fwd(g, H, 3, 0.9, 0.1)
    for c0, c1 in [(0, 3), (3, 4), (4, 10)]:
        Zs = propagate_fwd(g, np.ascontiguousarray(H[:, c0:c1]), 3, 0.9, 0.1)
        assert np.array_equal(Zs, Z[:, c0:c1])


def test_k0_identity_and_hop_rows():
    g = oracle.graph.graph_from_config(synth.get_config("tiny_dir"))
    H = np.random.default_rng(3).standard_normal((g.n, 4))
    assert np.array_equal(propagate_fwd(g, H, 0), H)
    Z1 = propagate_fwd(g, H, 1, 0.9, 0.1)
    rows = np.array([0, 5, g.n - 1, 17])
    assert np.array_equal(oracle.propagate.hop_rows(g, H, H, rows, 0.9, 0.1), Z1[rows])
    G1 = propagate_bwd(g, H, 1, 0.9, 0.1)
    assert np.array_equal(oracle.propagate.hop_rows(g, H, H, rows, 0.9, 0.1, transposed=True), G1[rows])
