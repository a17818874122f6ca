"""Pins of the decoupled-GAT oracle (oracle/gat.py; NEXT-2, Eq. 5, §4.1.1).

What fixes it without a second implementation: a hand-computed two-vertex example; the a = 0 special
case, where every attention row is uniform over N_in(v) + {v} and on a regular undirected graph the
attention matrix IS the pinned GCN operator A^ (oracle.propagate, O3); softmax rows summing to one and
identical scores giving equal weights; adjointness of the transposed operator; central
finite differences of every parameter; ln C at zero weights and lr = 0."""
import numpy as np
import pytest

import oracle
from oracle import gat
from oracle.graph import build_graph


def _graph(n, m, seed, symmetric):
    rng = np.random.default_rng(seed)
    return build_graph(rng.integers(0, n, m), rng.integers(0, n, m), n, symmetric=symmetric)


def _ring(n):
    v = np.arange(n)
    return build_graph(v, (v + 1) % n, n, symmetric=True)


def test_two_vertex_hand_computed():
    """Arc 0 -> 1 only, C = 1, z = (2, -1), a_src = 0.5, a_dst = 1:
    s_01 = 0.5*2 + 1*(-1) = 0 -> e = 0;  s_11 = 0.5*(-1) + 1*(-1) = -1.5 -> e = -0.3 (slope 0.2);
    alpha_01 = 1 / (1 + exp(-0.3)), alpha_11 = exp(-0.3) / (1 + exp(-0.3)); vertex 0 has only its self loop."""
    g = build_graph(np.array([0]), np.array([1]), 2, symmetric=False)
    z = np.array([[2.0], [-1.0]])
    alpha, s = gat.attention(g, z, [0.5], [1.0])
    src, dst = gat.arcs(g)                      # (0,0), (1,1), then the in-CSR arc (0,1)
    assert list(zip(src.tolist(), dst.tolist())) == [(0, 0), (1, 1), (0, 1)]
    a01 = 1.0 / (1.0 + np.exp(-0.3))
    np.testing.assert_allclose(s, [0.5 * 2 + 2.0, -1.5, 0.0], atol=1e-15)
    np.testing.assert_allclose(alpha, [1.0, 1.0 - a01, a01], atol=1e-15)
    Z = gat.propagate(g, alpha, z, 1, 0.5)[-1]
    np.testing.assert_allclose(Z, [[0.5 * 2.0], [0.5 * (a01 * 2.0 + (1.0 - a01) * -1.0)]], atol=1e-15)


@pytest.mark.parametrize("n,K,gamma", [(7, 1, 1.0), (12, 3, 0.9), (33, 2, 0.5)])
def test_zero_attention_vector_is_gcn_on_regular_graph(n, K, gamma):
    """a = 0: alpha_uv = 1/(deg_in(v)+1) for every arc of v.  On the ring (2-regular, undirected) that is
    1/3 = (d~_v d~_u)^{-1/2}: the attention operator equals the pinned GCN propagation O3."""
    g = _ring(n)
    rng = np.random.default_rng(n)
    H = rng.standard_normal((n, 4))
    alpha, _ = gat.attention(g, H, np.zeros(4), np.zeros(4))
    np.testing.assert_allclose(alpha, 1.0 / 3.0, atol=1e-16)
    got = gat.propagate(g, alpha, H, K, gamma)[-1]
    ref = oracle.propagate.propagate_fwd(g, H, K, gamma, 0.0)
    np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-14)


def test_zero_attention_vector_directed_random_walk():
    """a = 0 on a directed graph: A_att = D~_in^{-1} (A + I), built here from the raw arc set."""
    n = 20
    rng = np.random.default_rng(3)
    s_, d_ = rng.integers(0, n, 70), rng.integers(0, n, 70)
    g = build_graph(s_, d_, n, symmetric=False)
    A = np.eye(n)
    for u, v in zip(s_.tolist(), d_.tolist()):
        if u != v:
            A[v, u] = 1.0
    A /= A.sum(axis=1, keepdims=True)
    H = rng.standard_normal((n, 3))
    alpha, _ = gat.attention(g, H, np.zeros(3), np.zeros(3))
    np.testing.assert_allclose(gat.att_matrix(g, alpha).toarray(), A, atol=1e-16)


def test_rows_sum_to_one_and_identical_scores_uniform():
    g = _graph(40, 200, 5, False)
    rng = np.random.default_rng(1)
    z = rng.standard_normal((40, 5)) * 3
    alpha, _ = gat.attention(g, z, rng.standard_normal(5), rng.standard_normal(5))
    _, dst = gat.arcs(g)
    np.testing.assert_allclose(np.bincount(dst, weights=alpha, minlength=40), 1.0, atol=1e-14)
    # vertex 2 with in-neighbours 0 and 1 whose embeddings equal its own: three equal scores
    g2 = build_graph(np.array([0, 1]), np.array([2, 2]), 3, symmetric=False)
    z2 = np.ones((3, 2))
    alpha2, _ = gat.attention(g2, z2, np.array([0.3, -1.0]), np.array([2.0, 0.1]))
    np.testing.assert_allclose(alpha2[2::], [1 / 3, 1 / 3, 1 / 3], atol=1e-16)   # self of 2, then arcs 0->2, 1->2
    np.testing.assert_allclose(alpha2[:2], [1.0, 1.0], atol=1e-16)              # 0 and 1: only self loops


def test_transposed_operator_is_adjoint():
    g = _graph(30, 150, 8, False)
    rng = np.random.default_rng(2)
    z = rng.standard_normal((30, 4))
    alpha, _ = gat.attention(g, z, rng.standard_normal(4), rng.standard_normal(4))
    x, y = rng.standard_normal((30, 3)), rng.standard_normal((30, 3))
    fx = gat.propagate(g, alpha, x, 3, 0.7)[-1]
    by = gat.propagate(g, alpha, y, 3, 0.7, transposed=True)[-1]
    assert abs(np.sum(fx * y) - np.sum(x * by)) < 1e-12


def _setup(n, m, seed, symmetric, d_in=5, hid=6, C=4):
    g = _graph(n, m, seed, symmetric)
    rng = np.random.default_rng(seed + 100)
    X = rng.standard_normal((n, d_in))
    y = rng.integers(0, C, n)
    mask = (rng.random(n) < 0.7).astype(np.uint8)
    W0 = rng.standard_normal((d_in, hid)) * 0.5
    W1 = rng.standard_normal((hid, C)) * 0.5
    a_s = rng.standard_normal(C)
    a_d = rng.standard_normal(C)
    return g, X, y, mask, W0, W1, a_s, a_d


@pytest.mark.parametrize("n,m,seed,symmetric,K,gamma", [(6, 14, 1, False, 2, 1.0), (9, 30, 2, True, 3, 0.9),
                                                        (8, 20, 3, False, 1, 0.8)])
def test_finite_difference_gradients(n, m, seed, symmetric, K, gamma):
    g, X, y, mask, W0, W1, a_s, a_d = _setup(n, m, seed, symmetric)
    loss, dW0, dW1, das, dad, _ = gat.epoch_grads(g, X, y, mask, W0, W1, a_s, a_d, K, gamma)
    params = [W0, W1, a_s, a_d]
    grads = [dW0, dW1, das, dad]
    h = 1e-6
    for pi, (P, G) in enumerate(zip(params, grads)):
        num = np.zeros_like(P)
        for idx in np.ndindex(P.shape):
            for sgn in (1, -1):
                Q = [p.copy() for p in params]
                Q[pi][idx] += sgn * h
                num[idx] += sgn * gat.forward_loss(g, X, y, mask, *Q, K, gamma)
            num[idx] /= 2 * h
        err = np.abs(num - G).max() / max(np.abs(num).max(), 1e-8)
        assert err < 1e-4, (pi, err)


def test_zero_weights_loss_is_log_C_and_lr_zero_constant():
    g, X, y, mask, W0, W1, a_s, a_d = _setup(10, 30, 4, True)
    loss = gat.forward_loss(g, X, y, mask, W0, np.zeros_like(W1), a_s, a_d, 2, 1.0)
    assert loss == pytest.approx(np.log(4), abs=1e-14)
    losses, *_ = gat.train(g, X, y, mask, W0, W1, a_s, a_d, 2, 1.0, 0.0, 3)
    assert losses[0] == losses[1] == losses[2]
    losses, *_ = gat.train(g, X, y, mask, W0, W1, a_s, a_d, 2, 1.0, 0.5, 5)
    assert losses[-1] < losses[0]


@pytest.mark.parametrize("n,m,seed,symmetric,K,gamma,slope", [(9, 30, 2, True, 3, 0.9, 0.2),
                                                              (12, 40, 5, False, 2, 1.0, 0.2),
                                                              (8, 20, 3, False, 1, 0.8, 0.0)])
def test_backward_contraction_identity(n, m, seed, symmetric, K, gamma, slope):
    """The engine never forms the per-arc attention gradient (csrc/gat.cu): with beta = alpha * LeakyReLU'(s)
    and dalpha_uv = gamma sum_k G^k_v . Z^{k-1}_u, the oracle's per-arc sums ps_u = sum_v ds_uv and
    pd_v = sum_u ds_uv equal the per-vertex contractions
        w = sum_k G^k . Z^k,   pd = sum_k G^k . Y^k - w * b,   ps = sum_k Z^{k-1} . X^k - A_beta^T w
    with Y^k = gamma A_beta Z^{k-1}, X^k = gamma A_beta^T G^k, b = A_beta 1.  Checked here in fp64 against
    the oracle's own backward (a mistake in the algebra -- a dropped self loop, beta for alpha, Z^k for
    Z^{k-1} -- fails at 1e-10)."""
    g, X, y, mask, W0, W1, a_s, a_d = _setup(n, m, seed, symmetric)
    _, _, _, _, _, ex = gat.epoch_grads(g, X, y, mask, W0, W1, a_s, a_d, K, gamma, slope)
    src, dst = gat.arcs(g)
    alpha, s, Zs, ds = ex["alpha"], ex["s"], ex["Zs"], ex["ds"]
    ps_ref = np.zeros(g.n)
    pd_ref = np.zeros(g.n)
    np.add.at(ps_ref, src, ds)
    np.add.at(pd_ref, dst, ds)
    beta = alpha * np.where(s > 0, 1.0, slope)
    A = gat.att_matrix(g, alpha)
    B = gat.att_matrix(g, beta)
    _, _, dlog = oracle.model.softmax_xent(Zs[-1], y, mask)
    G = dlog / max(int(mask.sum()), 1)
    w = np.zeros(g.n)
    gy = np.zeros(g.n)
    zx = np.zeros(g.n)
    for k in range(K, 0, -1):
        Yk = gamma * (B @ Zs[k - 1])
        Xk = gamma * (B.T @ G)
        w += np.einsum("ij,ij->i", G, Zs[k])
        gy += np.einsum("ij,ij->i", G, Yk)
        zx += np.einsum("ij,ij->i", Zs[k - 1], Xk)
        G = gamma * (A.T @ G)
    b = np.asarray(B.sum(axis=1)).ravel()
    pd = gy - w * b
    ps = zx - B.T @ w
    scale = max(np.abs(ps_ref).max(), np.abs(pd_ref).max())
    assert np.abs(pd - pd_ref).max() <= 1e-10 * scale
    assert np.abs(ps - ps_ref).max() <= 1e-10 * scale
