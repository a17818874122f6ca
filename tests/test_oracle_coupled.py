"""Pins for oracle/coupled.py (NEXT-1: the coupled GCN of naive tensor parallelism) — CPU only."""
import numpy as np
import pytest

from oracle import coupled
from oracle.graph import build_graph


def _problem(seed, n=7, widths=(4, 3, 3), sym=False):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, 14)
    dst = rng.integers(0, n, 14)
    g = build_graph(src, dst, n, sym)
    X = rng.standard_normal((n, widths[0]))
    y = rng.integers(0, widths[-1], n)
    mask = (rng.random(n) < 0.7).astype(np.uint8)
    mask[0] = 1
    Ws = [rng.standard_normal((widths[i], widths[i + 1])) for i in range(len(widths) - 1)]
    return g, X, y, mask, Ws


def _dense_A(g):
    """A^ = D~_in^-1/2 (A + I) D~_out^-1/2 written out from the arc list (R1): entry [v, u] for arc u -> v."""
    n = g.n
    A = np.eye(n)
    for v in range(n):
        for k in range(g.row_ptr[v], g.row_ptr[v + 1]):
            A[v, g.col[k]] += 1.0
    din = A.sum(axis=1)        # in-degree + 1 (row sums of A + I)
    dout = A.sum(axis=0)       # out-degree + 1 (column sums)
    return A / np.sqrt(din)[:, None] / np.sqrt(dout)[None, :]


@pytest.mark.parametrize("seed", range(3))
@pytest.mark.parametrize("widths", [(4, 3, 3), (5, 4, 3, 2)])
def test_forward_equals_dense_layer_formula(seed, widths):
    """logits = A^ ReLU(... ReLU(A^ X W1) ...) W_L with a dense A^ built from the arcs: pins the layer
    order (aggregate, then update), the ReLU placement (none on the last layer) and the operand sides."""
    g, X, y, mask, Ws = _problem(seed, widths=widths, sym=bool(seed % 2))
    A = _dense_A(g)
    H = X
    for l, W in enumerate(Ws):
        H = A @ H @ W
        if l + 1 < len(Ws):
            H = np.maximum(H, 0.0)
    _, _, logits = coupled.forward(g, X, Ws)
    np.testing.assert_allclose(logits, H, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("seed", range(3))
@pytest.mark.parametrize("widths", [(4, 3, 3), (4, 3, 3, 2)])
def test_finite_difference_gradients(seed, widths):
    """Central differences (h = 1e-6) match every dW^l to 1e-4 relative."""
    g, X, y, mask, Ws = _problem(seed, widths=widths, sym=bool(seed % 2))
    loss, dWs = coupled.epoch_grads(g, X, y, mask, Ws)
    h = 1e-6
    for l, W in enumerate(Ws):
        num = np.zeros_like(W)
        for idx in np.ndindex(W.shape):
            Wp = [w.copy() for w in Ws]
            Wm = [w.copy() for w in Ws]
            Wp[l][idx] += h
            Wm[l][idx] -= h
            num[idx] = (coupled.forward_loss(g, X, y, mask, Wp) - coupled.forward_loss(g, X, y, mask, Wm)) / (2 * h)
        assert np.abs(num - dWs[l]).max() <= 1e-4 * max(1.0, np.abs(num).max()), l


def test_zero_last_weights_give_ln_C():
    g, X, y, mask, Ws = _problem(0, widths=(4, 3, 5))
    Ws[-1] = np.zeros_like(Ws[-1])
    assert abs(coupled.forward_loss(g, X, y, mask, Ws) - np.log(5)) < 1e-12


def test_layout_change_count_is_paper_constant():
    """Naive TP: 10 collective rounds for a 3-layer GNN, growing linearly with L; decoupled: 4."""
    assert coupled.layout_changes(3, 4) == 10
    assert [coupled.layout_changes(L, 8) for L in (1, 2, 3, 4)] == [2, 6, 10, 14]
    assert coupled.layout_changes(3, 1) == 0


def test_layout_bytes_closed_form():
    """(P-1) * V_p * d_s * b per change; widths (602, 256, 41) at P = 4, fp32, d_s = ceil(w/P) to 4."""
    ds = lambda w: -(-(-(-w // 4)) // 4) * 4
    got = coupled.layout_bytes((602, 256, 41), 100, ds, 4, 4)
    assert got == 3 * 100 * 4 * (2 * ds(602) + 4 * ds(256))


def test_training_lowers_loss():
    g, X, y, mask, Ws = _problem(4, n=7, widths=(4, 6, 3))
    losses, _ = coupled.train(g, X, y, mask, Ws, 0.5, 30)
    assert losses[-1] < losses[0]
