"""Pins for oracle/model.py (O5–O9) and oracle/layout.py (a1/a3/a5) — CPU only."""
import numpy as np
import pytest

import oracle
import synth
from oracle.graph import build_graph
from oracle import model, layout


def _tiny_problem(seed, n=6, d=4, hid=3, C=3, sym=False):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, 12)
    dst = rng.integers(0, n, 12)
    g = build_graph(src, dst, n, sym)
    X = rng.standard_normal((n, d))
    y = rng.integers(0, C, n)
    mask = np.array([1, 1, 0, 1, 1, 0][:n], dtype=np.uint8)
    W0 = rng.standard_normal((d, hid))
    W1 = rng.standard_normal((hid, C))
    return g, X, y, mask, W0, W1


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("K,gamma,alpha", [(2, 1.0, 0.0), (3, 0.9, 0.1)])
def test_finite_difference_gradients(seed, K, gamma, alpha):
    """Central differences, h = 1e-6, rel err < 1e-4 for every weight."""
    g, X, y, mask, W0, W1 = _tiny_problem(seed, sym=bool(seed % 2))
    loss, dW0, dW1, _ = model.epoch_grads(g, X, y, mask, W0, W1, K, gamma, alpha)
    h = 1e-6
    for W, dW, which in [(W0, dW0, 0), (W1, dW1, 1)]:
        num = np.zeros_like(W)
        for idx in np.ndindex(W.shape):
            Wp, Wm = W.copy(), W.copy()
            Wp[idx] += h
            Wm[idx] -= h
            args_p = (Wp, W1) if which == 0 else (W0, Wp)
            args_m = (Wm, W1) if which == 0 else (W0, Wm)
            lp = model.forward_loss(g, X, y, mask, *args_p, K, gamma, alpha)
            lm = model.forward_loss(g, X, y, mask, *args_m, K, gamma, alpha)
            num[idx] = (lp - lm) / (2 * h)
        err = np.abs(num - dW).max() / max(np.abs(num).max(), 1e-12)
        assert err < 1e-4


def test_zero_weights_loss_is_log_C():
    """All-zero features or weights -> uniform softmax -> loss = ln C."""
    g, X, y, mask, W0, W1 = _tiny_problem(0, C=5)
    assert abs(model.forward_loss(g, X, y, mask, W0, np.zeros_like(W1), 2, 1.0, 0.0) - np.log(5)) < 1e-15
    assert abs(model.forward_loss(g, np.zeros_like(X), y, mask, W0, W1, 2, 1.0, 0.0) - np.log(5)) < 1e-15


def test_lr_zero_constant_loss():
    g, X, y, mask, W0, W1 = _tiny_problem(1)
    losses, _, _ = model.train(g, X, y, mask, W0, W1, 2, 1.0, 0.0, 0.0, 3)
    assert losses[0] == losses[1] == losses[2]


def test_associativity_R3():
    """M (H1 W1) == (M H1) W1 (reading R3: the engine may propagate min(hid, C) columns)."""
    cfg = synth.get_config("tiny_dir")
    g = oracle.graph.graph_from_config(cfg)
    X, y, m = synth.config_inputs(cfg)
    W0, W1 = synth.model_weights(cfg)
    A1, H1, Lhat = model.mlp_forward(X, W0, W1)
    a = oracle.propagate.propagate_fwd(g, Lhat, cfg.K, cfg.gamma, cfg.alpha)
    b = oracle.propagate.propagate_fwd(g, H1, cfg.K, cfg.gamma, cfg.alpha) @ np.asarray(W1, np.float64)
    np.testing.assert_allclose(a, b, rtol=1e-11, atol=1e-12)


def test_two_cluster_convergence():
    """Planted two-cluster graph, labels = cluster, features = noisy one-hot of the
    cluster: decoupled GCN reaches >= 95% train accuracy within 200 epochs."""
    rng = np.random.default_rng(7)
    n = 40
    cl = np.repeat([0, 1], n // 2)
    src, dst = [], []
    for u in range(n):
        for v in range(n):
            if u != v and rng.random() < (0.4 if cl[u] == cl[v] else 0.02):
                src.append(u)
                dst.append(v)
    g = build_graph(np.array(src), np.array(dst), n, True)
    X = np.eye(2)[cl] + 0.8 * rng.standard_normal((n, 2))
    X = np.concatenate([X, rng.standard_normal((n, 2))], axis=1)
    mask = np.ones(n, dtype=np.uint8)
    W0 = 0.5 * rng.standard_normal((4, 8))
    W1 = 0.5 * rng.standard_normal((8, 2))
    for ep in range(200):
        loss, W0, W1 = model.train_epoch(g, X, cl, mask, W0, W1, 2, 1.0, 0.0, 0.5)
    _, _, Lhat = model.mlp_forward(X, W0, W1)
    logits = oracle.propagate.propagate_fwd(g, Lhat, 2, 1.0, 0.0)
    assert (logits.argmax(1) == cl).mean() >= 0.95


# ---------------------------------------------------------------- layout (a1/a3/a5)

@pytest.mark.parametrize("n,w,P", [(16, 8, 4), (17, 10, 3), (1000, 41, 8), (5, 3, 8), (233, 41, 1)])
def test_split_gather_roundtrip_bitwise(n, w, P):
    X = np.random.default_rng(n).standard_normal((n, w)).astype(np.float32)
    part = layout.partition(n, w, P, 4)
    vparts = [layout.vertex_part(X, n, w, P, q, 4) for q in range(P)]
    fparts = layout.split(vparts, P, part["d_s"])
    for q in range(P):
        assert np.array_equal(fparts[q], layout.feature_part(X, n, w, P, q, 4))
    back = layout.gather(fparts, P, part["V_p"])
    for q in range(P):
        assert np.array_equal(back[q], vparts[q])


def test_comm_volume_closed_form():
    """V=16, D=8, N=4: each worker sends (N-1)*V/N*D/N = 24 scalars per gather, 96 in total,
    384 over the 4 layout changes of an epoch."""
    per = layout.payload_scalars_per_layout_change(16, 8, 4, 4, align=4)
    assert per == [24, 24, 24, 24]
    assert 4 * sum(per) == 384
    # non-divisible case: V=17, D=10, N=3 -> ceil/floor blocks, counted exactly
    per = layout.payload_scalars_per_layout_change(17, 10, 3, 4, align=4)
    part = layout.partition(17, 10, 3, 4, align=4)
    assert part["V_p"] == 6 and part["d_s"] == 4
    # rank 2 owns rows 12..16 (5 rows) and columns 8..9 (2 real)
    assert per == [(6 + 5) * 4, (6 + 5) * 4, (6 + 6) * 2]


def test_partition_maps():
    part = layout.partition(232_965, 41, 8, 4, chunks=4)
    assert part["V_p"] == 29_121 and part["d_s"] == 8 and part["V_pad"] == 232_968
    assert part["owner_rows"][7] == (7 * 29_121, 232_965)
    rows = sorted(r for ch in part["chunk_rows"] for r in ch)
    # chunks tile every owner block exactly
    assert rows[0][0] == 0 and rows[-1][1] == 8 * 29_121
    assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
    assert layout.slice_width(41, 1, 4) == 44 and layout.slice_width(41, 1, 4, 32) == 48
    assert layout.slice_width(128, 8, 2) == 16 and layout.slice_width(41, 4, 4) == 12


def test_softmax_xent_train_mask_hand_computed():
    """O7/O8 on two hand-computed rows (masks P:919): a masked-out row -- even with extreme
    logits -- contributes neither loss, count nor gradient; an unmasked one does.  A consistent omission
    of the mask from loss, count and dlogits fails the first case, a wrong N_train the second."""
    y = np.array([0, 1])
    # row 0: uniform over 2 classes -> -log(1/2) = ln 2, dlogits = (1/2 - 1, 1/2)
    # row 1: extreme logits, masked out
    logits = np.array([[0.0, 0.0], [1000.0, -1000.0]])
    loss_sum, n_train, d = model.softmax_xent(logits, y, np.array([1, 0], dtype=np.uint8))
    assert n_train == 1
    assert loss_sum == pytest.approx(np.log(2.0), abs=1e-15)
    np.testing.assert_allclose(d, [[-0.5, 0.5], [0.0, 0.0]], atol=1e-15)
    # row 1 = (ln 3, 0), label 1, now in the train set: -log(1/4) = ln 4, dlogits = (3/4, 1/4 - 1)
    logits = np.array([[0.0, 0.0], [np.log(3.0), 0.0]])
    loss_sum, n_train, d = model.softmax_xent(logits, y, np.array([1, 1], dtype=np.uint8))
    assert n_train == 2
    assert loss_sum == pytest.approx(np.log(8.0), abs=1e-14)
    np.testing.assert_allclose(d, [[-0.5, 0.5], [0.75, -0.75]], atol=1e-15)


def test_forward_loss_divides_by_train_count():
    """O7's 1/N_train: on the empty graph (A^ = I) with K = 1, gamma = 1, alpha = 0 and W chosen so the
    logits are the hand-computed rows above, the mean loss over the one train row is ln 2."""
    g = build_graph(np.zeros(0, np.int64), np.zeros(0, np.int64), 2, symmetric=True)
    X = np.array([[0.0], [1.0]])
    W0 = np.array([[1.0]])
    W1 = np.array([[1000.0, -1000.0]])   # row 0: logits (0, 0); row 1: (1000, -1000), masked out
    loss = model.forward_loss(g, X, np.array([0, 1]), np.array([1, 0], np.uint8), W0, W1, 1, 1.0, 0.0)
    assert loss == pytest.approx(np.log(2.0), abs=1e-15)
