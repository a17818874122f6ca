"""Oracle coupled GCN ("naive GNN tensor parallelism") — TEST INFRASTRUCTURE ONLY.

NEXT-1: the paper's baseline for decoupled training is the coupled model trained with
naive tensor parallelism, which "involves more rounds of communication (i.e., twice per layer) to
gather and split vertex embeddings" — 4L - 2 layout changes per epoch against 4 for the
decoupled epoch (Fig. 6).  The model it trains is the ordinary L-layer GCN
(Eq. 3-4: AGG then UPDATE in every layer), written here as its plain definition:

    H^0 = X
    Z^l = A^ H^{l-1}                       (one hop, reading R1's two-sided A^, gamma = 1, alpha = 0)
    A^l = Z^l W^l;   H^l = ReLU(A^l)  for l < L;   logits = A^L      (no bias)
    loss = (1/N_train) sum_{train} [logsumexp(logits_v) - logits_{v, y_v}]        (O7)
  backward (chain rule, ReLU'(0) = 0 as R12):
    dA^L = (softmax - onehot) / N_train on train rows, 0 elsewhere
    dW^l = (Z^l)^T dA^l;   dZ^l = dA^l (W^l)^T;   dH^{l-1} = A^T dZ^l;   dA^{l-1} = dH^{l-1} * [A^{l-1} > 0]
    SGD: W^l <- W^l - lr dW^l; the reported loss is the pre-update loss (O9).
fp64; A^ and A^T are applied through oracle.propagate (K = 1), the pinned O3/O4 operators.
"""
from __future__ import annotations

import numpy as np

from .graph import Graph
from .model import softmax_xent
from .propagate import propagate_bwd, propagate_fwd


def forward(g: Graph, X, Ws):
    """Returns (Zs, As, logits): Zs[l] = A^ H^{l}, As[l] = Zs[l] W^{l+1} (0-based lists)."""
    H = np.asarray(X, dtype=np.float64)
    Zs, As = [], []
    for l, W in enumerate(Ws):
        Z = propagate_fwd(g, H, 1, 1.0, 0.0)
        A = Z @ np.asarray(W, dtype=np.float64)
        Zs.append(Z)
        As.append(A)
        H = np.maximum(A, 0.0) if l + 1 < len(Ws) else A
    return Zs, As, As[-1]


def forward_loss(g: Graph, X, y, mask, Ws):
    _, _, logits = forward(g, X, Ws)
    loss_sum, n_train, _ = softmax_xent(logits, y, mask)
    return loss_sum / max(n_train, 1)


def epoch_grads(g: Graph, X, y, mask, Ws):
    """(loss, [dW^1..dW^L])."""
    Zs, As, logits = forward(g, X, Ws)
    loss_sum, n_train, d = softmax_xent(logits, y, mask)
    N = max(n_train, 1)
    dA = d / N
    dWs = [None] * len(Ws)
    for l in range(len(Ws) - 1, -1, -1):
        dWs[l] = Zs[l].T @ dA
        if l > 0:
            dZ = dA @ np.asarray(Ws[l], dtype=np.float64).T
            dH = propagate_bwd(g, dZ, 1, 1.0, 0.0)
            dA = dH * (As[l - 1] > 0)
    return loss_sum / N, dWs


def train(g: Graph, X, y, mask, Ws, lr, epochs):
    Ws = [np.asarray(W, dtype=np.float64) for W in Ws]
    losses = []
    for _ in range(epochs):
        loss, dWs = epoch_grads(g, X, y, mask, Ws)
        losses.append(loss)
        Ws = [W - lr * dW for W, dW in zip(Ws, dWs)]
    return losses, Ws


def layout_changes(L: int, P: int) -> int:
    """Layout changes (split / gather all-to-alls) per epoch of naive TP: a split before and a gather
    after each layer's aggregation forward, the same for layers 2..L backward (the input layer's
    gradient is not propagated) -> 2L + 2(L - 1) = 4L - 2 (10 for L = 3).  0 on one worker."""
    return 0 if P <= 1 else 4 * L - 2


def layout_bytes(widths, V_p: int, d_s_of, P: int, elem: int) -> int:
    """Bytes one worker sends per epoch: (P-1) * V_p * d_s(w) * elem per layout change of width w;
    forward layer l moves width widths[l-1] twice, backward layer l >= 2 moves widths[l-1] twice."""
    if P <= 1:
        return 0
    L = len(widths) - 1
    tot = 0
    for l in range(1, L + 1):
        k = 2 if l == 1 else 4
        tot += k * (P - 1) * V_p * d_s_of(widths[l - 1]) * elem
    return tot
