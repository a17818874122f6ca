"""Oracle decoupled model, loss, gradients and SGD epoch — TEST INFRASTRUCTURE ONLY.

Follows SURVEY §8(c) O5–O9 in the paper's order (Alg. 1):
  O5  A1 = X W0;  H1 = ReLU(A1);  L^ = H1 W1            (Eq. 7 "L^ = MLP^k(X)"; no bias)
  O6  logits = M L^                                     (Eq. 8-9; M from oracle.propagate)
  O7  loss = (1/N_train) sum_{v in train} [logsumexp(logits_v) - logits_{v,y_v}]
  O8  dlogits = (softmax - onehot)/N_train on train rows, 0 elsewhere;
      dL^ = M^T dlogits (adjoint);  dW1 = H1^T dL^;
      dH1 = (dL^ W1^T) * [A1 > 0]  (ReLU'(0) = 0, R12);  dW0 = X^T dH1
  O9  W <- W - lr * dW; the reported loss is the pre-update loss.
All fp64.
"""
from __future__ import annotations

import numpy as np

from .graph import Graph
from .propagate import propagate_fwd, propagate_bwd


def mlp_forward(X, W0, W1):
    X = np.asarray(X, dtype=np.float64)
    A1 = X @ np.asarray(W0, dtype=np.float64)
    H1 = np.maximum(A1, 0.0)
    Lhat = H1 @ np.asarray(W1, dtype=np.float64)
    return A1, H1, Lhat


def softmax_xent(logits, y, mask):
    """(sum of per-row losses over train rows, N_train, dlogits_unnormalised).

    Max-subtraction for stability (S:249 style); dlogits rows = softmax - onehot on
    train rows, 0 elsewhere (not yet divided by N_train).
    """
    logits = np.asarray(logits, dtype=np.float64)
    y = np.asarray(y, dtype=np.int64)
    m = np.asarray(mask).astype(bool)
    mx = logits.max(axis=1, keepdims=True)
    ex = np.exp(logits - mx)
    se = ex.sum(axis=1, keepdims=True)
    lse = np.log(se) + mx
    rows = np.arange(logits.shape[0])
    per_row = lse[:, 0] - logits[rows, y]
    loss_sum = float(per_row[m].sum())
    p = ex / se
    d = p.copy()
    d[rows, y] -= 1.0
    d[~m] = 0.0
    return loss_sum, int(m.sum()), d


def forward_loss(g: Graph, X, y, mask, W0, W1, K, gamma, alpha):
    A1, H1, Lhat = mlp_forward(X, W0, W1)
    logits = propagate_fwd(g, Lhat, K, gamma, alpha)
    loss_sum, n_train, _ = softmax_xent(logits, y, mask)
    return loss_sum / max(n_train, 1)


def epoch_grads(g: Graph, X, y, mask, W0, W1, K, gamma, alpha):
    """One forward + backward pass: (loss, dW0, dW1, extras)."""
    X = np.asarray(X, dtype=np.float64)
    W1d = np.asarray(W1, dtype=np.float64)
    A1, H1, Lhat = mlp_forward(X, W0, W1)
    logits = propagate_fwd(g, Lhat, K, gamma, alpha)            # O6
    loss_sum, n_train, d = softmax_xent(logits, y, mask)        # O7
    N = max(n_train, 1)
    dlogits = d / N                                             # O8.1
    dLhat = propagate_bwd(g, dlogits, K, gamma, alpha)          # O8.2
    dW1 = H1.T @ dLhat                                          # O8.3
    dH1 = (dLhat @ W1d.T) * (A1 > 0)                            # O8.4
    dW0 = X.T @ dH1                                             # O8.5
    return loss_sum / N, dW0, dW1, dict(A1=A1, H1=H1, Lhat=Lhat, logits=logits,
                                        dlogits=dlogits, dLhat=dLhat, n_train=n_train)


def train_epoch(g: Graph, X, y, mask, W0, W1, K, gamma, alpha, lr):
    """O9: returns (pre-update loss, W0', W1') in fp64."""
    loss, dW0, dW1, _ = epoch_grads(g, X, y, mask, W0, W1, K, gamma, alpha)
    W0n = np.asarray(W0, dtype=np.float64) - lr * dW0
    W1n = np.asarray(W1, dtype=np.float64) - lr * dW1
    return loss, W0n, W1n


def train(g: Graph, X, y, mask, W0, W1, K, gamma, alpha, lr, epochs):
    losses = []
    for _ in range(epochs):
        loss, W0, W1 = train_epoch(g, X, y, mask, W0, W1, K, gamma, alpha, lr)
        losses.append(loss)
    return losses, W0, W1
