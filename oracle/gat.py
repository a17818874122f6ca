"""Oracle decoupled GAT (NEXT-2) — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper's second model class: "complex models incorporating edge-associated NN operations, such as
GAT" (Eq. 5), trained decoupled by "precomputing all the attention coefficients required for
each edge ... before the graph aggregation operation starts" (§4.1.1) and then aggregating
feature slices with them exactly like the simple models (§4.1.2).  Written as its plain
definition, in the paper's order (readings G1-G4 in DESIGN.md):

  G1  vertex NN first (decoupled):  A1 = X W0,  H1 = ReLU(A1),  z = H1 W1          [n x C]
  G2  attention once per epoch from z (Eq. 5 with the vertex NN already applied), over the in-arcs of
      every v plus its self loop (A~ = A + I, reading R1), a = [a_src ; a_dst]:
        s_uv = a_src . z_u + a_dst . z_v,   e_uv = LeakyReLU(s_uv) (slope 0.2, GAT's value),
        alpha_uv = exp(e_uv) / sum_{u' in N_in(v) + {v}} exp(e_u'v)        (softmax over v's in-arcs)
  G3  K hops with the attention matrix (A_att)_{v,u} = alpha_uv (Eq. 5 second line, Eq. 9's gamma):
        Z^0 = z,  Z^k = gamma A_att Z^{k-1};  logits = Z^K      (alpha mix 0: reading G3)
  G4  loss and every gradient of (W0, W1, a_src, a_dst) by the chain rule:
        G^K = dlogits (O8.1);  G^{k-1} = gamma A_att^T G^k
        dalpha_uv = gamma sum_{k=1..K} G^k_v . Z^{k-1}_u
        de_uv = alpha_uv (dalpha_uv - sum_{u'} alpha_u'v dalpha_u'v)           (softmax backward)
        ds_uv = de_uv * (1 if s_uv > 0 else slope)                             (LeakyReLU backward)
        dz = G^0 + sum_{arcs} ds_uv (a_src at u, a_dst at v);  da_src = sum ds_uv z_u, da_dst = sum ds_uv z_v
        dW1 = H1^T dz,  dH1 = (dz W1^T) * [A1 > 0],  dW0 = X^T dH1;   SGD on W0, W1, a (O9).
fp64.  The attention matrix is applied with scipy.sparse (a library SpMM as one step).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .graph import Graph
from .model import softmax_xent

SLOPE = 0.2


def arcs(g: Graph):
    """Every attention arc (self loop first, then the in-CSR arcs): (src u, dst v) int64 arrays, n + nnz long."""
    n = g.n
    dst_e = np.repeat(np.arange(n, dtype=np.int64), np.diff(g.row_ptr))
    src = np.concatenate([np.arange(n, dtype=np.int64), g.col.astype(np.int64)])
    dst = np.concatenate([np.arange(n, dtype=np.int64), dst_e])
    return src, dst


def leaky(x, slope=SLOPE):
    return np.where(x > 0, x, slope * x)


def attention(g: Graph, z, a_src, a_dst, slope=SLOPE):
    """G2: (alpha [n + nnz] in arcs() order, s [n + nnz]).  Softmax per destination with max-subtraction."""
    z = np.asarray(z, dtype=np.float64)
    src, dst = arcs(g)
    s = z[src] @ np.asarray(a_src, np.float64) + z[dst] @ np.asarray(a_dst, np.float64)
    e = leaky(s, slope)
    m = np.full(g.n, -np.inf)
    np.maximum.at(m, dst, e)
    ex = np.exp(e - m[dst])
    den = np.zeros(g.n)
    np.add.at(den, dst, ex)
    return ex / den[dst], s


def att_matrix(g: Graph, alpha):
    """A_att [n x n] sparse: row v = destination, column u = source, value alpha_uv."""
    src, dst = arcs(g)
    return sp.csr_matrix((np.asarray(alpha, np.float64), (dst, src)), shape=(g.n, g.n))


def propagate(g: Graph, alpha, Z, K: int, gamma: float = 1.0, transposed: bool = False):
    """G3: (gamma A_att)^K Z (or with A_att^T): K hops, returns the list [Z^0, ..., Z^K]."""
    A = att_matrix(g, alpha)
    if transposed:
        A = A.T.tocsr()
    out = [np.asarray(Z, dtype=np.float64)]
    for _ in range(K):
        out.append(gamma * (A @ out[-1]))
    return out


def forward(g: Graph, X, W0, W1, a_src, a_dst, K, gamma, slope=SLOPE):
    X = np.asarray(X, np.float64)
    A1 = X @ np.asarray(W0, np.float64)
    H1 = np.maximum(A1, 0.0)
    z = H1 @ np.asarray(W1, np.float64)
    alpha, s = attention(g, z, a_src, a_dst, slope)
    Zs = propagate(g, alpha, z, K, gamma)
    return dict(A1=A1, H1=H1, z=z, alpha=alpha, s=s, Zs=Zs, logits=Zs[-1])


def forward_loss(g: Graph, X, y, mask, W0, W1, a_src, a_dst, K, gamma, slope=SLOPE):
    f = forward(g, X, W0, W1, a_src, a_dst, K, gamma, slope)
    loss_sum, n_train, _ = softmax_xent(f["logits"], y, mask)
    return loss_sum / max(n_train, 1)


def epoch_grads(g: Graph, X, y, mask, W0, W1, a_src, a_dst, K, gamma, slope=SLOPE):
    """G4: (loss, dW0, dW1, da_src, da_dst, extras)."""
    X = np.asarray(X, np.float64)
    W1d = np.asarray(W1, np.float64)
    a_src = np.asarray(a_src, np.float64)
    a_dst = np.asarray(a_dst, np.float64)
    f = forward(g, X, W0, W1, a_src, a_dst, K, gamma, slope)
    loss_sum, n_train, d = softmax_xent(f["logits"], y, mask)
    N = max(n_train, 1)
    src, dst = arcs(g)
    alpha, s, Zs, z = f["alpha"], f["s"], f["Zs"], f["z"]
    AT = att_matrix(g, alpha).T.tocsr()
    G = d / N                                            # G^K
    dalpha = np.zeros_like(alpha)
    for k in range(K, 0, -1):
        dalpha += gamma * np.einsum("ij,ij->i", G[dst], Zs[k - 1][src])   # G^k_v . Z^{k-1}_u
        G = gamma * (AT @ G)                             # G^{k-1}
    dz = G                                               # G^0 (Z^0 = z)
    wsum = np.zeros(g.n)
    np.add.at(wsum, dst, alpha * dalpha)
    de = alpha * (dalpha - wsum[dst])
    ds = de * np.where(s > 0, 1.0, slope)
    ps = np.zeros(g.n)
    pd = np.zeros(g.n)
    np.add.at(ps, src, ds)                               # sum over arcs leaving u (its z_u terms)
    np.add.at(pd, dst, ds)                               # sum over arcs entering v (its z_v terms)
    dz = dz + np.outer(ps, a_src) + np.outer(pd, a_dst)
    da_src = ps @ z
    da_dst = pd @ z
    dW1 = f["H1"].T @ dz
    dH1 = (dz @ W1d.T) * (f["A1"] > 0)
    dW0 = X.T @ dH1
    return loss_sum / N, dW0, dW1, da_src, da_dst, dict(f, dalpha=dalpha, ds=ds, dz=dz, n_train=n_train)


def train_epoch(g: Graph, X, y, mask, W0, W1, a_src, a_dst, K, gamma, lr, slope=SLOPE):
    """O9 for the GAT parameters: returns (pre-update loss, W0', W1', a_src', a_dst')."""
    loss, dW0, dW1, das, dad, _ = epoch_grads(g, X, y, mask, W0, W1, a_src, a_dst, K, gamma, slope)
    return (loss, np.asarray(W0, np.float64) - lr * dW0, np.asarray(W1, np.float64) - lr * dW1,
            np.asarray(a_src, np.float64) - lr * das, np.asarray(a_dst, np.float64) - lr * dad)


def train(g: Graph, X, y, mask, W0, W1, a_src, a_dst, K, gamma, lr, epochs, slope=SLOPE):
    losses = []
    for _ in range(epochs):
        loss, W0, W1, a_src, a_dst = train_epoch(g, X, y, mask, W0, W1, a_src, a_dst, K, gamma, lr, slope)
        losses.append(loss)
    return losses, W0, W1, a_src, a_dst
