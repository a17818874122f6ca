"""Oracle K-hop propagation — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

O3 (forward, Eq. 9 + readings R1/R2):
    Z^0 = H;  Z^k = gamma * A^ Z^{k-1} + alpha * H,   A^ = D~_in^{-1/2} (A+I) D~_out^{-1/2}
O4 (backward = exact adjoint, "accumulate gradients along out-edges"):
    Y^0 = G;  Y^k = gamma * A^T Y^{k-1} + alpha * G   (over the out-CSR)
Both run in the C loop of oracle/csrc/oracle.c (fp64, fixed per-row order).
"""
from __future__ import annotations

import numpy as np

from ._lib import lib
from .graph import Graph


def _run(n, row_ptr, col, rs, cs, H, K, gamma, alpha):
    H = np.ascontiguousarray(H, dtype=np.float64)
    if H.ndim == 1:
        H = H[:, None]
    assert H.shape[0] == n
    d = H.shape[1]
    Z = np.empty_like(H)
    tmp = np.empty_like(H)
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    cl = np.ascontiguousarray(col, dtype=np.int32)
    rs = np.ascontiguousarray(rs, dtype=np.float64)
    cs = np.ascontiguousarray(cs, dtype=np.float64)
    lib.oracle_propagate(n, rp.ctypes.data, cl.ctypes.data, rs.ctypes.data, cs.ctypes.data, d,
                         H.ctypes.data, Z.ctypes.data, tmp.ctypes.data, int(K), float(gamma), float(alpha))
    return Z


def propagate_fwd(g: Graph, H, K: int, gamma: float = 1.0, alpha: float = 0.0) -> np.ndarray:
    """Z^K = M H with M = (gamma A^)^K + alpha * sum_{j<K} (gamma A^)^j  (O3)."""
    return _run(g.n, g.row_ptr, g.col, g.dinv_in, g.dinv_out, H, K, gamma, alpha)


def propagate_bwd(g: Graph, G, K: int, gamma: float = 1.0, alpha: float = 0.0) -> np.ndarray:
    """dH = M^T G via the out-CSR with row/column scales swapped (O4)."""
    return _run(g.n, g.row_ptr_t, g.col_t, g.dinv_out, g.dinv_in, G, K, gamma, alpha)


def hop_rows(g: Graph, zin, h, rows, gamma: float, alpha: float, transposed: bool = False) -> np.ndarray:
    """One hop evaluated only at output rows `rows` (for full-scale sampled checks)."""
    zin = np.ascontiguousarray(zin, dtype=np.float64)
    d = zin.shape[1]
    hh = None if h is None else np.ascontiguousarray(h, dtype=np.float64)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.empty((rows.size, d), dtype=np.float64)
    if transposed:
        rp, cl, rs, cs = g.row_ptr_t, g.col_t, g.dinv_out, g.dinv_in
    else:
        rp, cl, rs, cs = g.row_ptr, g.col, g.dinv_in, g.dinv_out
    rp = np.ascontiguousarray(rp, dtype=np.int64)
    cl = np.ascontiguousarray(cl, dtype=np.int32)
    rs = np.ascontiguousarray(rs)
    cs = np.ascontiguousarray(cs)
    lib.oracle_hop_rows(rp.ctypes.data, cl.ctypes.data, rs.ctypes.data, cs.ctypes.data, d,
                        zin.ctypes.data, None if hh is None else hh.ctypes.data,
                        float(gamma), float(alpha), rows.ctypes.data, rows.size, out.ctypes.data)
    return out
