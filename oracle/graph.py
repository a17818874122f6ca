"""Oracle graph setup — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

O1: arcs -> drop ids >= n and self loops -> (optionally append
reverse arcs) -> sort by (dst, src) and deduplicate -> in-CSR (row v =
destination, columns = ascending sources u of arcs u->v, "N_in(v)" of Eq. 1,
P:262) -> out-CSR the same way from (src, dst).  deg_in / deg_out = row lengths.
O2: D~ = D + I, so dinv = (deg + 1)^{-1/2} (isolated vertex -> 1, R8).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._lib import lib


@dataclass
class Graph:
    n: int
    symmetric: bool
    row_ptr: np.ndarray    # int64 [n+1], in-CSR
    col: np.ndarray        # int32 [nnz], sources, ascending per row
    row_ptr_t: np.ndarray  # int64 [n+1], out-CSR (transpose)
    col_t: np.ndarray      # int32 [nnz], destinations, ascending per row
    deg_in: np.ndarray     # int64 [n]
    deg_out: np.ndarray    # int64 [n]

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def dinv_in(self) -> np.ndarray:
        return dinv(self.deg_in)

    @property
    def dinv_out(self) -> np.ndarray:
        return dinv(self.deg_out)


def hash64(seed: int, stream: int, i: int) -> int:
    """The oracle's own h(seed, stream, i) (C implementation)."""
    return int(lib.oracle_hash(seed, stream, i))


def rmat_arcs(scale: int, thresholds, seed: int, i0: int, count: int):
    """Raw R-MAT arcs i in [i0, i0+count) as (src, dst) int64 arrays (before any rejection)."""
    src = np.empty(count, dtype=np.int64)
    dst = np.empty(count, dtype=np.int64)
    t0, t1, t2 = (int(t) for t in thresholds)
    lib.oracle_rmat_arcs(scale, t0, t1, t2, seed, i0, count,
                         src.ctypes.data, dst.ctypes.data)
    return src, dst


def _sort_dedup(keys: np.ndarray) -> np.ndarray:
    """Sort ascending and drop repeats (np.sort + adjacent-difference mask)."""
    s = np.sort(keys)
    if s.size == 0:
        return s
    keep = np.empty(s.size, dtype=bool)
    keep[0] = True
    np.not_equal(s[1:], s[:-1], out=keep[1:])
    return s[keep]


def _csr_from_keys(keys: np.ndarray, n: int):
    """keys = row<<32 | col, sorted & unique -> (row_ptr int64[n+1], col int32[nnz])."""
    rows = (keys >> np.int64(32)).astype(np.int64)
    cols = (keys & np.int64(0xFFFFFFFF)).astype(np.int32)
    counts = np.bincount(rows, minlength=n).astype(np.int64)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    return row_ptr, cols


def build_graph(src, dst, n: int, symmetric: bool) -> Graph:
    """O1 on an arc list."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    keep = (src >= 0) & (src < n) & (dst >= 0) & (dst < n) & (src != dst)
    s, d = src[keep], dst[keep]
    if symmetric:
        s, d = np.concatenate([s, d]), np.concatenate([d, s])
    keys_in = _sort_dedup((d << np.int64(32)) | s)          # sort by (dst, src), dedup
    row_ptr, col = _csr_from_keys(keys_in, n)
    keys_out = _sort_dedup((s << np.int64(32)) | d)         # sort by (src, dst), dedup
    row_ptr_t, col_t = _csr_from_keys(keys_out, n)
    deg_in = np.diff(row_ptr)
    deg_out = np.diff(row_ptr_t)
    return Graph(n, symmetric, row_ptr, col, row_ptr_t, col_t, deg_in, deg_out)


def from_csr(row_ptr, col, n: int, symmetric: bool = False) -> Graph:
    """Graph from an in-CSR given by the caller (the ntp_load_graph input form)."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    col = np.asarray(col, dtype=np.int64)
    dst = np.repeat(np.arange(n, dtype=np.int64), np.diff(row_ptr))
    g = build_graph(col, dst, n, symmetric=False)   # drops explicit self loops (R1), dedups
    g.symmetric = bool(symmetric)
    return g


def graph_from_config(cfg) -> Graph:
    """R-MAT graph of a synth config (O1 + O10)."""
    from synth import rmat_thresholds
    thr = rmat_thresholds(*cfg.abc)
    src, dst = rmat_arcs(cfg.scale, thr, cfg.seed, 0, cfg.m_raw)
    return build_graph(src, dst, cfg.n, cfg.symmetric)


def sampled_rows(cfg, rows, transposed: bool = False):
    """O1 restricted to sampled rows, for configs too large to build whole on the CPU:
    {v: sorted unique in-neighbours} (or out-neighbours if `transposed`) for v in `rows`,
    from a full regeneration of the raw arc stream filtered by a row bitmap."""
    from synth import rmat_thresholds
    rows = np.unique(np.asarray(rows, dtype=np.int64))
    bitmap = np.zeros((cfg.n + 63) // 64, dtype=np.uint64)
    np.bitwise_or.at(bitmap, rows >> 6, np.left_shift(np.uint64(1), (rows & 63).astype(np.uint64)))
    t0, t1, t2 = rmat_thresholds(*cfg.abc)
    cap = 1 << 20
    while True:
        src = np.empty(cap, dtype=np.int64)
        dst = np.empty(cap, dtype=np.int64)
        cnt = lib.oracle_rmat_filter(cfg.scale, t0, t1, t2, cfg.seed, cfg.m_raw, cfg.n, int(cfg.symmetric),
                                     bitmap.ctypes.data, 0 if transposed else 1, src.ctypes.data, dst.ctypes.data, cap)
        if cnt <= cap:
            break
        cap = int(cnt) + 1
    src, dst = src[:cnt], dst[:cnt]
    key_row, key_col = (src, dst) if transposed else (dst, src)
    keys = _sort_dedup((key_row << np.int64(32)) | key_col)
    kr = keys >> np.int64(32)
    kc = (keys & np.int64(0xFFFFFFFF)).astype(np.int32)
    out = {}
    bounds = np.searchsorted(kr, rows)
    ends = np.searchsorted(kr, rows, side="right")
    for v, a, b in zip(rows.tolist(), bounds.tolist(), ends.tolist()):
        out[v] = kc[a:b]
    return out


def dinv(deg) -> np.ndarray:
    """(deg + 1)^{-1/2} in fp64 (O2)."""
    return 1.0 / np.sqrt(np.asarray(deg, dtype=np.float64) + 1.0)


def dense_adjacency_hat(g: Graph) -> np.ndarray:
    """Explicit V x V  A^ = D~_in^{-1/2} (A + I) D~_out^{-1/2}  (row v, column u), V <= a few thousand."""
    n = g.n
    A = np.zeros((n, n), dtype=np.float64)
    rows = np.repeat(np.arange(n), np.diff(g.row_ptr))
    A[rows, g.col.astype(np.int64)] = 1.0
    A += np.eye(n)
    return g.dinv_in[:, None] * A * g.dinv_out[None, :]
