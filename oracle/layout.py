"""Oracle partition maps and layout changes — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

a1 (readings R6/R7):
  * vertex ownership: contiguous ranges R_q = [q*V_p, (q+1)*V_p), V_p = ceil(n/P),
    V padded to V_pad = P*V_p with zero rows ("each worker is responsible for
    ... V/N vertices"; contiguous ranges as SPEC S:405);
  * column ownership: [q*d_s, (q+1)*d_s), d_s = ceil(w/P) rounded up so that
    d_s*elem_bytes is a multiple of `align` bytes (16 by default, 32 optional;
    DESIGN.md reading D1), padded with zero columns ("each worker holds D/N
    dimensions"; SPEC ceil rule S:171, reading R7);
  * scheduling chunks: chunk j = union over q of [q*V_p + j*c, q*V_p + min((j+1)*c, V_p)),
    c = ceil(V_p / n_chunks)  ("evenly distribute its vertex-related
    communication tasks across all workers").
a3/a5: "split" (vertex -> feature layout) and "gather" (feature -> vertex
layout), written as their definitions on the padded matrix.
"""
from __future__ import annotations

import numpy as np


def slice_width(w: int, P: int, elem_bytes: int, align: int = 16) -> int:
    """d_s = ceil(w/P) rounded up to a multiple of align/elem_bytes elements."""
    q = align // elem_bytes
    base = -(-w // P)
    return -(-base // q) * q


def partition(n: int, w: int, P: int, elem_bytes: int, chunks: int = 1, align: int = 16) -> dict:
    V_p = -(-n // P) if n > 0 else 0
    d_s = slice_width(w, P, elem_bytes, align)
    c = -(-V_p // chunks) if chunks > 0 and V_p > 0 else 0
    owner_rows = [(q * V_p, min((q + 1) * V_p, n)) for q in range(P)]
    cols = [(q * d_s, (q + 1) * d_s) for q in range(P)]
    chunk_rows = []
    for j in range(chunks):
        chunk_rows.append([(q * V_p + min(j * c, V_p), q * V_p + min((j + 1) * c, V_p)) for q in range(P)])
    return dict(V_p=V_p, V_pad=P * V_p, d_s=d_s, w_pad=P * d_s, chunk=c,
                owner_rows=owner_rows, cols=cols, chunk_rows=chunk_rows)


def pad(X: np.ndarray, n: int, w: int, P: int, elem_bytes: int, align: int = 16) -> np.ndarray:
    part = partition(n, w, P, elem_bytes, align=align)
    out = np.zeros((part["V_pad"], part["w_pad"]), dtype=X.dtype)
    out[:n, :w] = X[:n, :w]
    return out


def vertex_part(X: np.ndarray, n: int, w: int, P: int, q: int, elem_bytes: int, align: int = 16) -> np.ndarray:
    """Rank q's vertex-layout rows R_q at full (padded) width."""
    part = partition(n, w, P, elem_bytes, align=align)
    Xp = pad(X, n, w, P, elem_bytes, align)
    return Xp[q * part["V_p"]:(q + 1) * part["V_p"], :]


def feature_part(X: np.ndarray, n: int, w: int, P: int, q: int, elem_bytes: int, align: int = 16) -> np.ndarray:
    """Rank q's feature-layout slice: all V_pad rows x columns [q*d_s, (q+1)*d_s)."""
    part = partition(n, w, P, elem_bytes, align=align)
    Xp = pad(X, n, w, P, elem_bytes, align)
    return Xp[:, q * part["d_s"]:(q + 1) * part["d_s"]]


def split(vertex_parts: list[np.ndarray], P: int, d_s: int) -> list[np.ndarray]:
    """v2f: from every rank's [V_p x P*d_s] rows to every rank's [V_pad x d_s] column slice."""
    full = np.concatenate(vertex_parts, axis=0)
    return [full[:, q * d_s:(q + 1) * d_s].copy() for q in range(P)]


def gather(feature_parts: list[np.ndarray], P: int, V_p: int) -> list[np.ndarray]:
    """f2v: from every rank's [V_pad x d_s] column slice to every rank's [V_p x P*d_s] rows."""
    full = np.concatenate(feature_parts, axis=1)
    return [full[q * V_p:(q + 1) * V_p, :].copy() for q in range(P)]


def bytes_per_layout_change(n: int, w: int, P: int, elem_bytes: int, align: int = 16) -> int:
    """Bytes each rank sends in one split or gather (padded wire volume): (P-1) * V_p * d_s * b."""
    part = partition(n, w, P, elem_bytes, align=align)
    return (P - 1) * part["V_p"] * part["d_s"] * elem_bytes


def payload_scalars_per_layout_change(n: int, w: int, P: int, elem_bytes: int, align: int = 16) -> list[int]:
    """Real (unpadded) scalars rank q sends in one gather: rows it owns that are real
    vertices of the OTHER ranks' blocks x real columns of its slice.  Equals the
    A11 closed form (N-1) * V/N * D/N when P divides n and w."""
    part = partition(n, w, P, elem_bytes, align=align)
    out = []
    for q in range(P):
        c0, c1 = part["cols"][q]
        real_cols = max(0, min(c1, w) - c0)
        rows_other = sum(max(0, r1 - r0) for p, (r0, r1) in enumerate(part["owner_rows"]) if p != q)
        out.append(rows_other * real_cols)
    return out
