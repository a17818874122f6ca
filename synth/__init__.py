"""Seeded synthetic-input generators shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no normalisation, no propagation,
no MLP, no loss).  It only turns (config, seed) into the raw inputs both sides
consume: the counter-based hash, R-MAT quadrant thresholds, feature matrices,
labels, masks and initial weights (SURVEY.md §8(d) "Synthetic input spec").

The R-MAT *arc generator* itself is NOT here: it is part of the library's graph
setup (§8(a) a0), so the CUDA library and the oracle each implement the same
counter-based generator independently (rule ③: "each side implements the same
counter-based generator"), and the tests compare them bit-exactly.

Hash:
    h(seed, stream, i) = splitmix64_finaliser(seed*G + stream*D + i)   (mod 2^64)
    G = 0x9E3779B97F4A7C15, D = 0xD1B54A32D192ED03
"""
from __future__ import annotations

import numpy as np

from .configs import CONFIGS, Config, get_config  # noqa: F401

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
STREAM_MUL = np.uint64(0xD1B54A32D192ED03)

# stream ids
S_RMAT, S_FEAT, S_LABEL, S_MASK, S_WEIGHT = 0, 1, 2, 3, 4


def _fin(z: np.ndarray) -> np.ndarray:
    """SplitMix64 output finaliser, vectorised over uint64 arrays (wrapping)."""
    z = z.copy()
    z ^= z >> np.uint64(30)
    z *= np.uint64(0xBF58476D1CE4E5B9)
    z ^= z >> np.uint64(27)
    z *= np.uint64(0x94D049BB133111EB)
    z ^= z >> np.uint64(31)
    return z


def hash64(seed: int, stream: int, idx) -> np.ndarray:
    """h(seed, stream, i) for an array (or scalar) of counters i."""
    with np.errstate(over="ignore"):
        base = np.uint64(seed) * GOLDEN + np.uint64(stream) * STREAM_MUL
        i = np.asarray(idx, dtype=np.uint64)
        return _fin(base + i)


def rmat_thresholds(a: float, b: float, c: float) -> tuple[int, int, int]:
    """Integer quadrant thresholds floor(a*2^32), floor((a+b)*2^32), floor((a+b+c)*2^32).

    Computed with exact rational arithmetic on the decimal strings so both sides
    receive the same integers.
    """
    from fractions import Fraction

    fa, fb, fc = Fraction(str(a)), Fraction(str(b)), Fraction(str(c))
    two32 = 1 << 32
    t = [int(fa * two32), int((fa + fb) * two32), int((fa + fb + fc) * two32)]
    return tuple(min(x, two32 - 1) for x in t)


def features(seed: int, n: int, d: int, binary_density: float | None = None,
             row0: int = 0, rows: int | None = None) -> np.ndarray:
    """X[v][j] for v in [row0, row0+rows): fp32.

    Dense:  x = ((h(seed,1,v*d+j) >> 40) / 2^23) - 1   (2^24-point grid in [-1,1), exact in fp32)
    Binary: x = [h(seed,1,v*d+j) < floor(density*2^64)]   (Cora shape)
    """
    if rows is None:
        rows = n - row0
    out = np.empty((rows, d), dtype=np.float32)
    step = max(1, (1 << 24) // max(d, 1))  # bound temporaries to ~16M elements
    for r in range(0, rows, step):
        rr = min(step, rows - r)
        idx = (np.arange(row0 + r, row0 + r + rr, dtype=np.uint64)[:, None] * np.uint64(d)
               + np.arange(d, dtype=np.uint64)[None, :])
        h = hash64(seed, S_FEAT, idx)
        if binary_density is None:
            out[r:r + rr] = ((h >> np.uint64(40)).astype(np.float64) / float(1 << 23) - 1.0).astype(np.float32)
        else:
            thr = np.uint64(int(binary_density * float(1 << 64)))
            out[r:r + rr] = (h < thr).astype(np.float32)
    return out


def labels(seed: int, n: int, C: int, row0: int = 0, rows: int | None = None) -> np.ndarray:
    """y[v] = h(seed,2,v) mod C, int32."""
    if rows is None:
        rows = n - row0
    h = hash64(seed, S_LABEL, np.arange(row0, row0 + rows, dtype=np.uint64))
    return (h % np.uint64(C)).astype(np.int32)


MASK_TRAIN, MASK_VAL, MASK_TEST = 1, 2, 3


def split_masks(seed: int, n: int, row0: int = 0, rows: int | None = None) -> np.ndarray:
    """Per-vertex split code (uint8): 1 = train (u < 0.65*2^64), 2 = val (< 0.90*2^64), 3 = test.

    65/25/10 train/val/test per P:919 ("randomly select 65%, 25%, 10%"), SURVEY O7.
    """
    if rows is None:
        rows = n - row0
    u = hash64(seed, S_MASK, np.arange(row0, row0 + rows, dtype=np.uint64))
    t_train = np.uint64(int(0.65 * float(1 << 64)))
    t_val = np.uint64(int(0.90 * float(1 << 64)))
    out = np.full(rows, MASK_TEST, dtype=np.uint8)
    out[u < t_val] = MASK_VAL
    out[u < t_train] = MASK_TRAIN
    return out


def train_mask(seed: int, n: int, row0: int = 0, rows: int | None = None) -> np.ndarray:
    """uint8 0/1 train-mask."""
    return (split_masks(seed, n, row0, rows) == MASK_TRAIN).astype(np.uint8)


def glorot(seed: int, fan_in: int, fan_out: int, offset: int = 0) -> np.ndarray:
    """Glorot-uniform [fan_in x fan_out] fp32 from stream 4 at counter offset `offset`.

    w = (2*(h>>40)/2^24 - 1) * sqrt(6/(fan_in+fan_out))
    """
    lim = np.sqrt(6.0 / (fan_in + fan_out))
    h = hash64(seed, S_WEIGHT, np.arange(offset, offset + fan_in * fan_out, dtype=np.uint64))
    u = (h >> np.uint64(40)).astype(np.float64) / float(1 << 24)
    return ((2.0 * u - 1.0) * lim).astype(np.float32).reshape(fan_in, fan_out)


def model_weights(cfg: "Config") -> tuple[np.ndarray, np.ndarray]:
    """(W0 [d_in x hid], W1 [hid x C]) for a config; W1 drawn after W0 on stream 4."""
    W0 = glorot(cfg.seed, cfg.d_in, cfg.hid, 0)
    W1 = glorot(cfg.seed, cfg.hid, cfg.C, cfg.d_in * cfg.hid)
    return W0, W1


def config_inputs(cfg: "Config", row0: int = 0, rows: int | None = None):
    """(X, y, train_mask) rows [row0, row0+rows) of config `cfg`."""
    X = features(cfg.seed, cfg.n, cfg.d_in, cfg.binary_density, row0, rows)
    y = labels(cfg.seed, cfg.n, cfg.C, row0, rows)
    m = train_mask(cfg.seed, cfg.n, row0, rows)
    return X, y, m


# ---------------------------------------------------------------- the same formulas on a torch device
# (bench inputs at papers scale: 14 G feature hashes take minutes in numpy).  int64 two's-complement
# arithmetic wraps like uint64; right shifts are made logical with a mask; unsigned compare / modulo
# are rewritten in signed terms.  Pinned against the numpy versions above (tests/test_gpu_graph.py).
def _i64(x: int) -> int:
    x &= (1 << 64) - 1
    return x - (1 << 64) if x >= 1 << 63 else x


def _srl(z, k: int):
    import torch
    return torch.bitwise_and(torch.bitwise_right_shift(z, k), (1 << (64 - k)) - 1)


def hash64_torch(seed: int, stream: int, idx):
    """h(seed, stream, i) for an int64 torch tensor of counters (result: int64 bit pattern of the uint64)."""
    base = _i64(seed * 0x9E3779B97F4A7C15 + stream * 0xD1B54A32D192ED03)
    z = idx + base
    z = torch_xor(z, _srl(z, 30)) * _i64(0xBF58476D1CE4E5B9)
    z = torch_xor(z, _srl(z, 27)) * _i64(0x94D049BB133111EB)
    return torch_xor(z, _srl(z, 31))


def torch_xor(a, b):
    import torch
    return torch.bitwise_xor(a, b)


def _ult(a, t: int):
    """unsigned a < t for int64 bit patterns a and a python int threshold t in [0, 2^64)."""
    return (a ^ _i64(1 << 63)) < _i64(t ^ (1 << 63))


def features_device(seed: int, n: int, d: int, device="cuda", row0: int = 0, rows: int | None = None):
    """features() (dense) computed on a torch device: fp32 [rows x d]."""
    import torch
    if rows is None:
        rows = n - row0
    X = torch.empty(rows, d, dtype=torch.float32, device=device)
    cols = torch.arange(d, dtype=torch.int64, device=device)
    step = max(1, (1 << 25) // max(d, 1))
    for r in range(0, rows, step):
        rr = min(step, rows - r)
        idx = (torch.arange(row0 + r, row0 + r + rr, dtype=torch.int64, device=device)[:, None] * d + cols[None, :])
        X[r:r + rr] = (_srl(hash64_torch(seed, S_FEAT, idx), 40).to(torch.float64) / float(1 << 23) - 1.0).to(torch.float32)
    return X


def config_inputs_device(cfg: "Config", row0: int = 0, rows: int | None = None, device="cuda", ld: int | None = None,
                         out=None):
    """config_inputs() computed on a torch device: (X [rows x ld][:, :d_in] fp32, y int32, train mask uint8).
    out=(X, y, m): write into these (first `rows` rows) instead of allocating."""
    import torch
    if rows is None:
        rows = cfg.n - row0
    d = cfg.d_in
    ld = ld or d
    X = out[0] if out is not None else torch.zeros(rows, ld, dtype=torch.float32, device=device)[:, :d]
    cols = torch.arange(d, dtype=torch.int64, device=device)
    step = max(1, (1 << 25) // max(d, 1))
    for r in range(0, rows, step):
        rr = min(step, rows - r)
        idx = (torch.arange(row0 + r, row0 + r + rr, dtype=torch.int64, device=device)[:, None] * d + cols[None, :])
        h = hash64_torch(cfg.seed, S_FEAT, idx)
        if cfg.binary_density is None:
            X[r:r + rr] = (_srl(h, 40).to(torch.float64) / float(1 << 23) - 1.0).to(torch.float32)
        else:
            X[r:r + rr] = _ult(h, int(cfg.binary_density * float(1 << 64))).to(torch.float32)
    v = torch.arange(row0, row0 + rows, dtype=torch.int64, device=device)
    hl = hash64_torch(cfg.seed, S_LABEL, v)
    hi, lo = _srl(hl, 32), torch.bitwise_and(hl, 0xFFFFFFFF)
    y = (((hi % cfg.C) * ((1 << 32) % cfg.C) + lo) % cfg.C).to(torch.int32)
    hm = hash64_torch(cfg.seed, S_MASK, v)
    m = _ult(hm, int(0.65 * float(1 << 64))).to(torch.uint8)
    if out is not None:
        out[1][:rows] = y
        out[2][:rows] = m
        return out
    return X, y, m
