"""Helpers shared by the GPU parity tests (test infrastructure)."""
from __future__ import annotations

import functools

import numpy as np

import oracle
import synth


@functools.lru_cache(maxsize=8)
def oracle_graph(name: str):
    return oracle.graph.graph_from_config(synth.get_config(name))


def ntp_ctx_for(name: str, device: int = 0, slice_align: int = 16, reorder: bool = False):
    """A world-1 context with the config's R-MAT graph generated ON THE DEVICE
    (reorder: the library's internal degree-ordered numbering, NTP_G_REORDER)."""
    from paper_2412_20379_b200 import ntp
    cfg = synth.get_config(name)
    ctx = ntp.Context(device=device, slice_align=slice_align)
    ctx.generate_rmat(cfg.n, cfg.scale, cfg.m_raw, synth.rmat_thresholds(*cfg.abc), cfg.seed, cfg.symmetric,
                      reorder=reorder)
    return ctx


def cond_bound(g, H, K, gamma, alpha, transposed=False):
    """M|H| (or M^T|H|): the forward-error denominator of reading R10."""
    f = oracle.propagate.propagate_bwd if transposed else oracle.propagate.propagate_fwd
    return f(g, np.abs(np.asarray(H, dtype=np.float64)), K, gamma, alpha)


def assert_r10(got, ref, denom, tol, what=""):
    got = np.asarray(got, dtype=np.float64)
    err = np.abs(got - ref)
    bound = tol * denom + 1e-30
    bad = err > bound
    if bad.any():
        i = np.argwhere(bad)[0]
        raise AssertionError(f"{what}: {bad.sum()} elements exceed R10 bound {tol}; first at {tuple(i)}: "
                             f"got {got[tuple(i)]!r} ref {ref[tuple(i)]!r} denom {denom[tuple(i)]!r}; "
                             f"max scaled err {(err / (denom + 1e-300)).max():.3e}")
    return float((err / (denom + 1e-300)).max())
