"""Loader for oracle/csrc/oracle.c (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py)."""
from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csrc", "oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")


def build_oracle_lib(force: bool = False) -> str:
    """Compile the C oracle with gcc (-O2 -fopenmp, no fast-math: IEEE fp64)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-fno-fast-math",
               "-ffp-contract=off", "-o", _SO, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _SO


def _load():
    build_oracle_lib()
    L = ctypes.CDLL(_SO)
    i64, i32, u32, u64, dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double
    vp = ctypes.c_void_p
    L.oracle_hash.argtypes = [u64, u64, u64]
    L.oracle_hash.restype = u64
    L.oracle_rmat_arcs.argtypes = [i32, u32, u32, u32, u64, i64, i64, vp, vp]
    L.oracle_rmat_arcs.restype = None
    L.oracle_propagate.argtypes = [i64, vp, vp, vp, vp, i64, vp, vp, vp, i32, dbl, dbl]
    L.oracle_propagate.restype = None
    L.oracle_hop_rows.argtypes = [vp, vp, vp, vp, i64, vp, vp, dbl, dbl, vp, i64, vp]
    L.oracle_hop_rows.restype = None
    L.oracle_rmat_filter.argtypes = [i32, u32, u32, u32, u64, i64, i64, i32, vp, i32, vp, vp, i64]
    L.oracle_rmat_filter.restype = i64
    L.oracle_num_threads.argtypes = []
    L.oracle_num_threads.restype = i32
    L.oracle_set_num_threads.argtypes = [i32]
    L.oracle_set_num_threads.restype = None
    return L


lib = _load()
