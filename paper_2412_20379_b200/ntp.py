"""ctypes binding of libntp (include/ntp.h) — argument marshalling only.

Every computation runs inside libntp.so (CUDA, sm_100a).  If the library is
missing this module raises at import time: there is no CPU fallback.
Tensors are torch tensors (device memory owned by the caller); NumPy arrays are
accepted only where the C call takes HOST pointers.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NTP_LIB") or os.path.join(_HERE, "libntp.so")   # NTP_LIB: dev A/B builds

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libntp.so not found at {LIB_PATH}: run `python -m paper_2412_20379_b200.build` "
                      "(there is no fallback implementation)")

_lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)

# ---------------------------------------------------------------- enums
NTP_OK, NTP_ERR_ARG, NTP_ERR_SHAPE, NTP_ERR_CONFIG, NTP_ERR_GRAPH, NTP_ERR_STATE, NTP_ERR_OOM, \
    NTP_ERR_CUDA, NTP_ERR_NCCL, NTP_ERR_TIMEOUT = 0, -1, -2, -3, -4, -5, -6, -7, -8, -9
NTP_F32, NTP_BF16 = 0, 1
NTP_LAYOUT_VERTEX, NTP_LAYOUT_FEATURE = 0, 1
NTP_G_SYMMETRIC, NTP_G_VALIDATE, NTP_G_REORDER = 1, 2, 4
NTP_M_W1_AFTER_PROP, NTP_M_OVERLAP, NTP_M_HOST_INPUTS, NTP_M_P2P_LAYOUTS = 1, 2, 4, 8
NTP_M_STAGED, NTP_M_SLOT_SHIFT, NTP_M_DATA_PARALLEL, NTP_M_HOST_STREAM = 16, 8, 32, 64
NTP_STAGE_SLOTS = 3
PHASES = ["mlp_fwd", "v2f_fwd", "prop_fwd", "f2v_fwd", "loss", "v2f_bwd", "prop_bwd", "f2v_bwd",
          "mlp_bwd", "allreduce", "sgd", "total"]

EXPORTED = ["ntp_abi_version", "ntp_status_string", "ntp_last_error", "ntp_get_unique_id", "ntp_create",
            "ntp_destroy", "ntp_load_graph", "ntp_build_graph", "ntp_generate_rmat", "ntp_rmat_arcs",
            "ntp_graph_info", "ntp_copy_csr", "ntp_copy_dinv", "ntp_partition", "ntp_scatter_features",
            "ntp_layout_v2f", "ntp_layout_f2v", "ntp_propagate_fwd", "ntp_propagate_bwd",
            "ntp_propagate_pipeline", "ntp_gemm_f32", "ntp_train_epoch", "ntp_train_epoch_coupled",
            "ntp_stage_inputs", "ntp_set_slices", "ntp_hop_timing", "ntp_train_epoch_gat",
            "ntp_set_timeout", "ntp_sync", "ntp_abort", "ntp_set_trace", "ntp_trace"]


class ntp_tensor(C.Structure):
    _fields_ = [("data", C.c_void_p), ("dtype", C.c_int), ("layout", C.c_int), ("rows", C.c_int64),
                ("cols", C.c_int32), ("ld", C.c_int64)]


class ntp_partition_info(C.Structure):
    _fields_ = [("n", C.c_int64), ("V_p", C.c_int64), ("V_pad", C.c_int64), ("w", C.c_int32), ("P", C.c_int32),
                ("d_s", C.c_int32), ("w_pad", C.c_int32), ("elem_bytes", C.c_int32), ("chunks", C.c_int32),
                ("chunk", C.c_int64)]


class ntp_model(C.Structure):
    _fields_ = [("d_in", C.c_int32), ("hid", C.c_int32), ("C", C.c_int32), ("K", C.c_int32),
                ("gamma", C.c_float), ("alpha", C.c_float), ("lr", C.c_float), ("dtype", C.c_int),
                ("chunks", C.c_int32), ("flags", C.c_uint32)]


class ntp_epoch_report(C.Structure):
    _fields_ = [("loss", C.c_double), ("n_train", C.c_int64), ("ms", C.c_double * 12),
                ("bytes_sent", C.c_int64 * 4), ("bytes_recv", C.c_int64 * 4), ("collectives", C.c_int64),
                ("kernel_launches", C.c_int64), ("spmm_ms", C.c_double), ("spmm_launches", C.c_int32),
                ("pad_", C.c_int32)]


class ntp_trace_rec(C.Structure):
    _fields_ = [("stream", C.c_int32), ("phase", C.c_int32), ("chunk", C.c_int32), ("begin_ms", C.c_float),
                ("end_ms", C.c_float)]


NTP_MAX_LAYERS = 8


class ntp_coupled_model(C.Structure):
    _fields_ = [("L", C.c_int32), ("widths", C.c_int32 * (NTP_MAX_LAYERS + 1)), ("lr", C.c_float),
                ("dtype", C.c_int), ("flags", C.c_uint32)]


class ntp_coupled_report(C.Structure):
    _fields_ = [("loss", C.c_double), ("n_train", C.c_int64), ("layout_changes", C.c_int32), ("hops", C.c_int32),
                ("bytes_sent", C.c_int64), ("bytes_recv", C.c_int64), ("ms_total", C.c_double),
                ("ms_agg", C.c_double), ("kernel_launches", C.c_int64)]


_vp, _i64, _i32, _u32, _u64, _f = C.c_void_p, C.c_int64, C.c_int32, C.c_uint32, C.c_uint64, C.c_float
_sig = {
    "ntp_abi_version": ([], C.c_int),
    "ntp_status_string": ([C.c_int], C.c_char_p),
    "ntp_last_error": ([_vp], C.c_char_p),
    "ntp_get_unique_id": ([_vp], C.c_int),
    "ntp_create": ([C.POINTER(_vp), C.c_int, C.c_int, C.c_int, _vp, C.c_int], C.c_int),
    "ntp_destroy": ([_vp], None),
    "ntp_load_graph": ([_vp, _vp, _vp, _i64, _i64, _u32], C.c_int),
    "ntp_build_graph": ([_vp, _vp, _vp, _i64, _i64, _u32], C.c_int),
    "ntp_generate_rmat": ([_vp, _i64, C.c_int, _i64, _vp, _u64, _u32], C.c_int),
    "ntp_rmat_arcs": ([_vp, C.c_int, _vp, _u64, _i64, _i64, _vp, _vp], C.c_int),
    "ntp_graph_info": ([_vp, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(C.c_int)], C.c_int),
    "ntp_copy_csr": ([_vp, C.c_int, _vp, _vp, _vp], C.c_int),
    "ntp_copy_dinv": ([_vp, _vp, _vp], C.c_int),
    "ntp_partition": ([_i64, _i32, _i32, C.c_int, _i32, C.c_int, C.POINTER(ntp_partition_info)], C.c_int),
    "ntp_scatter_features": ([_vp, _vp, C.c_int, _i64, _i32, C.c_int, C.POINTER(ntp_tensor)], C.c_int),
    "ntp_layout_v2f": ([_vp, C.POINTER(ntp_tensor), C.POINTER(ntp_tensor), _vp], C.c_int),
    "ntp_layout_f2v": ([_vp, C.POINTER(ntp_tensor), C.POINTER(ntp_tensor), _vp], C.c_int),
    "ntp_propagate_fwd": ([_vp, C.POINTER(ntp_tensor), C.POINTER(ntp_tensor), C.c_int, _f, _f, _vp], C.c_int),
    "ntp_propagate_bwd": ([_vp, C.POINTER(ntp_tensor), C.POINTER(ntp_tensor), C.c_int, _f, _f, _vp], C.c_int),
    "ntp_propagate_pipeline": ([_vp, C.POINTER(ntp_tensor), C.POINTER(ntp_tensor), C.c_int, _f, _f, C.c_int, C.c_int,
                                C.c_int32, C.c_uint32, _vp], C.c_int),
    "ntp_gemm_f32": ([_vp, _i64, _i64, _i64, _vp, _i64, C.c_int, _vp, _i64, C.c_int, _vp, _i64, C.c_int, _vp],
                     C.c_int),
    "ntp_train_epoch": ([_vp, C.POINTER(ntp_model), C.POINTER(ntp_tensor), _vp, _vp, C.POINTER(ntp_tensor),
                         C.POINTER(ntp_tensor), C.POINTER(ntp_epoch_report), _vp], C.c_int),
    "ntp_stage_inputs": ([_vp, C.c_int, _vp, _i64, _i32, _i64, _vp, _vp], C.c_int),
    "ntp_set_slices": ([_vp, _i32], C.c_int),
    "ntp_set_timeout": ([_vp, _i64], C.c_int),
    "ntp_sync": ([_vp, _vp], C.c_int),
    "ntp_abort": ([_vp], C.c_int),
    "ntp_train_epoch_gat": ([_vp, C.POINTER(ntp_model), C.POINTER(ntp_tensor), _vp, _vp, C.POINTER(ntp_tensor),
                             C.POINTER(ntp_tensor), C.POINTER(ntp_tensor), _f, C.POINTER(ntp_epoch_report), _vp],
                            C.c_int),
    "ntp_hop_timing": ([_vp, C.POINTER(C.c_double), C.POINTER(_i32)], C.c_int),
    "ntp_set_trace": ([_vp, C.c_int], C.c_int),
    "ntp_trace": ([_vp, C.POINTER(ntp_trace_rec), _i32, C.POINTER(_i32)], C.c_int),
    "ntp_train_epoch_coupled": ([_vp, C.POINTER(ntp_coupled_model), C.POINTER(ntp_tensor), _vp, _vp,
                                 C.POINTER(C.POINTER(ntp_tensor)), C.POINTER(ntp_coupled_report), _vp], C.c_int),
}
for _name, (_args, _res) in _sig.items():
    _fn = getattr(_lib, _name)
    _fn.argtypes = _args
    _fn.restype = _res


class NtpError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_lib.ntp_status_string(status).decode()}: {msg}")
        self.status = status


def abi_version() -> int:
    return _lib.ntp_abi_version()


def get_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    st = _lib.ntp_get_unique_id(buf)
    if st != NTP_OK:
        raise NtpError(st, _lib.ntp_last_error(None).decode())
    return bytes(buf)


def partition(n: int, w: int, P: int, dtype: int = NTP_F32, chunks: int = 1, slice_align: int = 16) -> dict:
    info = ntp_partition_info()
    st = _lib.ntp_partition(n, w, P, dtype, chunks, slice_align, C.byref(info))
    if st != NTP_OK:
        raise NtpError(st, "ntp_partition: bad arguments")
    return {k: getattr(info, k) for k, _ in ntp_partition_info._fields_}


def _dtype_code(t) -> int:
    import torch
    if t.dtype == torch.float32:
        return NTP_F32
    if t.dtype == torch.bfloat16:
        return NTP_BF16
    raise TypeError(f"unsupported dtype {t.dtype}")


def as_ntp_tensor(t, layout: int = NTP_LAYOUT_VERTEX) -> ntp_tensor:
    """Describe a 2-D torch tensor with unit column stride."""
    if t.dim() == 1:
        t = t.view(-1, 1)
    assert t.dim() == 2 and (t.stride(1) == 1 or t.shape[1] <= 1), "need a row-major 2-D tensor"
    return ntp_tensor(t.data_ptr(), _dtype_code(t), layout, t.shape[0], t.shape[1], max(t.stride(0), t.shape[1]))


def _stream_ptr(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def _ptr(a):
    return a.ctypes.data if isinstance(a, np.ndarray) else a.data_ptr()


class Context:
    """One libntp context per process/GPU (ntp_create / ntp_destroy)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, unique_id: bytes | None = None,
                 slice_align: int = 16):
        self._h = C.c_void_p()
        idbuf = None
        if unique_id is not None:
            idbuf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        st = _lib.ntp_create(C.byref(self._h), device, rank, world, idbuf, slice_align)
        if st != NTP_OK:
            raise NtpError(st, _lib.ntp_last_error(None).decode())
        self.device, self.rank, self.world, self.slice_align = device, rank, world, slice_align
        self.slices = world

    def set_slices(self, P: int):
        """ntp_set_slices: P = world * vs feature slices (vs virtual slices per rank, in sequence)."""
        self._chk(_lib.ntp_set_slices(self._h, int(P)))
        self.slices = int(P)

    def set_timeout(self, ms: int):
        """ntp_set_timeout: collective deadline of the synchronising calls (0 = none)."""
        self._chk(_lib.ntp_set_timeout(self._h, int(ms)))

    def abort(self):
        """ntp_abort: abort this rank's communicator (no further waits on peers)."""
        self._chk(_lib.ntp_abort(self._h))

    def sync(self, stream=None):
        """ntp_sync: wait for the stream's work under the timeout / abort contract."""
        self._chk(_lib.ntp_sync(self._h, _stream_ptr(stream)))

    def hop_timing(self):
        """ntp_hop_timing: (summed ms, launches) of the SpMM hops of the last propagation / epoch call."""
        ms, k = C.c_double(), C.c_int32()
        self._chk(_lib.ntp_hop_timing(self._h, C.byref(ms), C.byref(k)))
        return ms.value, k.value

    def set_trace(self, on: bool = True):
        """ntp_set_trace: record the overlap trace of the following epochs (they run eagerly)."""
        self._chk(_lib.ntp_set_trace(self._h, int(bool(on))))

    def trace(self) -> list:
        """ntp_trace: the last epoch's trace records as dicts (stream 'compute' / 'comm', phase, chunk, ms)."""
        k = C.c_int32()
        self._chk(_lib.ntp_trace(self._h, None, 0, C.byref(k)))
        buf = (ntp_trace_rec * max(k.value, 1))()
        self._chk(_lib.ntp_trace(self._h, buf, k.value, C.byref(k)))
        comm_ph = {0: "split", 1: "gather", 2: "gradient split", 3: "gradient gather"}
        comp_ph = {0: "mlp forward", 1: "head", 3: "mlp backward", 4: "forward hops", 5: "backward hops"}
        return [dict(stream="comm" if r.stream else "compute", phase=r.phase,
                     what=(comm_ph if r.stream else comp_ph).get(r.phase, str(r.phase)), chunk=r.chunk,
                     begin_ms=r.begin_ms, end_ms=r.end_ms) for r in buf[:k.value]]

    def close(self):
        if self._h:
            _lib.ntp_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, st):
        if st != NTP_OK:
            raise NtpError(st, _lib.ntp_last_error(self._h).decode())

    # -------------------------------------------------------------- graph
    def load_graph(self, row_ptr, col_idx, n: int, symmetric: bool = False, validate: bool = False,
                   reorder: bool = False):
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        cl = np.ascontiguousarray(col_idx, dtype=np.int32)
        flags = ((NTP_G_SYMMETRIC if symmetric else 0) | (NTP_G_VALIDATE if validate else 0)
                 | (NTP_G_REORDER if reorder else 0))
        self._chk(_lib.ntp_load_graph(self._h, rp.ctypes.data, cl.ctypes.data, n, int(rp[-1]) if n >= 0 else 0,
                                      flags))

    def build_graph(self, src, dst, n: int, symmetric: bool = False, reorder: bool = False):
        s = np.ascontiguousarray(src, dtype=np.int64)
        d = np.ascontiguousarray(dst, dtype=np.int64)
        self._chk(_lib.ntp_build_graph(self._h, s.ctypes.data, d.ctypes.data, s.size, n,
                                       (NTP_G_SYMMETRIC if symmetric else 0) | (NTP_G_REORDER if reorder else 0)))

    def generate_rmat(self, n: int, scale: int, m_raw: int, thresholds, seed: int, symmetric: bool,
                      reorder: bool = False):
        thr = (C.c_uint32 * 3)(*[int(t) for t in thresholds])
        self._chk(_lib.ntp_generate_rmat(self._h, n, scale, m_raw, thr, seed,
                                         (NTP_G_SYMMETRIC if symmetric else 0) | (NTP_G_REORDER if reorder else 0)))

    def rmat_arcs(self, scale: int, thresholds, seed: int, i0: int, count: int):
        thr = (C.c_uint32 * 3)(*[int(t) for t in thresholds])
        src = np.empty(count, dtype=np.int64)
        dst = np.empty(count, dtype=np.int64)
        self._chk(_lib.ntp_rmat_arcs(self._h, scale, thr, seed, i0, count, src.ctypes.data, dst.ctypes.data))
        return src, dst

    def graph_info(self):
        n, nnz, sym = C.c_int64(), C.c_int64(), C.c_int()
        self._chk(_lib.ntp_graph_info(self._h, C.byref(n), C.byref(nnz), C.byref(sym)))
        return n.value, nnz.value, bool(sym.value)

    def copy_csr(self, transposed: bool = False):
        n, nnz, _ = self.graph_info()
        rp = np.empty(n + 1, dtype=np.int64)
        cl = np.empty(max(nnz, 1), dtype=np.int32)
        deg = np.empty(max(n, 1), dtype=np.int32)
        self._chk(_lib.ntp_copy_csr(self._h, int(transposed), rp.ctypes.data, cl.ctypes.data, deg.ctypes.data))
        return rp, cl[:nnz], deg[:n]

    def copy_dinv(self):
        n, _, _ = self.graph_info()
        a = np.empty(max(n, 1), dtype=np.float32)
        b = np.empty(max(n, 1), dtype=np.float32)
        self._chk(_lib.ntp_copy_dinv(self._h, a.ctypes.data, b.ctypes.data))
        return a[:n], b[:n]

    # -------------------------------------------------------------- features / layouts
    def scatter_features(self, X: np.ndarray, layout: int, out):
        import torch
        code = NTP_BF16 if out.dtype == torch.bfloat16 else NTP_F32
        if code == NTP_BF16:
            Xh = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32)).to(torch.bfloat16).contiguous()
            ptr = Xh.data_ptr()
        else:
            Xh = np.ascontiguousarray(X, dtype=np.float32)
            ptr = Xh.ctypes.data
        t = as_ntp_tensor(out, layout)
        self._chk(_lib.ntp_scatter_features(self._h, ptr, code, X.shape[0], X.shape[1], layout, C.byref(t)))

    def layout_v2f(self, Hv, Hf, stream=None):
        a, b = as_ntp_tensor(Hv, NTP_LAYOUT_VERTEX), as_ntp_tensor(Hf, NTP_LAYOUT_FEATURE)
        self._chk(_lib.ntp_layout_v2f(self._h, C.byref(a), C.byref(b), _stream_ptr(stream)))

    def layout_f2v(self, Hf, Hv, stream=None):
        a, b = as_ntp_tensor(Hf, NTP_LAYOUT_FEATURE), as_ntp_tensor(Hv, NTP_LAYOUT_VERTEX)
        self._chk(_lib.ntp_layout_f2v(self._h, C.byref(a), C.byref(b), _stream_ptr(stream)))

    # -------------------------------------------------------------- propagation
    def propagate_fwd(self, H, Z, K: int, gamma: float = 1.0, alpha: float = 0.0, stream=None):
        a, b = as_ntp_tensor(H, NTP_LAYOUT_FEATURE), as_ntp_tensor(Z, NTP_LAYOUT_FEATURE)
        self._chk(_lib.ntp_propagate_fwd(self._h, C.byref(a), C.byref(b), K, gamma, alpha, _stream_ptr(stream)))

    def propagate_bwd(self, G, dH, K: int, gamma: float = 1.0, alpha: float = 0.0, stream=None):
        a, b = as_ntp_tensor(G, NTP_LAYOUT_FEATURE), as_ntp_tensor(dH, NTP_LAYOUT_FEATURE)
        self._chk(_lib.ntp_propagate_bwd(self._h, C.byref(a), C.byref(b), K, gamma, alpha, _stream_ptr(stream)))

    def propagate_pipeline(self, Hv, Zv, K: int, gamma: float = 1.0, alpha: float = 0.0, transposed: bool = False,
                           dtype: int = None, chunks: int = 1, overlap: bool = False, stream=None):
        """Vertex rows -> split -> K hops -> gather (ntp_propagate_pipeline); dtype = slice storage."""
        a, b = as_ntp_tensor(Hv, NTP_LAYOUT_VERTEX), as_ntp_tensor(Zv, NTP_LAYOUT_VERTEX)
        dt = NTP_F32 if dtype is None else dtype
        self._chk(_lib.ntp_propagate_pipeline(self._h, C.byref(a), C.byref(b), K, gamma, alpha, int(transposed), dt,
                                              chunks, NTP_M_OVERLAP if overlap else 0, _stream_ptr(stream)))

    # -------------------------------------------------------------- MLP GEMM
    def gemm(self, A, B, C, trans_a=False, trans_b=False, relu=False, stream=None):
        """C = op(A) op(B) on the tensor cores (fp32 tensors, row-major, ld = stride(0))."""
        M, N = C.shape
        K = A.shape[0] if trans_a else A.shape[1]
        self._chk(_lib.ntp_gemm_f32(self._h, M, N, K, A.data_ptr(), A.stride(0), int(trans_a), B.data_ptr(),
                                    B.stride(0), int(trans_b), C.data_ptr(), C.stride(0), int(relu),
                                    _stream_ptr(stream)))

    # -------------------------------------------------------------- epoch
    def train_epoch_coupled(self, widths, lr: float, X_v, labels_v, mask_v, Ws, dtype: int = NTP_F32,
                            stream=None) -> dict:
        """NEXT-1: one naive-tensor-parallel epoch of the coupled GCN (ntp_train_epoch_coupled);
        Ws (device fp32 [widths[l] x widths[l+1]]) are updated in place."""
        L = len(widths) - 1
        m = ntp_coupled_model()
        m.L = L
        for i, w in enumerate(widths):
            m.widths[i] = int(w)
        m.lr = float(lr)
        m.dtype = int(dtype)
        m.flags = 0
        xt = as_ntp_tensor(X_v, NTP_LAYOUT_VERTEX)
        wts = [as_ntp_tensor(W) for W in Ws]
        arr = (C.POINTER(ntp_tensor) * L)(*[C.pointer(w) for w in wts])
        rep = ntp_coupled_report()
        self._chk(_lib.ntp_train_epoch_coupled(self._h, C.byref(m), C.byref(xt), _ptr(labels_v), _ptr(mask_v), arr,
                                               C.byref(rep), _stream_ptr(stream)))
        return {"loss": rep.loss, "n_train": rep.n_train, "layout_changes": rep.layout_changes, "hops": rep.hops,
                "bytes_sent": rep.bytes_sent, "bytes_recv": rep.bytes_recv, "ms_total": rep.ms_total,
                "ms_agg": rep.ms_agg, "kernel_launches": rep.kernel_launches}

    def stage_inputs(self, slot: int, X_host, labels_host, mask_host):
        """ntp_stage_inputs: enqueue the host->device copy of one epoch's inputs into slot 0/1 (returns at
        once; pinned host tensors give an asynchronous copy that overlaps the running epoch)."""
        rows, d_in = X_host.shape
        ldx = X_host.stride(0) if hasattr(X_host, "stride") and callable(X_host.stride) else d_in
        self._chk(_lib.ntp_stage_inputs(self._h, int(slot), _ptr(X_host), rows, d_in, ldx, _ptr(labels_host),
                                        _ptr(mask_host)))

    def _report(self, rep) -> dict:
        return {"loss": rep.loss, "n_train": rep.n_train, "ms": dict(zip(PHASES, list(rep.ms))),
                "bytes_sent": list(rep.bytes_sent), "bytes_recv": list(rep.bytes_recv),
                "collectives": rep.collectives, "kernel_launches": rep.kernel_launches,
                "spmm_ms": rep.spmm_ms, "spmm_launches": rep.spmm_launches}

    def train_epoch_gat(self, model: dict, X_v, labels_v, mask_v, W0, W1, att, slope: float = 0.2,
                        stream=None) -> dict:
        """NEXT-2: one decoupled-GAT epoch (ntp_train_epoch_gat); W0, W1, att [2 x C] updated in place."""
        m = ntp_model(model["d_in"], model["hid"], model["C"], model["K"], model["gamma"], model.get("alpha", 0.0),
                      model["lr"], model.get("dtype", NTP_F32), model.get("chunks", 1), model.get("flags", 0))
        xt = as_ntp_tensor(X_v, NTP_LAYOUT_VERTEX)
        w0, w1, at = as_ntp_tensor(W0), as_ntp_tensor(W1), as_ntp_tensor(att)
        rep = ntp_epoch_report()
        self._chk(_lib.ntp_train_epoch_gat(self._h, C.byref(m), C.byref(xt), _ptr(labels_v), _ptr(mask_v),
                                           C.byref(w0), C.byref(w1), C.byref(at), float(slope), C.byref(rep),
                                           _stream_ptr(stream)))
        return self._report(rep)

    def train_epoch(self, model: dict, X_v, labels_v, mask_v, W0, W1, stream=None, host_inputs: bool = False,
                    staged_slot: int | None = None, host_stream: bool = False) -> dict:
        flags = (model.get("flags", 0) | (NTP_M_HOST_INPUTS if host_inputs else 0)
                 | (NTP_M_HOST_STREAM if host_stream else 0))
        if staged_slot is not None:   # inputs from ntp_stage_inputs slot (X_v gives the shape only)
            flags |= NTP_M_STAGED | (int(staged_slot) << NTP_M_SLOT_SHIFT)
        m = ntp_model(model["d_in"], model["hid"], model["C"], model["K"], model["gamma"], model["alpha"],
                      model["lr"], model.get("dtype", NTP_F32), model.get("chunks", 1), flags)
        xt = as_ntp_tensor(X_v, NTP_LAYOUT_VERTEX)
        w0, w1 = as_ntp_tensor(W0), as_ntp_tensor(W1)
        rep = ntp_epoch_report()
        self._chk(_lib.ntp_train_epoch(self._h, C.byref(m), C.byref(xt), _ptr(labels_v), _ptr(mask_v),
                                       C.byref(w0), C.byref(w1), C.byref(rep), _stream_ptr(stream)))
        return {"loss": rep.loss, "n_train": rep.n_train, "ms": dict(zip(PHASES, list(rep.ms))),
                "bytes_sent": list(rep.bytes_sent), "bytes_recv": list(rep.bytes_recv),
                "collectives": rep.collectives, "kernel_launches": rep.kernel_launches,
                "spmm_ms": rep.spmm_ms, "spmm_launches": rep.spmm_launches}
