// layout.cu — vertex <-> feature layout changes (K7-K9).
//
// "split" (v2f, Alg. 1 lines 9/22): rank q's vertex rows [V_p x w]
//   -> pack into [P][V_p][d_s] (block p = columns [p*d_s, (p+1)*d_s) of my rows,
//      optionally pre-scaled by a per-row D~^{-1/2} and cast to the storage dtype)
//   -> exchange (block p to rank p) -> receive [P][V_p][d_s] == feature slice
//      [V_pad][d_s] in row order (blocks arrive in rank order): no unpack.
// "gather" (f2v, Alg. 1 lines 12/25): feature slice [V_pad][d_s] is already
//   [P][V_p][d_s] (block p = rows R_p) -> exchange -> [P][V_p][d_s] (block p =
//   columns of rank p for my rows) -> unpack into [V_p x w].
// Pure data movement (plus the optional pre-scale): gather(split(x)) == x bitwise.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "ntp_internal.cuh"

namespace ntp {

namespace {

template <typename Tin, typename Tout>
__device__ __forceinline__ Tout cvt(Tin x);
template <> __device__ __forceinline__ float cvt<float, float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 cvt<float, __nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }
template <> __device__ __forceinline__ float cvt<__nv_bfloat16, float>(__nv_bfloat16 x) { return __bfloat162float(x); }
template <> __device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16, __nv_bfloat16>(__nv_bfloat16 x) { return x; }

template <typename T> struct Q4;   // 4 consecutive elements
template <> struct Q4<float> {
    __device__ __forceinline__ static void ld(const float* p, float (&v)[4]) {
        const float4 x = *reinterpret_cast<const float4*>(p);
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    }
    __device__ __forceinline__ static void st(float* p, const float (&v)[4]) {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    }
};
template <> struct Q4<__nv_bfloat16> {
    __device__ __forceinline__ static void ld(const __nv_bfloat16* p, float (&v)[4]) {
        const uint2 x = *reinterpret_cast<const uint2*>(p);
        v[0] = __uint_as_float(x.x << 16); v[1] = __uint_as_float(x.x & 0xFFFF0000u);
        v[2] = __uint_as_float(x.y << 16); v[3] = __uint_as_float(x.y & 0xFFFF0000u);
    }
    __device__ __forceinline__ static void st(__nv_bfloat16* p, const float (&v)[4]) {
        const __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]), b = __floats2bfloat162_rn(v[2], v[3]);
        *reinterpret_cast<uint2*>(p) = make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
    }
};

// One warp per vertex row (grid-stride), each lane 4 consecutive columns: block q of `send`
// gets columns [q*d_s, (q+1)*d_s) of the row (d_s is a multiple of 4, so a quad never straddles
// two blocks), pre-scaled by row_scale[row0 + v] and cast; columns >= w and rows >= n are zero.
// `vec`: Hv rows are 16-byte aligned with ld % 4 == 0 (quad loads), else element loads.
// Row chunk: Hv holds `rows` rows that are rows [vofs, vofs + rows) of this rank's block.
// `bits` (optional): [V_p][nw] words, bit k of row vofs + v = (Hv[v][k] > 0) -- the ReLU' mask of
// the MLP backward kept as 1 bit per element instead of the fp32 H1 (memory-lean epoch).
template <typename Tin, typename Tout>
__global__ void __launch_bounds__(256) pack_v2f_kernel(const Tin* __restrict__ Hv, int64_t ld_v, int32_t w,
                                                       Tout* __restrict__ send, int64_t V_p, int32_t d_s, int32_t P,
                                                       const float* __restrict__ row_scale, int64_t row0, int64_t n,
                                                       int vec, void* const* __restrict__ peer, int rank, int64_t rows,
                                                       int64_t vofs, uint32_t* __restrict__ bits, int32_t nw) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int wpad = P * d_s;
    for (int64_t vl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; vl < rows; vl += warps) {
        const int64_t v = vofs + vl;
        const int64_t gr = row0 + v;
        const bool real = gr < n;
        const float sc = (real && row_scale) ? row_scale[gr] : 1.f;
        const Tin* src = Hv + vl * ld_v;
        for (int k = lane * 4; k < wpad; k += 128) {
            float x[4] = {0.f, 0.f, 0.f, 0.f};
            if (real) {
                if (vec && k + 3 < w) {
                    Q4<Tin>::ld(src + k, x);
                } else {
#pragma unroll
                    for (int i = 0; i < 4; ++i) x[i] = (k + i < w) ? cvt<Tin, float>(src[k + i]) : 0.f;
                }
            }
            if (bits) {   // 4 bits per lane, 8 lanes per 32-column word (k advances by 128 per pass)
                uint32_t nib = 0;
#pragma unroll
                for (int i = 0; i < 4; ++i) nib |= (x[i] > 0.f ? 1u : 0u) << i;
                uint32_t word = nib << (4 * (lane & 7));
                word |= __shfl_xor_sync(0xffffffffu, word, 1);
                word |= __shfl_xor_sync(0xffffffffu, word, 2);
                word |= __shfl_xor_sync(0xffffffffu, word, 4);
                const int wi = k >> 5;
                if ((lane & 7) == 0 && wi < nw) bits[v * nw + wi] = word;
            }
            if (real) {
#pragma unroll
                for (int i = 0; i < 4; ++i) x[i] *= sc;
            }
            const int q = k / d_s;
            // peer-direct split: block q lands in rank q's window as block `rank` (row row0 + v of
            // q's feature slice) -- the all-to-all fused into the pack
            Tout* dst = peer ? static_cast<Tout*>(peer[q]) + ((int64_t)rank * V_p + v) * d_s + (k - q * d_s)
                             : send + ((int64_t)q * V_p + v) * d_s + (k - q * d_s);
            Q4<Tout>::st(dst, x);
        }
    }
#ifndef NTP_NO_P2P_FENCE
    if (peer) __threadfence_system();
#endif
}

// One warp per vertex row: columns [4k, 4k+4) of the row come from block q = 4k / d_s of `recv`.
// `keep` (optional, same row/column indexing as Hv, ld_keep): zero where keep <= 0 (the fused
// ReLU' mask of the MLP backward, reading R12).
// Row chunk: rows [vofs, vofs + rows) of the block layout -> Hv rows [0, rows).  `keep_bits`
// ([V_p][nw] words, block-row indexed): the same mask as `keep`, one bit per element.
template <typename Tin, typename Tout>
__global__ void __launch_bounds__(256) unpack_f2v_kernel(const Tin* __restrict__ recv, int64_t V_p, int32_t d_s,
                                                         Tout* __restrict__ Hv, int64_t ld_v, int32_t w, int vec,
                                                         const float* __restrict__ keep, int64_t ld_keep, int64_t rows,
                                                         int64_t vofs, const uint32_t* __restrict__ keep_bits,
                                                         int32_t nw) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t vl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; vl < rows; vl += warps) {
        const int64_t v = vofs + vl;
        Tout* dst = Hv + vl * ld_v;
        for (int k = lane * 4; k < w; k += 128) {
            const int q = k / d_s;
            float x[4];
            Q4<Tin>::ld(recv + ((int64_t)q * V_p + v) * d_s + (k - q * d_s), x);
            if (keep) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (k + i < w && !(keep[vl * ld_keep + k + i] > 0.f)) x[i] = 0.f;
            }
            if (keep_bits) {
                const uint32_t word = keep_bits[v * nw + (k >> 5)];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (!((word >> ((k + i) & 31)) & 1u)) x[i] = 0.f;
            }
            if (vec && k + 3 < w) {
                Q4<Tout>::st(dst + k, x);
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (k + i < w) dst[k + i] = cvt<float, Tout>(x[i]);
            }
        }
    }
}

int row_blocks(int64_t rows) { return (int)std::min<int64_t>(std::max<int64_t>(cdiv(rows, 8), 1), 148 * 16); }
template <typename T> bool quad_ok(const void* p, int64_t ld) {
    return (reinterpret_cast<uintptr_t>(p) % (4 * sizeof(T))) == 0 && (ld % 4) == 0;
}

}  // namespace

void pack_v2f(ntp_ctx* c, const void* Hv, int64_t ld_v, int32_t w, void* send, int64_t V_p, int32_t d_s, int32_t P,
              const float* row_scale, int64_t row0, int64_t n, ntp_dtype dt_in, ntp_dtype dt_out, cudaStream_t s,
              void* const* peer, int64_t rows, int64_t vofs, uint32_t* bits, int32_t nw) {
    const int rk = c->rank;
    if (rows < 0) rows = V_p;
    if (rows == 0 || d_s == 0) return;
    const int b = row_blocks(rows);
    const int vec = (dt_in == NTP_F32) ? quad_ok<float>(Hv, ld_v) : quad_ok<__nv_bfloat16>(Hv, ld_v);
    if (dt_in == NTP_F32 && dt_out == NTP_F32)
        pack_v2f_kernel<float, float><<<b, 256, 0, s>>>((const float*)Hv, ld_v, w, (float*)send, V_p, d_s, P, row_scale, row0, n, vec, peer, rk, rows, vofs, bits, nw);
    else if (dt_in == NTP_F32 && dt_out == NTP_BF16)
        pack_v2f_kernel<float, __nv_bfloat16><<<b, 256, 0, s>>>((const float*)Hv, ld_v, w, (__nv_bfloat16*)send, V_p, d_s, P,
                                                                row_scale, row0, n, vec, peer, rk, rows, vofs, bits, nw);
    else if (dt_in == NTP_BF16 && dt_out == NTP_BF16)
        pack_v2f_kernel<__nv_bfloat16, __nv_bfloat16><<<b, 256, 0, s>>>((const __nv_bfloat16*)Hv, ld_v, w,
                                                                        (__nv_bfloat16*)send, V_p, d_s, P, row_scale, row0, n, vec, peer, rk, rows, vofs, bits, nw);
    else
        pack_v2f_kernel<__nv_bfloat16, float><<<b, 256, 0, s>>>((const __nv_bfloat16*)Hv, ld_v, w, (float*)send, V_p, d_s,
                                                                P, row_scale, row0, n, vec, peer, rk, rows, vofs, bits, nw);
    NTP_LAUNCH_CHECK();
    count_launch(c);
}

void unpack_f2v(ntp_ctx* c, const void* recv, int64_t V_p, int32_t d_s, int32_t P, void* Hv, int64_t ld_v, int32_t w,
                ntp_dtype dt_in, ntp_dtype dt_out, cudaStream_t s, const float* keep, int64_t ld_keep, int64_t rows,
                int64_t vofs, const uint32_t* keep_bits, int32_t nw) {
    (void)P;
    if (rows < 0) rows = V_p;
    if (rows == 0 || w == 0) return;
    const int b = row_blocks(rows);
    const int vec = (dt_out == NTP_F32) ? quad_ok<float>(Hv, ld_v) : quad_ok<__nv_bfloat16>(Hv, ld_v);
    if (dt_in == NTP_F32 && dt_out == NTP_F32)
        unpack_f2v_kernel<float, float><<<b, 256, 0, s>>>((const float*)recv, V_p, d_s, (float*)Hv, ld_v, w, vec, keep, ld_keep, rows, vofs, keep_bits, nw);
    else if (dt_in == NTP_BF16 && dt_out == NTP_F32)
        unpack_f2v_kernel<__nv_bfloat16, float><<<b, 256, 0, s>>>((const __nv_bfloat16*)recv, V_p, d_s, (float*)Hv, ld_v, w, vec, keep, ld_keep, rows, vofs, keep_bits, nw);
    else if (dt_in == NTP_BF16 && dt_out == NTP_BF16)
        unpack_f2v_kernel<__nv_bfloat16, __nv_bfloat16><<<b, 256, 0, s>>>((const __nv_bfloat16*)recv, V_p, d_s,
                                                                          (__nv_bfloat16*)Hv, ld_v, w, vec, keep, ld_keep, rows, vofs, keep_bits, nw);
    else
        unpack_f2v_kernel<float, __nv_bfloat16><<<b, 256, 0, s>>>((const float*)recv, V_p, d_s, (__nv_bfloat16*)Hv, ld_v, w, vec, keep, ld_keep, rows, vofs, keep_bits, nw);
    NTP_LAUNCH_CHECK();
    count_launch(c);
}

// ---------------------------------------------------------------- peer-direct layouts
// Each rank exposes two windows by CUDA IPC: the split target ([P][V_p][d_s]: the feature slice the
// hops read) and the gather target ([P][V_p][d_s]: the last hop's rows for this rank's vertices).
// Producers store straight into the owner's window over NVLink (pack for the split, the last
// hop's epilogue for the gather, the loss kernel for the gradient split); a stream-ordered barrier
// (1-int allreduce) after each producer replaces the all-to-all.  Handles are exchanged with the
// library's own NCCL communicator whenever a window has to grow (collective, outside capture).
void p2p_barrier(ntp_ctx* c, cudaStream_t s) {
    NTP_NCCL(ncclAllReduce(c->p2p_bar.p, c->p2p_bar.p, 1, ncclInt32, ncclSum, c->comm, s));
}

static void p2p_close(ntp_ctx* c) {
    for (int q = 0; q < (int)c->p2p_peer_split.size(); ++q) {
        if (q == c->rank) continue;
        if (c->p2p_peer_split[q]) cudaIpcCloseMemHandle(c->p2p_peer_split[q]);
        if (c->p2p_peer_gath[q]) cudaIpcCloseMemHandle(c->p2p_peer_gath[q]);
    }
    c->p2p_peer_split.clear();
    c->p2p_peer_gath.clear();
}

void p2p_shutdown(ntp_ctx* c) { p2p_close(c); }

bool p2p_ensure(ntp_ctx* c, size_t sb, size_t gb, cudaStream_t s) {
    const int P = c->world;
    static const bool enabled = [] { const char* e = getenv("NTP_P2P"); return !(e && atoi(e) == 0); }();
    if (P <= 1 || c->p2p_state < 0 || !enabled) return false;
    if (c->p2p_state == 1 && sb <= c->p2p_split_bytes && gb <= c->p2p_gath_bytes) {
        if (sb == c->p2p_used_sb && gb == c->p2p_used_gb) return true;
        if (c->capturing) return false;
        // same windows, new layout (another dtype or slice width): bytes of the old layout would show
        // through as this layout's never-written padding rows (a bf16 view of fp32 data can hold NaN
        // patterns), so the windows are cleared -- collectively, between two barriers
        p2p_barrier(c, s);
        NTP_CUDA(cudaMemsetAsync(c->p2p_split.p, 0, c->p2p_split_bytes, s));
        NTP_CUDA(cudaMemsetAsync(c->p2p_gath.p, 0, c->p2p_gath_bytes, s));
        p2p_barrier(c, s);
        c->p2p_used_sb = sb;
        c->p2p_used_gb = gb;
        return true;
    }
    if (c->capturing) return false;
    c->p2p_bar.ensure(16);
    NTP_CUDA(cudaMemsetAsync(c->p2p_bar.p, 0, 16, s));
    p2p_barrier(c, s);                         // nobody writes into the old windows any more
    wait_stream(c, s);
    p2p_close(c);
    const size_t nsb = std::max(sb, c->p2p_split_bytes), ngb = std::max(gb, c->p2p_gath_bytes);
    c->p2p_split.release();
    c->p2p_gath.release();
    c->p2p_split.ensure(nsb);
    c->p2p_gath.ensure(ngb + kCeFlagBytes);                  // + the copy-engine layout flags (inbox)
    NTP_CUDA(cudaMemsetAsync(c->p2p_split.p, 0, nsb, s));   // padding rows are never written
    NTP_CUDA(cudaMemsetAsync(c->p2p_gath.p, 0, ngb + kCeFlagBytes, s));
    cudaIpcMemHandle_t own[2];
    NTP_CUDA(cudaIpcGetMemHandle(&own[0], c->p2p_split.p));
    NTP_CUDA(cudaIpcGetMemHandle(&own[1], c->p2p_gath.p));
    const size_t hb = sizeof(own);
    DevBuf dh;
    dh.ensure(hb * (P + 1));
    NTP_CUDA(cudaMemcpyAsync(static_cast<char*>(dh.p) + hb * P, own, hb, cudaMemcpyHostToDevice, s));
    NTP_NCCL(ncclAllGather(static_cast<char*>(dh.p) + hb * P, dh.p, hb, ncclUint8, c->comm, s));
    std::vector<cudaIpcMemHandle_t> all(2 * P);
    NTP_CUDA(cudaMemcpyAsync(all.data(), dh.p, hb * P, cudaMemcpyDeviceToHost, s));
    wait_stream(c, s);
    c->p2p_peer_split.assign(P, nullptr);
    c->p2p_peer_gath.assign(P, nullptr);
    int ok = 1;
    for (int q = 0; q < P; ++q) {
        if (q == c->rank) {
            c->p2p_peer_split[q] = c->p2p_split.p;
            c->p2p_peer_gath[q] = c->p2p_gath.p;
            continue;
        }
        if (cudaIpcOpenMemHandle(&c->p2p_peer_split[q], all[2 * q], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
            cudaIpcOpenMemHandle(&c->p2p_peer_gath[q], all[2 * q + 1], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            cudaGetLastError();
            ok = 0;
        }
    }
    // every rank must take the same path: agree on the minimum
    NTP_CUDA(cudaMemcpyAsync(dh.p, &ok, sizeof(int), cudaMemcpyHostToDevice, s));
    NTP_NCCL(ncclAllReduce(dh.p, dh.p, 1, ncclInt32, ncclMin, c->comm, s));
    NTP_CUDA(cudaMemcpyAsync(&ok, dh.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    wait_stream(c, s);
    if (!ok) {
        p2p_close(c);
        c->p2p_state = -1;
        return false;
    }
    std::vector<void*> tab(2 * P);
    for (int q = 0; q < P; ++q) {
        tab[q] = c->p2p_peer_split[q];
        tab[P + q] = c->p2p_peer_gath[q];
    }
    c->p2p_tab.ensure(2 * P * sizeof(void*));
    NTP_CUDA(cudaMemcpy(c->p2p_tab.p, tab.data(), 2 * P * sizeof(void*), cudaMemcpyHostToDevice));
    c->p2p_split_bytes = nsb;
    c->p2p_gath_bytes = ngb;
    c->p2p_used_sb = sb;
    c->p2p_used_gb = gb;
    c->p2p_state = 1;
    return true;
}

uint32_t* ce_flags(ntp_ctx* c, int q) {
    return reinterpret_cast<uint32_t*>(static_cast<char*>(c->p2p_peer_gath[q]) + c->p2p_gath_bytes);
}

namespace {
PFN_cuStreamWriteValue32_v8000 write_u32_fn() {
    static PFN_cuStreamWriteValue32_v8000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        return (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) == cudaSuccess &&
                q == cudaDriverEntryPointSuccess)
                   ? reinterpret_cast<PFN_cuStreamWriteValue32_v8000>(f)
                   : nullptr;
    }();
    NTP_CHECK(fn != nullptr, NTP_ERR_CUDA, "cuStreamWriteValue32 not available");
    return fn;
}
PFN_cuStreamWaitValue32_v8000 wait_u32_fn() {
    static PFN_cuStreamWaitValue32_v8000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        return (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) == cudaSuccess &&
                q == cudaDriverEntryPointSuccess)
                   ? reinterpret_cast<PFN_cuStreamWaitValue32_v8000>(f)
                   : nullptr;
    }();
    NTP_CHECK(fn != nullptr, NTP_ERR_CUDA, "cuStreamWaitValue32 not available");
    return fn;
}
}  // namespace

void stream_write_u32(cudaStream_t s, void* addr, uint32_t v) {
    const CUresult r = write_u32_fn()((CUstream)s, (CUdeviceptr)(uintptr_t)addr, v, CU_STREAM_WRITE_VALUE_DEFAULT);
    NTP_CHECK(r == CUDA_SUCCESS, NTP_ERR_CUDA, "cuStreamWriteValue32 failed: %d", (int)r);
}

void stream_wait_u32_geq(cudaStream_t s, void* addr, uint32_t v) {
    const CUresult r = wait_u32_fn()((CUstream)s, (CUdeviceptr)(uintptr_t)addr, v, CU_STREAM_WAIT_VALUE_GEQ);
    NTP_CHECK(r == CUDA_SUCCESS, NTP_ERR_CUDA, "cuStreamWaitValue32 failed: %d", (int)r);
}

// Block exchange: block q of `send` goes to rank q and lands as block `rank` of
// rank q's `recv` (an all-to-all of equal blocks).  world == 1: a local copy.
void alltoall_blocks(ntp_ctx* c, const void* send, void* recv, int64_t block_elems, ntp_dtype dt, cudaStream_t s) {
    const size_t es = esize(dt);
    if (c->world == 1) {
        if (send != recv && block_elems > 0)
            NTP_CUDA(cudaMemcpyAsync(recv, send, block_elems * es, cudaMemcpyDeviceToDevice, s));
        return;
    }
    const ncclDataType_t t = dt == NTP_BF16 ? ncclBfloat16 : ncclFloat32;
    NTP_NCCL(ncclGroupStart());
    for (int q = 0; q < c->world; ++q) {
        NTP_NCCL(ncclSend(static_cast<const char*>(send) + q * block_elems * es, block_elems, t, q, c->comm, s));
        NTP_NCCL(ncclRecv(static_cast<char*>(recv) + q * block_elems * es, block_elems, t, q, c->comm, s));
        if (q != c->rank) wire_add(c, block_elems * (int64_t)es, block_elems * (int64_t)es);
    }
    NTP_NCCL(ncclGroupEnd());
}

// Split / gather with vs slices per rank: per (peer q, local slice j) one send/recv of blk elements, issued in
// the same (q, j) order on every rank so NCCL pairs them.  vs == 1: the block all-to-all above.
static void exchange_sliced(ntp_ctx* c, const void* src, void* dst, int64_t blk, ntp_dtype dt, cudaStream_t s,
                            bool v2f) {
    const int W = c->world, vs = c->vs;
    const size_t es = esize(dt);
    if (vs == 1) {
        alltoall_blocks(c, src, dst, blk, dt, s);
        return;
    }
    if (W == 1) {   // slice j of my rows is block j on both sides
        if (src != dst && blk > 0)
            NTP_CUDA(cudaMemcpyAsync(dst, src, (size_t)vs * blk * es, cudaMemcpyDeviceToDevice, s));
        return;
    }
    const ncclDataType_t t = dt == NTP_BF16 ? ncclBfloat16 : ncclFloat32;
    const char* sp = static_cast<const char*>(src);
    char* dp = static_cast<char*>(dst);
    NTP_NCCL(ncclGroupStart());
    for (int q = 0; q < W; ++q)
        for (int j = 0; j < vs; ++j) {
            // v2f: send block (q*vs + j) of my rows, receive rank q's rows of my slice j (block j*W + q);
            // f2v: the reverse
            const int64_t sb = v2f ? (int64_t)q * vs + j : (int64_t)j * W + q;
            const int64_t rb = v2f ? (int64_t)j * W + q : (int64_t)q * vs + j;
            NTP_NCCL(ncclSend(sp + sb * blk * es, blk, t, q, c->comm, s));
            NTP_NCCL(ncclRecv(dp + rb * blk * es, blk, t, q, c->comm, s));
            if (q != c->rank) wire_add(c, blk * (int64_t)es, blk * (int64_t)es);
        }
    NTP_NCCL(ncclGroupEnd());
}

void exchange_v2f(ntp_ctx* c, const void* send, void* feat, int64_t blk, ntp_dtype dt, cudaStream_t s) {
    exchange_sliced(c, send, feat, blk, dt, s, true);
}
void exchange_f2v(ntp_ctx* c, const void* feat, void* recv, int64_t blk, ntp_dtype dt, cudaStream_t s) {
    exchange_sliced(c, feat, recv, blk, dt, s, false);
}

}  // namespace ntp
