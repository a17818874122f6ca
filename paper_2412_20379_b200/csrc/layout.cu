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

#include "ntp_internal.cuh"

namespace ntp {

namespace {

template <typename Tin, typename Tout>
__device__ __forceinline__ Tout cvt(Tin x);
template <> __device__ __forceinline__ float cvt<float, float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 cvt<float, __nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }
template <> __device__ __forceinline__ float cvt<__nv_bfloat16, float>(__nv_bfloat16 x) { return __bfloat162float(x); }
template <> __device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16, __nv_bfloat16>(__nv_bfloat16 x) { return x; }

template <typename Tin, typename Tout>
__global__ void pack_v2f_kernel(const Tin* __restrict__ Hv, int64_t ld_v, int32_t w, Tout* __restrict__ send,
                                int64_t V_p, int32_t d_s, int32_t P, const float* __restrict__ row_scale,
                                int64_t row0, int64_t n) {
    const int64_t total = (int64_t)P * V_p * d_s;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = (int32_t)(i % d_s);
        const int64_t v = (i / d_s) % V_p;
        const int32_t q = (int32_t)(i / ((int64_t)d_s * V_p));
        const int32_t col = q * d_s + c;
        const int64_t gr = row0 + v;
        float x = 0.f;
        if (col < w && gr < n) {
            x = cvt<Tin, float>(Hv[v * ld_v + col]);
            if (row_scale) x *= row_scale[gr];
        }
        send[i] = cvt<float, Tout>(x);
    }
}

template <typename Tin, typename Tout>
__global__ void unpack_f2v_kernel(const Tin* __restrict__ recv, int64_t V_p, int32_t d_s, Tout* __restrict__ Hv,
                                  int64_t ld_v, int32_t w) {
    const int64_t total = V_p * (int64_t)w;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i / w;
        const int32_t col = (int32_t)(i % w);
        const int32_t q = col / d_s, c = col % d_s;
        Hv[v * ld_v + col] = cvt<Tin, Tout>(recv[((int64_t)q * V_p + v) * d_s + c]);
    }
}

int blocks_for(int64_t total) { return (int)std::min<int64_t>(std::max<int64_t>(cdiv(total, 256), 1), 148 * 16); }

}  // namespace

void pack_v2f(ntp_ctx* c, const void* Hv, int64_t ld_v, int32_t w, void* send, int64_t V_p, int32_t d_s, int32_t P,
              const float* row_scale, int64_t row0, int64_t n, ntp_dtype dt_in, ntp_dtype dt_out, cudaStream_t s) {
    const int64_t total = (int64_t)P * V_p * d_s;
    if (total == 0) return;
    const int b = blocks_for(total);
    if (dt_in == NTP_F32 && dt_out == NTP_F32)
        pack_v2f_kernel<float, float><<<b, 256, 0, s>>>((const float*)Hv, ld_v, w, (float*)send, V_p, d_s, P, row_scale, row0, n);
    else if (dt_in == NTP_F32 && dt_out == NTP_BF16)
        pack_v2f_kernel<float, __nv_bfloat16><<<b, 256, 0, s>>>((const float*)Hv, ld_v, w, (__nv_bfloat16*)send, V_p, d_s, P,
                                                                row_scale, row0, n);
    else if (dt_in == NTP_BF16 && dt_out == NTP_BF16)
        pack_v2f_kernel<__nv_bfloat16, __nv_bfloat16><<<b, 256, 0, s>>>((const __nv_bfloat16*)Hv, ld_v, w,
                                                                        (__nv_bfloat16*)send, V_p, d_s, P, row_scale, row0, n);
    else
        pack_v2f_kernel<__nv_bfloat16, float><<<b, 256, 0, s>>>((const __nv_bfloat16*)Hv, ld_v, w, (float*)send, V_p, d_s,
                                                                P, row_scale, row0, n);
    NTP_LAUNCH_CHECK();
    count_launch(c);
}

void unpack_f2v(ntp_ctx* c, const void* recv, int64_t V_p, int32_t d_s, int32_t P, void* Hv, int64_t ld_v, int32_t w,
                ntp_dtype dt_in, ntp_dtype dt_out, cudaStream_t s) {
    (void)P;
    const int64_t total = V_p * (int64_t)w;
    if (total == 0) return;
    const int b = blocks_for(total);
    if (dt_in == NTP_F32 && dt_out == NTP_F32)
        unpack_f2v_kernel<float, float><<<b, 256, 0, s>>>((const float*)recv, V_p, d_s, (float*)Hv, ld_v, w);
    else if (dt_in == NTP_BF16 && dt_out == NTP_F32)
        unpack_f2v_kernel<__nv_bfloat16, float><<<b, 256, 0, s>>>((const __nv_bfloat16*)recv, V_p, d_s, (float*)Hv, ld_v, w);
    else if (dt_in == NTP_BF16 && dt_out == NTP_BF16)
        unpack_f2v_kernel<__nv_bfloat16, __nv_bfloat16><<<b, 256, 0, s>>>((const __nv_bfloat16*)recv, V_p, d_s,
                                                                          (__nv_bfloat16*)Hv, ld_v, w);
    else
        unpack_f2v_kernel<float, __nv_bfloat16><<<b, 256, 0, s>>>((const float*)recv, V_p, d_s, (__nv_bfloat16*)Hv, ld_v, w);
    NTP_LAUNCH_CHECK();
    count_launch(c);
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
    }
    NTP_NCCL(ncclGroupEnd());
}

}  // namespace ntp
