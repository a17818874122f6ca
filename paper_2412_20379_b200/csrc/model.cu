// model.cu — one decoupled-TP training epoch (Alg. 1).
//
//   a2  H1 = ReLU(X_v W0);  L^ = H1 W1 (unless W1 is applied after propagation, R3)
//   a3  split L^ (pack with column-side pre-scale D~_out^{-1/2}) -> S^0 feature slice
//   a4  K forward hops (spmm.cu)
//   a5  gather Z^K -> logits rows (read in place by the loss kernel, or unpacked + W1)
//   a6  softmax-xent on train rows; dlogits = softmax - onehot (1/N_train folded into SGD)
//   a7  split dlogits (pre-scale D~_in^{-1/2}: the backward's column side)
//   a8  K backward hops over the out-CSR
//   a9  gather -> dL^ rows
//   a10 dW1 = H1^T dL^, dH1 = (dL^ W1^T) .* [H1 > 0], dW0 = X^T dH1
//   a11 allreduce(dW0 | dW1) + allreduce(loss_sum, n_train) ; W -= lr/N_train * dW
// Dense GEMMs: tcgen05 3xTF32 (gemm.cu; fp32-level accuracy, parity reading R11).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "ntp_internal.cuh"

namespace ntp {

namespace {

template <typename T> __device__ __forceinline__ float ldf(const T* p);
template <> __device__ __forceinline__ float ldf<float>(const float* p) { return *p; }
template <> __device__ __forceinline__ float ldf<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }
template <typename T> __device__ __forceinline__ void stf(T* p, float v);
template <> __device__ __forceinline__ void stf<float>(float* p, float v) { *p = v; }
template <> __device__ __forceinline__ void stf<__nv_bfloat16>(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

// LPR lanes per vertex row (32/LPR rows per warp, so short rows do not leave a warp's
// dependent load -> max -> exp -> sum chain idle).  Input logits: blocked [P][V_p][d_s]
// (TIn = storage dtype) when `in_blocked`, else plain fp32 [V_p x ld_plain].  Output gradient
// rows: blocked with per-row scale `gscale` (the split's pre-scale) when `out_blocked`, else
// plain fp32.  Each lane keeps its <= MAXK logits in registers (one read, one exp per logit;
// LPR*MAXK >= C is guaranteed by the launcher).  Per-block loss partials (fp64, fixed order)
// -> part[blockIdx.x]; train counts -> cnt[blockIdx.x].
template <typename TIn, typename TOut, int LPR>
__global__ void __launch_bounds__(256) softmax_xent_kernel(const TIn* __restrict__ in, int in_blocked, int64_t V_p,
                                                           int32_t d_s, int32_t C, const int32_t* __restrict__ y,
                                                           const uint8_t* __restrict__ mask, int64_t row0, int64_t n,
                                                           TOut* __restrict__ out, int out_blocked,
                                                           const float* __restrict__ gscale, double* __restrict__ part,
                                                           int64_t* __restrict__ cnt, int64_t ld_plain,
                                                           void* const* __restrict__ peer, int rank) {
    constexpr int MAXK = 8;
    constexpr int RPB = 256 / LPR;                     // rows per block
    __shared__ double s_loss[RPB];
    __shared__ int64_t s_cnt[RPB];
    const int sub = threadIdx.x % LPR;
    const int rloc = threadIdx.x / LPR;
    const unsigned smask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << ((threadIdx.x & 31) / LPR * LPR));
    double my_loss = 0.0;
    int64_t my_cnt = 0;
    // grid-stride over row groups: a fixed grid keeps the partials few (the fixed-order
    // reduce stays one small pass) and the per-thread accumulation order fixed.
    for (int64_t v = (int64_t)blockIdx.x * RPB + rloc; v < V_p; v += (int64_t)gridDim.x * RPB) {
        const int64_t gr = row0 + v;
        const bool train = gr < n && mask[v] != 0;
        auto addr = [&](int col) -> int64_t {
            if (in_blocked) {
                const int q = col / d_s;
                return ((int64_t)q * V_p + v) * d_s + (col - q * d_s);
            }
            return v * ld_plain + col;
        };
        float x[MAXK];
        float mx = -INFINITY;
#pragma unroll
        for (int k = 0; k < MAXK; ++k) {
            const int col = sub + LPR * k;
            x[k] = col < C ? ldf<TIn>(in + addr(col)) : -INFINITY;
            mx = fmaxf(mx, x[k]);
        }
        for (int o = LPR / 2; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(smask, mx, o));
        float se = 0.f;
#pragma unroll
        for (int k = 0; k < MAXK; ++k) {
            x[k] = (sub + LPR * k < C) ? expf(x[k] - mx) : 0.f;
            se += x[k];
        }
        for (int o = LPR / 2; o > 0; o >>= 1) se += __shfl_xor_sync(smask, se, o);
        const int yv = train ? y[v] : -1;
        if (train && sub == 0) {
            const float ly = ldf<TIn>(in + addr(yv));
            my_loss += (double)(logf(se) + mx - ly);
            my_cnt += 1;
        }
        const float inv = 1.f / se;
        const float sc = (gscale && gr < n) ? gscale[gr] : 1.f;
#pragma unroll
        for (int k = 0; k < MAXK; ++k) {
            const int col = sub + LPR * k;
            if (col < C) {
                const float gval = train ? (x[k] * inv - (col == yv ? 1.f : 0.f)) * sc : 0.f;
                if (out_blocked) {
                    const int q = col / d_s;
                    // peer-direct: straight into rank q's split window (the gradient v2f fused in)
                    TOut* dst = peer ? static_cast<TOut*>(peer[q]) + ((int64_t)rank * V_p + v) * d_s + (col - q * d_s)
                                     : out + ((int64_t)q * V_p + v) * d_s + (col - q * d_s);
                    stf<TOut>(dst, gval);
                } else {
                    stf<TOut>(out + v * ld_plain + col, gval);
                }
            }
        }
    }
#ifndef NTP_NO_P2P_FENCE
    if (peer) __threadfence_system();
#endif
    if (sub == 0) {
        s_loss[rloc] = my_loss;
        s_cnt[rloc] = my_cnt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double l = 0.0;
        int64_t k = 0;
        for (int i = 0; i < RPB; ++i) {  // fixed order
            l += s_loss[i];
            k += s_cnt[i];
        }
        part[blockIdx.x] = l;
        cnt[blockIdx.x] = k;
    }
}

// Launches the loss kernel with the narrowest row group that holds C logits in registers.
template <typename TIn, typename TOut>
int64_t launch_softmax_xent(ntp_ctx* c, const TIn* in, int in_blocked, int64_t V_p, int32_t d_s, int32_t C,
                            const int32_t* y, const uint8_t* mask, int64_t row0, int64_t n, TOut* out,
                            int out_blocked, const float* gscale, double* part, int64_t* cnt, int64_t ld_plain,
                            cudaStream_t s, void* const* peer = nullptr) {
    NTP_CHECK(C <= 256, NTP_ERR_CONFIG, "C = %d > 256 classes is not supported", C);
    int64_t nb;
#define NTP_LOSS_LAUNCH(LPR)                                                                                    \
    nb = std::min<int64_t>(std::max<int64_t>(cdiv(V_p, 256 / LPR), 1), 148 * 8);                              \
    softmax_xent_kernel<TIn, TOut, LPR><<<(unsigned)nb, 256, 0, s>>>(in, in_blocked, V_p, d_s, C, y, mask, row0, n, \
                                                                     out, out_blocked, gscale, part, cnt, ld_plain, \
                                                                     peer, c->rank)
    if (C <= 32) { NTP_LOSS_LAUNCH(4); }
    else if (C <= 64) { NTP_LOSS_LAUNCH(8); }
    else if (C <= 128) { NTP_LOSS_LAUNCH(16); }
    else { NTP_LOSS_LAUNCH(32); }
#undef NTP_LOSS_LAUNCH
    NTP_LAUNCH_CHECK();
    count_launch(c);
    return nb;
}

// Zero the padded gradient columns [C, P*d_s) of blocked output (left untouched by the loss kernel).
template <typename T>
__global__ void zero_pad_cols_kernel(T* __restrict__ buf, int64_t V_p, int32_t d_s, int32_t P, int32_t C,
                                     void* const* __restrict__ peer, int rank) {
    const int32_t pad = P * d_s - C;
    const int64_t total = V_p * pad;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i / pad;
        const int32_t col = C + (int32_t)(i % pad);
        const int32_t q = col / d_s;
        T* dst = peer ? static_cast<T*>(peer[q]) + ((int64_t)rank * V_p + v) * d_s + col % d_s
                      : buf + ((int64_t)q * V_p + v) * d_s + col % d_s;
        stf<T>(dst, 0.f);
    }
#ifndef NTP_NO_P2P_FENCE
    if (peer) __threadfence_system();
#endif
}

// Fixed-order sum of block partials -> scal[0] = loss_sum, scal[1] = n_train (as double).
__global__ void reduce_partials_kernel(const double* __restrict__ part, const int64_t* __restrict__ cnt, int64_t nb,
                                       double* __restrict__ scal) {
    __shared__ double sl[256];
    __shared__ int64_t sk[256];
    double l = 0.0;
    int64_t k = 0;
    for (int64_t i = threadIdx.x; i < nb; i += 256) {
        l += part[i];
        k += cnt[i];
    }
    sl[threadIdx.x] = l;
    sk[threadIdx.x] = k;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            sl[threadIdx.x] += sl[threadIdx.x + o];
            sk[threadIdx.x] += sk[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        scal[0] = sl[0];
        scal[1] = (double)sk[0];
    }
}

__global__ void sgd_kernel(float* __restrict__ W0, int64_t n0, float* __restrict__ W1, int64_t n1,
                           const float* __restrict__ dW, const double* __restrict__ scal, float lr) {
    const double N = scal[1] > 0.0 ? scal[1] : 1.0;
    const float step = (float)((double)lr / N);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n0 + n1; i += (int64_t)gridDim.x * blockDim.x) {
        if (i < n0) W0[i] -= step * dW[i];
        else W1[i - n0] -= step * dW[i];
    }
}

// out[i] = sum_ch part[ch][i] in chunk order (deterministic weight gradients of the chunked epoch)
__global__ void sum_chunks_kernel(const float* __restrict__ part, int64_t nch, int64_t len, float* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
        float acc = part[i];
        for (int64_t ch = 1; ch < nch; ++ch) acc += part[ch * len + i];
        out[i] = acc;
    }
}

int eblocks(int64_t total) { return (int)std::min<int64_t>(std::max<int64_t>(cdiv(total, 256), 1), 148 * 16); }

// MLP GEMM C = op(A) op(B) (+ epilogue: 1 ReLU, 2 keep where aux > 0) on the tensor cores
// (gemm.cu, tcgen05 3xTF32; Bs: optional pre-split {hi, lo} copy of B, same layout and ldb).
struct Split { const float* hi = nullptr; const float* lo = nullptr; };
void mlp_gemm(ntp_ctx* c, bool ta, bool tb, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
              const float* B, int64_t ldb, float* C, int64_t ldc, cudaStream_t s, int epi = 0,
              const float* aux = nullptr, int64_t ldaux = 0, Split Bs = Split{}) {
    if (Bs.hi) gemm_tf32x3(c, M, N, K, A, lda, ta, Bs.hi, ldb, !tb, C, ldc, epi, aux, ldaux, s, Bs.lo);
    else gemm_tf32x3(c, M, N, K, A, lda, ta, B, ldb, !tb, C, ldc, epi, aux, ldaux, s);
}

inline int64_t round4(int64_t x) { return (x + 3) / 4 * 4; }

}  // namespace

// ---- epoch building blocks shared with the GAT epoch (gat.cu)
// Phase times from the epoch's events: E0 start, E1 mlp fwd, E2 v2f, E[10] fwd hops done, E3 f2v, E4 loss,
// E5 v2f bwd, E[11] bwd hops done, E6 f2v bwd (+ unpack), E7 mlp bwd, E8 allreduce, E9 sgd.
void epoch_phases(cudaEvent_t* E, double* ms) {
    struct { int a, b, ph; } tab[] = {{0, 1, NTP_PH_MLP_FWD}, {1, 2, NTP_PH_V2F_FWD}, {2, 10, NTP_PH_PROP_FWD},
                                      {10, 3, NTP_PH_F2V_FWD}, {3, 4, NTP_PH_LOSS},    {4, 5, NTP_PH_V2F_BWD},
                                      {5, 11, NTP_PH_PROP_BWD}, {11, 6, NTP_PH_F2V_BWD}, {6, 7, NTP_PH_MLP_BWD},
                                      {7, 8, NTP_PH_ALLREDUCE}, {8, 9, NTP_PH_SGD},     {0, 9, NTP_PH_TOTAL}};
    for (int i = 0; i < NTP_PH_COUNT; ++i) ms[i] = 0.0;
    for (const auto& t : tab) {
        float x = 0.f;
        NTP_CUDA(cudaEventElapsedTime(&x, E[t.a], E[t.b]));
        ms[t.ph] = x;
    }
}

void epoch_gemm(ntp_ctx* c, bool ta, bool tb, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                const float* B, int64_t ldb, float* C, int64_t ldc, cudaStream_t s, int epi, const float* aux,
                int64_t ldaux, const float* B_hi, const float* B_lo) {
    mlp_gemm(c, ta, tb, M, N, K, A, lda, B, ldb, C, ldc, s, epi, aux, ldaux, Split{B_hi, B_lo});
}

int64_t epoch_loss(ntp_ctx* c, const void* in, ntp_dtype tin, int in_blocked, int64_t V_p, int32_t d_s, int32_t C,
                   const int32_t* y, const uint8_t* mask, int64_t row0, int64_t n, void* out, ntp_dtype tout,
                   int out_blocked, const float* gscale, double* part, int64_t* cnt, int64_t ld_plain, cudaStream_t s) {
    NTP_CHECK(tin == tout, NTP_ERR_CONFIG, "loss kernel: input and gradient storage must match");
    if (tin == NTP_F32)
        return launch_softmax_xent(c, (const float*)in, in_blocked, V_p, d_s, C, y, mask, row0, n, (float*)out,
                                   out_blocked, gscale, part, cnt, ld_plain, s);
    return launch_softmax_xent(c, (const __nv_bfloat16*)in, in_blocked, V_p, d_s, C, y, mask, row0, n,
                               (__nv_bfloat16*)out, out_blocked, gscale, part, cnt, ld_plain, s);
}

void epoch_zero_pad_cols(ntp_ctx* c, void* buf, ntp_dtype dt, int64_t V_p, int32_t d_s, int32_t P, int32_t C,
                         cudaStream_t s) {
    if (P * d_s <= C) return;
    if (dt == NTP_F32)
        zero_pad_cols_kernel<float><<<eblocks(V_p * (P * d_s - C)), 256, 0, s>>>((float*)buf, V_p, d_s, P, C, nullptr, 0);
    else
        zero_pad_cols_kernel<__nv_bfloat16><<<eblocks(V_p * (P * d_s - C)), 256, 0, s>>>((__nv_bfloat16*)buf, V_p, d_s,
                                                                                        P, C, nullptr, 0);
    NTP_LAUNCH_CHECK();
    count_launch(c);
}

void epoch_reduce_loss(ntp_ctx* c, const double* part, const int64_t* cnt, int64_t nb, double* scal, cudaStream_t s) {
    reduce_partials_kernel<<<1, 256, 0, s>>>(part, cnt, nb, scal);
    NTP_LAUNCH_CHECK();
    count_launch(c);
}

void epoch_sgd(ntp_ctx* c, float* W, int64_t n, const float* dW, const double* scal, float lr, cudaStream_t s) {
    sgd_kernel<<<eblocks(n), 256, 0, s>>>(W, n, nullptr, 0, dW, scal, lr);
    NTP_LAUNCH_CHECK();
    count_launch(c);
}

// Propagate K hops on this rank's feature slice (a.Z = output slice [V_pad x d_s])
// and gather the result into `recv` ([P][V_p][d_s], block p = rank p's columns of
// my rows).  overlap == false: all hops, then one block exchange on `s`.
// overlap == true (a12, Fig. 7(c)): hops 1..K-1, then the last hop chunk by
// chunk -- peer blocks in the rotated order rank+1, rank+2, ..., rank (own block
// last), each split into `chunks` row ranges -- and every finished chunk is sent to
// its owner on the comm stream while the next chunk computes.  At step s rank r
// sends block (r+s)%P and receives from (r-s)%P, so each step is a permutation and
// all ranks issue the same NCCL sequence.  Arithmetic is unchanged.
static void propagate_and_gather(ntp_ctx* c, const PropArgs& a, void* recv, bool overlap, int chunks, int64_t V_p,
                                 int32_t d_s, bool timed, cudaStream_t s, cudaEvent_t mid = nullptr) {
    const int P = c->world;
    const size_t es = esize(a.dtype);
    const int64_t n = c->g.n;
    const int64_t V_pad = (int64_t)P * V_p;
    if (V_pad > n)   // padding rows of the slice travel to the last owner: keep them zero
        NTP_CUDA(cudaMemsetAsync(static_cast<char*>(a.Z) + n * a.ld_z * es, 0, (V_pad - n) * a.ld_z * es, s));
    if (!overlap || P == 1) {
        propagate(c, a, s, timed, true);
        if (mid) NTP_CUDA(record_timing(c, mid, s));   // hops done, the gather follows
        alltoall_blocks(c, a.Z, recv, V_p * d_s, a.dtype, s);
        return;
    }
    // the chunked gather writes `recv` while later chunks of the last hop still read S^0 -- for the
    // alpha term, and with K == 1 as the gathered state itself: when they are the same buffer, keep
    // S^0 in a copy
    PropArgs ao = a;
    if (recv == a.H && (a.alpha != 0.f || a.K == 1)) {
        const size_t bytes = (size_t)V_pad * a.ld_h * es;
        c->prop_s0.ensure(bytes + 16);
        NTP_CUDA(cudaMemcpyAsync(c->prop_s0.p, a.H, bytes, cudaMemcpyDeviceToDevice, s));
        ao.H = c->prop_s0.p;
    }
    LastHop lh;
    propagate(c, ao, s, timed, true, &lh);
    if (mid) NTP_CUDA(record_timing(c, mid, s));   // overlap: the "gather" phase holds the chunked last hop
    const int64_t csz = cdiv(V_p, std::max(chunks, 1));
    const ncclDataType_t t = a.dtype == NTP_BF16 ? ncclBfloat16 : ncclFloat32;
    char* zf = static_cast<char*>(a.Z);
    char* rv = static_cast<char*>(recv);
    cudaEvent_t ev = c->ev[50];
    for (int st = 1; st <= P; ++st) {
        const int sidx = st % P;
        const int q = (c->rank + sidx) % P;          // block computed and sent
        const int pr = (c->rank - sidx + P) % P;     // block received from
        for (int64_t r = 0; r < V_p; r += csz) {
            const int64_t lo = (int64_t)q * V_p + r;
            const int64_t hi = (int64_t)q * V_p + std::min(r + csz, V_p);
            if (lo < n) run_last_hop(c, lh, lo, std::min(hi, n), s, timed);
            NTP_CUDA(cudaEventRecord(ev, s));
            NTP_CUDA(cudaStreamWaitEvent(c->s_comm, ev, 0));
            const int64_t cnt = (hi - lo) * d_s;
            char* dst = rv + ((int64_t)pr * V_p + r) * d_s * es;
            if (sidx == 0) {
                NTP_CUDA(cudaMemcpyAsync(dst, zf + lo * d_s * es, cnt * es, cudaMemcpyDeviceToDevice, c->s_comm));
            } else {
                NTP_NCCL(ncclGroupStart());
                NTP_NCCL(ncclSend(zf + lo * d_s * es, cnt, t, q, c->comm, c->s_comm));
                NTP_NCCL(ncclRecv(dst, cnt, t, pr, c->comm, c->s_comm));
                NTP_NCCL(ncclGroupEnd());
                wire_add(c, cnt * (int64_t)es, cnt * (int64_t)es);
            }
        }
    }
    NTP_CUDA(cudaEventRecord(c->ev[51], c->s_comm));
    NTP_CUDA(cudaStreamWaitEvent(s, c->ev[51], 0));
}

static void enqueue_epoch_dp(ntp_ctx* c, const ntp_model* m, const float* X, int64_t ldx, const int32_t* lab,
                             const uint8_t* msk, float* W0u, float* W1u, const float* W0g, int64_t ldw0,
                             const float* W1g, int64_t ldw1, Split W0s, Split W1s, bool timed);

// Rows per vertex-side chunk of the W1-after-propagation epoch: NTP_HEAD_CHUNK, else the model's chunk count
// (the a12 schedule's chunks), capped at 2^23 rows; V_p (one chunk) otherwise.
int64_t epoch_row_chunk(const ntp_model* m, int64_t V_p) {
    if (!(m->flags & NTP_M_W1_AFTER_PROP) || V_p <= 0) return std::max<int64_t>(V_p, 1);
    const char* hce = getenv("NTP_HEAD_CHUNK");   // read per call (tests vary it)
    const int64_t head_chunk_env = hce ? atoll(hce) : 0;
    const int64_t hc_def = m->chunks > 1 ? std::min<int64_t>(cdiv(V_p, m->chunks), (int64_t)1 << 23) : (int64_t)1 << 23;
    return std::max<int64_t>(1, std::min<int64_t>(V_p, head_chunk_env > 0 ? head_chunk_env : hc_def));
}

// Overlap trace (ntp_set_trace): a timed event on `st` (its index), or -1 when tracing is off / full.
static int trace_mark(ntp_ctx* c, cudaStream_t st) {
    if (!c->trace_on || c->tr_used >= kTrEvents) return -1;
    const int i = c->tr_used++;
    NTP_CUDA(cudaEventRecord(c->tr_ev[i], st));
    return i;
}
static void trace_add(ntp_ctx* c, int stream, int phase, int chunk, int e0, int e1) {
    if (e0 >= 0 && e1 >= 0) c->tr_recs.push_back({stream, phase, chunk, e0, e1});
}

// Enqueues one epoch (everything between events E0 and E9) on c->s_comp; capturable.
static void enqueue_epoch(ntp_ctx* c, const ntp_model* m, const ntp_tensor* X_v, const int32_t* labels_v,
                          const uint8_t* mask_v, ntp_tensor* W0, ntp_tensor* W1, bool timed) {
    const Graph& g = c->g;
    cudaStream_t s = c->s_comp;
    c->tr_used = 0;   // overlap trace of this epoch (ntp_set_trace)
    c->tr_recs.clear();
    // P feature slices over `world` ranks, vs = P / world per rank (virtual slices, processed in sequence).
    // V_pad = P * ceil(n / P); this rank's vertex rows are the contiguous V_p = V_pad / world = vs * ceil(n/P)
    // rows from row0, and every blocked buffer is [P][V_p][d_s] (block q = slice q of these rows).
    const int32_t P = nslices(c);
    const int32_t vs = c->vs;
    const int64_t n = g.n;
    const int64_t V_pad = (int64_t)P * cdiv(n, P);
    const int64_t V_p = V_pad / c->world;
    const int64_t row0 = (int64_t)c->rank * V_p;
    const bool after = (m->flags & NTP_M_W1_AFTER_PROP) != 0;
    const int32_t w = after ? m->hid : m->C;
    const int32_t d_s = slice_width(w, P, m->dtype, c->slice_align);
    const ntp_dtype dt = m->dtype;
    const size_t es = esize(dt);
    const int64_t feat_elems = (int64_t)vs * V_pad * d_s;   // this rank's slices [vs][V_pad][d_s]
    auto slice_at = [&](void* base, int j) -> void* { return static_cast<char*>(base) + (size_t)j * V_pad * d_s * es; };

    cudaEvent_t* E = c->ev;
    int ei = 0;
    wire_reset(c);
    NTP_CUDA(record_timing(c, E[ei++], s));   // E0 start (input staging counts as mlp_fwd)

    // ---- inputs (e2e: copy host inputs in).  GEMM operands need 16-byte row pitch (TMA).
    const int64_t ldXp = round4(m->d_in), ldH = round4(m->hid), ldL = round4(std::max(m->C, m->hid));
    const int64_t ldC1 = round4(m->C);
    const float* X = static_cast<const float*>(X_v->data);
    int64_t ldx = X_v->ld;
    const int32_t* lab = labels_v;
    const uint8_t* msk = mask_v;
    if (m->flags & NTP_M_STAGED) {
        // inputs staged by ntp_stage_inputs (copy stream); this epoch waits for that copy
        const int slot = (int)((m->flags >> NTP_M_SLOT_SHIFT) & NTP_M_SLOT_MASK);
        NTP_CHECK(c->st_rows[slot] == V_p && c->st_d_in[slot] == m->d_in, NTP_ERR_STATE,
                  "staging slot %d holds no inputs of this shape", slot);
        NTP_CUDA(cudaStreamWaitEvent(s, c->st_ready[slot], c->capturing ? cudaEventWaitExternal : 0));
        X = c->st_X[slot].as<float>();
        ldx = c->st_ld[slot];
        lab = c->st_y[slot].as<int32_t>();
        msk = c->st_m[slot].as<uint8_t>();
    } else if (m->flags & NTP_M_HOST_INPUTS) {
        c->m_Xs.ensure((size_t)V_p * ldXp * sizeof(float));
        c->m_lab.ensure((size_t)V_p * sizeof(int32_t));
        c->m_mask.ensure((size_t)V_p);
        if (ldx == ldXp) {
            NTP_CUDA(cudaMemcpyAsync(c->m_Xs.p, X_v->data, (size_t)V_p * ldx * sizeof(float), cudaMemcpyHostToDevice, s));
        } else {
            // one contiguous DMA in the host pitch (a 2-D host copy with ~2 KB rows runs at a third of
            // the link rate), then the 16-byte GEMM pitch on the device
            c->m_Xh.ensure((size_t)V_p * ldx * sizeof(float));
            NTP_CUDA(cudaMemcpyAsync(c->m_Xh.p, X_v->data, (size_t)V_p * ldx * sizeof(float), cudaMemcpyHostToDevice, s));
            NTP_CUDA(cudaMemcpy2DAsync(c->m_Xs.p, ldXp * sizeof(float), c->m_Xh.p, ldx * sizeof(float),
                                       m->d_in * sizeof(float), V_p, cudaMemcpyDeviceToDevice, s));
        }
        NTP_CUDA(cudaMemcpyAsync(c->m_lab.p, labels_v, V_p * sizeof(int32_t), cudaMemcpyHostToDevice, s));
        NTP_CUDA(cudaMemcpyAsync(c->m_mask.p, mask_v, V_p, cudaMemcpyHostToDevice, s));
        X = c->m_Xs.as<float>();
        ldx = ldXp;
        lab = c->m_lab.as<int32_t>();
        msk = c->m_mask.as<uint8_t>();
    } else if (m->flags & NTP_M_HOST_STREAM) {
        // X stays in host memory: the row-chunk loops below stream it through c->hs_ring
    } else if ((ldx % 4) != 0 || (reinterpret_cast<uintptr_t>(X) % 16) != 0) {
        c->m_Xs.ensure((size_t)V_p * ldXp * sizeof(float));
        NTP_CUDA(cudaMemcpy2DAsync(c->m_Xs.p, ldXp * sizeof(float), X, ldx * sizeof(float), m->d_in * sizeof(float),
                                   V_p, cudaMemcpyDeviceToDevice, s));
        X = c->m_Xs.as<float>();
        ldx = ldXp;
    }
    float* W0u = static_cast<float*>(W0->data);   // updated in place by SGD
    float* W1u = static_cast<float*>(W1->data);
    const float* W0g = W0u;                       // GEMM views (16-byte pitch)
    int64_t ldw0 = m->hid;
    if ((m->hid % 4) != 0 || (reinterpret_cast<uintptr_t>(W0u) % 16) != 0) {
        c->m_W0p.ensure((size_t)m->d_in * ldH * sizeof(float));
        NTP_CUDA(cudaMemcpy2DAsync(c->m_W0p.p, ldH * sizeof(float), W0u, m->hid * sizeof(float),
                                   m->hid * sizeof(float), m->d_in, cudaMemcpyDeviceToDevice, s));
        W0g = c->m_W0p.as<float>();
        ldw0 = ldH;
    }
    const float* W1g = W1u;
    int64_t ldw1 = m->C;
    if ((m->C % 4) != 0 || (reinterpret_cast<uintptr_t>(W1u) % 16) != 0) {
        c->m_W1p.ensure((size_t)m->hid * ldC1 * sizeof(float));
        NTP_CUDA(cudaMemcpy2DAsync(c->m_W1p.p, ldC1 * sizeof(float), W1u, m->C * sizeof(float), m->C * sizeof(float),
                                   m->hid, cudaMemcpyDeviceToDevice, s));
        W1g = c->m_W1p.as<float>();
        ldw1 = ldC1;
    }

    // weights split once per epoch into {rn_tf32(W), rn_tf32(W - hi)} for the tensor-core GEMMs
    c->m_Wsplit.ensure((size_t)2 * ((int64_t)m->d_in * ldw0 + (int64_t)m->hid * ldw1) * sizeof(float));
    Split W0s, W1s;
    {
        float* w = c->m_Wsplit.as<float>();
        float* w0h = w;
        float* w0l = w0h + (int64_t)m->d_in * ldw0;
        float* w1h = w0l + (int64_t)m->d_in * ldw0;
        float* w1l = w1h + (int64_t)m->hid * ldw1;
        tf32_split(c, W0g, m->d_in, m->hid, ldw0, w0h, w0l, s);
        tf32_split(c, W1g, m->hid, m->C, ldw1, w1h, w1l, s);
        W0s = Split{w0h, w0l};
        W1s = Split{w1h, w1l};
    }

    if (m->flags & NTP_M_DATA_PARALLEL) {   // NEXT-4 baseline: full-width rows, all-gather before each hop
        NTP_CHECK(!after && !(m->flags & (NTP_M_OVERLAP | NTP_M_P2P_LAYOUTS)) && !g.reordered, NTP_ERR_CONFIG,
                  "NTP_M_DATA_PARALLEL: W1 before propagation, NCCL layouts, original vertex order only");
        c->hop_ev_used = 0;
        enqueue_epoch_dp(c, m, X, ldx, lab, msk, W0u, W1u, W0g, ldw0, W1g, ldw1, W0s, W1s, timed);
        return;
    }

    // ---- scratch.  One GPU (P = 1): the layout changes are identities, so the producers write the
    // feature slice directly and the hops ping-pong between two slices (propagate_consume) -- no
    // exchange copies, no send buffer, no scratch slice.  W1 after propagation (R3, papers shape):
    // the vertex-side work runs in row chunks of `hc` rows (H1, logits, gradients chunk-sized; the
    // ReLU' mask kept as bits) so the epoch's footprint is the slices plus X (memory-lean plan).
    const bool local = (c->world == 1);
    const int64_t hc = epoch_row_chunk(m, V_p);
    const int64_t nch = cdiv(V_p, hc);
    // NTP_M_HOST_STREAM (memory-efficient scheduling: inputs stay in host memory): every row chunk of
    // X is copied into one slot of a 2-slot device ring on the copy stream right before the kernel that reads
    // it; the copy of chunk ch+1 waits only for the slot's previous reader (chunk ch-1), so it runs under the
    // GEMM of chunk ch.  X_v is read twice per epoch (MLP forward, dW0).
    const bool hstream = (m->flags & NTP_M_HOST_STREAM) != 0;
    if (hstream) c->hs_ring.ensure((size_t)2 * hc * ldXp * sizeof(float) + 16);
    int hs_next = 0;
    auto x_rows = [&](int64_t r, int64_t h, int& slot) -> const float* {
        if (!hstream) {
            slot = -1;
            return X + r * ldx;
        }
        slot = hs_next;
        hs_next ^= 1;
        float* dst = c->hs_ring.as<float>() + (size_t)slot * hc * ldXp;
        if (c->hs_used[slot]) NTP_CUDA(cudaStreamWaitEvent(c->s_copy, c->hs_free[slot], 0));
        if (ldx == ldXp)
            NTP_CUDA(cudaMemcpyAsync(dst, X + r * ldx, (size_t)h * ldx * sizeof(float), cudaMemcpyHostToDevice, c->s_copy));
        else
            NTP_CUDA(cudaMemcpy2DAsync(dst, ldXp * sizeof(float), X + r * ldx, ldx * sizeof(float), m->d_in * sizeof(float),
                                       h, cudaMemcpyHostToDevice, c->s_copy));
        NTP_CUDA(cudaEventRecord(c->hs_ready[slot], c->s_copy));
        NTP_CUDA(cudaStreamWaitEvent(s, c->hs_ready[slot], 0));
        return dst;
    };
    auto x_done = [&](int slot) {
        if (slot < 0) return;
        NTP_CUDA(cudaEventRecord(c->hs_free[slot], s));
        c->hs_used[slot] = true;
    };
    const int64_t ldxc = hstream ? ldXp : ldx;      // row pitch of a chunk as the kernels see it
    const int32_t nwb = (m->hid + 31) / 32;          // mask words per row
    const int64_t rowsH = after ? hc : V_p;
    c->m_H1.ensure((size_t)rowsH * ldH * sizeof(float));
    c->m_L.ensure((size_t)rowsH * ldL * sizeof(float));
    c->m_dL.ensure((size_t)rowsH * ldL * sizeof(float));
    c->m_dH1.ensure((size_t)rowsH * ldH * sizeof(float));
    if (after) c->m_bits.ensure((size_t)V_p * nwb * sizeof(uint32_t) + 16);
    const int64_t n_w = (int64_t)m->d_in * m->hid + (int64_t)m->hid * m->C;
    c->m_dW.ensure((size_t)n_w * sizeof(float));
    if (nch > 1) c->m_dWp.ensure((size_t)nch * n_w * sizeof(float));
    c->m_scal.ensure(4 * sizeof(double));
    if (!local) c->send.ensure((size_t)feat_elems * es + 16);
    c->recv.ensure((size_t)feat_elems * es + 16);
    c->xfer.ensure((size_t)feat_elems * es + 16);     // propagation output (feature slice)
    const int64_t loss_blocks = std::min<int64_t>(cdiv(V_p, 8), 148 * 8) * nch;   // loss-kernel grid bound per chunk
    c->m_part.ensure((size_t)loss_blocks * (sizeof(double) + sizeof(int64_t)) + 16);
    double* part = c->m_part.as<double>();
    int64_t* cnt = reinterpret_cast<int64_t*>(part + loss_blocks);
    float* H1 = c->m_H1.as<float>();
    float* L = c->m_L.as<float>();
    float* dL = c->m_dL.as<float>();
    float* dH1 = c->m_dH1.as<float>();
    uint32_t* bits = after ? c->m_bits.as<uint32_t>() : nullptr;
    float* dW0 = c->m_dW.as<float>();
    float* dW1 = dW0 + (int64_t)m->d_in * m->hid;
    double* scal = c->m_scal.as<double>();
    // chunk ch's weight-gradient partials (dW0 | dW1), summed in chunk order afterwards
    auto dw0_at = [&](int64_t ch) { return nch > 1 ? c->m_dWp.as<float>() + ch * n_w : dW0; };
    auto dw1_at = [&](int64_t ch) { return dw0_at(ch) + (int64_t)m->d_in * m->hid; };

    // Peer-direct layouts (NTP_M_P2P_LAYOUTS, P > 1, CUDA IPC available): the producers store into
    // the owners' windows and a barrier replaces each all-to-all; otherwise the NCCL block exchange.
    const bool overlap = (m->flags & NTP_M_OVERLAP) != 0;
    const size_t win = (size_t)feat_elems * es;
    const bool p2p = !local && !overlap && (m->flags & NTP_M_P2P_LAYOUTS) && p2p_ensure(c, win, win, s);
    // copy-engine layout changes (a12 with NTP_M_OVERLAP | NTP_M_P2P_LAYOUTS, W1 after propagation): every
    // row chunk of every layout change is one cudaMemcpyAsync per peer straight into the owner's IPC window on
    // the comm stream -- copy engines over NVLink, no SMs -- followed by a flag write into the owner's inbox
    // (cuStreamWriteValue32, fenced); consumers wait on their inbox (cuStreamWaitValue32).  Eager epochs only.
    const bool ce = !local && overlap && after && (m->flags & NTP_M_P2P_LAYOUTS) && vs == 1 && !c->capturing &&
                    nch <= kCeChunks && c->world <= kCeRanks && p2p_ensure(c, win, win, s);
    if (ce) ++c->ce_seq;
    const uint32_t seq = c->ce_seq;
    void* const* tab_split = p2p ? c->p2p_tab.as<void*>() : nullptr;
    void* const* tab_gath = p2p ? c->p2p_tab.as<void*>() + P : nullptr;
    // Rows [n, V_pad) of every buffer that serves as a feature slice are padding: no hop writes them,
    // and every consumer multiplies them by zero (dl = 0, X = 0, mask bits 0) -- so they must hold
    // zeros, not stale bytes of an earlier allocation (a bf16 view of old fp32 data can be NaN, and
    // 0 * NaN = NaN in dW1).  Cleared every epoch (< P rows per slice).
    if (V_pad > n) {
        const size_t off = (size_t)n * d_s * es, len = (size_t)(V_pad - n) * d_s * es;
        for (int j = 0; j < vs; ++j)
            for (void* b : {c->recv.p, c->xfer.p, local ? nullptr : c->send.p})
                if (b) NTP_CUDA(cudaMemsetAsync(static_cast<char*>(slice_at(b, j)) + off, 0, len, s));
        if (p2p || ce)
            for (void* b : {c->p2p_split.p, c->p2p_gath.p})
                NTP_CUDA(cudaMemsetAsync(static_cast<char*>(b) + off, 0, len, s));
    }
    // a12 for the W1-after-propagation epoch (P > 1, NCCL layouts): every layout change runs per row chunk
    // on the comm stream -- split chunk ch while the MLP computes chunk ch+1, gather chunk ch while the head
    // consumes chunk ch-1, gradient split behind the head, backward gather ahead of the MLP backward --
    // with the same arithmetic (chunks are the same with and without the overlap).
    const bool ovl = overlap && after && !local && !p2p;   // (ce: the same chunk schedule, copy-engine transfers)
    int ovi = 0;                                   // next free overlap event
    auto ov_event = [&]() -> cudaEvent_t {
        NTP_CHECK(ovi < kOvEvents, NTP_ERR_CONFIG, "too many overlap chunks (%d events)", kOvEvents);
        return c->ov_ev[ovi++];
    };
    // rows [r, r+h) of every block: block q of `src` -> rank q; rank q's block `rank` -> block q of `dst`
    auto exchange_rows = [&](const void* src, void* dst, int64_t r, int64_t h, cudaStream_t st) {
        const ncclDataType_t t = dt == NTP_BF16 ? ncclBfloat16 : ncclFloat32;
        const size_t cnt = (size_t)h * d_s;
        NTP_NCCL(ncclGroupStart());
        for (int q = 0; q < P; ++q) {
            const size_t off = ((size_t)q * V_p + r) * d_s * es;
            if (q == c->rank) {
                NTP_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, cnt * es,
                                         cudaMemcpyDeviceToDevice, st));
                continue;
            }
            NTP_NCCL(ncclSend(static_cast<const char*>(src) + off, cnt, t, q, c->comm, st));
            NTP_NCCL(ncclRecv(static_cast<char*>(dst) + off, cnt, t, q, c->comm, st));
            wire_add(c, (int64_t)(cnt * es), (int64_t)(cnt * es));
        }
        NTP_NCCL(ncclGroupEnd());
    };
    // copy-engine variant of exchange_rows: rows [r, r+h) of block q of `src` -> block `rank` of rank q's
    // window (split windows for phases 0 / 2, gather windows for 1 / 3), then flag (phase, rank, ch) := seq
    // in every peer's inbox
    auto ce_rows = [&](const void* src, int phase, int64_t r, int64_t h, int ch, cudaStream_t st) {
        const std::vector<void*>& dst = (phase == 0 || phase == 2) ? c->p2p_peer_split : c->p2p_peer_gath;
        const size_t bytes = (size_t)h * d_s * es;
        for (int k = 1; k <= P; ++k) {   // peers first (rotated, so ranks do not all target the same peer), own last
            const int q = (c->rank + k) % P;
            NTP_CUDA(cudaMemcpyAsync(static_cast<char*>(dst[q]) + ((size_t)c->rank * V_p + r) * d_s * es,
                                     static_cast<const char*>(src) + ((size_t)q * V_p + r) * d_s * es, bytes,
                                     cudaMemcpyDeviceToDevice, st));
            if (q != c->rank) wire_add(c, (int64_t)bytes, (int64_t)bytes);
        }
        for (int q = 0; q < P; ++q)
            if (q != c->rank) stream_write_u32(st, ce_flags(c, q) + ce_flag_slot(phase, c->rank, ch), seq);
    };
    // this rank's chunk ch of `phase` has landed: own block (event) and every peer's (inbox flags)
    auto ce_wait = [&](cudaEvent_t own, int phase, int ch) {
        NTP_CUDA(cudaStreamWaitEvent(s, own, 0));
        for (int q = 0; q < P; ++q)
            if (q != c->rank) stream_wait_u32_geq(s, ce_flags(c, c->rank) + ce_flag_slot(phase, q, ch), seq);
    };
    int ce_phase = 0, ce_ch = 0;   // phase / chunk of the next async_exchange (copy-engine mode)
    int tr_ch[4] = {0, 0, 0, 0};   // trace: chunks exchanged per phase
    // comm stream: after `s` reaches this point, exchange rows [r, r+h); returns the completion event
    auto async_exchange = [&](const void* src, void* dst, int64_t r, int64_t h) -> cudaEvent_t {
        cudaEvent_t a = ov_event(), b = ov_event();
        NTP_CUDA(cudaEventRecord(a, s));
        NTP_CUDA(cudaStreamWaitEvent(c->s_comm, a, 0));
        const int t0 = trace_mark(c, c->s_comm);
        if (ce) ce_rows(src, ce_phase, r, h, ce_ch++, c->s_comm);
        else exchange_rows(src, dst, r, h, c->s_comm);
        trace_add(c, 1, ce_phase, tr_ch[ce_phase]++, t0, trace_mark(c, c->s_comm));
        NTP_CUDA(cudaEventRecord(b, c->s_comm));
        return b;
    };
    // consumer side of chunk ch (NCCL: the comm stream's event; copy engines: plus the peers' flags)
    auto wait_chunk = [&](cudaEvent_t ev, int phase, int ch) {
        if (ce) ce_wait(ev, phase, ch);
        else NTP_CUDA(cudaStreamWaitEvent(s, ev, 0));
    };
    void* slice_in = (p2p || ce) ? c->p2p_split.p : c->recv.p;   // this rank's feature slice after a split
    void* split_dst = p2p ? nullptr : (local ? c->recv.p : c->send.p);   // where the split's producer writes

    // one GPU on a reordered graph: producers that can scatter write S^0 / the gradient straight into the
    // internal vertex order, so the hops skip the permutation pass (propagate_consume input_internal)
    const int32_t* perm_local = (local && g.reordered && m->alpha == 0.f) ? g.perm.as<int32_t>() : nullptr;
    bool fwd_internal = false, bwd_internal = false;

    // a2 (+ a3's pack): MLP forward (ReLU fused into the GEMM epilogue)
    const float* prop_src = H1;             // rows propagated (w columns)
    int64_t ld_src = ldH;
    if (!after) {
        mlp_gemm(c, false, false, V_p, m->hid, m->d_in, X, ldx, W0g, ldw0, H1, ldH, s, /*relu*/ 1, nullptr, 0, W0s);
        mlp_gemm(c, false, false, V_p, m->C, m->hid, H1, ldH, W1g, ldw1, L, ldL, s, 0, nullptr, 0, W1s);
        prop_src = L;
        ld_src = ldL;
        NTP_CUDA(record_timing(c, E[ei++], s));   // E1 mlp_fwd done
        pack_v2f(c, prop_src, ld_src, w, split_dst, V_p, d_s, P, g.dinv_out_orig(), row0, n, NTP_F32, dt, s, tab_split);
    } else {
        cudaEvent_t last = nullptr;
        // bf16 slice, no padding columns: the split's pack runs in the GEMM epilogue (gemm_tf32x3_pack)
        const char* pfe = getenv("NTP_PACK_FUSED");
        const bool fuse_pack = !(pfe && atoi(pfe) == 0) && dt == NTP_BF16 &&
                               (int64_t)P * d_s == m->hid && m->hid % 32 == 0 && d_s % 8 == 0 && !p2p;
        for (int64_t r = 0; r < V_p; r += hc) {      // H1 chunk -> pre-scaled slice rows + ReLU' bits
            const int64_t h = std::min(hc, V_p - r);
            const int t0 = ovl ? trace_mark(c, s) : -1;
            int slot;
            const float* Xc = x_rows(r, h, slot);
            if (fuse_pack) {
                const PackEpi pk{static_cast<__nv_bfloat16*>(split_dst), V_p, d_s, g.dinv_out_orig(), row0, n, bits,
                                 nwb, r, perm_local};
                fwd_internal = perm_local != nullptr;
                gemm_tf32x3_pack(c, h, m->hid, m->d_in, Xc, ldxc, W0s.hi, W0s.lo, ldw0, pk, s);
            } else {
                mlp_gemm(c, false, false, h, m->hid, m->d_in, Xc, ldxc, W0g, ldw0, H1, ldH, s, 1, nullptr, 0, W0s);
                pack_v2f(c, H1, ldH, w, split_dst, V_p, d_s, P, g.dinv_out_orig(), row0, n, NTP_F32, dt, s, tab_split,
                         h, r, bits, nwb);
            }
            x_done(slot);
            if (ovl) trace_add(c, 0, 0, (int)(r / hc), t0, trace_mark(c, s));
            if (ovl) last = async_exchange(c->send.p, c->recv.p, r, h);   // a3 of chunk ch under a2 of ch+1
        }
        if (ovl) wait_chunk(last, 0, (int)nch - 1);   // every chunk (a peer's copies land in stream order)
        NTP_CUDA(record_timing(c, E[ei++], s));   // E1 mlp_fwd (+ pack) done
    }

    // peer-direct layout change: the producer stored (P-1) blocks of V_p x d_s into the peers' windows
    const int64_t p2p_wire = (int64_t)(P - 1) * V_p * d_s * (int64_t)es;
    // a3: split (pre-scaled by the forward column side D~_out^{-1/2})
    if (p2p) p2p_barrier(c, s), wire_add(c, p2p_wire, p2p_wire);
    else if (!local && !ovl) exchange_v2f(c, c->send.p, c->recv.p, V_p * d_s, dt, s);
    NTP_CUDA(record_timing(c, E[ei++], s));   // E2 v2f done

    // a4 + a5: K forward hops on S^0 (pre-scaled) -> Z^K, gathered into this rank's rows
    c->hop_ev_used = 0;
    c->wire_phase = 1;
    void* gathered = (p2p || ce) ? c->p2p_gath.p : c->recv.p;
    {
        PropArgs a{};
        a.H = slice_in;
        a.Z = c->xfer.p;
        a.ld_h = d_s;
        a.ld_z = d_s;
        a.cols = d_s;
        a.dtype = dt;
        a.K = m->K;
        a.gamma = m->gamma;
        a.alpha = m->alpha;
        a.transposed = false;
        if (local) {   // slice j of recv -> slice j of recv / xfer (the same buffer for every slice)
            for (int j = 0; j < vs; ++j) {
                PropArgs aj = a;
                aj.H = slice_at(c->recv.p, j);
                aj.Z = slice_at(c->xfer.p, j);
                gathered = propagate_consume(c, aj, s, timed, fwd_internal) == aj.H ? c->recv.p : c->xfer.p;
            }
            NTP_CUDA(record_timing(c, E[10], s));   // one GPU: the gather is the identity
        } else if (vs > 1) {   // every slice in sequence, then one gather
            for (int j = 0; j < vs; ++j) {
                PropArgs aj = a;
                aj.H = slice_at(slice_in, j);
                aj.Z = slice_at(c->xfer.p, j);
                propagate(c, aj, s, timed, true);
            }
            NTP_CUDA(record_timing(c, E[10], s));
            exchange_f2v(c, c->xfer.p, c->recv.p, V_p * d_s, dt, s);
        } else if (p2p) {
            a.po = PeerOut{tab_gath, V_p, c->rank};
            propagate(c, a, s, timed, true);
            NTP_CUDA(record_timing(c, E[10], s));   // stores done by the last hop; the barrier completes them
            p2p_barrier(c, s);
            wire_add(c, p2p_wire, p2p_wire);
        } else if (ovl) {
            const int t0 = trace_mark(c, s);
            propagate(c, a, s, timed, true);     // a5 per chunk below, consumed chunk by chunk by the head
            trace_add(c, 0, 4, -1, t0, trace_mark(c, s));
            NTP_CUDA(record_timing(c, E[10], s));
        } else {
            propagate_and_gather(c, a, c->recv.p, overlap && !after, m->chunks, V_p, d_s, timed, s, E[10]);
        }
    }
    std::vector<cudaEvent_t> g_ev;                 // forward gather of row chunk ch done (ovl)
    ce_phase = 1, ce_ch = 0;
    if (ovl)
        for (int64_t r = 0; r < V_p; r += hc) g_ev.push_back(async_exchange(c->xfer.p, c->recv.p, r, std::min(hc, V_p - r)));
    ce_phase = 2, ce_ch = 0;
    NTP_CUDA(record_timing(c, E[ei++], s));   // E3 prop fwd + f2v done
    // the gradient split's producer target: the send buffer, or on one GPU the slice the forward no
    // longer needs
    void* gsend = local ? (gathered == c->recv.p ? c->xfer.p : c->recv.p) : c->send.p;

    // a6: loss + gradient, written straight into the backward split's send buffer (or windows)
    c->wire_phase = 2;
    const float* gscale_bwd = g.dinv_in_orig();   // backward column side (original vertex order)
    int64_t nb_loss = 0;
    if (!after) {
        if (dt == NTP_F32)
            nb_loss = launch_softmax_xent(c, (const float*)gathered, 1, V_p, d_s, m->C, lab, msk, row0, n,
                                          (float*)gsend, 1, gscale_bwd, part, cnt, 0, s, tab_split);
        else
            nb_loss = launch_softmax_xent(c, (const __nv_bfloat16*)gathered, 1, V_p, d_s, m->C, lab, msk, row0, n,
                                          (__nv_bfloat16*)gsend, 1, gscale_bwd, part, cnt, 0, s, tab_split);
        if (P * d_s > m->C) {
            if (dt == NTP_F32)
                zero_pad_cols_kernel<float><<<eblocks(V_p * (P * d_s - m->C)), 256, 0, s>>>((float*)gsend, V_p, d_s,
                                                                                          P, m->C, tab_split, c->rank);
            else
                zero_pad_cols_kernel<__nv_bfloat16><<<eblocks(V_p * (P * d_s - m->C)), 256, 0, s>>>(
                    (__nv_bfloat16*)gsend, V_p, d_s, P, m->C, tab_split, c->rank);
            NTP_LAUNCH_CHECK();
            count_launch(c);
        }
    } else {
        // per row chunk: Z_v = unpack(gathered) [h x hid]; logits = Z_v W1; dlogits; dW1 += Z_v^T dlogits;
        // dZ_v = dlogits W1^T -> pack into the gradient split
        float* Zv = dH1;   // reuse [hc x ldH]
        cudaEvent_t last = nullptr;
        const bool fused = head_fused_supported(P, d_s, m->hid, m->C, dt);
        for (int64_t r = 0, ch = 0; r < V_p; r += hc, ++ch) {
            const int64_t h = std::min(hc, V_p - r);
            if (ovl) wait_chunk(g_ev[ch], 1, (int)ch);
            const int t0 = ovl ? trace_mark(c, s) : -1;
            if (fused) {
                // one tcgen05 pass over the chunk's rows (head.cu): logits, dl and dZ stay on chip
                nb_loss += head_fused(c, gathered, V_p, d_s, P, m->hid, m->C, W1g, ldw1, lab, msk, row0, n, gscale_bwd,
                                      p2p ? nullptr : gsend, tab_split, dw1_at(ch), part + nb_loss, cnt + nb_loss, s,
                                      r, r + h, perm_local);
                bwd_internal = perm_local != nullptr;
                if (ovl) trace_add(c, 0, 1, (int)ch, t0, trace_mark(c, s));
                if (ovl) last = async_exchange(c->send.p, c->recv.p, r, h);   // a7 of chunk ch
                continue;
            }
            unpack_f2v(c, gathered, V_p, d_s, P, Zv, ldH, m->hid, dt, NTP_F32, s, nullptr, 0, h, r);
            mlp_gemm(c, false, false, h, m->C, m->hid, Zv, ldH, W1g, ldw1, L, ldL, s, 0, nullptr, 0, W1s);
            nb_loss += launch_softmax_xent(c, (const float*)L, 0, h, d_s, m->C, lab + r, msk + r, row0 + r, n, dL, 0,
                                           nullptr, part + nb_loss, cnt + nb_loss, ldL, s);
            mlp_gemm(c, true, false, m->hid, m->C, h, Zv, ldH, dL, ldL, dw1_at(ch), m->C, s);          // dW1 = Z_v^T dlogits
            mlp_gemm(c, false, true, h, m->hid, m->C, dL, ldL, W1g, ldw1, L, ldL, s, 0, nullptr, 0, W1s);  // dZ_v -> L
            pack_v2f(c, L, ldL, m->hid, p2p ? nullptr : gsend, V_p, d_s, P, gscale_bwd, row0, n, NTP_F32, dt, s,
                     tab_split, h, r);
            if (ovl) trace_add(c, 0, 1, (int)ch, t0, trace_mark(c, s));
            if (ovl) last = async_exchange(c->send.p, c->recv.p, r, h);       // a7 of chunk ch
        }
        if (ovl) wait_chunk(last, 2, (int)nch - 1);
    }
    reduce_partials_kernel<<<1, 256, 0, s>>>(part, cnt, nb_loss, scal);
    NTP_LAUNCH_CHECK();
    count_launch(c);
    NTP_CUDA(record_timing(c, E[ei++], s));   // E4 loss done

    // a7: split the gradient
    if (p2p) p2p_barrier(c, s), wire_add(c, p2p_wire, p2p_wire);
    else if (!local && !ovl) exchange_v2f(c, c->send.p, c->recv.p, V_p * d_s, dt, s);
    NTP_CUDA(record_timing(c, E[ei++], s));   // E5 v2f bwd

    // a8 + a9: K backward hops on the split gradient, gathered -> dL^ rows [V_p x w]
    c->wire_phase = 3;
    void* gathered_b = (p2p || ce) ? c->p2p_gath.p : c->send.p;
    {
        PropArgs a{};
        a.H = local ? gsend : slice_in;
        a.Z = local ? (gsend == c->recv.p ? c->xfer.p : c->recv.p) : c->xfer.p;
        a.ld_h = d_s;
        a.ld_z = d_s;
        a.cols = d_s;
        a.dtype = dt;
        a.K = m->K;
        a.gamma = m->gamma;
        a.alpha = m->alpha;
        a.transposed = true;
        if (local) {
            void* hb = const_cast<void*>(a.H);
            void* zb = a.Z;
            for (int j = 0; j < vs; ++j) {
                PropArgs aj = a;
                aj.H = slice_at(hb, j);
                aj.Z = slice_at(zb, j);
                gathered_b = propagate_consume(c, aj, s, timed, bwd_internal) == aj.H ? hb : zb;
            }
            NTP_CUDA(record_timing(c, E[11], s));
        } else if (vs > 1) {
            for (int j = 0; j < vs; ++j) {
                PropArgs aj = a;
                aj.H = slice_at(slice_in, j);
                aj.Z = slice_at(c->xfer.p, j);
                propagate(c, aj, s, timed, true);
            }
            NTP_CUDA(record_timing(c, E[11], s));
            exchange_f2v(c, c->xfer.p, c->send.p, V_p * d_s, dt, s);
        } else if (p2p) {
            a.po = PeerOut{tab_gath, V_p, c->rank};
            propagate(c, a, s, timed, true);
            NTP_CUDA(record_timing(c, E[11], s));
            p2p_barrier(c, s);
            wire_add(c, p2p_wire, p2p_wire);
        } else if (ovl) {
            const int t0 = trace_mark(c, s);
            propagate(c, a, s, timed, true);     // a9 per chunk below, consumed chunk by chunk by a10
            trace_add(c, 0, 5, -1, t0, trace_mark(c, s));
            NTP_CUDA(record_timing(c, E[11], s));
        } else {
            propagate_and_gather(c, a, c->send.p, overlap && !after, m->chunks, V_p, d_s, timed, s, E[11]);
        }
    }
    std::vector<cudaEvent_t> b_ev;                 // backward gather of row chunk ch done (ovl)
    ce_phase = 3, ce_ch = 0;
    if (ovl)
        for (int64_t r = 0; r < V_p; r += hc) b_ev.push_back(async_exchange(c->xfer.p, c->send.p, r, std::min(hc, V_p - r)));
    if (!after) unpack_f2v(c, gathered_b, V_p, d_s, P, dL, ldL, w, dt, NTP_F32, s);
    NTP_CUDA(record_timing(c, E[ei++], s));   // E6 prop bwd + f2v bwd

    // a10: MLP backward (ReLU' mask fused into the dH1 GEMM epilogue, or into the unpack from bits)
    if (!after) {
        mlp_gemm(c, true, false, m->hid, m->C, V_p, H1, ldH, dL, ldL, dW1, m->C, s);              // dW1 = H1^T dL^
        mlp_gemm(c, false, true, V_p, m->hid, m->C, dL, ldL, W1g, ldw1, dH1, ldH, s, 2, H1, ldH, W1s);  // dH1
        mlp_gemm(c, true, false, m->d_in, m->hid, V_p, X, ldx, dH1, ldH, dW0, m->hid, s);            // dW0 = X^T dH1
    } else {
        for (int64_t r = 0, ch = 0; r < V_p; r += hc, ++ch) {
            const int64_t h = std::min(hc, V_p - r);
            if (ovl) wait_chunk(b_ev[ch], 3, (int)ch);
            const int t0 = ovl ? trace_mark(c, s) : -1;
            if (!hstream && wgrad_fused_supported(P, d_s, m->d_in, m->hid, dt)) {   // unpack + dW0 GEMM in one kernel
                wgrad_fused(c, X, ldx, V_p, m->d_in, gathered_b, d_s, P, m->hid, bits, nwb, r, r + h, dw0_at(ch), s);
                if (ovl) trace_add(c, 0, 3, (int)ch, t0, trace_mark(c, s));
                continue;
            }
            unpack_f2v(c, gathered_b, V_p, d_s, P, dH1, ldH, w, dt, NTP_F32, s, nullptr, 0, h, r, bits, nwb);
            int slot;
            const float* Xc = x_rows(r, h, slot);
            mlp_gemm(c, true, false, m->d_in, m->hid, h, Xc, ldxc, dH1, ldH, dw0_at(ch), m->hid, s);
            x_done(slot);
            if (ovl) trace_add(c, 0, 3, (int)ch, t0, trace_mark(c, s));
        }
        if (nch > 1) {
            sum_chunks_kernel<<<eblocks(n_w), 256, 0, s>>>(c->m_dWp.as<float>(), nch, n_w, dW0);
            NTP_LAUNCH_CHECK();
            count_launch(c);
        }
    }
    NTP_CUDA(record_timing(c, E[ei++], s));   // E7 mlp bwd

    // a11: allreduce (sync_and_update)
    if (!local) {
        NTP_NCCL(ncclGroupStart());
        NTP_NCCL(ncclAllReduce(dW0, dW0, n_w, ncclFloat32, ncclSum, c->comm, s));
        NTP_NCCL(ncclAllReduce(scal, scal, 2, ncclFloat64, ncclSum, c->comm, s));
        NTP_NCCL(ncclGroupEnd());
    }
    NTP_CUDA(record_timing(c, E[ei++], s));   // E8 allreduce
    sgd_kernel<<<eblocks(n_w), 256, 0, s>>>(W0u, (int64_t)m->d_in * m->hid, W1u, (int64_t)m->hid * m->C, dW0, scal,
                                            m->lr);
    NTP_LAUNCH_CHECK();
    count_launch(c);
    if (m->flags & NTP_M_STAGED) {   // the slot may be refilled once this epoch is done with it
        const int slot = (int)((m->flags >> NTP_M_SLOT_SHIFT) & NTP_M_SLOT_MASK);
        NTP_CUDA(cudaEventRecordWithFlags(c->st_free[slot], s, c->capturing ? cudaEventRecordExternal : cudaEventRecordDefault));
        c->st_free_rec[slot] = true;
    }
    NTP_CUDA(record_timing(c, E[ei++], s));   // E9 sgd
}

namespace {
bool graphs_enabled() {
    static const bool v = [] { const char* e = getenv("NTP_GRAPH"); return e ? atoi(e) != 0 : true; }();
    return v;
}
}  // namespace

void drop_epoch_graph(ntp_ctx* c) {
    if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
    c->graph_exec = nullptr;
    c->graph_valid = false;
    for (int i = 0; i < NTP_STAGE_SLOTS; ++i) {
        if (c->sg_exec[i]) cudaGraphExecDestroy(c->sg_exec[i]);
        c->sg_exec[i] = nullptr;
        c->sg_valid[i] = false;
    }
}

// One epoch.  The enqueue sequence is captured into a CUDA graph on the second call with the same
// key (model + every pointer it bakes in) and replayed afterwards: one launch instead of ~60, so
// the GPU does not idle while the host re-issues the epoch.  Any eager call invalidates the graph
// (it may have grown scratch buffers the graph points into).  NTP_GRAPH=0 disables capture.
// Vertex-layout pipeline (a3 -> a4 -> a5; transposed: a7 -> a8 -> a9): this rank's rows Hv [V_p x w]
// (fp32) -> pack with the column-side pre-scale + block exchange -> K hops on the feature slice
// (storage dtype dt) -> gather (chunked and overlapped with the last hop when `overlap`) -> Zv.
void propagate_pipeline(ntp_ctx* c, const ntp_tensor* Hv, ntp_tensor* Zv, int K, float gamma, float alpha,
                        bool transposed, ntp_dtype dt, int chunks, bool overlap, cudaStream_t user) {
    const Graph& g = c->g;
    NTP_CHECK(!(overlap && g.reordered), NTP_ERR_CONFIG,
              "the overlapped gather sends last-hop chunks by destination block: needs a graph without NTP_G_REORDER");
    NTP_CHECK(!(overlap && c->vs > 1), NTP_ERR_CONFIG, "the overlapped gather needs one slice per rank");
    cudaStream_t s = c->s_comp;
    const int32_t P = nslices(c);
    const int32_t vs = c->vs;
    const int64_t n = g.n;
    const int64_t V_pad = (int64_t)P * cdiv(n, P);
    const int64_t V_p = V_pad / c->world;                 // this rank's rows (vs slice blocks)
    const int64_t row0 = (int64_t)c->rank * V_p;
    const int32_t w = Hv->cols;
    const int32_t d_s = slice_width(w, P, dt, c->slice_align);
    const size_t es = esize(dt);
    const int64_t feat = (int64_t)P * V_p * d_s;
    c->hop_ev_used = 0;
    c->send.ensure((size_t)feat * es + 16);
    c->recv.ensure((size_t)feat * es + 16);
    c->xfer.ensure((size_t)feat * es + 16);
    NTP_CUDA(cudaEventRecord(c->ev[40], user));
    NTP_CUDA(cudaStreamWaitEvent(s, c->ev[40], 0));
    const float* cs = transposed ? g.dinv_in_orig() : g.dinv_out_orig();   // column side of this direction
    pack_v2f(c, Hv->data, Hv->ld, w, c->send.p, V_p, d_s, P, cs, row0, n, NTP_F32, dt, s);
    exchange_v2f(c, c->send.p, c->recv.p, V_p * d_s, dt, s);
    PropArgs a{};
    a.H = c->recv.p;
    a.Z = c->xfer.p;
    a.ld_h = d_s;
    a.ld_z = d_s;
    a.cols = d_s;
    a.dtype = dt;
    a.K = K;
    a.gamma = gamma;
    a.alpha = alpha;
    a.transposed = transposed;
    if (vs == 1) {
        propagate_and_gather(c, a, c->send.p, overlap, chunks, V_p, d_s, true, s);
    } else {   // virtual slices: each slice in sequence, then one gather
        for (int j = 0; j < vs; ++j) {
            PropArgs aj = a;
            const size_t off = (size_t)j * V_pad * d_s * es;
            aj.H = static_cast<char*>(c->recv.p) + off;
            aj.Z = static_cast<char*>(c->xfer.p) + off;
            if (V_pad > n)   // padding rows of every slice travel in the gather: keep them zero
                NTP_CUDA(cudaMemsetAsync(static_cast<char*>(aj.Z) + n * d_s * es, 0, (V_pad - n) * d_s * es, s));
            propagate(c, aj, s, true, true);
        }
        exchange_f2v(c, c->xfer.p, c->send.p, V_p * d_s, dt, s);
    }
    unpack_f2v(c, c->send.p, V_p, d_s, P, Zv->data, Zv->ld, w, dt, NTP_F32, s);
    NTP_CUDA(cudaEventRecord(c->ev[41], s));
    NTP_CUDA(cudaStreamWaitEvent(user, c->ev[41], 0));
}

void train_epoch(ntp_ctx* c, const ntp_model* m, const ntp_tensor* X_v, const int32_t* labels_v,
                 const uint8_t* mask_v, ntp_tensor* W0, ntp_tensor* W1, ntp_epoch_report* rep, cudaStream_t user) {
    const Graph& g = c->g;
    cudaStream_t s = c->s_comp;
    const int64_t launches0 = c->launches;
    const int32_t P = c->world;
    const bool after = (m->flags & NTP_M_W1_AFTER_PROP) != 0;
    const bool timed = true;
    cudaEvent_t* E = c->ev;
    NTP_CHECK(c->vs == 1 || !(m->flags & (NTP_M_OVERLAP | NTP_M_P2P_LAYOUTS | NTP_M_DATA_PARALLEL)), NTP_ERR_CONFIG,
              "virtual slices (ntp_set_slices P > world) run the plain layout path: no NTP_M_OVERLAP, "
              "NTP_M_P2P_LAYOUTS or NTP_M_DATA_PARALLEL");
    NTP_CHECK(!((m->flags & NTP_M_OVERLAP) && g.reordered && !after), NTP_ERR_CONFIG,
              "NTP_M_OVERLAP sends last-hop chunks by destination block: needs a graph without NTP_G_REORDER "
              "(the W1-after-propagation epoch overlaps its layout changes by row chunk instead)");

    // ---- order after the caller's stream
    NTP_CUDA(cudaEventRecord(c->ev[40], user ? user : (cudaStream_t)0));
    NTP_CUDA(cudaStreamWaitEvent(s, c->ev[40], 0));

    EpochKey key{};
    key.m = *m;
    key.ptrs[0] = X_v->data;
    key.ptrs[1] = labels_v;
    key.ptrs[2] = mask_v;
    key.ptrs[3] = W0->data;
    key.ptrs[4] = W1->data;
    key.ld = X_v->ld;
    key.graph_version = c->g_version;
    key.head_chunk = getenv("NTP_HEAD_CHUNK") ? atoll(getenv("NTP_HEAD_CHUNK")) : 0;
    key.head_fused = (getenv("NTP_HEAD_FUSED") ? atoll(getenv("NTP_HEAD_FUSED")) : 1) +
                     2 * (getenv("NTP_HEAD_TMA") ? atoll(getenv("NTP_HEAD_TMA")) : 1) +
                     4 * (getenv("NTP_PACK_FUSED") ? atoll(getenv("NTP_PACK_FUSED")) : 1) +
                     8 * (getenv("NTP_WGRAD_FUSED") ? atoll(getenv("NTP_WGRAD_FUSED")) : 1);
    // graph cache entry: the plain epoch, or one per staging slot (whose buffers the graph bakes in; the
    // copy stream's ready / free events become external event nodes)
    const bool staged = (m->flags & NTP_M_STAGED) != 0;
    const int sl = staged ? (int)((m->flags >> NTP_M_SLOT_SHIFT) & NTP_M_SLOT_MASK) : 0;
    if (staged) {
        key.ptrs[0] = c->st_X[sl].p;
        key.ptrs[1] = c->st_y[sl].p;
        key.ptrs[2] = c->st_m[sl].p;
        key.ld = c->st_ld[sl];
    }
    EpochKey& gkey = staged ? c->sg_key[sl] : c->graph_key;
    bool& gwarm = staged ? c->sg_warm[sl] : c->graph_warm;
    bool& gvalid = staged ? c->sg_valid[sl] : c->graph_valid;
    cudaGraphExec_t& gexec = staged ? c->sg_exec[sl] : c->graph_exec;
    int& ghops = staged ? c->sg_hops[sl] : c->graph_hops;
    int64_t& glaunches = staged ? c->sg_launches[sl] : c->graph_launches;
    int64_t* gwire = staged ? c->sg_wire[sl] : c->graph_wire;
    int64_t& ggen = staged ? c->sg_gen[sl] : c->graph_gen;
    int64_t epoch_launches = 0;
    // A captured graph bakes in every scratch pointer: it is replayed only while no library buffer has been
    // (re)allocated or freed since its capture (alloc_generation), whatever entry point moved it.
    // host-streamed and copy-engine-overlap epochs run eagerly
    const bool ce_mode = (m->flags & NTP_M_OVERLAP) && (m->flags & NTP_M_P2P_LAYOUTS) && after && P > 1;
    const bool capturable = graphs_enabled() && !(m->flags & NTP_M_HOST_STREAM) && !ce_mode && !c->trace_on;
    if (capturable && gvalid && gkey == key && ggen == alloc_generation()) {
        NTP_CUDA(cudaGraphLaunch(gexec, s));
        c->hop_ev_used = ghops;
        epoch_launches = glaunches;
        for (int i = 0; i < 4; ++i) c->wire_sent[i] = gwire[i], c->wire_recv[i] = gwire[4 + i];
        if (staged) c->st_free_rec[sl] = true;
    } else if (capturable && gwarm && gkey == key) {
        if (gexec) cudaGraphExecDestroy(gexec);
        gexec = nullptr;
        gvalid = false;
        cudaGraph_t graph = nullptr;
        const int64_t gen0 = alloc_generation();
        NTP_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
        c->capturing = true;
        try {
            enqueue_epoch(c, m, X_v, labels_v, mask_v, W0, W1, timed);
        } catch (...) {
            c->capturing = false;
            cudaStreamEndCapture(s, &graph);
            if (graph) cudaGraphDestroy(graph);
            gwarm = false;
            throw;
        }
        c->capturing = false;
        NTP_CUDA(cudaStreamEndCapture(s, &graph));
        if (alloc_generation() != gen0) {
            // a buffer moved while the epoch was being recorded: earlier nodes may hold the old pointer.
            // Discard the recording and run the epoch eagerly (the buffers now have their final size).
            cudaGraphDestroy(graph);
            enqueue_epoch(c, m, X_v, labels_v, mask_v, W0, W1, timed);
            epoch_launches = c->launches - launches0;
        } else {
            cudaError_t ie = cudaGraphInstantiate(&gexec, graph, 0);
            cudaGraphDestroy(graph);
            NTP_CUDA(ie);
            gvalid = true;
            ggen = gen0;
            ghops = c->hop_ev_used;
            glaunches = c->launches - launches0;
            for (int i = 0; i < 4; ++i) gwire[i] = c->wire_sent[i], gwire[4 + i] = c->wire_recv[i];
            epoch_launches = glaunches;
            NTP_CUDA(cudaGraphLaunch(gexec, s));
        }
    } else {
        // a different key (or capture disabled): this entry's recording no longer matches it
        if (gexec) cudaGraphExecDestroy(gexec);
        gexec = nullptr;
        gvalid = false;
        enqueue_epoch(c, m, X_v, labels_v, mask_v, W0, W1, timed);
        epoch_launches = c->launches - launches0;
        gwarm = true;
        gkey = key;
    }
    double* scal = c->m_scal.as<double>();
    double h_scal[2] = {0, 0};
    NTP_CUDA(cudaMemcpyAsync(h_scal, scal, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    NTP_CUDA(cudaEventRecord(c->ev[41], s));
    NTP_CUDA(cudaStreamWaitEvent(user ? user : (cudaStream_t)0, c->ev[41], 0));
    wait_stream(c, s);

    if (rep) {
        rep->loss = h_scal[1] > 0 ? h_scal[0] / h_scal[1] : 0.0;
        rep->n_train = (int64_t)h_scal[1];
        // E0 start, E1 mlp fwd, E2 v2f, E3 prop fwd (+gather), E4 loss, E5 v2f bwd,
        // E6 prop bwd (+gather, unpack), E7 mlp bwd, E8 allreduce, E9 sgd.
        epoch_phases(E, rep->ms);
        float tot = 0.f;
        NTP_CUDA(cudaEventElapsedTime(&tot, E[0], E[9]));
        rep->ms[NTP_PH_TOTAL] = tot;
        // counted where the transfers are issued (NCCL counts, peer-store extents); DP: all in entry 0
        for (int i = 0; i < 4; ++i) {
            rep->bytes_sent[i] = c->wire_sent[i];
            rep->bytes_recv[i] = c->wire_recv[i];
        }
        rep->collectives = P > 1 ? 5 : 0;
        if ((m->flags & NTP_M_DATA_PARALLEL) && P > 1) rep->collectives = 2 * m->K + 1;   // 2K all-gathers + allreduce
        rep->kernel_launches = epoch_launches;
        int nh = 0;
        rep->spmm_ms = collect_hop_ms(c, &nh);
        rep->spmm_launches = nh;
    }
}


// NEXT-4: the data-parallel baseline the paper compares against (P:338-368,
// "DepComm"-style).  Each rank owns the vertex rows R_q at FULL width and computes the
// same decoupled model: before every hop the current state is all-gathered (every rank needs the
// rows of all in-neighbours), then the rank aggregates only its own destination rows.  Same
// function as the tensor-parallel epoch -- parity against the same oracle -- but the work per rank
// follows the degree distribution of its rows (load imbalance, Fig. 10) and the traffic is 2K
// all-gathers of full-width rows instead of 4 exchanges of slices.  Non-W1-after path, original
// vertex order, fp32 or bf16 storage.
static void enqueue_epoch_dp(ntp_ctx* c, const ntp_model* m, const float* X, int64_t ldx, const int32_t* lab,
                             const uint8_t* msk, float* W0u, float* W1u, const float* W0g, int64_t ldw0,
                             const float* W1g, int64_t ldw1, Split W0s, Split W1s, bool timed) {
    const Graph& g = c->g;
    cudaStream_t s = c->s_comp;
    const int32_t P = c->world;
    const int64_t n = g.n;
    const int64_t V_p = cdiv(n, P);
    const int64_t V_pad = (int64_t)P * V_p;
    const int64_t row0 = (int64_t)c->rank * V_p;
    const int64_t row_hi = std::min(row0 + V_p, n);
    const ntp_dtype dt = m->dtype;
    const size_t es = esize(dt);
    const int32_t ws = slice_width(m->C, 1, dt, c->slice_align);   // full row width, 16-byte padded
    const int64_t ldH = round4(m->hid), ldL = round4(std::max(m->C, m->hid));
    cudaEvent_t* E = c->ev;
    int ei = 1;
    c->m_H1.ensure((size_t)V_p * ldH * sizeof(float));
    c->m_L.ensure((size_t)V_p * ldL * sizeof(float));
    c->m_dL.ensure((size_t)V_p * ldL * sizeof(float));
    c->m_dH1.ensure((size_t)V_p * ldH * sizeof(float));
    const int64_t n_w = (int64_t)m->d_in * m->hid + (int64_t)m->hid * m->C;
    c->m_dW.ensure((size_t)n_w * sizeof(float));
    c->m_scal.ensure(4 * sizeof(double));
    const size_t full = (size_t)V_pad * ws * es;
    c->recv.ensure(full + 16);
    c->xfer.ensure(full + 16);
    c->send.ensure(full + 16);      // S^0 (alpha term) / gradient rows
    const int64_t loss_blocks = std::min<int64_t>(cdiv(V_p, 8), 148 * 8);
    c->m_part.ensure((size_t)loss_blocks * (sizeof(double) + sizeof(int64_t)) + 16);
    double* part = c->m_part.as<double>();
    int64_t* cnt = reinterpret_cast<int64_t*>(part + loss_blocks);
    float* H1 = c->m_H1.as<float>();
    float* L = c->m_L.as<float>();
    float* dL = c->m_dL.as<float>();
    float* dH1 = c->m_dH1.as<float>();
    float* dW0 = c->m_dW.as<float>();
    float* dW1 = dW0 + (int64_t)m->d_in * m->hid;
    double* scal = c->m_scal.as<double>();
    char* A = static_cast<char*>(c->recv.p);
    char* B = static_cast<char*>(c->xfer.p);
    char* S0 = static_cast<char*>(c->send.p);
    const size_t own = (size_t)row0 * ws * es;
    if (V_pad > n)   // padding rows: never written by a hop, multiplied by zero downstream -> keep them zero
        for (char* b : {A, B, S0}) NTP_CUDA(cudaMemsetAsync(b + (size_t)n * ws * es, 0, (V_pad - n) * ws * es, s));
    const ncclDataType_t t = dt == NTP_BF16 ? ncclBfloat16 : ncclFloat32;
    auto allgather = [&](char* buf) {   // own rows -> every rank's copy of the full matrix
        if (P > 1) {
            NTP_NCCL(ncclAllGather(buf + own, buf, (size_t)V_p * ws, t, c->comm, s));
            wire_add(c, (int64_t)(P - 1) * V_p * ws * (int64_t)es, (int64_t)(P - 1) * V_p * ws * (int64_t)es);
        }
    };
    // K hops of one direction on full-width rows: S^0 own rows in `A` (pre-scaled); returns the buffer
    // holding Z^K own rows (unscaled, storage dtype)
    auto hops = [&](bool transposed) -> char* {
        const Csr& csr = transposed ? g.bwd() : g.fwd();
        const float* rs = transposed ? g.dinv_out_p() : g.dinv_in_p();
        const float* cs = transposed ? g.dinv_in_p() : g.dinv_out_p();
        if (m->alpha != 0.f) NTP_CUDA(cudaMemcpyAsync(S0 + own, A + own, (size_t)V_p * ws * es, cudaMemcpyDeviceToDevice, s));
        char* cur = A;
        char* nxt = B;
        for (int k = 1; k <= m->K; ++k) {
            allgather(cur);
            const bool tm = timed && c->hop_ev_used + 2 <= kHopEvents;
            if (tm) NTP_CUDA(record_timing(c, c->hop_ev[c->hop_ev_used], s));
            spmm_hop(c, csr, rs, cs, cur, nxt, m->alpha != 0.f ? (const void*)S0 : (const void*)cur, ws, ws, ws, ws,
                     dt, m->gamma, m->alpha, k == m->K ? 1 : 0, row0, row_hi, s);
            if (tm) {
                NTP_CUDA(record_timing(c, c->hop_ev[c->hop_ev_used + 1], s));
                c->hop_ev_used += 2;
            }
            std::swap(cur, nxt);
        }
        return cur;
    };
    // a2: MLP forward on own rows; S^0 own rows = D~_out^{-1/2} L^ (storage dtype)
    mlp_gemm(c, false, false, V_p, m->hid, m->d_in, X, ldx, W0g, ldw0, H1, ldH, s, 1, nullptr, 0, W0s);
    mlp_gemm(c, false, false, V_p, m->C, m->hid, H1, ldH, W1g, ldw1, L, ldL, s, 0, nullptr, 0, W1s);
    NTP_CUDA(record_timing(c, E[ei++], s));   // E1 mlp_fwd
    pack_v2f(c, L, ldL, m->C, A + own, V_p, ws, 1, g.dinv_out_orig(), row0, n, NTP_F32, dt, s);
    NTP_CUDA(record_timing(c, E[ei++], s));   // E2 (no split)
    char* Z = hops(false);
    NTP_CUDA(record_timing(c, E[10], s));
    NTP_CUDA(record_timing(c, E[ei++], s));   // E3 prop fwd (incl. all-gathers)
    // a6: loss on own rows; gradient rows (pre-scaled by the backward column side) into A's own rows
    char* G = (Z == A) ? B : A;
    int64_t nb = 0;
    if (dt == NTP_F32)
        nb = launch_softmax_xent(c, (const float*)(Z + own), 0, V_p, ws, m->C, lab, msk, row0, n, (float*)(G + own), 1,
                                 g.dinv_in_orig(), part, cnt, ws, s);
    else
        nb = launch_softmax_xent(c, (const __nv_bfloat16*)(Z + own), 0, V_p, ws, m->C, lab, msk, row0, n,
                                 (__nv_bfloat16*)(G + own), 1, g.dinv_in_orig(), part, cnt, ws, s);
    if (ws > m->C) {
        if (dt == NTP_F32)
            zero_pad_cols_kernel<float><<<eblocks(V_p * (ws - m->C)), 256, 0, s>>>((float*)(G + own), V_p, ws, 1, m->C,
                                                                                  nullptr, 0);
        else
            zero_pad_cols_kernel<__nv_bfloat16><<<eblocks(V_p * (ws - m->C)), 256, 0, s>>>(
                (__nv_bfloat16*)(G + own), V_p, ws, 1, m->C, nullptr, 0);
        NTP_LAUNCH_CHECK();
        count_launch(c);
    }
    reduce_partials_kernel<<<1, 256, 0, s>>>(part, cnt, nb, scal);
    NTP_LAUNCH_CHECK();
    count_launch(c);
    NTP_CUDA(record_timing(c, E[ei++], s));   // E4 loss
    NTP_CUDA(record_timing(c, E[ei++], s));   // E5 (no split)
    if (G != A) NTP_CUDA(cudaMemcpyAsync(A + own, G + own, (size_t)V_p * ws * es, cudaMemcpyDeviceToDevice, s));
    char* dZ = hops(true);
    NTP_CUDA(record_timing(c, E[11], s));
    unpack_f2v(c, dZ + own, V_p, ws, 1, dL, ldL, m->C, dt, NTP_F32, s);
    NTP_CUDA(record_timing(c, E[ei++], s));   // E6 prop bwd
    // a10: MLP backward on own rows
    mlp_gemm(c, true, false, m->hid, m->C, V_p, H1, ldH, dL, ldL, dW1, m->C, s);
    mlp_gemm(c, false, true, V_p, m->hid, m->C, dL, ldL, W1g, ldw1, dH1, ldH, s, 2, H1, ldH, W1s);
    mlp_gemm(c, true, false, m->d_in, m->hid, V_p, X, ldx, dH1, ldH, dW0, m->hid, s);
    NTP_CUDA(record_timing(c, E[ei++], s));   // E7 mlp bwd
    if (P > 1) {
        NTP_NCCL(ncclGroupStart());
        NTP_NCCL(ncclAllReduce(dW0, dW0, n_w, ncclFloat32, ncclSum, c->comm, s));
        NTP_NCCL(ncclAllReduce(scal, scal, 2, ncclFloat64, ncclSum, c->comm, s));
        NTP_NCCL(ncclGroupEnd());
    }
    NTP_CUDA(record_timing(c, E[ei++], s));   // E8 allreduce
    sgd_kernel<<<eblocks(n_w), 256, 0, s>>>(W0u, (int64_t)m->d_in * m->hid, W1u, (int64_t)m->hid * m->C, dW0, scal,
                                            m->lr);
    NTP_LAUNCH_CHECK();
    count_launch(c);
    NTP_CUDA(record_timing(c, E[ei++], s));   // E9 sgd
}

// Input staging (e2e loops): host -> slot copy on the copy stream, after the last epoch that read
// the slot.  One contiguous DMA in the host pitch, then the 16-byte GEMM pitch on the device (a 2-D
// host copy with ~2 KB rows runs at a third of the link rate).
void stage_inputs(ntp_ctx* c, int slot, const float* X, int64_t rows, int32_t d_in, int64_t ldx, const int32_t* y,
                  const uint8_t* m) {
    cudaStream_t s = c->s_copy;
    const int64_t ld = round4(d_in);
    c->st_X[slot].ensure((size_t)rows * ld * sizeof(float) + 16);
    c->st_y[slot].ensure((size_t)rows * sizeof(int32_t) + 16);
    c->st_m[slot].ensure((size_t)rows + 16);
    if (c->st_free_rec[slot]) NTP_CUDA(cudaStreamWaitEvent(s, c->st_free[slot], 0));
    if (ldx == ld) {
        NTP_CUDA(cudaMemcpyAsync(c->st_X[slot].p, X, (size_t)rows * ldx * sizeof(float), cudaMemcpyHostToDevice, s));
    } else {
        c->st_raw[slot].ensure((size_t)rows * ldx * sizeof(float) + 16);
        NTP_CUDA(cudaMemcpyAsync(c->st_raw[slot].p, X, (size_t)rows * ldx * sizeof(float), cudaMemcpyHostToDevice, s));
        NTP_CUDA(cudaMemcpy2DAsync(c->st_X[slot].p, ld * sizeof(float), c->st_raw[slot].p, ldx * sizeof(float),
                                   d_in * sizeof(float), rows, cudaMemcpyDeviceToDevice, s));
    }
    NTP_CUDA(cudaMemcpyAsync(c->st_y[slot].p, y, (size_t)rows * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    NTP_CUDA(cudaMemcpyAsync(c->st_m[slot].p, m, (size_t)rows, cudaMemcpyHostToDevice, s));
    NTP_CUDA(cudaEventRecord(c->st_ready[slot], s));
    c->st_rows[slot] = rows;
    c->st_d_in[slot] = d_in;
    c->st_ld[slot] = ld;
}

// ------------------------------------------------------------------------------------------------
// NEXT-1: naive (coupled) GNN tensor parallelism, the paper's baseline (P:574,
// Fig. 6).  An L-layer GCN  H^l = ReLU(A^ H^{l-1} W^l)  (logits = A^ H^{L-1} W^L) trained
// layer by layer with each aggregation on feature slices: every layer pays a split before and a
// gather after its hop -- 2L layout changes forward and 2(L-1) backward, 4L - 2 per epoch against
// the decoupled epoch's 4.  Reuses the decoupled path's kernels unchanged: pack (split with
// the column-side pre-scale), block all-to-all, one-hop propagation, unpack (gather; with the ReLU'
// mask on the backward), tensor-core GEMMs, loss, fixed-order reductions, SGD.
void train_epoch_coupled(ntp_ctx* c, const ntp_coupled_model* m, const ntp_tensor* X_v, const int32_t* labels_v,
                         const uint8_t* mask_v, ntp_tensor* const* W, ntp_coupled_report* rep, cudaStream_t user) {
    const Graph& g = c->g;
    cudaStream_t s = c->s_comp;
    const int64_t launches0 = c->launches;
    const int32_t P = c->world;
    const int64_t n = g.n;
    const int64_t V_p = cdiv(n, P);
    const int64_t row0 = (int64_t)c->rank * V_p;
    const int L = m->L;
    const ntp_dtype dt = m->dtype;
    const size_t es = esize(dt);
    const bool local = (P == 1);
    NTP_CHECK(c->vs == 1, NTP_ERR_CONFIG, "the coupled epoch runs one slice per rank (no virtual slices)");
    drop_epoch_graph(c);   // the buffers below may move ones a captured decoupled epoch points into
    NTP_CUDA(cudaEventRecord(c->ev[40], user ? user : (cudaStream_t)0));
    NTP_CUDA(cudaStreamWaitEvent(s, c->ev[40], 0));
    cudaEvent_t* E = c->ev;
    NTP_CUDA(record_timing(c, E[0], s));
    c->hop_ev_used = 0;

    // ---- buffers: Z^l [V_p x w_{l-1}], H^l [V_p x w_l] (l < L), logits / dA [V_p x w_L], dZ / dA scratch
    int64_t ldw[kMaxLayers + 1];
    for (int l = 0; l <= L; ++l) ldw[l] = round4(m->widths[l]);
    int64_t maxw = 0, nw = 0, nwp = 0;
    for (int l = 0; l <= L; ++l) maxw = std::max<int64_t>(maxw, ldw[l]);
    for (int l = 1; l <= L; ++l) nw += (int64_t)m->widths[l - 1] * m->widths[l];
    for (int l = 1; l <= L; ++l) nwp += (int64_t)m->widths[l - 1] * ldw[l];
    for (int l = 1; l <= L; ++l) c->cp_Z[l].ensure((size_t)V_p * ldw[l - 1] * sizeof(float) + 16);
    for (int l = 1; l < L; ++l) c->cp_H[l].ensure((size_t)V_p * ldw[l] * sizeof(float) + 16);
    c->cp_A.ensure((size_t)V_p * maxw * sizeof(float) + 16);     // logits, then dA^l
    c->cp_B.ensure((size_t)V_p * maxw * sizeof(float) + 16);     // dZ^l
    c->cp_W.ensure((size_t)nwp * sizeof(float) + 16);            // 16-byte-pitch copies of W^l
    c->m_dW.ensure((size_t)nw * sizeof(float) + 16);
    c->m_scal.ensure(4 * sizeof(double));
    int64_t maxfeat = 0;
    for (int l = 0; l < L; ++l)
        maxfeat = std::max<int64_t>(maxfeat, (int64_t)P * V_p * slice_width(m->widths[l], P, dt, c->slice_align));
    if (!local) c->send.ensure((size_t)maxfeat * es + 16);
    c->recv.ensure((size_t)maxfeat * es + 16);
    c->xfer.ensure((size_t)maxfeat * es + 16);
    const int64_t loss_blocks = std::min<int64_t>(cdiv(V_p, 8), 148 * 8);
    c->m_part.ensure((size_t)loss_blocks * (sizeof(double) + sizeof(int64_t)) + 16);
    double* part = c->m_part.as<double>();
    int64_t* cnt = reinterpret_cast<int64_t*>(part + loss_blocks);
    double* scal = c->m_scal.as<double>();
    float* Wp[kMaxLayers + 1];
    float* dWl[kMaxLayers + 1];
    {
        float* w = c->cp_W.as<float>();
        float* d = c->m_dW.as<float>();
        for (int l = 1; l <= L; ++l) {
            Wp[l] = w;
            dWl[l] = d;
            // padded GEMM copy (16-byte pitch) of the caller's dense W^l (ld == cols)
            NTP_CUDA(cudaMemcpy2DAsync(w, ldw[l] * sizeof(float), W[l - 1]->data, m->widths[l] * sizeof(float),
                                       m->widths[l] * sizeof(float), m->widths[l - 1], cudaMemcpyDeviceToDevice, s));
            w += (int64_t)m->widths[l - 1] * ldw[l];
            d += (int64_t)m->widths[l - 1] * m->widths[l];
        }
    }
    const float* X = static_cast<const float*>(X_v->data);
    int64_t ldx = X_v->ld;
    if ((ldx % 4) != 0 || (reinterpret_cast<uintptr_t>(X) % 16) != 0) {
        c->m_Xs.ensure((size_t)V_p * ldw[0] * sizeof(float));
        NTP_CUDA(cudaMemcpy2DAsync(c->m_Xs.p, ldw[0] * sizeof(float), X, ldx * sizeof(float), m->widths[0] * sizeof(float),
                                   V_p, cudaMemcpyDeviceToDevice, s));
        X = c->m_Xs.as<float>();
        ldx = ldw[0];
    }
    int changes = 0;
    wire_reset(c);
    // one layout round trip around a single hop: vertex rows Hv [V_p x w] -> split (pre-scaled) -> hop
    // (transposed = backward) -> gather -> out [V_p x w] (with keep: the ReLU' mask)
    auto agg = [&](const float* Hv, int64_t ldh, int w, bool transposed, float* out, int64_t ldo, const float* keep,
                   int64_t ldk) {
        const int32_t d_s = slice_width(w, P, dt, c->slice_align);
        const float* cs = transposed ? g.dinv_in_orig() : g.dinv_out_orig();
        pack_v2f(c, Hv, ldh, w, local ? c->recv.p : c->send.p, V_p, d_s, P, cs, row0, n, NTP_F32, dt, s);
        if (!local) alltoall_blocks(c, c->send.p, c->recv.p, V_p * d_s, dt, s);
        PropArgs a{};
        a.H = c->recv.p;
        a.Z = c->xfer.p;
        a.ld_h = d_s;
        a.ld_z = d_s;
        a.cols = d_s;
        a.dtype = dt;
        a.K = 1;
        a.gamma = 1.f;
        a.alpha = 0.f;
        a.transposed = transposed;
        void* gathered = c->recv.p;
        if (local) gathered = propagate_consume(c, a, s, true);
        else propagate_and_gather(c, a, c->recv.p, false, 1, V_p, d_s, true, s);
        unpack_f2v(c, gathered, V_p, d_s, P, out, ldo, w, dt, NTP_F32, s, keep, ldk);
        if (!local) changes += 2;
    };
    // ---- forward: Z^l = A^ H^{l-1} (sliced), H^l = ReLU(Z^l W^l), logits = Z^L W^L
    float* logits = c->cp_B.as<float>();
    for (int l = 1; l <= L; ++l) {
        const float* Hin = (l == 1) ? X : c->cp_H[l - 1].as<float>();
        const int64_t ldin = (l == 1) ? ldx : ldw[l - 1];
        agg(Hin, ldin, m->widths[l - 1], false, c->cp_Z[l].as<float>(), ldw[l - 1], nullptr, 0);
        float* out = (l < L) ? c->cp_H[l].as<float>() : logits;
        mlp_gemm(c, false, false, V_p, m->widths[l], m->widths[l - 1], c->cp_Z[l].as<float>(), ldw[l - 1], Wp[l],
                 ldw[l], out, ldw[l], s, l < L ? 1 : 0);
    }
    // ---- loss and dA^L (softmax - onehot on train rows; 1/N_train folded into SGD, R12), in place
    float* dA = c->cp_A.as<float>();
    const int64_t nb = launch_softmax_xent(c, (const float*)logits, 0, V_p, 0, m->widths[L], labels_v, mask_v, row0, n,
                                           dA, 0, nullptr, part, cnt, ldw[L], s);
    reduce_partials_kernel<<<1, 256, 0, s>>>(part, cnt, nb, scal);
    NTP_LAUNCH_CHECK();
    count_launch(c);
    // ---- backward (dA^l in cp_A, dZ^l in cp_B: the logits are consumed by the loss)
    for (int l = L; l >= 1; --l) {
        mlp_gemm(c, true, false, m->widths[l - 1], m->widths[l], V_p, c->cp_Z[l].as<float>(), ldw[l - 1], dA, ldw[l],
                 dWl[l], m->widths[l], s);                                               // dW^l = Z^l^T dA^l
        if (l == 1) break;
        float* dZ = c->cp_B.as<float>();
        mlp_gemm(c, false, true, V_p, m->widths[l - 1], m->widths[l], dA, ldw[l], Wp[l], ldw[l], dZ, ldw[l - 1], s);
        // dA^{l-1} = (A^T dZ^l) * [H^{l-1} > 0], into the logits / dA buffer (dA^l is consumed)
        agg(dZ, ldw[l - 1], m->widths[l - 1], true, dA, ldw[l - 1], c->cp_H[l - 1].as<float>(), ldw[l - 1]);
    }
    if (P > 1) {
        NTP_NCCL(ncclGroupStart());
        NTP_NCCL(ncclAllReduce(c->m_dW.p, c->m_dW.p, nw, ncclFloat32, ncclSum, c->comm, s));
        NTP_NCCL(ncclAllReduce(scal, scal, 2, ncclFloat64, ncclSum, c->comm, s));
        NTP_NCCL(ncclGroupEnd());
    }
    for (int l = 1; l <= L; ++l) {
        const int64_t len = (int64_t)m->widths[l - 1] * m->widths[l];
        sgd_kernel<<<eblocks(len), 256, 0, s>>>(static_cast<float*>(W[l - 1]->data), len, nullptr, 0, dWl[l], scal,
                                                m->lr);
        NTP_LAUNCH_CHECK();
        count_launch(c);
    }
    NTP_CUDA(record_timing(c, E[1], s));
    double h_scal[2] = {0, 0};
    NTP_CUDA(cudaMemcpyAsync(h_scal, scal, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    NTP_CUDA(cudaEventRecord(c->ev[41], s));
    NTP_CUDA(cudaStreamWaitEvent(user ? user : (cudaStream_t)0, c->ev[41], 0));
    wait_stream(c, s);
    if (rep) {
        rep->loss = h_scal[1] > 0 ? h_scal[0] / h_scal[1] : 0.0;
        rep->n_train = (int64_t)h_scal[1];
        rep->layout_changes = changes;
        rep->bytes_sent = c->wire_sent[0];   // every layout change of the coupled epoch counts in entry 0
        rep->bytes_recv = c->wire_recv[0];
        float tot = 0.f;
        NTP_CUDA(cudaEventElapsedTime(&tot, E[0], E[1]));
        rep->ms_total = tot;
        int nh = 0;
        rep->ms_agg = collect_hop_ms(c, &nh);
        rep->hops = nh;
        rep->kernel_launches = c->launches - launches0;
    }
}

}  // namespace ntp
