// gat.cu — NEXT-2: decoupled GAT training epoch on feature slices.
//
// Paper: GAT's aggregation carries an edge-associated NN operation (Eq. 5):
//   a_uv = softmax_v( LeakyReLU( a^T [W h_u || W h_v] ) ),  a_v = sum_{u in N_in(v)} a_uv h_u
// NeutronTP decouples it by "precomputing all the attention coefficients required for each edge" before
// the aggregation starts, with data parallelism over the vertices' in-edges, then "the attention
// coefficients are shared among all workers" and the aggregation runs on feature slices like the simple
// models (§4.1.1, §4.1.2).  Readings G1-G4: z = ReLU(X W0) W1 (vertex NN
// first), attention over N_in(v) + {v} (A~ = A + I, R1) with a = [a_src ; a_dst] and LeakyReLU slope 0.2,
// K hops Z^k = gamma A_att Z^{k-1}, softmax cross-entropy on Z^K, and the full backward including the
// attention parameters.
//
// B200 design:
//   * a_src.z_u + a_dst.z_v splits into two per-vertex scalars (f_u, g_v): each rank computes them for its
//     own rows and one all-gather of 2 floats per vertex replaces the paper's all-share of nnz coefficients;
//     every rank then evaluates the softmax of every destination itself (identical arithmetic, so the
//     coefficients are bitwise equal on all ranks).  (Re-deriving nnz coefficients from 8 bytes per vertex
//     costs one pass over col_idx; shipping them would move 4 bytes per arc over NVLink.)
//   * The weighted hop is the merge-path SpMM kernel's WT variant (spmm.cu): per-arc coefficients loaded
//     with the column indices, same pipeline and fixed reduction order; the backward runs over the out-CSR
//     with the coefficients in its order, re-derived from each destination's softmax (max, sum).
//   * Backward without per-arc gradients.  With beta_uv = alpha_uv LeakyReLU'(s_uv) the softmax / LeakyReLU
//     backward ds_uv = beta_uv (dalpha_uv - w_v), w_v = sum_u alpha_uv dalpha_uv, only enters through the sums
//     ps_u = sum_v ds_uv and pd_v = sum_u ds_uv, and since dalpha_uv = gamma sum_k G^k_v . Z^{k-1}_u these are
//     per-vertex dot products of hop outputs: w_v = sum_k G^k.Z^k, pd_v = sum_k G^k.Y^k - w_v b_v and
//     ps_u = sum_k Z^{k-1}.X^k - sum_v beta_uv w_v, where Y^k = gamma A_beta Z^{k-1} (forward, one more
//     weighted hop per level) and X^k = gamma A_beta^T G^k (backward, likewise), b_v = sum_u beta_uv.  Each
//     slice contributes partial dots; one allreduce of 3n floats sums them over ranks (the SDDMM form moved
//     n + nnz).  dz += ps a_src + pd a_dst and da_src = sum ps z, da_dst = sum pd z (rank-1 terms).
// Coefficient layout everywhere: [n self loops | nnz arcs in in-CSR order] (the oracle's arcs() order).
#include <algorithm>
#include <cmath>

#include "ntp_internal.cuh"

namespace ntp {

namespace {

__device__ __forceinline__ float leaky(float x, float slope) { return x > 0.f ? x : slope * x; }

// Coefficient words: alpha_uv with the sign bit set where s_uv <= 0, so one word gives alpha = |w| and
// beta = alpha * LeakyReLU'(s) = (w < 0 ? slope : 1) * |w| (the dual hop decodes it the same way, spmm.cu)
__device__ __forceinline__ float coef_word(float a, bool pos) { return pos ? a : -a; }
__device__ __forceinline__ float word_beta(float w, float slope) {
    const float a = __int_as_float(__float_as_int(w) & 0x7fffffff);
    return __float_as_int(w) < 0 ? slope * a : a;
}

// one 16-byte vector of a slice row as fp32 values (fp32: 4, bf16: 8 widened exactly)
template <typename T> __device__ __forceinline__ void load16(const void* p, float (&v)[16 / sizeof(T)]) {
    const uint4 x = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
    if constexpr (sizeof(T) == 4) {
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(w[i]);
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __uint_as_float((i & 1) ? (w[i >> 1] & 0xFFFF0000u) : (w[i >> 1] << 16));
    }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// G2 per-vertex halves of the score: fg[2v] = a_src . z_v, fg[2v+1] = a_dst . z_v (own rows, 0 on padding)
__global__ void gat_fg_kernel(const float* __restrict__ z, int64_t ldz, int32_t C, const float* __restrict__ att,
                              int64_t rows, int64_t row0, int64_t n, float* __restrict__ fg) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < rows; v += warps) {
        float f = 0.f, g = 0.f;
        for (int c = lane; c < C; c += 32) {
            const float x = z[v * ldz + c];
            f = fmaf(x, att[c], f);
            g = fmaf(x, att[C + c], g);
        }
        f = warp_sum(f);
        g = warp_sum(g);
        if (lane == 0) {
            const bool real = row0 + v < n;
            fg[2 * (row0 + v)] = real ? f : 0.f;
            fg[2 * (row0 + v) + 1] = real ? g : 0.f;
        }
    }
}

// Per-row reductions run on a warp (rows of <= kBigDeg arcs, grid-stride over rows) or, for hub rows (up to
// ~50K in-arcs on the Reddit shape, ~700K on papers), on a whole 256-thread CTA (one row per CTA, rows from
// a per-graph list): one warp walking a hub row alone would hold up the kernel for its ~1.5K iterations.
constexpr int kBigDeg = 4096;

struct WarpRed {
    int t, T;
    __device__ WarpRed() : t(threadIdx.x & 31), T(32) {}
    __device__ float sum(float v) const { return warp_sum(v); }
    __device__ float max(float v) const { return warp_max(v); }
    __device__ void combine(float& m, float& sm) const {   // online softmax (max, sum) over the group
        const float M = warp_max(m);
        sm = warp_sum(sm == 0.f ? 0.f : sm * expf(m - M));
        m = M;
    }
};
struct BlockRed {
    float* sh;   // >= 32 floats of shared memory
    int t, T;
    __device__ explicit BlockRed(float* s_) : sh(s_), t(threadIdx.x), T(blockDim.x) {}
    __device__ float all(float v, bool is_max) const {
        v = is_max ? warp_max(v) : warp_sum(v);
        __syncthreads();
        if ((t & 31) == 0) sh[t >> 5] = v;
        __syncthreads();
        float r = (t & 31) < (T >> 5) ? sh[t & 31] : (is_max ? -INFINITY : 0.f);
        return is_max ? warp_max(r) : warp_sum(r);   // fixed order: warp partials, then a fixed tree
    }
    __device__ float sum(float v) const { return all(v, false); }
    __device__ float max(float v) const { return all(v, true); }
    __device__ void combine(float& m, float& sm) const {
        const float M = all(m, true);
        sm = all(sm == 0.f ? 0.f : sm * expf(m - M), false);
        m = M;
    }
};

// G2 softmax over a destination's self loop + in-arcs, two passes: (1) e = LeakyReLU(f_u + g_v) -- the only
// gather of f -- stored in alpha's slot and an online max / sum per thread combined over the group; (2)
// alpha = exp(e - m) / sum from the stored e (coalesced), beta = alpha * LeakyReLU'(s) (1 where s > 0, i.e.
// where e > 0, else the slope) and b_v = sum of v's betas (fixed order).  (max, sum) are kept per
// destination: the out-CSR order re-derives its coefficients from them (gat_coef_t_kernel).
__device__ __forceinline__ void online_add(float& m, float& sm, float e) {
    if (e > m) {
        sm = sm * expf(m - e) + 1.f;
        m = e;
    } else {
        sm += expf(e - m);
    }
}

template <class Red>
__device__ void softmax_row(const Red& R, int64_t v, const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                            const float* __restrict__ fg, int64_t n, float slope, float* __restrict__ alpha,
                            float* __restrict__ msum, float* __restrict__ bsum) {
    const float gv = fg[2 * v + 1];
    const float ss = fg[2 * v] + gv;
    const float es = leaky(ss, slope);
    const int b = rp[v], e = rp[v + 1];
    float m = -INFINITY, sm = 0.f;
    if (R.t == 0) m = es, sm = 1.f;
    for (int j = b + R.t; j < e; j += R.T) {
        const float ej = leaky(fg[2 * (int64_t)col[j]] + gv, slope);
        alpha[n + j] = ej;
        online_add(m, sm, ej);
    }
    R.combine(m, sm);
    float bs = 0.f;
    if (R.t == 0) {
        const float a = expf(es - m) / sm;
        alpha[v] = coef_word(a, ss > 0.f);
        bs = ss > 0.f ? a : slope * a;
        msum[2 * v] = m;
        msum[2 * v + 1] = sm;
    }
    for (int j = b + R.t; j < e; j += R.T) {
        const float ej = alpha[n + j];
        const float a = expf(ej - m) / sm;
        alpha[n + j] = coef_word(a, ej > 0.f);
        bs += ej > 0.f ? a : slope * a;
    }
    bs = R.sum(bs);
    if (R.t == 0) bsum[v] = bs;
}

__global__ void gat_softmax_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                   const float* __restrict__ fg, int64_t n, float slope, float* __restrict__ alpha,
                                   float* __restrict__ msum, float* __restrict__ bsum) {
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const WarpRed R;
    for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += warps)
        if (rp[v + 1] - rp[v] <= kBigDeg) softmax_row(R, v, rp, col, fg, n, slope, alpha, msum, bsum);
}

__global__ void __launch_bounds__(256) gat_softmax_big_kernel(const int32_t* __restrict__ big, int32_t nbig,
                                                              const int32_t* __restrict__ rp,
                                                              const int32_t* __restrict__ col,
                                                              const float* __restrict__ fg, int64_t n, float slope,
                                                              float* __restrict__ alpha, float* __restrict__ msum,
                                                              float* __restrict__ bsum) {
    __shared__ float sh[32];
    const BlockRed R(sh);
    for (int i = blockIdx.x; i < nbig; i += gridDim.x) softmax_row(R, big[i], rp, col, fg, n, slope, alpha, msum, bsum);
}

// rows of more than kBigDeg arcs (list built once per graph; order irrelevant: rows are independent)
__global__ void gat_big_rows_kernel(const int32_t* __restrict__ rp, int64_t n, int32_t* __restrict__ list,
                                    int32_t* __restrict__ cnt) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        if (rp[v + 1] - rp[v] > kBigDeg) list[atomicAdd(cnt, 1)] = (int32_t)v;
}

// out-CSR arc j' (row u, column v) -> its in-CSR index (u's position in row v); dev switch NTP_GAT_PERMUTE only
__global__ void gat_perm_kernel(const int32_t* __restrict__ rp_in, const int32_t* __restrict__ col_in,
                                const int32_t* __restrict__ rp_out, const int32_t* __restrict__ col_out, int64_t n,
                                int32_t* __restrict__ perm) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n; u += warps) {
        for (int j = rp_out[u] + lane; j < rp_out[u + 1]; j += 32) {
            const int v = col_out[j];
            int lo = rp_in[v], hi = rp_in[v + 1];
            while (lo < hi) {   // first position with col_in >= u (u is present: the CSRs are transposes)
                const int mid = (lo + hi) >> 1;
                if (col_in[mid] < u) lo = mid + 1;
                else hi = mid;
            }
            perm[j] = lo;
        }
    }
}

// Dev switch NTP_GAT_PERMUTE=1: the plain permutation (the re-derivation below must match it bitwise;
// tests/test_gpu_gat.py).
__global__ void gat_permute_kernel(const float* __restrict__ a, const int32_t* __restrict__ perm, int64_t n, int64_t nnz,
                                   float* __restrict__ at) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n + nnz; i += (int64_t)gridDim.x * blockDim.x)
        at[i] = i < n ? a[i] : a[n + perm[i - n]];
}

// The coefficient words in out-CSR order, re-derived rather than permuted: arc j' (row u, column v) gets
// alpha = exp(LeakyReLU(f_u + g_v) - m_v) / sum_v from the destination's stored (max, sum), signed by
// f_u + g_v -- the very operands and operations of softmax_row, so at[n + j'] is bitwise a[n + perm[j']] --
// with col_out streamed and fg / msum (16 bytes per vertex,
// L2-resident) gathered, instead of a random 4-byte gather from the nnz-long arrays.  Warps take ranges of
// kAtArcs consecutive out-arcs (hub rows spread over many warps); self loops are copied.
constexpr int kAtArcs = 2048;
__global__ void gat_coef_t_kernel(const int32_t* __restrict__ rp_out, const int32_t* __restrict__ col_out,
                                  const float* __restrict__ fg, const float* __restrict__ msum,
                                  const float* __restrict__ a, int64_t n, int64_t nnz, float slope,
                                  float* __restrict__ at) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t v = warp * 32 + lane; v < n; v += nwarps * 32) at[v] = a[v];
    const int64_t nranges = (nnz + kAtArcs - 1) / kAtArcs;
    for (int64_t rg = warp; rg < nranges; rg += nwarps) {
        const int64_t a0 = rg * kAtArcs, a1 = min(a0 + (int64_t)kAtArcs, nnz);
        int64_t lo = 0, hi = n;   // u = last row with rp_out[u] <= a0
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (rp_out[mid] <= a0) lo = mid;
            else hi = mid;
        }
        int64_t u = lo;
        for (int64_t j = a0 + lane; j < a1; j += 32) {
            while (rp_out[u + 1] <= j) ++u;
            const int64_t v = __ldg(col_out + j);
            const float sj = fg[2 * u] + fg[2 * v + 1];
            const float ej = leaky(sj, slope);
            const float2 ms = *reinterpret_cast<const float2*>(msum + 2 * v);
            // __fsub_rn: no contraction of slope * s - m into one FMA (softmax_row subtracts from the stored e)
            at[n + j] = coef_word(expf(__fsub_rn(ej, ms.x)) / ms.y, ej > 0.f);
        }
    }
}

// G4 per-vertex dot products of one level k and one slice (d_s columns), accumulated over levels and slices:
//   w_v  += G^k_v . Z^k_v        (= sum_u alpha_uv dalpha_uv: Z^k = gamma A_att Z^{k-1})
//   gy_v += G^k_v . Y^k_v        (= sum_u beta_uv dalpha_uv,  Y^k = gamma A_beta Z^{k-1})
//   zx_v += Z^{k-1}_v . X^k_v    (= sum_w beta_vw dalpha_vw over v's out-arcs, X^k = gamma A_beta^T G^k)
// Eight lanes per row (16-byte vectors strided by 8), a fixed xor tree over the eight: deterministic.
template <typename T>
__global__ void gat_dots_kernel(const char* __restrict__ G, const char* __restrict__ Z, const char* __restrict__ Y,
                                const char* __restrict__ Zp, const char* __restrict__ X, int64_t n, int32_t nvec,
                                float* __restrict__ w, float* __restrict__ gy, float* __restrict__ zx, int accumulate) {
    constexpr int VALS = 16 / sizeof(T);
    const int sub = threadIdx.x & 7;
    const int64_t ld = (int64_t)nvec * 16;
    const int64_t groups = (int64_t)gridDim.x * (blockDim.x >> 3);
    for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3; v < n; v += groups) {
        float a = 0.f, b = 0.f, c = 0.f;
        for (int k = sub; k < nvec; k += 8) {
            const int64_t off = v * ld + 16 * k;
            float g[VALS], z[VALS], y[VALS], zp[VALS], x[VALS];
            load16<T>(G + off, g);
            load16<T>(Z + off, z);
            load16<T>(Y + off, y);
            load16<T>(Zp + off, zp);
            load16<T>(X + off, x);
#pragma unroll
            for (int i = 0; i < VALS; ++i) {
                a = fmaf(g[i], z[i], a);
                b = fmaf(g[i], y[i], b);
                c = fmaf(zp[i], x[i], c);
            }
        }
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
            c += __shfl_xor_sync(0xffffffffu, c, o);
        }
        if (sub == 0) {
            w[v] = accumulate ? w[v] + a : a;
            gy[v] = accumulate ? gy[v] + b : b;
            zx[v] = accumulate ? zx[v] + c : c;
        }
    }
}

// G4 softmax + LeakyReLU backward without per-arc gradients: with ds_uv = beta_uv (dalpha_uv - w_v),
//   ps_u = sum_v ds_uv = zx_u - q_u,  q_u = sum_v beta_uv w_v (out-CSR row u, self loop included)
//   pd_v = sum_u ds_uv = gy_v - w_v b_v
template <class Red>
__device__ void pspd_row(const Red& R, int64_t u, const int32_t* __restrict__ rp_out, const int32_t* __restrict__ col_out,
                         const float* __restrict__ bt, const float* __restrict__ w, const float* __restrict__ gy,
                         const float* __restrict__ zx, const float* __restrict__ bsum, int64_t n, float slope,
                         float* __restrict__ ps, float* __restrict__ pd) {
    float q = R.t == 0 ? word_beta(bt[u], slope) * w[u] : 0.f;
    for (int j = rp_out[u] + R.t; j < rp_out[u + 1]; j += R.T) q = fmaf(word_beta(bt[n + j], slope), w[col_out[j]], q);
    q = R.sum(q);
    if (R.t == 0) {
        ps[u] = zx[u] - q;
        pd[u] = gy[u] - w[u] * bsum[u];
    }
}

// rows [lo, hi) only: ps / pd feed this rank's own rows (dz, da), so each rank evaluates its own share
__global__ void gat_pspd_kernel(const int32_t* __restrict__ rp_out, const int32_t* __restrict__ col_out,
                                const float* __restrict__ bt, const float* __restrict__ w, const float* __restrict__ gy,
                                const float* __restrict__ zx, const float* __restrict__ bsum, int64_t n, float slope,
                                float* __restrict__ ps, float* __restrict__ pd, int64_t lo, int64_t hi) {
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const WarpRed R;
    for (int64_t u = lo + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); u < hi; u += warps)
        if (rp_out[u + 1] - rp_out[u] <= kBigDeg) pspd_row(R, u, rp_out, col_out, bt, w, gy, zx, bsum, n, slope, ps, pd);
}

__global__ void __launch_bounds__(256) gat_pspd_big_kernel(const int32_t* __restrict__ big, int32_t nbig,
                                                           const int32_t* __restrict__ rp_out,
                                                           const int32_t* __restrict__ col_out,
                                                           const float* __restrict__ bt, const float* __restrict__ w,
                                                           const float* __restrict__ gy, const float* __restrict__ zx,
                                                           const float* __restrict__ bsum, int64_t n, float slope,
                                                           float* __restrict__ ps, float* __restrict__ pd, int64_t lo,
                                                           int64_t hi) {
    __shared__ float sh[32];
    const BlockRed R(sh);
    for (int i = blockIdx.x; i < nbig; i += gridDim.x)
        if (big[i] >= lo && big[i] < hi) pspd_row(R, big[i], rp_out, col_out, bt, w, gy, zx, bsum, n, slope, ps, pd);
}

// dz[v] += ps_v a_src + pd_v a_dst (own rows)
__global__ void gat_dz_kernel(float* __restrict__ dz, int64_t ld, int32_t C, const float* __restrict__ att,
                              const float* __restrict__ ps, const float* __restrict__ pd, int64_t rows, int64_t row0,
                              int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * C; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i / C;
        const int c = (int)(i % C);
        const int64_t gr = row0 + v;
        if (gr >= n) continue;
        dz[v * ld + c] = fmaf(pd[gr], att[C + c], fmaf(ps[gr], att[c], dz[v * ld + c]));
    }
}

// da partials: block b sums own rows v = b, b + nb, ...: part[b][c] = sum ps_v z_v[c], part[b][C + c] = sum pd_v z_v[c]
__global__ void gat_da_partial_kernel(const float* __restrict__ z, int64_t ldz, int32_t C, const float* __restrict__ ps,
                                      const float* __restrict__ pd, int64_t rows, int64_t row0, int64_t n,
                                      float* __restrict__ part) {
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
        float as = 0.f, ad = 0.f;
        for (int64_t v = blockIdx.x; v < rows && row0 + v < n; v += gridDim.x) {
            const float x = z[v * ldz + c];
            as = fmaf(ps[row0 + v], x, as);
            ad = fmaf(pd[row0 + v], x, ad);
        }
        part[(int64_t)blockIdx.x * 2 * C + c] = as;
        part[(int64_t)blockIdx.x * 2 * C + C + c] = ad;
    }
}

__global__ void gat_sum_parts_kernel(const float* __restrict__ part, int nb, int len, float* __restrict__ out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) {
        float acc = 0.f;
        for (int b = 0; b < nb; ++b) acc += part[(int64_t)b * len + i];   // fixed block order
        out[i] = acc;
    }
}

int wblocks(int64_t rows) { return (int)std::min<int64_t>(std::max<int64_t>(cdiv(rows, 8), 1), 148 * 16); }
int eblk(int64_t total) { return (int)std::min<int64_t>(std::max<int64_t>(cdiv(total, 256), 1), 148 * 16); }
inline int64_t r4(int64_t x) { return (x + 3) / 4 * 4; }

}  // namespace

void train_epoch_gat(ntp_ctx* c, const ntp_model* m, const ntp_tensor* X_v, const int32_t* lab, const uint8_t* msk,
                     ntp_tensor* W0, ntp_tensor* W1, ntp_tensor* att, float slope, ntp_epoch_report* rep,
                     cudaStream_t user) {
    const Graph& g = c->g;
    NTP_CHECK(!g.reordered, NTP_ERR_CONFIG, "the GAT epoch needs a graph without NTP_G_REORDER");
    drop_epoch_graph(c);   // buffers below may move ones a captured decoupled epoch points into
    cudaStream_t s = c->s_comp;
    const int64_t launches0 = c->launches;
    const int W = c->world, vs = c->vs, P = nslices(c);
    const int64_t n = g.n, nnz = g.nnz, na = n + nnz;
    const int64_t V_pad = (int64_t)P * cdiv(n, P), V_p = V_pad / W, row0 = (int64_t)c->rank * V_p;
    const int32_t C = m->C;
    const ntp_dtype dt = m->dtype;
    const size_t es = esize(dt);
    const int32_t d_s = slice_width(C, P, dt, c->slice_align);
    const int64_t slice = V_pad * d_s, feat = (int64_t)vs * slice;   // elements: one slice / this rank's slices
    const bool local = W == 1;
    auto sl = [&](void* base, int64_t i) -> void* { return static_cast<char*>(base) + (size_t)i * slice * es; };

    NTP_CUDA(cudaEventRecord(c->ev[40], user ? user : (cudaStream_t)0));
    NTP_CUDA(cudaStreamWaitEvent(s, c->ev[40], 0));
    cudaEvent_t* E = c->ev;
    int ei = 0;
    wire_reset(c);
    c->hop_ev_used = 0;
    NTP_CUDA(record_timing(c, E[ei++], s));   // E0

    // ---- operands: 16-byte pitches for the TMA GEMMs, weights split once into {hi, lo} tf32
    const int64_t ldXp = r4(m->d_in), ldH = r4(m->hid), ldL = r4(C);
    const float* X = static_cast<const float*>(X_v->data);
    int64_t ldx = X_v->ld;
    if ((ldx % 4) != 0 || (reinterpret_cast<uintptr_t>(X) % 16) != 0) {
        c->m_Xs.ensure((size_t)V_p * ldXp * sizeof(float));
        NTP_CUDA(cudaMemcpy2DAsync(c->m_Xs.p, ldXp * sizeof(float), X, ldx * sizeof(float), m->d_in * sizeof(float),
                                   V_p, cudaMemcpyDeviceToDevice, s));
        X = c->m_Xs.as<float>();
        ldx = ldXp;
    }
    float* W0u = static_cast<float*>(W0->data);
    float* W1u = static_cast<float*>(W1->data);
    float* attu = static_cast<float*>(att->data);
    c->m_W0p.ensure((size_t)m->d_in * ldH * sizeof(float));
    c->m_W1p.ensure((size_t)m->hid * ldL * sizeof(float));
    NTP_CUDA(cudaMemcpy2DAsync(c->m_W0p.p, ldH * sizeof(float), W0u, m->hid * sizeof(float), m->hid * sizeof(float),
                               m->d_in, cudaMemcpyDeviceToDevice, s));
    NTP_CUDA(cudaMemcpy2DAsync(c->m_W1p.p, ldL * sizeof(float), W1u, C * sizeof(float), C * sizeof(float), m->hid,
                               cudaMemcpyDeviceToDevice, s));
    const float* W0g = c->m_W0p.as<float>();
    const float* W1g = c->m_W1p.as<float>();
    c->m_Wsplit.ensure((size_t)2 * ((int64_t)m->d_in * ldH + (int64_t)m->hid * ldL) * sizeof(float));
    float* w0h = c->m_Wsplit.as<float>();
    float* w0l = w0h + (int64_t)m->d_in * ldH;
    float* w1h = w0l + (int64_t)m->d_in * ldH;
    float* w1l = w1h + (int64_t)m->hid * ldL;
    tf32_split(c, W0g, m->d_in, m->hid, ldH, w0h, w0l, s);
    tf32_split(c, W1g, m->hid, C, ldL, w1h, w1l, s);

    // ---- buffers
    c->m_H1.ensure((size_t)V_p * ldH * sizeof(float));
    c->m_L.ensure((size_t)V_p * ldL * sizeof(float));
    c->m_dL.ensure((size_t)V_p * ldL * sizeof(float));
    c->m_dH1.ensure((size_t)V_p * ldH * sizeof(float));
    const int64_t n_w = (int64_t)m->d_in * m->hid + (int64_t)m->hid * C;
    c->m_dW.ensure((size_t)(n_w + 2 * C) * sizeof(float));
    c->m_scal.ensure(4 * sizeof(double));
    c->gat_fg.ensure((size_t)2 * V_pad * sizeof(float) + 16);
    c->gat_msum.ensure((size_t)2 * n * sizeof(float) + 16);
    c->gat_alpha.ensure((size_t)na * sizeof(float) + 16);     // coefficient words, in-CSR order
    c->gat_alpha_t.ensure((size_t)na * sizeof(float) + 16);   // coefficient words, out-CSR order
    c->gat_pspd.ensure((size_t)6 * n * sizeof(float) + 16);       // ps | pd | w | gy | zx | b
    c->gat_Z.ensure((size_t)(2 * m->K + 1) * feat * es + 16);     // Z^0..Z^K, Y^1..Y^K
    c->gat_X.ensure((size_t)slice * es + 16);
    c->recv.ensure((size_t)feat * es + 16);
    c->xfer.ensure((size_t)feat * es + 16);
    c->send.ensure((size_t)feat * es + 16);
    const int nbda = 148 * 2;
    c->gat_da.ensure((size_t)nbda * 2 * C * sizeof(float) + 16);
    const int64_t loss_blocks = std::min<int64_t>(cdiv(V_p, 8), 148 * 8);
    c->m_part.ensure((size_t)loss_blocks * (sizeof(double) + sizeof(int64_t)) + 16);
    const char* gpe = getenv("NTP_GAT_PERMUTE");   // dev switch, read per call (tests compare both)
    const bool permute = gpe && atoi(gpe) != 0;
    if (permute && c->gat_perm_version != c->g_version) {   // out-CSR arc -> in-CSR arc
        c->gat_perm.ensure((size_t)std::max<int64_t>(nnz, 1) * sizeof(int32_t));
        gat_perm_kernel<<<wblocks(n), 256, 0, s>>>(g.fwd().row_ptr.as<int32_t>(), g.fwd().col.as<int32_t>(),
                                                  g.bwd().row_ptr.as<int32_t>(), g.bwd().col.as<int32_t>(), n,
                                                  c->gat_perm.as<int32_t>());
        NTP_LAUNCH_CHECK();
        count_launch(c);
        c->gat_perm_version = c->g_version;
    }
    if (c->gat_big_version != c->g_version) {
        const Csr& in = g.fwd();
        const Csr& out = g.bwd();
        // hub rows (> kBigDeg arcs) of both CSRs: one CTA each in the per-row reductions
        c->gat_big.ensure((size_t)2 * (n + 1) * sizeof(int32_t) + 16);
        DevBuf cnt;
        cnt.ensure(2 * sizeof(int32_t));
        NTP_CUDA(cudaMemsetAsync(cnt.p, 0, 2 * sizeof(int32_t), s));
        gat_big_rows_kernel<<<eblk(n), 256, 0, s>>>(in.row_ptr.as<int32_t>(), n, c->gat_big.as<int32_t>(), cnt.as<int32_t>());
        gat_big_rows_kernel<<<eblk(n), 256, 0, s>>>(out.row_ptr.as<int32_t>(), n, c->gat_big.as<int32_t>() + n + 1,
                                                   cnt.as<int32_t>() + 1);
        NTP_LAUNCH_CHECK();
        int32_t h[2];
        NTP_CUDA(cudaMemcpyAsync(h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, s));
        NTP_CUDA(cudaStreamSynchronize(s));
        c->gat_nbig[0] = h[0];
        c->gat_nbig[1] = h[1];
        count_launch(c, 2);
        c->gat_big_version = c->g_version;
    }
    const int32_t* big_in = c->gat_big.as<int32_t>();
    const int32_t* big_out = big_in + n + 1;
    float* H1 = c->m_H1.as<float>();
    float* z = c->m_L.as<float>();
    float* dz = c->m_dL.as<float>();
    float* dH1 = c->m_dH1.as<float>();
    float* dW0 = c->m_dW.as<float>();
    float* dW1 = dW0 + (int64_t)m->d_in * m->hid;
    float* da = dW0 + n_w;
    double* scal = c->m_scal.as<double>();
    double* part = c->m_part.as<double>();
    int64_t* cnt = reinterpret_cast<int64_t*>(part + loss_blocks);
    float* fg = c->gat_fg.as<float>();
    float* alpha = c->gat_alpha.as<float>();
    float* alpha_t = c->gat_alpha_t.as<float>();
    float* ps = c->gat_pspd.as<float>();
    float* pd = ps + n;
    float* wv = ps + 2 * n;
    float* gy = ps + 3 * n;
    float* zx = ps + 4 * n;
    float* bsum = ps + 5 * n;
    const int32_t* perm = c->gat_perm.as<int32_t>();
    void* Zst = c->gat_Z.p;   // Z^k slice j at sl(Zst, k*vs + j); Y^k slice j at sl(Zst, (K + k)*vs + j)
    void* Xs = c->gat_X.p;

    // rows [n, V_pad) of every slice are padding (never written by a hop, exchanged as zeros)
    if (V_pad > n)
        for (int64_t i = 0; i < (int64_t)(2 * m->K + 1) * vs; ++i)
            NTP_CUDA(cudaMemsetAsync(static_cast<char*>(sl(Zst, i)) + n * d_s * es, 0, (V_pad - n) * d_s * es, s));
    if (V_pad > n)
        for (int j = 0; j < vs; ++j)
            for (void* b : {c->recv.p, c->xfer.p})
                NTP_CUDA(cudaMemsetAsync(static_cast<char*>(sl(b, j)) + n * d_s * es, 0, (V_pad - n) * d_s * es, s));

    // ---- G1: z = ReLU(X W0) W1 on this rank's rows
    epoch_gemm(c, false, false, V_p, m->hid, m->d_in, X, ldx, W0g, ldH, H1, ldH, s, 1, nullptr, 0, w0h, w0l);
    epoch_gemm(c, false, false, V_p, C, m->hid, H1, ldH, W1g, ldL, z, ldL, s, 0, nullptr, 0, w1h, w1l);
    NTP_CUDA(record_timing(c, E[ei++], s));   // E1 mlp fwd

    // ---- G2: attention, data-parallel halves then every destination's softmax
    gat_fg_kernel<<<wblocks(V_p), 256, 0, s>>>(z, ldL, C, attu, V_p, row0, n, fg);
    NTP_LAUNCH_CHECK();
    count_launch(c);
    if (!local) NTP_NCCL(ncclAllGather(fg + 2 * row0, fg, (size_t)2 * V_p, ncclFloat32, c->comm, s));
    float* msum = c->gat_msum.as<float>();
    gat_softmax_kernel<<<wblocks(n), 256, 0, s>>>(g.fwd().row_ptr.as<int32_t>(), g.fwd().col.as<int32_t>(), fg, n, slope,
                                                 alpha, msum, bsum);
    if (c->gat_nbig[0] > 0)
        gat_softmax_big_kernel<<<std::min(c->gat_nbig[0], 148 * 8), 256, 0, s>>>(
            big_in, c->gat_nbig[0], g.fwd().row_ptr.as<int32_t>(), g.fwd().col.as<int32_t>(), fg, n, slope, alpha,
            msum, bsum);
    NTP_LAUNCH_CHECK();
    if (permute) {
        gat_permute_kernel<<<eblk(na), 256, 0, s>>>(alpha, perm, n, nnz, alpha_t);
    } else {
        const int at_blocks = (int)std::min<int64_t>(std::max<int64_t>(cdiv(nnz, kAtArcs * 8), 1) + 64, 148 * 16);
        gat_coef_t_kernel<<<at_blocks, 256, 0, s>>>(g.bwd().row_ptr.as<int32_t>(), g.bwd().col.as<int32_t>(), fg, msum,
                                                    alpha, n, nnz, slope, alpha_t);
    }
    NTP_LAUNCH_CHECK();
    count_launch(c, 2 + (c->gat_nbig[0] > 0 ? 1 : 0));

    // ---- a3: split z (no pre-scale: the attention operator carries its own normalisation)
    pack_v2f(c, z, ldL, C, local ? Zst : c->send.p, V_p, d_s, P, nullptr, row0, n, NTP_F32, dt, s);
    if (!local) exchange_v2f(c, c->send.p, Zst, V_p * d_s, dt, s);
    NTP_CUDA(record_timing(c, E[ei++], s));   // E2 v2f

    // ---- G3 / a4: K weighted hops per slice, every level kept for the backward's SDDMM
    // one pass, two sums: out = gamma A_att in (alpha) and out2 = gamma A_beta in (beta), from the signed words
    auto hop = [&](const void* in, void* out, void* out2, bool transposed) {
        const bool tm = c->hop_ev_used + 2 <= kHopEvents;
        if (tm) NTP_CUDA(record_timing(c, c->hop_ev[c->hop_ev_used], s));
        const float* co = transposed ? alpha_t : alpha;
        spmm_hop(c, transposed ? g.bwd() : g.fwd(), nullptr, nullptr, in, out, nullptr, d_s, d_s, d_s, d_s, dt,
                 m->gamma, 0.f, 1, 0, -1, s, nullptr, nullptr, co + n, co, out2, slope);
        if (tm) {
            NTP_CUDA(record_timing(c, c->hop_ev[c->hop_ev_used + 1], s));
            c->hop_ev_used += 2;
        }
    };
    // ... and, in the same pass, Y^k = gamma A_beta Z^{k-1} (beta = alpha * LeakyReLU'): the attention
    // backward's per-vertex form needs it (below)
    for (int k = 1; k <= m->K; ++k)
        for (int j = 0; j < vs; ++j)
            hop(sl(Zst, (int64_t)(k - 1) * vs + j), sl(Zst, (int64_t)k * vs + j), sl(Zst, (int64_t)(m->K + k) * vs + j),
                false);
    NTP_CUDA(record_timing(c, E[10], s));   // fwd hops done
    // a5: gather Z^K into this rank's rows, blocked [P][V_p][d_s]
    c->wire_phase = 1;
    void* ZK = sl(Zst, (int64_t)m->K * vs);
    void* gathered = ZK;
    if (!local) {
        exchange_f2v(c, ZK, c->send.p, V_p * d_s, dt, s);
        gathered = c->send.p;
    }
    NTP_CUDA(record_timing(c, E[ei++], s));   // E3 prop fwd + f2v

    // ---- a6: loss and dlogits (1/N_train folded into SGD), blocked gradient -> split
    c->wire_phase = 2;
    void* gsend = local ? c->recv.p : c->xfer.p;
    const int64_t nb = epoch_loss(c, gathered, dt, 1, V_p, d_s, C, lab, msk, row0, n, gsend, dt, 1, nullptr, part, cnt, 0, s);
    epoch_zero_pad_cols(c, gsend, dt, V_p, d_s, P, C, s);
    epoch_reduce_loss(c, part, cnt, nb, scal, s);
    NTP_CUDA(record_timing(c, E[ei++], s));   // E4 loss
    if (!local) {
        exchange_v2f(c, c->xfer.p, c->recv.p, V_p * d_s, dt, s);
        if (V_pad > n)   // xfer held the blocked gradient; as a slice its padding rows must read zero again
            for (int j = 0; j < vs; ++j)
                NTP_CUDA(cudaMemsetAsync(static_cast<char*>(sl(c->xfer.p, j)) + n * d_s * es, 0, (V_pad - n) * d_s * es, s));
    }
    NTP_CUDA(record_timing(c, E[ei++], s));   // E5 v2f bwd

    // per-vertex dot products of one level / slice (gat_dots_kernel), accumulated over levels and slices
    const int32_t nvec = (int32_t)(d_s * es / 16);
    auto dots = [&](const void* Gk, const void* Zk, const void* Yk, const void* Zp, int acc) {
        const int blocks = (int)std::min<int64_t>(cdiv(n, 32), 148 * 16);
        if (dt == NTP_F32)
            gat_dots_kernel<float><<<blocks, 256, 0, s>>>(static_cast<const char*>(Gk), static_cast<const char*>(Zk),
                                                          static_cast<const char*>(Yk), static_cast<const char*>(Zp),
                                                          static_cast<const char*>(Xs), n, nvec, wv, gy, zx, acc);
        else
            gat_dots_kernel<__nv_bfloat16><<<blocks, 256, 0, s>>>(
                static_cast<const char*>(Gk), static_cast<const char*>(Zk), static_cast<const char*>(Yk),
                static_cast<const char*>(Zp), static_cast<const char*>(Xs), n, nvec, wv, gy, zx, acc);
        NTP_LAUNCH_CHECK();
        count_launch(c);
    };

    // ---- G4 / a8: G^{k-1} = gamma A_att^T G^k per slice, X^k = gamma A_beta^T G^k, and the per-vertex dots.
    // The attention gradient dalpha_uv = gamma sum_k G^k_v . Z^{k-1}_u is never formed per arc: the softmax /
    // LeakyReLU backward needs only its contractions with alpha and beta, which the hops already carry --
    //   w_v = sum_u alpha_uv dalpha_uv = sum_k G^k_v . Z^k_v,   sum_u beta_uv dalpha_uv = sum_k G^k_v . Y^k_v,
    //   sum_v beta_uv dalpha_uv = sum_k Z^{k-1}_u . X^k_u
    // -- n-long partial sums per slice instead of an nnz-long SDDMM (and its allreduce).
    c->wire_phase = 3;
    void* cur = c->recv.p;
    void* nxt = c->xfer.p;
    for (int i = 0; i < m->K; ++i) {
        const int k = m->K - i;
        for (int j = 0; j < vs; ++j) {
            const void* Gj = sl(cur, j);
            hop(Gj, sl(nxt, j), Xs, true);
            dots(Gj, sl(Zst, (int64_t)k * vs + j), sl(Zst, (int64_t)(m->K + k) * vs + j),
                 sl(Zst, (int64_t)(k - 1) * vs + j), (i > 0 || j > 0) ? 1 : 0);
        }
        std::swap(cur, nxt);
    }
    NTP_CUDA(record_timing(c, E[11], s));   // bwd hops (+ dots) done
    // a9: gather G^0 -> dz rows
    void* gathered_b = cur;
    if (!local) {
        exchange_f2v(c, cur, c->send.p, V_p * d_s, dt, s);
        gathered_b = c->send.p;
    }
    unpack_f2v(c, gathered_b, V_p, d_s, P, dz, ldL, C, dt, NTP_F32, s);
    NTP_CUDA(record_timing(c, E[ei++], s));   // E6 prop bwd + f2v

    // ---- attention backward (every rank holds every coefficient): the dots summed over ranks (3n floats),
    // then ps / pd per vertex
    if (!local) NTP_NCCL(ncclAllReduce(wv, wv, (size_t)3 * n, ncclFloat32, ncclSum, c->comm, s));
    const int64_t own_lo = std::min(row0, n), own_hi = std::min(row0 + V_p, n);   // this rank's rows
    gat_pspd_kernel<<<wblocks(std::max<int64_t>(own_hi - own_lo, 1)), 256, 0, s>>>(
        g.bwd().row_ptr.as<int32_t>(), g.bwd().col.as<int32_t>(), alpha_t, wv, gy, zx, bsum, n, slope, ps, pd, own_lo,
        own_hi);
    if (c->gat_nbig[1] > 0)
        gat_pspd_big_kernel<<<std::min(c->gat_nbig[1], 148 * 8), 256, 0, s>>>(
            big_out, c->gat_nbig[1], g.bwd().row_ptr.as<int32_t>(), g.bwd().col.as<int32_t>(), alpha_t, wv, gy, zx, bsum,
            n, slope, ps, pd, own_lo, own_hi);
    NTP_LAUNCH_CHECK();
    gat_dz_kernel<<<eblk(V_p * C), 256, 0, s>>>(dz, ldL, C, attu, ps, pd, V_p, row0, n);
    NTP_LAUNCH_CHECK();
    gat_da_partial_kernel<<<nbda, 256, 0, s>>>(z, ldL, C, ps, pd, V_p, row0, n, c->gat_da.as<float>());
    NTP_LAUNCH_CHECK();
    gat_sum_parts_kernel<<<eblk(2 * C), 256, 0, s>>>(c->gat_da.as<float>(), nbda, 2 * C, da);
    NTP_LAUNCH_CHECK();
    count_launch(c, 4 + (c->gat_nbig[1] > 0 ? 1 : 0));

    // ---- a10: MLP backward
    epoch_gemm(c, true, false, m->hid, C, V_p, H1, ldH, dz, ldL, dW1, C, s, 0, nullptr, 0, nullptr, nullptr);
    epoch_gemm(c, false, true, V_p, m->hid, C, dz, ldL, W1g, ldL, dH1, ldH, s, 2, H1, ldH, w1h, w1l);
    epoch_gemm(c, true, false, m->d_in, m->hid, V_p, X, ldx, dH1, ldH, dW0, m->hid, s, 0, nullptr, 0, nullptr, nullptr);
    NTP_CUDA(record_timing(c, E[ei++], s));   // E7 mlp bwd

    // ---- a11: allreduce (dW0 | dW1 | da_src | da_dst) and the loss; SGD on W0, W1, a
    if (!local) {
        NTP_NCCL(ncclGroupStart());
        NTP_NCCL(ncclAllReduce(dW0, dW0, (size_t)(n_w + 2 * C), ncclFloat32, ncclSum, c->comm, s));
        NTP_NCCL(ncclAllReduce(scal, scal, 2, ncclFloat64, ncclSum, c->comm, s));
        NTP_NCCL(ncclGroupEnd());
    }
    NTP_CUDA(record_timing(c, E[ei++], s));   // E8 allreduce
    epoch_sgd(c, W0u, (int64_t)m->d_in * m->hid, dW0, scal, m->lr, s);
    epoch_sgd(c, W1u, (int64_t)m->hid * C, dW1, scal, m->lr, s);
    epoch_sgd(c, attu, 2 * C, da, scal, m->lr, s);
    NTP_CUDA(record_timing(c, E[ei++], s));   // E9 sgd

    double h_scal[2] = {0, 0};
    NTP_CUDA(cudaMemcpyAsync(h_scal, scal, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    NTP_CUDA(cudaEventRecord(c->ev[41], s));
    NTP_CUDA(cudaStreamWaitEvent(user ? user : (cudaStream_t)0, c->ev[41], 0));
    wait_stream(c, s);
    if (rep) {
        rep->loss = h_scal[1] > 0 ? h_scal[0] / h_scal[1] : 0.0;
        rep->n_train = (int64_t)h_scal[1];
        epoch_phases(E, rep->ms);
        for (int i = 0; i < 4; ++i) {
            rep->bytes_sent[i] = c->wire_sent[i];
            rep->bytes_recv[i] = c->wire_recv[i];
        }
        rep->collectives = local ? 0 : 7;   // 4 layout changes, all-gather (f, g), allreduce dalpha, allreduce dW
        rep->kernel_launches = c->launches - launches0;
        int nh = 0;
        rep->spmm_ms = collect_hop_ms(c, &nh);
        rep->spmm_launches = nh;
    }
}

}  // namespace ntp
