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
//     with the coefficients permuted into its order (perm: out-CSR arc -> in-CSR arc, built once).
//   * Backward: dalpha_uv = gamma sum_k G^k_v . Z^{k-1}_u is an SDDMM on every slice (partial dot products
//     over d_s columns), summed over slices and -- one allreduce of n + nnz floats -- over ranks; softmax /
//     LeakyReLU backward and the per-vertex sums ps (over out-arcs, via the out-CSR) and pd (over in-arcs)
//     then give dz += ps a_src + pd a_dst and da_src = sum ps z, da_dst = sum pd z (rank-1 terms).
// Coefficient layout everywhere: [n self loops | nnz arcs in in-CSR order] (the oracle's arcs() order).
#include <algorithm>
#include <cmath>

#include "ntp_internal.cuh"

namespace ntp {

namespace {

__device__ __forceinline__ float leaky(float x, float slope) { return x > 0.f ? x : slope * x; }

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
// gather of f -- stored in alpha's slot, an online max / sum per thread combined over the group, and the
// sign of s_uv (> 0) as one bit per arc (the backward's LeakyReLU'), ballot-packed per warp; (2) alpha =
// exp(e - m) / sum from the stored e (coalesced).
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
                            uint32_t* __restrict__ pos_bits) {
    const int lane = threadIdx.x & 31;
    const float gv = fg[2 * v + 1];
    const float ss = fg[2 * v] + gv;
    const float es = leaky(ss, slope);
    if (R.t == 0 && ss > 0.f) atomicOr(pos_bits + (v >> 5), 1u << (v & 31));
    const int b = rp[v], e = rp[v + 1];
    float m = -INFINITY, sm = 0.f;
    if (R.t == 0) m = es, sm = 1.f;
    for (int jb = b + (R.t - lane); jb < e; jb += R.T) {   // this warp's 32 consecutive arcs jb .. jb + 31
        const int j = jb + lane;
        bool pos = false;
        if (j < e) {
            const float sj = fg[2 * (int64_t)col[j]] + gv;
            const float ej = leaky(sj, slope);
            pos = sj > 0.f;
            alpha[n + j] = ej;
            online_add(m, sm, ej);
        }
        const uint32_t word = __ballot_sync(0xffffffffu, pos);
        if (lane == 0 && word) {
            const int64_t a = n + jb;                                // bit index of arc jb
            atomicOr(pos_bits + (a >> 5), word << (a & 31));
            if (a & 31) atomicOr(pos_bits + (a >> 5) + 1, word >> (32 - (a & 31)));
        }
    }
    R.combine(m, sm);
    if (R.t == 0) alpha[v] = expf(es - m) / sm;
    for (int j = b + R.t; j < e; j += R.T) alpha[n + j] = expf(alpha[n + j] - m) / sm;
}

__global__ void gat_softmax_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                   const float* __restrict__ fg, int64_t n, float slope, float* __restrict__ alpha,
                                   uint32_t* __restrict__ pos_bits) {
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const WarpRed R;
    for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += warps)
        if (rp[v + 1] - rp[v] <= kBigDeg) softmax_row(R, v, rp, col, fg, n, slope, alpha, pos_bits);
}

__global__ void __launch_bounds__(256) gat_softmax_big_kernel(const int32_t* __restrict__ big, int32_t nbig,
                                                              const int32_t* __restrict__ rp,
                                                              const int32_t* __restrict__ col,
                                                              const float* __restrict__ fg, int64_t n, float slope,
                                                              float* __restrict__ alpha, uint32_t* __restrict__ pos_bits) {
    __shared__ float sh[32];
    const BlockRed R(sh);
    for (int i = blockIdx.x; i < nbig; i += gridDim.x) softmax_row(R, big[i], rp, col, fg, n, slope, alpha, pos_bits);
}

// rows of more than kBigDeg arcs (list built once per graph; order irrelevant: rows are independent)
__global__ void gat_big_rows_kernel(const int32_t* __restrict__ rp, int64_t n, int32_t* __restrict__ list,
                                    int32_t* __restrict__ cnt) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        if (rp[v + 1] - rp[v] > kBigDeg) list[atomicAdd(cnt, 1)] = (int32_t)v;
}

// out-CSR arc j' (row u, column v) -> its in-CSR index (u's position in row v)
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

__global__ void gat_permute_kernel(const float* __restrict__ a, const int32_t* __restrict__ perm, int64_t n, int64_t nnz,
                                   float* __restrict__ at) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n + nnz; i += (int64_t)gridDim.x * blockDim.x)
        at[i] = i < n ? a[i] : a[n + perm[i - n]];
}

template <typename T> __device__ __forceinline__ float ldx(const T* p);
template <> __device__ __forceinline__ float ldx<float>(const float* p) { return *p; }
template <> __device__ __forceinline__ float ldx<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }

// G4 SDDMM: dalpha[j] (+)= gamma * G_v . Z_u over this slice's d_s columns (arc j: self loops first).
// Arcs are cut into ranges of kSdArcs consecutive in-CSR arcs, one warp per range (hubs spread over many
// warps).  A step covers E arcs: lane = e * VPP + c holds 16-byte vector c of arc e's two rows (G_v cached
// in L1 across a row's arcs, Z_u a random row gather like the hop's), multiplies in fp32 and reduces its
// group with a fixed xor tree; lane c = 0 of the group writes the arc.  The self loops are a separate
// streaming pass (j < n).
constexpr int kSdArcs = 2048;

// One arc per lane: lanes take consecutive arcs of a kSdArcs range (coalesced col / dalpha, the row of a lane
// advances monotonically), each lane reads the whole slice rows of its arc (NV 16-byte vectors of G_v --
// shared by the lanes of a row, so L1 -- and of the gathered Z_u) and sums the dot product in column order.
template <typename T, int NV>
__global__ void __launch_bounds__(256) gat_sddmm_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                        int64_t n, int64_t nnz, const char* __restrict__ G,
                                                        const char* __restrict__ Z, int32_t nvec, float gamma,
                                                        float* __restrict__ dalpha, int accumulate) {
    constexpr int VALS = 16 / sizeof(T);
    const int64_t ld = (int64_t)nvec * 16;   // NV == nvec, or NV = 16 chunks of a wider row
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    auto elem = [](const uint4& x, int i) {
        const uint32_t w[4] = {x.x, x.y, x.z, x.w};
        if (sizeof(T) == 4) return __uint_as_float(w[i]);
        return __uint_as_float((i & 1) ? (w[i >> 1] & 0xFFFF0000u) : (w[i >> 1] << 16));
    };
    auto dot = [&](const char* a, const char* b) {
        float d = 0.f;
        for (int k0 = 0; k0 < nvec; k0 += NV) {
            uint4 xa[NV], xb[NV];
#pragma unroll
            for (int k = 0; k < NV; ++k) {
                const bool ok = k0 + k < nvec;
                xa[k] = ok ? *reinterpret_cast<const uint4*>(a + 16 * (k0 + k)) : make_uint4(0, 0, 0, 0);
                xb[k] = ok ? __ldg(reinterpret_cast<const uint4*>(b + 16 * (k0 + k))) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int k = 0; k < NV; ++k)
#pragma unroll
                for (int i = 0; i < VALS; ++i) d = fmaf(elem(xa[k], i), elem(xb[k], i), d);
        }
        return d;
    };
    // self loops: arc v = G_v . Z_v
    for (int64_t v = warp * 32 + lane; v < n; v += nwarps * 32)
        dalpha[v] = (accumulate ? dalpha[v] : 0.f) + gamma * dot(G + v * ld, Z + v * ld);
    const int64_t nranges = (nnz + kSdArcs - 1) / kSdArcs;
    for (int64_t rg = warp; rg < nranges; rg += nwarps) {
        const int64_t a0 = rg * kSdArcs, a1 = min(a0 + (int64_t)kSdArcs, nnz);
        int64_t lo = 0, hi = n;   // v = last row with rp[v] <= a0
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (rp[mid] <= a0) lo = mid;
            else hi = mid;
        }
        int64_t v = lo;
        for (int64_t j = a0 + lane; j < a1; j += 32) {
            while (rp[v + 1] <= j) ++v;   // this lane's row (arcs are sorted by destination)
            const float d = dot(G + v * ld, Z + (int64_t)__ldg(col + j) * ld);
            dalpha[n + j] = (accumulate ? dalpha[n + j] : 0.f) + gamma * d;
        }
    }
}

// G4 softmax + LeakyReLU backward per destination: ds[j]; pd[v] = sum of v's ds (self + in-arcs).  The
// LeakyReLU' of every arc comes from the forward's sign bits: no gather of f.
template <class Red>
__device__ void softmax_bwd_row(const Red& R, int64_t v, const int32_t* __restrict__ rp,
                                const uint32_t* __restrict__ pos_bits, const float* __restrict__ alpha,
                                const float* __restrict__ dalpha, int64_t n, float slope, float* __restrict__ ds,
                                float* __restrict__ pd) {
    auto pos = [&](int64_t a) { return (pos_bits[a >> 5] >> (a & 31)) & 1u; };
    const int b = rp[v], e = rp[v + 1];
    float w = R.t == 0 ? alpha[v] * dalpha[v] : 0.f;
    for (int j = b + R.t; j < e; j += R.T) w = fmaf(alpha[n + j], dalpha[n + j], w);
    w = R.sum(w);
    float acc = 0.f;
    if (R.t == 0) {
        const float d = alpha[v] * (dalpha[v] - w) * (pos(v) ? 1.f : slope);
        ds[v] = d;
        acc = d;
    }
    for (int j = b + R.t; j < e; j += R.T) {
        const float d = alpha[n + j] * (dalpha[n + j] - w) * (pos(n + j) ? 1.f : slope);
        ds[n + j] = d;
        acc += d;
    }
    acc = R.sum(acc);
    if (R.t == 0) pd[v] = acc;
}

__global__ void gat_softmax_bwd_kernel(const int32_t* __restrict__ rp, const uint32_t* __restrict__ pos_bits,
                                       const float* __restrict__ alpha, const float* __restrict__ dalpha, int64_t n,
                                       float slope, float* __restrict__ ds, float* __restrict__ pd) {
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const WarpRed R;
    for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += warps)
        if (rp[v + 1] - rp[v] <= kBigDeg) softmax_bwd_row(R, v, rp, pos_bits, alpha, dalpha, n, slope, ds, pd);
}

__global__ void __launch_bounds__(256) gat_softmax_bwd_big_kernel(const int32_t* __restrict__ big, int32_t nbig,
                                                                  const int32_t* __restrict__ rp,
                                                                  const uint32_t* __restrict__ pos_bits,
                                                                  const float* __restrict__ alpha,
                                                                  const float* __restrict__ dalpha, int64_t n,
                                                                  float slope, float* __restrict__ ds,
                                                                  float* __restrict__ pd) {
    __shared__ float sh[32];
    const BlockRed R(sh);
    for (int i = blockIdx.x; i < nbig; i += gridDim.x) softmax_bwd_row(R, big[i], rp, pos_bits, alpha, dalpha, n, slope, ds, pd);
}

// ps[u] = ds of u's self loop + ds of every arc leaving u (out-CSR rows, coefficients through perm)
template <class Red>
__device__ void ps_row(const Red& R, int64_t u, const int32_t* __restrict__ rp_out, const int32_t* __restrict__ perm,
                       const float* __restrict__ ds, int64_t n, float* __restrict__ ps) {
    float acc = R.t == 0 ? ds[u] : 0.f;
    for (int j = rp_out[u] + R.t; j < rp_out[u + 1]; j += R.T) acc += ds[n + perm[j]];
    acc = R.sum(acc);
    if (R.t == 0) ps[u] = acc;
}

__global__ void gat_ps_kernel(const int32_t* __restrict__ rp_out, const int32_t* __restrict__ perm,
                              const float* __restrict__ ds, int64_t n, float* __restrict__ ps) {
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const WarpRed R;
    for (int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n; u += warps)
        if (rp_out[u + 1] - rp_out[u] <= kBigDeg) ps_row(R, u, rp_out, perm, ds, n, ps);
}

__global__ void __launch_bounds__(256) gat_ps_big_kernel(const int32_t* __restrict__ big, int32_t nbig,
                                                         const int32_t* __restrict__ rp_out,
                                                         const int32_t* __restrict__ perm, const float* __restrict__ ds,
                                                         int64_t n, float* __restrict__ ps) {
    __shared__ float sh[32];
    const BlockRed R(sh);
    for (int i = blockIdx.x; i < nbig; i += gridDim.x) ps_row(R, big[i], rp_out, perm, ds, n, ps);
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
    c->gat_alpha.ensure((size_t)na * sizeof(float) + 16);
    c->gat_alpha_t.ensure((size_t)na * sizeof(float) + 16);
    c->gat_dalpha.ensure((size_t)na * sizeof(float) + 16);
    c->gat_ds.ensure((size_t)na * sizeof(float) + 16);
    c->gat_pspd.ensure((size_t)2 * n * sizeof(float) + 16);
    c->gat_bits.ensure((size_t)cdiv(na, 32) * sizeof(uint32_t) + 16);
    c->gat_Z.ensure((size_t)(m->K + 1) * feat * es + 16);
    c->recv.ensure((size_t)feat * es + 16);
    c->xfer.ensure((size_t)feat * es + 16);
    c->send.ensure((size_t)feat * es + 16);
    const int nbda = 148 * 2;
    c->gat_da.ensure((size_t)nbda * 2 * C * sizeof(float) + 16);
    const int64_t loss_blocks = std::min<int64_t>(cdiv(V_p, 8), 148 * 8);
    c->m_part.ensure((size_t)loss_blocks * (sizeof(double) + sizeof(int64_t)) + 16);
    if (c->gat_perm_version != c->g_version) {   // out-CSR arc -> in-CSR arc, once per graph
        c->gat_perm.ensure((size_t)std::max<int64_t>(nnz, 1) * sizeof(int32_t));
        const Csr& in = g.fwd();
        const Csr& out = g.bwd();
        gat_perm_kernel<<<wblocks(n), 256, 0, s>>>(in.row_ptr.as<int32_t>(), in.col.as<int32_t>(),
                                                  out.row_ptr.as<int32_t>(), out.col.as<int32_t>(), n,
                                                  c->gat_perm.as<int32_t>());
        NTP_LAUNCH_CHECK();
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
        count_launch(c, 3);
        c->gat_perm_version = c->g_version;
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
    float* dalpha = c->gat_dalpha.as<float>();
    float* ds = c->gat_ds.as<float>();
    float* ps = c->gat_pspd.as<float>();
    float* pd = ps + n;
    const int32_t* perm = c->gat_perm.as<int32_t>();
    void* Zst = c->gat_Z.p;   // Z^k slice j at sl(Zst, k*vs + j)

    // rows [n, V_pad) of every slice are padding (never written by a hop, exchanged as zeros)
    if (V_pad > n)
        for (int64_t i = 0; i < (int64_t)(m->K + 1) * vs; ++i)
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
    NTP_CUDA(cudaMemsetAsync(c->gat_bits.p, 0, (size_t)cdiv(na, 32) * sizeof(uint32_t), s));
    gat_softmax_kernel<<<wblocks(n), 256, 0, s>>>(g.fwd().row_ptr.as<int32_t>(), g.fwd().col.as<int32_t>(), fg, n, slope,
                                                 alpha, c->gat_bits.as<uint32_t>());
    if (c->gat_nbig[0] > 0)
        gat_softmax_big_kernel<<<std::min(c->gat_nbig[0], 148 * 8), 256, 0, s>>>(
            big_in, c->gat_nbig[0], g.fwd().row_ptr.as<int32_t>(), g.fwd().col.as<int32_t>(), fg, n, slope, alpha,
            c->gat_bits.as<uint32_t>());
    NTP_LAUNCH_CHECK();
    gat_permute_kernel<<<eblk(na), 256, 0, s>>>(alpha, perm, n, nnz, alpha_t);
    NTP_LAUNCH_CHECK();
    count_launch(c, 2);

    // ---- a3: split z (no pre-scale: the attention operator carries its own normalisation)
    pack_v2f(c, z, ldL, C, local ? Zst : c->send.p, V_p, d_s, P, nullptr, row0, n, NTP_F32, dt, s);
    if (!local) exchange_v2f(c, c->send.p, Zst, V_p * d_s, dt, s);
    NTP_CUDA(record_timing(c, E[ei++], s));   // E2 v2f

    // ---- G3 / a4: K weighted hops per slice, every level kept for the backward's SDDMM
    auto hop = [&](const void* in, void* out, bool transposed) {
        const bool tm = c->hop_ev_used + 2 <= kHopEvents;
        if (tm) NTP_CUDA(record_timing(c, c->hop_ev[c->hop_ev_used], s));
        const float* co = transposed ? alpha_t : alpha;
        spmm_hop(c, transposed ? g.bwd() : g.fwd(), nullptr, nullptr, in, out, nullptr, d_s, d_s, d_s, d_s, dt,
                 m->gamma, 0.f, 1, 0, -1, s, nullptr, nullptr, co + n, co);
        if (tm) {
            NTP_CUDA(record_timing(c, c->hop_ev[c->hop_ev_used + 1], s));
            c->hop_ev_used += 2;
        }
    };
    for (int k = 1; k <= m->K; ++k)
        for (int j = 0; j < vs; ++j) hop(sl(Zst, (int64_t)(k - 1) * vs + j), sl(Zst, (int64_t)k * vs + j), false);
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

    // SDDMM launcher: E arcs per warp step by the slice's 16-byte vectors per row
    const int32_t nvec = (int32_t)(d_s * es / 16);
    const int sd_blocks = (int)std::min<int64_t>(std::max<int64_t>(cdiv(nnz, kSdArcs * 8), 1) + 64, 148 * 16);
    auto sddmm = [&](const void* Gj, const void* Zj, int acc) {
        const int64_t rp_n = n;
        const int32_t* rp = g.fwd().row_ptr.as<int32_t>();
        const int32_t* cl = g.fwd().col.as<int32_t>();
        const char* Gc = static_cast<const char*>(Gj);
        const char* Zc = static_cast<const char*>(Zj);
#define NTP_SDDMM(T, NV_) gat_sddmm_kernel<T, NV_><<<sd_blocks, 256, 0, s>>>(rp, cl, rp_n, nnz, Gc, Zc, nvec, m->gamma, dalpha, acc)
#define NTP_SDDMM_T(T) switch (nvec) { \
            case 1: NTP_SDDMM(T, 1); break; case 2: NTP_SDDMM(T, 2); break; case 3: NTP_SDDMM(T, 3); break; \
            case 4: NTP_SDDMM(T, 4); break; case 5: NTP_SDDMM(T, 5); break; case 6: NTP_SDDMM(T, 6); break; \
            case 7: NTP_SDDMM(T, 7); break; case 8: NTP_SDDMM(T, 8); break; case 9: NTP_SDDMM(T, 9); break; \
            case 10: NTP_SDDMM(T, 10); break; case 11: NTP_SDDMM(T, 11); break; case 12: NTP_SDDMM(T, 12); break; \
            case 13: NTP_SDDMM(T, 13); break; case 14: NTP_SDDMM(T, 14); break; case 15: NTP_SDDMM(T, 15); break; \
            default: NTP_SDDMM(T, 16); }
        if (dt == NTP_F32) { NTP_SDDMM_T(float) }
        else { NTP_SDDMM_T(__nv_bfloat16) }
#undef NTP_SDDMM_T
#undef NTP_SDDMM
        NTP_LAUNCH_CHECK();
    };

    // ---- G4 / a8: G^{k-1} = gamma A_att^T G^k per slice, with dalpha += gamma G^k_v . Z^{k-1}_u on the way
    c->wire_phase = 3;
    void* cur = c->recv.p;
    void* nxt = c->xfer.p;
    for (int i = 0; i < m->K; ++i) {
        const int k = m->K - i;
        for (int j = 0; j < vs; ++j) {
            const void* Gj = sl(cur, j);
            const void* Zj = sl(Zst, (int64_t)(k - 1) * vs + j);
            const int acc = (i > 0 || j > 0) ? 1 : 0;
            sddmm(Gj, Zj, acc);
            count_launch(c);
            hop(Gj, sl(nxt, j), true);
        }
        std::swap(cur, nxt);
    }
    NTP_CUDA(record_timing(c, E[11], s));   // bwd hops (+ SDDMM) done
    // a9: gather G^0 -> dz rows
    void* gathered_b = cur;
    if (!local) {
        exchange_f2v(c, cur, c->send.p, V_p * d_s, dt, s);
        gathered_b = c->send.p;
    }
    unpack_f2v(c, gathered_b, V_p, d_s, P, dz, ldL, C, dt, NTP_F32, s);
    NTP_CUDA(record_timing(c, E[ei++], s));   // E6 prop bwd + f2v

    // ---- attention backward (every rank holds every coefficient): dalpha summed over ranks
    if (!local) NTP_NCCL(ncclAllReduce(dalpha, dalpha, (size_t)na, ncclFloat32, ncclSum, c->comm, s));
    gat_softmax_bwd_kernel<<<wblocks(n), 256, 0, s>>>(g.fwd().row_ptr.as<int32_t>(), c->gat_bits.as<uint32_t>(), alpha,
                                                     dalpha, n, slope, ds, pd);
    if (c->gat_nbig[0] > 0)
        gat_softmax_bwd_big_kernel<<<std::min(c->gat_nbig[0], 148 * 8), 256, 0, s>>>(
            big_in, c->gat_nbig[0], g.fwd().row_ptr.as<int32_t>(), c->gat_bits.as<uint32_t>(), alpha, dalpha, n, slope,
            ds, pd);
    NTP_LAUNCH_CHECK();
    gat_ps_kernel<<<wblocks(n), 256, 0, s>>>(g.bwd().row_ptr.as<int32_t>(), perm, ds, n, ps);
    if (c->gat_nbig[1] > 0)
        gat_ps_big_kernel<<<std::min(c->gat_nbig[1], 148 * 8), 256, 0, s>>>(big_out, c->gat_nbig[1],
                                                                           g.bwd().row_ptr.as<int32_t>(), perm, ds, n, ps);
    NTP_LAUNCH_CHECK();
    gat_dz_kernel<<<eblk(V_p * C), 256, 0, s>>>(dz, ldL, C, attu, ps, pd, V_p, row0, n);
    NTP_LAUNCH_CHECK();
    gat_da_partial_kernel<<<nbda, 256, 0, s>>>(z, ldL, C, ps, pd, V_p, row0, n, c->gat_da.as<float>());
    NTP_LAUNCH_CHECK();
    gat_sum_parts_kernel<<<eblk(2 * C), 256, 0, s>>>(c->gat_da.as<float>(), nbda, 2 * C, da);
    NTP_LAUNCH_CHECK();
    count_launch(c, 5);

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
