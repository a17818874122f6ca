// spmm.cu — K-hop feature-sliced propagation (K1-K3).
//
// Paper: Z^k = gamma * A^ Z^{k-1} (Eq. 9) with A^ = D~^{-1/2}(A+I)D~^{-1/2}
// (P:738-739), two-sided for directed graphs (R1), plus the alpha*H mix (R2);
// the backward is the same recurrence with A^T over the out-CSR.
//
// Pre-scaled form (no per-edge coefficient array; SURVEY §8(a) design notes):
//   S^k = cs .* Z^k (column-side scaled state):  S^0 = cs .* H
//   intermediate hop:  S^k_v = gamma*rs_v*cs_v * (S_v + sum_{u in N(v)} S_u) + alpha*S^0_v
//   last hop:          Z^K_v = gamma*rs_v       * (S_v + sum_{u in N(v)} S_u) + (alpha/cs_v)*S^0_v
//   (alpha*cs_v*H_v = alpha*S^0_v, alpha*H_v = alpha*S^0_v/cs_v: only S^0 is kept.)
//   (rs, cs) = (dinv_in, dinv_out) forward, (dinv_out, dinv_in) backward.
// The gather is therefore an unweighted row-sum of 16-byte vectors.
//
// Work split: merge path over (row-ends + nnz), fixed T items per unit (a
// graph-level constant).  A unit is processed by a lane group of G=8 edge
// lanes x CW column lanes (16-byte vectors); lane g takes edges j = g mod 8 of
// the row, accumulates in fp32 in ascending order, and the 8 partials are
// combined by a fixed xor-tree.  Rows cut by a unit boundary write head/tail
// partials to a carry buffer, summed in unit order by the fix-up kernel.
// The per-row order depends only on (G, T, graph), not on the slice width or
// P, so every column's result is bitwise independent of the slicing.
#include <algorithm>

#include "ntp_internal.cuh"

namespace ntp {

namespace {

constexpr int kG = 8;           // edge lanes per group (fixed: part of the reduction order)
constexpr int kBlock = 256;

template <typename T> struct V16;
template <> struct V16<float> {
    static constexpr int N = 4;
    __device__ __forceinline__ static void load(const void* p, float (&v)[4]) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(p));
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    }
    __device__ __forceinline__ static void add(const void* p, float (&a)[4]) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(p));
        a[0] += x.x; a[1] += x.y; a[2] += x.z; a[3] += x.w;
    }
    __device__ __forceinline__ static void store(void* p, const float (&v)[4]) {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    }
};
template <> struct V16<__nv_bfloat16> {
    static constexpr int N = 8;
    __device__ __forceinline__ static void unpack(const uint4 x, float (&v)[8]) {
        const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            v[2 * i] = __uint_as_float(w[i] << 16);
            v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
        }
    }
    __device__ __forceinline__ static void load(const void* p, float (&v)[8]) {
        unpack(__ldg(reinterpret_cast<const uint4*>(p)), v);
    }
    __device__ __forceinline__ static void add(const void* p, float (&a)[8]) {
        float v[8];
        unpack(__ldg(reinterpret_cast<const uint4*>(p)), v);
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] += v[i];
    }
    __device__ __forceinline__ static void store(void* p, const float (&v)[8]) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
            w[i] = *reinterpret_cast<const uint32_t*>(&h);
        }
        *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
    }
};

struct HopParams {
    const int32_t* __restrict__ rp;
    const int32_t* __restrict__ col;
    const int32_t* __restrict__ unit_row;
    const int32_t* __restrict__ unit_e;
    const float* __restrict__ rs;      // row-side D~^{-1/2}
    const float* __restrict__ cs;      // column-side D~^{-1/2}
    const char* __restrict__ S_in;     // pre-scaled state, row stride ld_in bytes
    char* __restrict__ S_out;
    const char* __restrict__ S0;       // alpha term input S^0 = cs .* H (may be null if alpha == 0)
    float* __restrict__ carry;         // [U][2][nvec*VALS] fp32
    int64_t ld_in, ld_out, ld_s0;      // bytes
    int64_t n;
    int64_t u_begin, u_end;
    int64_t row_lo, row_hi;
    int32_t nvec;                      // 16-byte vectors per row
    float gamma, alpha;
    int mode;                          // 0 intermediate, 1 last
};

template <typename T, int CW>
__global__ void __launch_bounds__(kBlock) spmm_hop_kernel(const HopParams p) {
    constexpr int L = kG * CW;
    constexpr int VALS = V16<T>::N;
    const int lane = threadIdx.x & 31;
    const int gl = lane % L;
    const int g = gl % kG;
    const int c = gl / kG;
    const int64_t group = ((int64_t)blockIdx.x * kBlock + threadIdx.x) / L;
    const int64_t u = p.u_begin + group;
    if (u >= p.u_end) return;                           // group-uniform exit
    const unsigned gmask = (L == 32) ? 0xffffffffu : (((1u << L) - 1u) << ((lane / L) * L));

    const int r0 = p.unit_row[u], r1 = p.unit_row[u + 1];
    const int e0 = p.unit_e[u], e1 = p.unit_e[u + 1];
    const bool has_tail = (r1 < p.n) && (e1 > max(p.rp[r1], e0));
    const int r_end = has_tail ? r1 + 1 : r1;
    const int row_vals = p.nvec * VALS;
    const int npass = (p.nvec + CW - 1) / CW;

    for (int r = max((int64_t)r0, p.row_lo); r < min((int64_t)r_end, p.row_hi); ++r) {
        const int rs_e = p.rp[r], re_e = p.rp[r + 1];
        const int eb = max(rs_e, e0), ee = min(re_e, e1);
        const bool head = (r == r0) && (rs_e < e0);
        const bool tail = (r == r1);
        for (int pass = 0; pass < npass; ++pass) {
            const int vcol = pass * CW + c;
            const bool col_ok = vcol < p.nvec;
            const int64_t voff = (int64_t)vcol * 16;
            float acc[VALS];
#pragma unroll
            for (int i = 0; i < VALS; ++i) acc[i] = 0.f;
            if (col_ok) {
                int j = eb + g;
                for (; j + 3 * kG < ee; j += 4 * kG) {
                    const int s0 = __ldg(p.col + j), s1 = __ldg(p.col + j + kG);
                    const int s2 = __ldg(p.col + j + 2 * kG), s3 = __ldg(p.col + j + 3 * kG);
                    float v0[VALS], v1[VALS], v2[VALS], v3[VALS];
                    V16<T>::load(p.S_in + (int64_t)s0 * p.ld_in + voff, v0);
                    V16<T>::load(p.S_in + (int64_t)s1 * p.ld_in + voff, v1);
                    V16<T>::load(p.S_in + (int64_t)s2 * p.ld_in + voff, v2);
                    V16<T>::load(p.S_in + (int64_t)s3 * p.ld_in + voff, v3);
#pragma unroll
                    for (int i = 0; i < VALS; ++i) acc[i] = (((acc[i] + v0[i]) + v1[i]) + v2[i]) + v3[i];
                }
                for (; j < ee; j += kG) {
                    const int s0 = __ldg(p.col + j);
                    V16<T>::add(p.S_in + (int64_t)s0 * p.ld_in + voff, acc);
                }
            }
            // fixed xor-tree over the 8 edge lanes (lane g == 0 holds the canonical order)
#pragma unroll
            for (int o = 1; o < kG; o <<= 1) {
#pragma unroll
                for (int i = 0; i < VALS; ++i) acc[i] += __shfl_xor_sync(gmask, acc[i], o);
            }
            if (g != 0 || !col_ok) continue;
            if (head || tail) {
                float* dst = p.carry + ((u * 2 + (head ? 0 : 1)) * (int64_t)row_vals) + vcol * VALS;
#pragma unroll
                for (int i = 0; i < VALS; ++i) dst[i] = acc[i];
                continue;
            }
            float self[VALS];
            V16<T>::load(p.S_in + (int64_t)r * p.ld_in + voff, self);
            const float a = p.rs[r];
            float out[VALS];
            const float b = p.cs[r];
            const float sig = (p.mode == 0) ? p.gamma * a * b : p.gamma * a;
            if (p.alpha != 0.f) {
                float h[VALS];
                V16<T>::load(p.S0 + (int64_t)r * p.ld_s0 + voff, h);
                const float beta = (p.mode == 0) ? p.alpha : p.alpha / b;
#pragma unroll
                for (int i = 0; i < VALS; ++i) out[i] = sig * (acc[i] + self[i]) + beta * h[i];
            } else {
#pragma unroll
                for (int i = 0; i < VALS; ++i) out[i] = sig * (acc[i] + self[i]);
            }
            V16<T>::store(p.S_out + (int64_t)r * p.ld_out + voff, out);
        }
    }
}

// Fix-up: one warp per unit that STARTS a split row (its tail).  Sums tail[u],
// head[u+1], ..., head[u_last] in unit order, then applies the epilogue.
template <typename T>
__global__ void __launch_bounds__(kBlock) spmm_fixup_kernel(const HopParams p) {
    const int64_t u = p.u_begin + ((int64_t)blockIdx.x * kBlock + threadIdx.x) / 32;
    const int lane = threadIdx.x & 31;
    if (u >= p.u_end) return;
    const int r = p.unit_row[u + 1];
    const int e0 = p.unit_e[u], e1 = p.unit_e[u + 1];
    if (r >= p.n || r < p.row_lo || r >= p.row_hi) return;
    const int rs_e = p.rp[r];
    if (!(rs_e >= e0 && rs_e < e1)) return;            // row r does not start (with edges) in unit u
    constexpr int VALS = V16<T>::N;
    const int row_vals = p.nvec * VALS;
    const float a = p.rs[r];
    const float b = p.cs[r];
    for (int k = lane; k < row_vals; k += 32) {
        float acc = p.carry[(u * 2 + 1) * (int64_t)row_vals + k];
        for (int64_t v = u + 1;; ++v) {
            acc += p.carry[(v * 2 + 0) * (int64_t)row_vals + k];
            if (p.unit_row[v + 1] > r) break;
        }
        const int vcol = k / VALS, comp = k % VALS;
        float self[VALS];
        V16<T>::load(p.S_in + (int64_t)r * p.ld_in + (int64_t)vcol * 16, self);
        const float sig = (p.mode == 0) ? p.gamma * a * b : p.gamma * a;
        float out = sig * (acc + self[comp]);
        if (p.alpha != 0.f) {
            float h[VALS];
            V16<T>::load(p.S0 + (int64_t)r * p.ld_s0 + (int64_t)vcol * 16, h);
            out += ((p.mode == 0) ? p.alpha : p.alpha / b) * h[comp];
        }
        if (sizeof(T) == 4) {
            reinterpret_cast<float*>(p.S_out + (int64_t)r * p.ld_out)[k] = out;
        } else {
            reinterpret_cast<__nv_bfloat16*>(p.S_out + (int64_t)r * p.ld_out)[k] = __float2bfloat16_rn(out);
        }
    }
}

template <typename T>
__global__ void prescale_kernel(const char* __restrict__ H, int64_t ld_h, char* __restrict__ S, int64_t ld_s,
                                int32_t nvec, const float* __restrict__ scale, int64_t rows) {
    constexpr int VALS = V16<T>::N;
    const int64_t total = rows * nvec;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / nvec;
        const int64_t vc = i % nvec;
        float v[VALS];
        V16<T>::load(H + r * ld_h + vc * 16, v);
        const float s = scale[r];
#pragma unroll
        for (int k = 0; k < VALS; ++k) v[k] *= s;
        V16<T>::store(S + r * ld_s + vc * 16, v);
    }
}

template <typename T, int CW>
void launch_hop(const HopParams& p, cudaStream_t s) {
    constexpr int L = kG * CW;
    const int64_t groups = p.u_end - p.u_begin;
    const int64_t blocks = cdiv(groups * L, kBlock);
    spmm_hop_kernel<T, CW><<<(unsigned)blocks, kBlock, 0, s>>>(p);
    NTP_LAUNCH_CHECK();
}

}  // namespace

static void unit_range(const Csr& csr, int64_t row_lo, int64_t row_hi, int64_t& ub, int64_t& ue) {
    const auto& h = csr.h_unit_row;      // U+1 entries, non-decreasing
    // first unit whose row-end range reaches row_lo: unit_row[u+1] >= row_lo
    ub = std::lower_bound(h.begin() + 1, h.end(), (int32_t)row_lo) - (h.begin() + 1);
    // first unit starting at a row >= row_hi
    ue = std::lower_bound(h.begin(), h.end() - 1, (int32_t)row_hi) - h.begin();
    ub = std::min(ub, csr.U);
    ue = std::min(std::max(ue, ub), csr.U);
}

void spmm_hop(ntp_ctx* c, const Csr& csr, const float* rs, const float* cs, const void* S_in, void* S_out,
              const void* S0, int64_t ld_in, int64_t ld_out, int64_t ld_s0, int32_t cols, ntp_dtype dt,
              float gamma, float alpha, int mode, int64_t row_lo, int64_t row_hi, cudaStream_t s) {
    const Graph& g = c->g;
    if (row_hi < 0) row_hi = g.n;
    row_lo = std::max<int64_t>(row_lo, 0);
    row_hi = std::min<int64_t>(row_hi, g.n);
    if (row_hi <= row_lo) return;
    const size_t es = esize(dt);
    const int32_t nvec = (int32_t)(cols * es / 16);
    const int vals = 16 / (int)es;
    HopParams p;
    p.rp = csr.row_ptr.as<int32_t>();
    p.col = csr.col.as<int32_t>();
    p.unit_row = csr.unit_row.as<int32_t>();
    p.unit_e = csr.unit_e.as<int32_t>();
    p.rs = rs;
    p.cs = cs;
    p.S_in = static_cast<const char*>(S_in);
    p.S_out = static_cast<char*>(S_out);
    p.S0 = static_cast<const char*>(S0);
    p.ld_in = ld_in * es;
    p.ld_out = ld_out * es;
    p.ld_s0 = ld_s0 * es;
    p.n = g.n;
    unit_range(csr, row_lo, row_hi, p.u_begin, p.u_end);
    p.row_lo = row_lo;
    p.row_hi = row_hi;
    p.nvec = nvec;
    p.gamma = gamma;
    p.alpha = alpha;
    p.mode = mode;
    c->carry.ensure((size_t)(csr.U * 2) * nvec * vals * sizeof(float) + 16);
    p.carry = c->carry.as<float>();
    if (p.u_end <= p.u_begin) return;
    const int CW = nvec >= 3 ? 4 : (nvec == 2 ? 2 : 1);
    if (dt == NTP_F32) {
        if (CW == 4) launch_hop<float, 4>(p, s);
        else if (CW == 2) launch_hop<float, 2>(p, s);
        else launch_hop<float, 1>(p, s);
    } else {
        if (CW == 4) launch_hop<__nv_bfloat16, 4>(p, s);
        else if (CW == 2) launch_hop<__nv_bfloat16, 2>(p, s);
        else launch_hop<__nv_bfloat16, 1>(p, s);
    }
    const int64_t fblocks = cdiv((p.u_end - p.u_begin) * 32, kBlock);
    if (dt == NTP_F32) spmm_fixup_kernel<float><<<(unsigned)fblocks, kBlock, 0, s>>>(p);
    else spmm_fixup_kernel<__nv_bfloat16><<<(unsigned)fblocks, kBlock, 0, s>>>(p);
    NTP_LAUNCH_CHECK();
    count_launch(c, 2);
}

void prescale(ntp_ctx* c, const void* H, int64_t ld_h, void* S, int64_t ld_s, int32_t cols, const float* scale,
              int64_t rows, ntp_dtype dt, cudaStream_t s) {
    if (rows <= 0) return;
    const size_t es = esize(dt);
    const int32_t nvec = (int32_t)(cols * es / 16);
    const int64_t total = rows * nvec;
    const int blocks = (int)std::min<int64_t>(cdiv(total, 256), 148 * 16);
    if (dt == NTP_F32)
        prescale_kernel<float><<<blocks, 256, 0, s>>>((const char*)H, ld_h * es, (char*)S, ld_s * es, nvec, scale, rows);
    else
        prescale_kernel<__nv_bfloat16><<<blocks, 256, 0, s>>>((const char*)H, ld_h * es, (char*)S, ld_s * es, nvec,
                                                              scale, rows);
    NTP_LAUNCH_CHECK();
    count_launch(c);
}

// K hops.  Hop k writes bufs[(K-k) % 2] (bufs = {Z, scratch}) so hop K lands in Z.
// S^0 = cs .* H is formed by `prescale` unless the caller already holds it
// (prescaled_input: a.H points at S^0, e.g. the pack epilogue of the split).
// With alpha != 0, S^0 must outlive hop 1, so it gets its own buffer.
void propagate(ntp_ctx* c, const PropArgs& a, cudaStream_t s, bool time_hops, bool prescaled_input,
               int64_t last_row_lo, int64_t last_row_hi) {
    const Graph& g = c->g;
    const Csr& csr = a.transposed ? g.bwd() : g.fwd();
    const float* rs = a.transposed ? g.dinv_out_p() : g.dinv_in_p();
    const float* cs = a.transposed ? g.dinv_in_p() : g.dinv_out_p();
    const size_t es = esize(a.dtype);
    const int64_t n = g.n;
    if (a.K == 0) {
        NTP_CHECK(!prescaled_input, NTP_ERR_ARG, "K == 0 with pre-scaled input");
        if (n > 0)
            NTP_CUDA(cudaMemcpy2DAsync(a.Z, a.ld_z * es, a.H, a.ld_h * es, a.cols * es, n,
                                       cudaMemcpyDeviceToDevice, s));
        return;
    }
    const int64_t ld_t = a.cols;     // scratch is dense
    c->prop_tmp.ensure((size_t)n * ld_t * es + 16);
    void* bufs[2] = {a.Z, c->prop_tmp.p};
    const int64_t lds[2] = {a.ld_z, ld_t};
    const void* S0;
    int64_t ld_s0;
    if (prescaled_input) {
        S0 = a.H;
        ld_s0 = a.ld_h;
    } else if (a.alpha != 0.f) {
        c->prop_s0.ensure((size_t)n * ld_t * es + 16);
        prescale(c, a.H, a.ld_h, c->prop_s0.p, ld_t, a.cols, cs, n, a.dtype, s);
        S0 = c->prop_s0.p;
        ld_s0 = ld_t;
    } else {
        const int b0 = a.K % 2;       // hop 1 writes bufs[(K-1)%2], so S^0 may live in bufs[K%2]
        prescale(c, a.H, a.ld_h, bufs[b0], lds[b0], a.cols, cs, n, a.dtype, s);
        S0 = bufs[b0];
        ld_s0 = lds[b0];
    }
    const void* sin = S0;
    int64_t ld_sin = ld_s0;
    for (int k = 1; k <= a.K; ++k) {
        const int nxt = (a.K - k) % 2;
        const bool last = (k == a.K);
        const bool timed = time_hops && c->hop_ev_used + 2 <= 256;
        if (timed) NTP_CUDA(cudaEventRecord(c->hop_ev[c->hop_ev_used], s));
        const int64_t lo = last ? last_row_lo : 0;
        const int64_t hi = last ? last_row_hi : -1;
        spmm_hop(c, csr, rs, cs, sin, bufs[nxt], S0, ld_sin, lds[nxt], ld_s0, a.cols, a.dtype, a.gamma, a.alpha,
                 last ? 1 : 0, lo, hi, s);
        if (timed) {
            NTP_CUDA(cudaEventRecord(c->hop_ev[c->hop_ev_used + 1], s));
            c->hop_ev_used += 2;
        }
        sin = bufs[nxt];
        ld_sin = lds[nxt];
    }
}

double collect_hop_ms(ntp_ctx* c, int* n_hops) {
    double tot = 0.0;
    for (int i = 0; i + 1 < c->hop_ev_used; i += 2) {
        float ms = 0.f;
        NTP_CUDA(cudaEventElapsedTime(&ms, c->hop_ev[i], c->hop_ev[i + 1]));
        tot += ms;
    }
    if (n_hops) *n_hops = c->hop_ev_used / 2;
    c->hop_ev_used = 0;
    return tot;
}

}  // namespace ntp
