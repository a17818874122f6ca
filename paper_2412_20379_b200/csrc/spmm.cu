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
#include <cstdlib>

#include "ntp_internal.cuh"
#include "ptx.cuh"

namespace ntp {

namespace {

constexpr int kG = 8;           // edge lanes per group (fixed: part of the reduction order)
constexpr int kBlock = 256;

// Vector of VB bytes (16: LDG.128, 32: LDG.E.ENL2.256, sm_100) held as raw 32-bit words.
template <int VB> struct Raw { uint32_t w[VB / 4]; };

template <int VB> __device__ __forceinline__ Raw<VB> ldv(const void* p);
template <> __device__ __forceinline__ Raw<16> ldv<16>(const void* p) {
    const uint4 x = __ldg(reinterpret_cast<const uint4*>(p));
    return Raw<16>{{x.x, x.y, x.z, x.w}};
}
template <> __device__ __forceinline__ Raw<32> ldv<32>(const void* p) {
    Raw<32> r;
    asm volatile("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]),
                   "=r"(r.w[7])
                 : "l"(p));
    return r;
}
template <int VB> __device__ __forceinline__ void stv(void* p, const Raw<VB>& r);
template <> __device__ __forceinline__ void stv<16>(void* p, const Raw<16>& r) {
    *reinterpret_cast<uint4*>(p) = make_uint4(r.w[0], r.w[1], r.w[2], r.w[3]);
}
template <> __device__ __forceinline__ void stv<32>(void* p, const Raw<32>& r) {
    asm volatile("st.global.v8.u32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(r.w[0]), "r"(r.w[1]),
                 "r"(r.w[2]), "r"(r.w[3]), "r"(r.w[4]), "r"(r.w[5]), "r"(r.w[6]), "r"(r.w[7])
                 : "memory");
}
template <int VB> __device__ __forceinline__ Raw<VB> zero_raw() {
    Raw<VB> r;
#pragma unroll
    for (int i = 0; i < VB / 4; ++i) r.w[i] = 0u;
    return r;
}

// Element view of a vector: fp32 (VB/4 values) or bf16 (VB/2 values, widened exactly to fp32).
template <typename T, int VB> struct Vec;
template <int VB> struct Vec<float, VB> {
    static constexpr int N = VB / 4;
    __device__ __forceinline__ static float elem(const Raw<VB>& x, int i) { return __uint_as_float(x.w[i]); }
    __device__ __forceinline__ static Raw<VB> pack(const float (&v)[N]) {
        Raw<VB> r;
#pragma unroll
        for (int i = 0; i < N; ++i) r.w[i] = __float_as_uint(v[i]);
        return r;
    }
};
template <int VB> struct Vec<__nv_bfloat16, VB> {
    static constexpr int N = VB / 2;
    __device__ __forceinline__ static float elem(const Raw<VB>& x, int i) {
        const uint32_t w = x.w[i >> 1];
        return __uint_as_float((i & 1) ? (w & 0xFFFF0000u) : (w << 16));
    }
    __device__ __forceinline__ static Raw<VB> pack(const float (&v)[N]) {
        Raw<VB> r;
#pragma unroll
        for (int i = 0; i < N / 2; ++i) {
            const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
            r.w[i] = *reinterpret_cast<const uint32_t*>(&h);
        }
        return r;
    }
};
template <typename T, int VB>
__device__ __forceinline__ void vadd(float (&a)[Vec<T, VB>::N], const Raw<VB>& x) {
#pragma unroll
    for (int i = 0; i < Vec<T, VB>::N; ++i) a[i] += Vec<T, VB>::elem(x, i);
}
// weighted hop (per-arc coefficient, e.g. GAT attention): a += w * x as one rounding (explicit fma, so the
// accumulation is the same instruction sequence for every slice width)
template <typename T, int VB>
__device__ __forceinline__ void vfma(float (&a)[Vec<T, VB>::N], const Raw<VB>& x, float w) {
#pragma unroll
    for (int i = 0; i < Vec<T, VB>::N; ++i) a[i] = __fmaf_rn(w, Vec<T, VB>::elem(x, i), a[i]);
}

// 16-byte element loads for the fix-up / prescale kernels
template <typename T> __device__ __forceinline__ void load16(const void* p, float (&v)[16 / sizeof(T)]) {
    const Raw<16> x = ldv<16>(p);
#pragma unroll
    for (int i = 0; i < (int)(16 / sizeof(T)); ++i) v[i] = Vec<T, 16>::elem(x, i);
}
template <typename T> __device__ __forceinline__ void store16(void* p, const float (&v)[16 / sizeof(T)]) {
    stv<16>(p, Vec<T, 16>::pack(v));
}


// resident 256-thread CTAs per SM (register budget)
// MODE bits 2-3 (OCC, high-degree graphs): 1 = half-length batches at 3 CTAs/SM, 2 = half-length batches
// at 4 CTAs/SM -- the same bytes in flight per warp spread over more warps, so row ends, butterflies
// and epilogues of one warp hide behind the loads of the others.
template <int E, int VB, int MODE>
__host__ __device__ constexpr int hop_ctas() {
    return ((MODE >> 2) & 3) == 2 ? 4 : ((MODE >> 2) & 3) == 1 ? 3 : ((MODE & 1) && E == 8 && VB == 16) ? 3 : 2;
}

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
    float* __restrict__ carry;         // [U][2][row_vals] fp32
    int64_t ld_in, ld_out, ld_s0;      // bytes
    int64_t n;
    int64_t u_begin, u_end;
    int64_t row_lo, row_hi;
    int32_t nvec;                      // 16-byte vectors per row
    float gamma, alpha;
    int mode;                          // 0 intermediate, 1 last
    int64_t nnz;
    const int32_t* __restrict__ out_rows;   // last hop of a reordered graph: output row r goes to out_rows[r]
    void* const* __restrict__ peer_out;     // last hop, peer-direct gather: window table [P] (else null)
    int64_t po_V_p;
    int po_rank;
    const float* __restrict__ ew;      // weighted hop: per-arc coefficients in CSR order (else null)
    const float* __restrict__ sw;      // weighted hop: per-row self-loop coefficients
    // dual weighted hop (GAT): the coefficient words are signed, |w| = alpha and the sign bit marks the arcs
    // whose second coefficient is slope2 * alpha (else alpha); the second sum goes to S_out2 (row stride ld_out)
    char* __restrict__ S_out2;
    float* __restrict__ carry2;
    float slope2;
};

// dual weighted hop: (alpha, beta) from one signed coefficient word
__device__ __forceinline__ float coef_a(float w) { return __int_as_float(__float_as_int(w) & 0x7fffffff); }
__device__ __forceinline__ float coef_b(float w, float slope) {
    const float a = coef_a(w);
    return __float_as_int(w) < 0 ? slope * a : a;
}

// Where output row r (internal order) is stored: its original row (out_rows), locally or -- peer-direct
// gather -- in block po_rank of the owner's window: the f2v all-to-all fused into the epilogue.
__device__ __forceinline__ char* out_row_ptr(const HopParams& p, int64_t r) {
    const int64_t orow = p.out_rows ? (int64_t)__ldg(p.out_rows + r) : r;
    if (p.peer_out) {
        const int64_t q = orow / p.po_V_p;
        return static_cast<char*>(p.peer_out[q]) + ((int64_t)p.po_rank * p.po_V_p + orow - q * p.po_V_p) * p.ld_out;
    }
    return p.S_out + orow * p.ld_out;
}

// Lane layout ("full row per edge"): a group of L lanes works on one unit.  Lane
// gl = e*VP + c holds edge slot e in [0, E) and VB-byte column vector c in [0, VP):
// one load instruction fetches the complete row slices of E edges with
// consecutive lanes.  The per-instruction cost of a gather (not its bytes) is what
// bounds the hop, so rows whose width is a multiple of 32 bytes use
// 32-byte loads (VB = 32, LDG.E.ENL2.256): twice the edges per instruction.
// Edge j of a unit piece starting at eb belongs to reduction group g = (j - eb) mod 8,
// g = e + E*k: lane slot e keeps 8/E accumulators acc[k].  The 8 groups are combined by
// the fixed butterfly ((a0+a1)+(a2+a3))+((a4+a5)+(a6+a7)) -- cross-lane for the bits
// of e, in-lane for the bits of k -- so the per-column order is the same for every
// (E, VP, VB), i.e. for every slice width.  Column indices are loaded coalesced (one
// per lane) and distributed with shuffles.
// MODE (low-degree graphs, average degree < 32): bit 0 = short batches (E >= 4): 8-16-edge
// batches so a ~15-arc row does not pay for a 64-slot batch, and fewer registers for 3 CTAs per
// SM; bit 1 = tiny-row path (E >= 2, below).  Neither enters the reduction order (groups are
// (j - eb) mod 8 for any batch that is a multiple of 8), and the tiny path's registers are only
// paid where it is used.
// WT (weighted hop): the row sum carries a per-arc coefficient p.ew[j] (loaded with the column index and
// shuffled with it) and the self term p.sw[r]; no row / column D~^{-1/2} (rs = cs = 1).  GAT's attention
// aggregation (Eq. 5) -- the same merge-path split, pipeline and fixed reduction order; it is
// instantiated only as the DUAL variant, the one the GAT epoch runs.
// DUAL (implies WT): two sums per row from one pass over the arcs, with the coefficients alpha and beta
// decoded from one signed word per arc (coef_a / coef_b): the second accumulator set costs registers and
// FMAs, not a second gather.
template <typename T, int VB, int E, int L, int MODE, bool WT = false, bool DUAL = false>
__global__ void __launch_bounds__(kBlock, DUAL ? 3 : hop_ctas<E, VB, MODE>()) spmm_hop_kernel(const HopParams p) {
    constexpr bool SHORT = (MODE & 1) != 0;
    constexpr bool TINY = (MODE & 2) != 0 && E >= 2;
    // one accumulator per lane slot in the dual hop: its two sums (GAT) need no slice-width invariance, and
    // the registers saved buy a third resident CTA per SM (launch bounds below; measured on the Reddit-shape
    // GAT epoch, ms per dual hop: 8 groups at 2 CTAs/SM 3.79, one group at 2 CTAs 3.71, at 3 CTAs 2.98,
    // at 4 CTAs 3.38 -- the last two with some local-memory spills)
    constexpr int LOG_E = (E == 1) ? 0 : (E == 2) ? 1 : (E == 4) ? 2 : 3;
    constexpr int VALS = Vec<T, VB>::N;
    // edges per pipeline batch (a multiple of 8); loads per lane per batch LPB = BATCH / E:
    // 8 x 16 B (2-4 x 16 B short), or 4 x 32 B (2 x 32 B short) -- the same bytes in flight
    constexpr bool OCC = ((MODE >> 2) & 3) != 0;
    // MODE bit 5 (ONEACC) and the dual hop: one accumulator per lane slot instead of the 8 / E groups of
    // the slice-width-invariant order (below), for the registers of a 4th (3rd) resident CTA per SM
    constexpr int NACC = (DUAL || (MODE & 32)) ? 1 : kG / E;
    constexpr int BATCH0 = (VB == 16) ? (SHORT ? ((E >= 4) ? 16 : 8) : ((E == 8) ? 64 : (E == 4) ? 32 : 8 * E))
                                      : (SHORT ? ((E >= 4) ? 2 * E : 8) : ((E >= 2) ? 4 * E : 8));
    // half-length batches for the weighted hop too: its per-arc coefficients ride along with the loads
    // (full-length batches spilled ~30 registers to local memory at 128 registers)
    constexpr int BATCH = ((OCC || DUAL) && !SHORT && BATCH0 >= 16) ? BATCH0 / 2 : BATCH0;
    constexpr int LPB = BATCH / E;                        // loads per lane per batch
    constexpr int ISL = (BATCH + L - 1) / L;              // column indices held per lane
    constexpr int ISLW = WT ? ISL : 1, LPBW = WT ? LPB : 1;   // arc coefficients held per lane (weighted)
    static_assert(BATCH % 8 == 0, "batch must preserve the (j - eb) mod 8 grouping");
    static_assert(!(WT && MODE != 0), "the weighted hop has only the general path");
    static_assert(!DUAL || WT, "the dual hop is weighted");
    constexpr int NACC2 = DUAL ? NACC : 1;
    const int lane = threadIdx.x & 31;
    const int gl = lane % L;
    const int gbase = lane - gl;
    const int64_t u = p.u_begin + ((int64_t)blockIdx.x * kBlock + threadIdx.x) / L;
    if (u >= p.u_end) return;                           // group-uniform exit
    const unsigned gmask = (L == 32) ? 0xffffffffu : (((1u << L) - 1u) << gbase);
    const int nv = p.nvec / (VB / 16);                   // VB-byte vectors per row
    const int VP = (E == 1) ? min(nv, 32) : nv;          // vectors per pass
    // lane stride of an edge slot: VP rounded up to 8 lanes when that still fits, so no 8-lane
    // phase of a load straddles two rows (idle lanes mirror the row's last vector: same line)
    const int VPP = (E > 1 && E * ((VP + 7) & ~7) <= L) ? ((VP + 7) & ~7) : VP;
    const int e_raw = gl / VPP;
    const int c_raw = gl - e_raw * VPP;
    const bool active = e_raw < E && c_raw < VP;
    const int e = min(e_raw, E - 1);
    const int c = min(c_raw, VP - 1);
    const int32_t* __restrict__ colp = p.col;
    const uint32_t ld_in = (uint32_t)p.ld_in;
    const int r0 = p.unit_row[u], r1 = p.unit_row[u + 1];
    const int e0 = p.unit_e[u], e1 = p.unit_e[u + 1];
    const bool has_tail = (r1 < p.n) && (e1 > max(p.rp[r1], e0));
    const int r_end = has_tail ? r1 + 1 : r1;
    const int row_vals = p.nvec * (16 / (int)sizeof(T));
    const int npass = (nv + VP - 1) / VP;

    const int r_stop = (int)min((int64_t)r_end, p.row_hi);
    for (int r = max((int64_t)r0, p.row_lo); r < r_stop; ++r) {
        // ---- tiny-row fast path: E consecutive rows with <= 8 arcs each, wholly inside this unit,
        // one row per edge slot.  With <= 8 arcs every reduction group holds at most one arc, so
        // acc_g = 0 + v_g and the in-lane tree ((v0+v1)+(v2+v3))+((v4+v5)+(v6+v7)) is exactly the
        // canonical butterfly: results are bitwise those of the general path.
        if constexpr (TINY) {
            if (npass == 1 && r + E <= r1 && r + E <= r_stop) {
                const int my_r = r + e;
                const int trs = __ldg(p.rp + my_r), tre = __ldg(p.rp + my_r + 1);
                const int deg = tre - trs;
                const bool ok = deg <= 8 && !(my_r == r0 && trs < e0);
                if (__all_sync(gmask, ok)) {
                    const bool cok = active && c < nv;
                    const int64_t voff = (int64_t)min(c, nv - 1) * VB;
                    const Raw<VB> self_raw = ldv<VB>(p.S_in + (int64_t)my_r * p.ld_in + voff);
                    const Raw<VB> s0_raw =
                        (p.alpha != 0.f) ? ldv<VB>(p.S0 + (int64_t)my_r * p.ld_s0 + voff) : zero_raw<VB>();
                    const float ra = __ldg(p.rs + my_r), rb = __ldg(p.cs + my_r);
                    int src[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) src[k] = (k < deg) ? __ldg(colp + trs + k) : 0;
                    Raw<VB> x8[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        x8[k] = (k < deg) ? ldv<VB>(p.S_in + (int64_t)src[k] * p.ld_in + voff) : zero_raw<VB>();
                    const float sig = (p.mode == 0) ? p.gamma * ra * rb : p.gamma * ra;
                    const float beta = (p.mode == 0) ? p.alpha : p.alpha / rb;
                    float out[VALS];
#pragma unroll
                    for (int i = 0; i < VALS; ++i) {
                        float g[8];
#pragma unroll
                        for (int k = 0; k < 8; ++k) g[k] = 0.f + Vec<T, VB>::elem(x8[k], i);   // acc_g = 0 + v_g
                        const float tot = ((g[0] + g[1]) + (g[2] + g[3])) + ((g[4] + g[5]) + (g[6] + g[7]));
                        const float self = 0.f + Vec<T, VB>::elem(self_raw, i);
                        out[i] = (p.alpha != 0.f) ? sig * (tot + self) + beta * (0.f + Vec<T, VB>::elem(s0_raw, i))
                                                  : sig * (tot + self);
                    }
                    if (cok) stv<VB>(out_row_ptr(p, my_r) + voff, Vec<T, VB>::pack(out));
                    r += E - 1;
                    continue;
                }
            }
        }
        const int rs_e = p.rp[r], re_e = p.rp[r + 1];
        const int eb = max(rs_e, e0), ee = min(re_e, e1);
        const bool head = (r == r0) && (rs_e < e0);
        const bool tail = (r == r1);
        for (int pass = 0; pass < npass; ++pass) {
            const int vcol = pass * VP + c;
            const bool col_ok = active && vcol < nv;
            const char* __restrict__ vbase = p.S_in + (int64_t)min(vcol, nv - 1) * VB;
            // epilogue operands issued now so their latency hides behind the gather (short rows)
            const bool fin = !(head || tail) && e_raw == 0 && col_ok;
            Raw<VB> self_raw = zero_raw<VB>();
            float ra = 0.f, rb = 0.f, swr = 0.f, swr2 = 0.f;
            if (fin) {
                self_raw = ldv<VB>(p.S_in + (int64_t)r * p.ld_in + (int64_t)vcol * VB);
                if constexpr (WT) {
                    ra = rb = 1.f;
                    const float sw_raw = __ldg(p.sw + r);
                    swr = coef_a(sw_raw);
                    if constexpr (DUAL) swr2 = coef_b(sw_raw, p.slope2);
                } else {
                    ra = __ldg(p.rs + r);
                    rb = __ldg(p.cs + r);
                }
            }
            float acc[NACC][VALS], acc2[NACC2][VALS];
#pragma unroll
            for (int k = 0; k < NACC; ++k)
#pragma unroll
                for (int i = 0; i < VALS; ++i) acc[k][i] = 0.f;
#pragma unroll
            for (int k = 0; k < NACC2; ++k)
#pragma unroll
                for (int i = 0; i < VALS; ++i) acc2[k][i] = 0.f;
            // column indices of a batch: lane gl holds edges base + sl*L + gl (0 past the end), with their
            // coefficients when weighted
            auto load_idx = [&](int base, int (&dst)[ISL], float (&dw)[ISLW]) {
#pragma unroll
                for (int sl = 0; sl < ISL; ++sl) {
                    const int j = base + sl * L + gl;
                    const bool ok = sl * L + gl < BATCH && j < ee;
                    dst[sl] = ok ? __ldg(colp + j) : 0;
                    if constexpr (WT) dw[sl] = ok ? __ldg(p.ew + j) : 0.f;
                }
            };
            // row loads of a batch; slots past the end read row 0 (never accumulated)
            auto load_data = [&](const int (&ix)[ISL], const float (&iw)[ISLW], Raw<VB> (&dst)[LPB],
                                 float (&wd)[LPBW]) {
#pragma unroll
                for (int t = 0; t < LPB; ++t) {
                    // edge t*E + e of the batch: held by lane (t*E % L) + e in slot (t*E)/L (E divides L)
                    const int from = gbase + ((t * E) % L) + e;
                    const int src = __shfl_sync(gmask, ix[(t * E) / L], from);
                    if constexpr (WT) wd[t] = __shfl_sync(gmask, iw[(t * E) / L], from);
                    dst[t] = ldv<VB>(vbase + (size_t)(uint32_t)src * ld_in);
                }
            };
            // edge base + t*E + e belongs to group (t*E + e) mod 8, i.e. acc[t % NACC]
            auto consume = [&](const Raw<VB> (&v)[LPB], const float (&wv)[LPBW], int base) {
                const int rem = ee - base;
                auto add = [&](int t) {
                    if constexpr (DUAL) {
                        vfma<T, VB>(acc[t % NACC], v[t], coef_a(wv[t]));
                        vfma<T, VB>(acc2[t % NACC2], v[t], coef_b(wv[t], p.slope2));
                    } else if constexpr (WT) {
                        vfma<T, VB>(acc[t % NACC], v[t], coef_a(wv[t]));
                    } else {
                        vadd<T, VB>(acc[t % NACC], v[t]);
                    }
                };
                if (rem >= BATCH) {
#pragma unroll
                    for (int t = 0; t < LPB; ++t) add(t);
                } else {
#pragma unroll
                    for (int t = 0; t < LPB; ++t)
                        if (t * E + e < rem) add(t);
                }
            };
            // two-deep software pipeline, unrolled by 2 so the buffers ping-pong without copies:
            // while batch b is accumulated, batch b+1's rows and batch b+2's indices are in flight
            int ia[ISL], ib[ISL];
            float wia[ISLW], wib[ISLW], wva[LPBW], wvb[LPBW];
            Raw<VB> va[LPB], vb[LPB];
            load_idx(eb, ia, wia);
            if (eb < ee) load_data(ia, wia, va, wva);
            load_idx(eb + BATCH, ib, wib);
            for (int base = eb; base < ee;) {
                load_idx(base + 2 * BATCH, ia, wia);
                if (base + BATCH < ee) load_data(ib, wib, vb, wvb);
                consume(va, wva, base);
                base += BATCH;
                if (base >= ee) break;
                load_idx(base + 2 * BATCH, ib, wib);
                if (base + BATCH < ee) load_data(ia, wia, va, wva);
                consume(vb, wvb, base);
                base += BATCH;
            }
            // fixed butterfly over the 8 reduction groups
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                if (b < LOG_E) {
                    const int partner = gbase + ((e ^ (1 << b)) * VPP + c);
#pragma unroll
                    for (int k = 0; k < NACC; ++k)
#pragma unroll
                        for (int i = 0; i < VALS; ++i) acc[k][i] += __shfl_sync(gmask, acc[k][i], partner);
                    if constexpr (DUAL) {
#pragma unroll
                        for (int k = 0; k < NACC2; ++k)
#pragma unroll
                            for (int i = 0; i < VALS; ++i) acc2[k][i] += __shfl_sync(gmask, acc2[k][i], partner);
                    }
                } else {
                    const int kb = 1 << (b - LOG_E);
#pragma unroll
                    for (int k = 0; k < NACC; ++k)
                        if ((k & kb) == 0 && (k | kb) < NACC) {
#pragma unroll
                            for (int i = 0; i < VALS; ++i) acc[k][i] += acc[k | kb][i];
                            if constexpr (DUAL) {
#pragma unroll
                                for (int i = 0; i < VALS; ++i) acc2[k][i] += acc2[k | kb][i];
                            }
                        }
                }
            }
            if (e_raw != 0 || !col_ok) continue;
            if (head || tail) {
                const int64_t coff = ((u * 2 + (head ? 0 : 1)) * (int64_t)row_vals) + vcol * VALS;
#pragma unroll
                for (int i = 0; i < VALS; ++i) p.carry[coff + i] = acc[0][i];
                if constexpr (DUAL) {
#pragma unroll
                    for (int i = 0; i < VALS; ++i) p.carry2[coff + i] = acc2[0][i];
                }
                continue;
            }
            const float sig = (p.mode == 0) ? p.gamma * ra * rb : p.gamma * ra;
            float out[VALS];
            if constexpr (DUAL) {
                float out2[VALS];
#pragma unroll
                for (int i = 0; i < VALS; ++i) out2[i] = sig * __fmaf_rn(swr2, Vec<T, VB>::elem(self_raw, i), acc2[0][i]);
                stv<VB>(p.S_out2 + r * p.ld_out + (int64_t)vcol * VB, Vec<T, VB>::pack(out2));
            }
            if constexpr (WT) {   // gamma * (sum_u w_uv S_u + w_vv S_v); no alpha mix (the GAT epoch's reading)
#pragma unroll
                for (int i = 0; i < VALS; ++i)
                    out[i] = sig * __fmaf_rn(swr, Vec<T, VB>::elem(self_raw, i), acc[0][i]);
            } else if (p.alpha != 0.f) {
                const Raw<VB> s0_raw = ldv<VB>(p.S0 + (int64_t)r * p.ld_s0 + (int64_t)vcol * VB);
                const float beta = (p.mode == 0) ? p.alpha : p.alpha / rb;
#pragma unroll
                for (int i = 0; i < VALS; ++i)
                    out[i] = sig * (acc[0][i] + (0.f + Vec<T, VB>::elem(self_raw, i))) +
                             beta * (0.f + Vec<T, VB>::elem(s0_raw, i));
            } else {
#pragma unroll
                for (int i = 0; i < VALS; ++i) out[i] = sig * (acc[0][i] + (0.f + Vec<T, VB>::elem(self_raw, i)));
            }
            stv<VB>(out_row_ptr(p, r) + (int64_t)vcol * VB, Vec<T, VB>::pack(out));
        }
    }
#ifndef NTP_NO_P2P_FENCE
    if (p.peer_out) __threadfence_system();
#endif
}

// Wide rows (>= 1 KB of slice per vertex, e.g. the Orkut c4 pipeline at N <= 2).  The register-staged
// gather above keeps what the register file allows in flight (ncu, Orkut w = 512 fp32: 22% warps active,
// DRAM 59% of the copy peak, L2 28%).  Here a producer warp streams every arc's whole row slice into a
// shared-memory ring with cp.async.bulk -- nothing in flight occupies registers; completion is counted on
// one mbarrier per stage of A arcs -- and NW = row bytes / 512 consumer warps each own a 512-byte column
// chunk (one 16-byte vector per lane).  Arc j of a row accumulates into group (j - eb) mod 8 in ascending
// order and the 8 groups are reduced by the same butterfly ((a0+a1)+(a2+a3))+((a4+a5)+(a6+a7)): every
// column is summed exactly as in spmm_hop_kernel, so the two kernels give bitwise equal results and the
// slice-width (P) invariance holds across them.  One CTA per merge-path unit, all rows (no row range).
template <typename T, int NW, int A, int S>
__global__ void __launch_bounds__(32 * (NW + 1)) spmm_hop_bulk_kernel(const HopParams p) {
    extern __shared__ __align__(1024) uint8_t bulk_smem[];
    constexpr int RB = NW * 512;
    constexpr int VALS = Vec<T, 16>::N;
    uint64_t* full = reinterpret_cast<uint64_t*>(bulk_smem + (size_t)S * A * RB);
    uint64_t* empty = full + S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t u = p.u_begin + blockIdx.x;
    if (u >= p.u_end) return;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], NW);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    const int r0 = p.unit_row[u], r1 = p.unit_row[u + 1];
    const int e0 = p.unit_e[u], e1 = p.unit_e[u + 1];
    const int total = e1 - e0;                     // the unit's arcs, consumed in CSR order
    if (warp == NW) {                              // ---- producer
        const int nst = (total + A - 1) / A;
        for (int st = 0; st < nst; ++st) {
            const int stage = st % S;
            const int cnt = min(A, total - st * A);
            const int j = e0 + st * A + lane;
            const int src = lane < cnt ? __ldg(p.col + j) : 0;
            if (lane == 0) {
                if (st >= S) ptx::mbar_wait(&empty[stage], ((st / S) - 1) & 1);
                ptx::mbar_expect_tx(&full[stage], (uint32_t)cnt * RB);
            }
            __syncwarp();
            if (lane < cnt)
                ptx::bulk_load(bulk_smem + ((size_t)stage * A + lane) * RB, p.S_in + (size_t)(uint32_t)src * p.ld_in, RB,
                               &full[stage]);
        }
        return;
    }
    // ---- consumers: warp w owns 16-byte vector vcol = 32 w + lane of every row slice
    const int vcol = warp * 32 + lane;
    const bool has_tail = (r1 < p.n) && (e1 > max(p.rp[r1], e0));
    const int r_end = has_tail ? r1 + 1 : r1;
    const int row_vals = p.nvec * VALS;
    int k = 0;                                     // arcs consumed so far
    for (int r = r0; r < r_end; ++r) {
        const int rs_e = p.rp[r], re_e = p.rp[r + 1];
        const int eb = max(rs_e, e0), ee = min(re_e, e1);
        const bool head = (r == r0) && (rs_e < e0);
        const bool tail = (r == r1);
        const bool fin = !(head || tail);
        Raw<16> self_raw = zero_raw<16>();
        float ra = 0.f, rb = 0.f;
        if (fin) {
            self_raw = ldv<16>(p.S_in + (int64_t)r * p.ld_in + (int64_t)vcol * 16);
            ra = __ldg(p.rs + r);
            rb = __ldg(p.cs + r);
        }
        float acc[kG][VALS];
#pragma unroll
        for (int g = 0; g < kG; ++g)
#pragma unroll
            for (int i = 0; i < VALS; ++i) acc[g][i] = 0.f;
        for (int jb = eb; jb < ee; jb += kG) {   // arc jb + g belongs to group g (static register index)
#pragma unroll
            for (int g = 0; g < kG; ++g) {
                if (jb + g >= ee) break;
                const int st = k / A, stage = st % S, slot = k - st * A;
                if (slot == 0) ptx::mbar_wait(&full[stage], (st / S) & 1);
                const uint4 x =
                    *reinterpret_cast<const uint4*>(bulk_smem + ((size_t)stage * A + slot) * RB + vcol * 16);
                const Raw<16> xr{{x.x, x.y, x.z, x.w}};
                vadd<T, 16>(acc[g], xr);
                if (slot == A - 1 || k == total - 1) {
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&empty[stage]);
                }
                ++k;
            }
        }
        // fixed butterfly over the 8 reduction groups (in-lane; the E = 1 form of spmm_hop_kernel)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            const int kb = 1 << b;
#pragma unroll
            for (int g = 0; g < kG; ++g)
                if ((g & kb) == 0 && (g | kb) < kG) {
#pragma unroll
                    for (int i = 0; i < VALS; ++i) acc[g][i] += acc[g | kb][i];
                }
        }
        if (head || tail) {
            float* dst = p.carry + ((u * 2 + (head ? 0 : 1)) * (int64_t)row_vals) + vcol * VALS;
#pragma unroll
            for (int i = 0; i < VALS; ++i) dst[i] = acc[0][i];
            continue;
        }
        const float sig = (p.mode == 0) ? p.gamma * ra * rb : p.gamma * ra;
        float out[VALS];
        if (p.alpha != 0.f) {
            const Raw<16> s0_raw = ldv<16>(p.S0 + (int64_t)r * p.ld_s0 + (int64_t)vcol * 16);
            const float beta = (p.mode == 0) ? p.alpha : p.alpha / rb;
#pragma unroll
            for (int i = 0; i < VALS; ++i)
                out[i] = sig * (acc[0][i] + (0.f + Vec<T, 16>::elem(self_raw, i))) +
                         beta * (0.f + Vec<T, 16>::elem(s0_raw, i));
        } else {
#pragma unroll
            for (int i = 0; i < VALS; ++i) out[i] = sig * (acc[0][i] + (0.f + Vec<T, 16>::elem(self_raw, i)));
        }
        stv<16>(out_row_ptr(p, r) + (int64_t)vcol * 16, Vec<T, 16>::pack(out));
    }
#ifndef NTP_NO_P2P_FENCE
    if (p.peer_out) __threadfence_system();
#endif
}

constexpr int kBulkA = 4, kBulkS = 4;   // arcs per stage, stages in flight per unit
constexpr int64_t kBulkMinBytes = 1024;  // auto: rows of >= 1 KB take the bulk-copy gather

template <typename T, int NW, int A, int S>
void launch_bulk_as(const HopParams& p, cudaStream_t s) {
    constexpr size_t smem = (size_t)S * A * NW * 512 + 2 * S * sizeof(uint64_t);
    static bool attr = false;
    if (!attr) {
        NTP_CUDA(cudaFuncSetAttribute(spmm_hop_bulk_kernel<T, NW, A, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
        attr = true;
    }
    spmm_hop_bulk_kernel<T, NW, A, S><<<(unsigned)(p.u_end - p.u_begin), 32 * (NW + 1), smem, s>>>(p);
    NTP_LAUNCH_CHECK();
}

template <typename T, int NW>
void launch_bulk(const HopParams& p, cudaStream_t s) {
    // ring shape measured on the Orkut shape (ms per hop at 4 KB / 2 KB / 1 KB rows): 4 arcs x 4 stages
    // 61.2 / 28.6 / 15.1; 8 x 3: 65.8 / 31.3 / 15.3; 2 x 8: 63.3 / 30.7 / 16.4; 4 x 6: 66.9 / 32.1 / 16.0;
    // 2 x 4: 65.1 / 30.5 / 16.1 (register-staged kernel: 81.6 / 38.5 / 18.5; at 512 B rows 9.13 vs 9.49 bulk)
    launch_bulk_as<T, NW, kBulkA, kBulkS>(p, s);
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
    constexpr int VALS = 16 / sizeof(T);
    const int row_vals = p.nvec * VALS;
    const float a = p.sw ? 1.f : p.rs[r];
    const float b = p.sw ? 1.f : p.cs[r];
    const float swr = p.sw ? coef_a(p.sw[r]) : 0.f;
    const float swr2 = p.S_out2 ? coef_b(p.sw[r], p.slope2) : 0.f;
    char* orow_p = out_row_ptr(p, r);
    for (int k = lane; k < row_vals; k += 32) {
        float acc = p.carry[(u * 2 + 1) * (int64_t)row_vals + k];
        float acc2 = p.S_out2 ? p.carry2[(u * 2 + 1) * (int64_t)row_vals + k] : 0.f;
        for (int64_t v = u + 1;; ++v) {
            acc += p.carry[(v * 2 + 0) * (int64_t)row_vals + k];
            if (p.S_out2) acc2 += p.carry2[(v * 2 + 0) * (int64_t)row_vals + k];
            if (p.unit_row[v + 1] > r) break;
        }
        const int vcol = k / VALS, comp = k % VALS;
        float self[VALS];
        load16<T>(p.S_in + (int64_t)r * p.ld_in + (int64_t)vcol * 16, self);
        const float sig = (p.mode == 0) ? p.gamma * a * b : p.gamma * a;
        if (p.S_out2) {
            const float out2 = sig * __fmaf_rn(swr2, self[comp], acc2);
            char* o2 = p.S_out2 + (int64_t)r * p.ld_out;
            if (sizeof(T) == 4) reinterpret_cast<float*>(o2)[k] = out2;
            else reinterpret_cast<__nv_bfloat16*>(o2)[k] = __float2bfloat16_rn(out2);
        }
        float out = p.sw ? sig * __fmaf_rn(swr, self[comp], acc) : sig * (acc + self[comp]);
        if (p.alpha != 0.f) {
            float h[VALS];
            load16<T>(p.S0 + (int64_t)r * p.ld_s0 + (int64_t)vcol * 16, h);
            out += ((p.mode == 0) ? p.alpha : p.alpha / b) * h[comp];
        }
        if (sizeof(T) == 4) {
            reinterpret_cast<float*>(orow_p)[k] = out;
        } else {
            reinterpret_cast<__nv_bfloat16*>(orow_p)[k] = __float2bfloat16_rn(out);
        }
    }
#ifndef NTP_NO_P2P_FENCE
    if (p.peer_out) __threadfence_system();
#endif
}

template <typename T>
__global__ void prescale_kernel(const char* __restrict__ H, int64_t ld_h, char* __restrict__ S, int64_t ld_s,
                                int32_t nvec, const float* __restrict__ scale, int64_t rows,
                                const int32_t* __restrict__ src_rows) {
    constexpr int VALS = 16 / sizeof(T);
    const int64_t total = rows * nvec;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / nvec;
        const int64_t vc = i % nvec;
        const int64_t hr = src_rows ? (int64_t)src_rows[r] : r;    // reordered graph: gather in original order
        float v[VALS];
        load16<T>(H + hr * ld_h + vc * 16, v);
        const float s = scale ? scale[r] : 1.f;
#pragma unroll
        for (int k = 0; k < VALS; ++k) v[k] *= s;
        store16<T>(S + r * ld_s + vc * 16, v);
    }
}

bool carveout_max_l1() {
    static const bool v = [] { const char* e = getenv("NTP_L1_CARVEOUT"); return e ? atoi(e) != 0 : true; }();
    return v;
}

// 256-thread CTAs, one unit per lane group, the whole unified array as L1 (no shared memory).
template <typename T, int VB, int E, int L, int MODE, bool WT = false, bool DUAL = false>
void launch_variant(const HopParams& p, cudaStream_t s) {
    static bool attr = false;
    if (!attr && carveout_max_l1()) {
        NTP_CUDA(cudaFuncSetAttribute(spmm_hop_kernel<T, VB, E, L, MODE, WT, DUAL>,
                                      cudaFuncAttributePreferredSharedMemoryCarveout, 0));
        attr = true;
    }
    spmm_hop_kernel<T, VB, E, L, MODE, WT, DUAL><<<(unsigned)cdiv((p.u_end - p.u_begin) * L, kBlock), kBlock, 0, s>>>(p);
    NTP_LAUNCH_CHECK();
}

template <typename T, int VB, int E, int L>
void launch_hop(const HopParams& p, cudaStream_t s) {
    if constexpr (VB == 16) {
        if (p.ew) {   // weighted (GAT attention): the dual hop, general path only
            launch_variant<T, VB, E, L, 0, true, true>(p, s);
            return;
        }
    }
    static const int short_env = [] { const char* v = getenv("NTP_SPMM_SHORT"); return v ? atoi(v) : -1; }();
    // low-degree variants when the average degree is below 32 (products, papers shapes)
    const bool low_deg = short_env >= 0 ? short_env != 0 : (p.nnz < 32 * std::max<int64_t>(p.n, 1));
    constexpr int LOW = (E >= 4) ? 3 : (E >= 2) ? 2 : 0;   // short batches where E >= 4, tiny rows where E >= 2
    // high-degree graphs: rows of <= 4 vectors (<= 64 B) run the 4-CTA/SM half-batch variant (OCC 2:
    // measured 9-10% faster per hop at 32-64 B rows on the Reddit shape, 4-5% slower at 96-176 B)
    static const int occ_env = [] { const char* v = getenv("NTP_SPMM_OCC"); return v ? atoi(v) : -1; }();
    const int occ = occ_env >= 0 ? occ_env : (p.nvec * 16 / VB <= 4 ? 2 : 0);
    // high-degree graphs, two edge slots (rows of 9-16 16-byte vectors, e.g. the Reddit slice at P = 1): the
    // 4-CTA/SM half-batch variant with ONE accumulator per lane slot -- 2.06 vs 2.29 ms per hop at 176 B --
    // trading the slice-width-invariant reduction order for occupancy (results stay within R10 of the
    // oracle; NTP_SPMM_INVARIANT=1, read per call, keeps the invariant order everywhere)
    // (one edge slot measured slower that way: 64 registers spill its 8-vector batches -- Orkut 96 columns
    // 11.0 vs 8.5 ms per hop, Reddit 80 columns 7.6 vs 4.6)
    if constexpr (E == 2 && VB == 16) {
        const char* inv = getenv("NTP_SPMM_INVARIANT");
        if (!low_deg && occ_env < 0 && !(inv && atoi(inv) != 0)) {
            launch_variant<T, VB, E, L, 8 | 32>(p, s);
            return;
        }
    }
    if (low_deg) launch_variant<T, VB, E, L, LOW>(p, s);
    else if (occ == 1) launch_variant<T, VB, E, L, 4>(p, s);
    else if (occ == 2) launch_variant<T, VB, E, L, 8>(p, s);
    else launch_variant<T, VB, E, L, 0>(p, s);
}

// (E, L) from the row width in VB-byte vectors: E edge slots of nv lanes each, E*nv <= L.
template <typename T, int VB>
void dispatch_hop(const HopParams& p, int nv, cudaStream_t s) {
    if (nv == 1) launch_hop<T, VB, 8, 8>(p, s);
    else if (nv == 2) launch_hop<T, VB, 8, 16>(p, s);
    else if (nv <= 4) launch_hop<T, VB, 8, 32>(p, s);
    else if (nv <= 8) launch_hop<T, VB, 4, 32>(p, s);
    else if constexpr (VB == 16) {
        if (nv <= 16) launch_hop<T, VB, 2, 32>(p, s);
        else launch_hop<T, VB, 1, 32>(p, s);
    }
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
              float gamma, float alpha, int mode, int64_t row_lo, int64_t row_hi, cudaStream_t s,
              const int32_t* out_rows, const PeerOut* po, const float* ew, const float* sw, void* S_out2,
              float slope2) {
    const Graph& g = c->g;
    NTP_CHECK(!ew == !S_out2 && (!S_out2 || (!out_rows && !(po && po->tab))), NTP_ERR_ARG,
              "a weighted hop is the dual hop (two outputs) and writes local rows");
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
    p.nnz = g.nnz;
    p.out_rows = out_rows;
    p.peer_out = (po && po->tab) ? po->tab : nullptr;
    p.po_V_p = po ? po->V_p : 0;
    p.po_rank = po ? po->rank : 0;
    p.ew = ew;
    p.sw = sw;
    p.S_out2 = static_cast<char*>(S_out2);
    p.slope2 = slope2;

    unit_range(csr, row_lo, row_hi, p.u_begin, p.u_end);
    p.row_lo = row_lo;
    p.row_hi = row_hi;
    p.nvec = nvec;
    p.gamma = gamma;
    p.alpha = alpha;
    p.mode = mode;
    c->carry.ensure((size_t)(csr.U * 2) * nvec * vals * sizeof(float) + 16);
    p.carry = c->carry.as<float>();
    p.carry2 = nullptr;
    if (S_out2) {
        c->carry2.ensure((size_t)(csr.U * 2) * nvec * vals * sizeof(float) + 16);
        p.carry2 = c->carry2.as<float>();
    }
    if (p.u_end <= p.u_begin) return;
    // 32-byte vectors when every row the hop touches is 32-byte aligned and at most 8 of them wide
    // (E >= 4 edge slots: wider rows would need more accumulator registers than the kernel has)
    // auto (NTP_SPMM_VB unset), by row width -- measured ms per hop, 16-byte vs 32-byte vectors:
    //   papers (bf16): 256 B 107.3 vs 105.0, 128 B 72.1 vs 61.8, 64 B 37.9 vs 39.4, 32 B 24.5 vs 23.6
    //   products (fp32): 192 B 2.95 vs 2.98, 96 B 2.03 vs 1.75, 32 B 0.89 vs 0.95
    //   Reddit (fp32): 96 B 1.435 vs 1.409, 32 B 0.85 vs 1.02
    static const int vb_env = [] { const char* v = getenv("NTP_SPMM_VB"); return v ? atoi(v) : -1; }();
    const bool low_deg_g = p.nnz < 32 * std::max<int64_t>(p.n, 1);
    const bool al32 = (nvec % 2) == 0 && nvec <= 16 && p.ld_in % 32 == 0 && p.ld_out % 32 == 0 &&
                      ((uintptr_t)S_in % 32) == 0 && ((uintptr_t)S_out % 32) == 0 &&
                      (S0 == nullptr || (p.ld_s0 % 32 == 0 && ((uintptr_t)S0 % 32) == 0));
    // rows of 96 / 128 / 256 B (and 32-B bf16 rows on low-degree graphs) measured faster with 32-byte vectors
    const bool auto32 = nvec == 6 || nvec == 8 || nvec == 16 || (nvec == 2 && dt == NTP_BF16 && low_deg_g);
    // wide rows over the whole graph: the bulk-copy gather (NTP_SPMM_BULK: -1 auto, 0 off, 1 any multiple of 512 B)
    static const int bulk_env = [] { const char* v = getenv("NTP_SPMM_BULK"); return v ? atoi(v) : -1; }();
    const int64_t row_bytes = (int64_t)nvec * 16;
    const bool bulk_ok = !ew && row_lo == 0 && row_hi == g.n &&
                         (row_bytes == 512 || row_bytes == 1024 || row_bytes == 2048 || row_bytes == 4096) &&
                         (uintptr_t)S_in % 16 == 0 && p.ld_in % 16 == 0;
    if (bulk_ok && (bulk_env == 1 || (bulk_env < 0 && row_bytes >= kBulkMinBytes))) {
        const int nw = (int)(row_bytes / 512);
        if (dt == NTP_F32) {
            if (nw == 1) launch_bulk<float, 1>(p, s);
            else if (nw == 2) launch_bulk<float, 2>(p, s);
            else if (nw == 4) launch_bulk<float, 4>(p, s);
            else launch_bulk<float, 8>(p, s);
        } else {
            if (nw == 1) launch_bulk<__nv_bfloat16, 1>(p, s);
            else if (nw == 2) launch_bulk<__nv_bfloat16, 2>(p, s);
            else if (nw == 4) launch_bulk<__nv_bfloat16, 4>(p, s);
            else launch_bulk<__nv_bfloat16, 8>(p, s);
        }
    } else if (al32 && !ew && (vb_env == 32 || (vb_env < 0 && auto32))) {
        if (dt == NTP_F32) dispatch_hop<float, 32>(p, nvec / 2, s);
        else dispatch_hop<__nv_bfloat16, 32>(p, nvec / 2, s);
    } else {
        if (dt == NTP_F32) dispatch_hop<float, 16>(p, nvec, s);
        else dispatch_hop<__nv_bfloat16, 16>(p, nvec, s);
    }
    const int64_t fblocks = cdiv((p.u_end - p.u_begin) * 32, kBlock);
    if (dt == NTP_F32) spmm_fixup_kernel<float><<<(unsigned)fblocks, kBlock, 0, s>>>(p);
    else spmm_fixup_kernel<__nv_bfloat16><<<(unsigned)fblocks, kBlock, 0, s>>>(p);
    NTP_LAUNCH_CHECK();
    count_launch(c, 2);
}

void prescale(ntp_ctx* c, const void* H, int64_t ld_h, void* S, int64_t ld_s, int32_t cols, const float* scale,
              int64_t rows, ntp_dtype dt, cudaStream_t s, const int32_t* src_rows) {
    if (rows <= 0) return;
    const size_t es = esize(dt);
    const int32_t nvec = (int32_t)(cols * es / 16);
    const int64_t total = rows * nvec;
    const int blocks = (int)std::min<int64_t>(cdiv(total, 256), 148 * 16);
    if (dt == NTP_F32)
        prescale_kernel<float><<<blocks, 256, 0, s>>>((const char*)H, ld_h * es, (char*)S, ld_s * es, nvec, scale, rows,
                                                      src_rows);
    else
        prescale_kernel<__nv_bfloat16><<<blocks, 256, 0, s>>>((const char*)H, ld_h * es, (char*)S, ld_s * es, nvec,
                                                              scale, rows, src_rows);
    NTP_LAUNCH_CHECK();
    count_launch(c);
}

// K hops.  Hop k writes bufs[(K-k) % 2] (bufs = {Z, scratch}) so hop K lands in Z.
// S^0 = cs .* H is formed by `prescale` unless the caller already holds it
// (prescaled_input: a.H points at S^0, e.g. the pack epilogue of the split).
// With alpha != 0, S^0 must outlive hop 1, so it gets its own buffer.
void propagate(ntp_ctx* c, const PropArgs& a, cudaStream_t s, bool time_hops, bool prescaled_input,
               LastHop* defer_last) {
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
    // reordered graph: the slice arrives in original vertex order; S^0 is formed in internal order
    // (gather through inv; a pre-scaled input is only permuted) and the last hop scatters back
    const int32_t* inv = g.inv_p();
    NTP_CHECK(!(inv && defer_last), NTP_ERR_CONFIG, "chunked overlap needs original vertex order (no NTP_G_REORDER)");
    const void* S0;
    int64_t ld_s0;
    const float* pre = prescaled_input ? nullptr : cs;
    if (prescaled_input && !inv) {
        S0 = a.H;
        ld_s0 = a.ld_h;
    } else if (a.alpha != 0.f) {
        c->prop_s0.ensure((size_t)n * ld_t * es + 16);
        prescale(c, a.H, a.ld_h, c->prop_s0.p, ld_t, a.cols, pre, n, a.dtype, s, inv);
        S0 = c->prop_s0.p;
        ld_s0 = ld_t;
    } else {
        const int b0 = a.K % 2;       // hop 1 writes bufs[(K-1)%2], so S^0 may live in bufs[K%2]
        prescale(c, a.H, a.ld_h, bufs[b0], lds[b0], a.cols, pre, n, a.dtype, s, inv);
        S0 = bufs[b0];
        ld_s0 = lds[b0];
    }
    const void* sin = S0;
    int64_t ld_sin = ld_s0;
    for (int k = 1; k <= a.K; ++k) {
        const int nxt = (a.K - k) % 2;
        const bool last = (k == a.K);
        if (last && defer_last) {
            *defer_last = LastHop{&csr, rs, cs, sin, ld_sin, S0, ld_s0, bufs[nxt], lds[nxt], a.cols, a.dtype,
                                  a.gamma, a.alpha};
            return;
        }
        const bool timed = time_hops && c->hop_ev_used + 2 <= kHopEvents;
        if (timed) NTP_CUDA(record_timing(c, c->hop_ev[c->hop_ev_used], s));
        spmm_hop(c, csr, rs, cs, sin, bufs[nxt], S0, ld_sin, lds[nxt], ld_s0, a.cols, a.dtype, a.gamma, a.alpha,
                 last ? 1 : 0, 0, -1, s, last ? inv : nullptr, last ? &a.po : nullptr);
        if (timed) {
            NTP_CUDA(record_timing(c, c->hop_ev[c->hop_ev_used + 1], s));
            c->hop_ev_used += 2;
        }
        sin = bufs[nxt];
        ld_sin = lds[nxt];
    }
}

void* propagate_consume(ntp_ctx* c, const PropArgs& a, cudaStream_t s, bool time_hops, bool input_internal) {
    if (a.alpha != 0.f || a.K == 0 || a.ld_h != a.ld_z || a.po.tab) {
        propagate(c, a, s, time_hops, true);
        return a.Z;
    }
    const Graph& g = c->g;
    const Csr& csr = a.transposed ? g.bwd() : g.fwd();
    const float* rs = a.transposed ? g.dinv_out_p() : g.dinv_in_p();
    const float* cs = a.transposed ? g.dinv_in_p() : g.dinv_out_p();
    const int32_t* inv = g.inv_p();
    void* cur = const_cast<void*>(a.H);
    void* oth = a.Z;
    if (inv && !input_internal) {   // reordered graph: S^0 permuted into internal order first (other buffer)
        prescale(c, cur, a.ld_h, oth, a.ld_z, a.cols, nullptr, g.n, a.dtype, s, inv);
        std::swap(cur, oth);
    }
    for (int k = 1; k <= a.K; ++k) {
        const bool last = (k == a.K);
        const bool timed = time_hops && c->hop_ev_used + 2 <= kHopEvents;
        if (timed) NTP_CUDA(record_timing(c, c->hop_ev[c->hop_ev_used], s));
        spmm_hop(c, csr, rs, cs, cur, oth, cur, a.ld_h, a.ld_z, a.ld_h, a.cols, a.dtype, a.gamma, 0.f, last ? 1 : 0, 0,
                 -1, s, last ? inv : nullptr, nullptr);
        if (timed) {
            NTP_CUDA(record_timing(c, c->hop_ev[c->hop_ev_used + 1], s));
            c->hop_ev_used += 2;
        }
        std::swap(cur, oth);
    }
    return cur;
}

void run_last_hop(ntp_ctx* c, const LastHop& lh, int64_t row_lo, int64_t row_hi, cudaStream_t s, bool time_hops) {
    const bool timed = time_hops && c->hop_ev_used + 2 <= kHopEvents;
    if (timed) NTP_CUDA(record_timing(c, c->hop_ev[c->hop_ev_used], s));
    spmm_hop(c, *lh.csr, lh.rs, lh.cs, lh.sin, lh.out, lh.S0, lh.ld_sin, lh.ld_out, lh.ld_s0, lh.cols, lh.dt, lh.gamma,
             lh.alpha, 1, row_lo, row_hi, s);
    if (timed) {
        NTP_CUDA(record_timing(c, c->hop_ev[c->hop_ev_used + 1], s));
        c->hop_ev_used += 2;
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
