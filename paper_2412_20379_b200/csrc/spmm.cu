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

template <typename T> struct V16;
__device__ __forceinline__ uint4 ld_raw(const void* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }

// Gather load with a cache policy: 0 = ld.global.nc (L1 allocate), 1 = ld.global.nc.L1::no_allocate,
// 2 = ld.global.cg (L2 only).
template <int POL>
__device__ __forceinline__ uint4 ld_gather(const void* p) {
    uint4 r;
    if constexpr (POL == 0) {
        r = __ldg(reinterpret_cast<const uint4*>(p));
    } else if constexpr (POL == 1) {
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    } else {
        asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    }
    return r;
}

template <> struct V16<float> {
    static constexpr int N = 4;
    __device__ __forceinline__ static float elem(const uint4 x, int i) {
        return __uint_as_float(i == 0 ? x.x : i == 1 ? x.y : i == 2 ? x.z : x.w);
    }
    __device__ __forceinline__ static void add_raw(float (&a)[4], const uint4 x) {
        a[0] += __uint_as_float(x.x); a[1] += __uint_as_float(x.y);
        a[2] += __uint_as_float(x.z); a[3] += __uint_as_float(x.w);
    }
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
    __device__ __forceinline__ static uint4 pack(const float (&v)[4]) {
        return make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]), __float_as_uint(v[3]));
    }
};
template <> struct V16<__nv_bfloat16> {
    static constexpr int N = 8;
    __device__ __forceinline__ static float elem(const uint4 x, int i) {
        const uint32_t w = (i >> 1) == 0 ? x.x : (i >> 1) == 1 ? x.y : (i >> 1) == 2 ? x.z : x.w;
        return __uint_as_float((i & 1) ? (w & 0xFFFF0000u) : (w << 16));
    }
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
    __device__ __forceinline__ static void add_raw(float (&a)[8], const uint4 x) {
        float v[8];
        unpack(x, v);
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] += v[i];
    }
    __device__ __forceinline__ static void add(const void* p, float (&a)[8]) {
        float v[8];
        unpack(__ldg(reinterpret_cast<const uint4*>(p)), v);
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] += v[i];
    }
    __device__ __forceinline__ static uint4 pack(const float (&v)[8]) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
            w[i] = *reinterpret_cast<const uint32_t*>(&h);
        }
        return make_uint4(w[0], w[1], w[2], w[3]);
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
    int tma_per8;                      // groups (out of every 8) that gather with TMA gather4
    int64_t nnz;
};

// Lane layout ("full row per edge"): a group of L lanes works on one unit.  Lane
// gl = e*VP + c holds edge slot e in [0, E) and 16-byte column vector c in [0, VP):
// one load instruction fetches the complete row slices of E edges with
// consecutive lanes, so it touches the fewest distinct 128-byte lines (the L1TEX
// wavefront count is what bounds a gather).  Edge j of a unit piece
// starting at eb belongs to reduction group g = (j - eb) mod 8, g = e + E*k: lane
// slot e keeps 8/E accumulators acc[k].  The 8 groups are combined by the fixed
// butterfly ((a0+a1)+(a2+a3))+((a4+a5)+(a6+a7)) -- cross-lane for the bits of e,
// in-lane for the bits of k -- so the per-column order is the same for every
// (E, VP), i.e. for every slice width.  Column indices are loaded coalesced (one
// per lane) and distributed with shuffles.
// GATHER: 0 = LSU loads (ld.global, policy POL), 1 = TMA tile::gather4 into a per-group
// double-buffered shared-memory ring (no L1 data-pipe fill), read back with LDS.
// MODE (low-degree graphs, average degree < 32): bit 0 = short batches (E >= 4): 8-16-edge
// batches so a ~15-arc row does not pay for a 64-slot batch, and fewer registers for 3 CTAs per
// SM; bit 1 = tiny-row path (E >= 2, below).  Neither enters the reduction order (groups are
// (j - eb) mod 8 for any batch that is a multiple of 8), and the tiny path's registers are only
// paid where it is used.
template <typename T, int E, int L, int POL, int GATHER, int MODE = 0>
__global__ void __launch_bounds__(kBlock, ((MODE & 1) && E == 8) ? 3 : 2) spmm_hop_kernel(const HopParams p, const __grid_constant__ CUtensorMap tmS) {
    constexpr bool SHORT = (MODE & 1) != 0;
    constexpr bool TINY = (MODE & 2) != 0 && E >= 2;
    // GATHER == 1: mixed mode -- groups with (gidx % 8) < p.tma_per8 use the TMA engine, the others
    // the LSU path, so both units pull rows from L2 concurrently (same reduction order either way).
    constexpr int NACC = kG / E;
    constexpr int LOG_E = (E == 1) ? 0 : (E == 2) ? 1 : (E == 4) ? 2 : 3;
    constexpr int VALS = V16<T>::N;
    // edges per pipeline batch: 16-byte loads per lane per batch = BATCH / E (4 or 8)
    constexpr int BATCH = SHORT ? ((E >= 4) ? 16 : 8) : ((E == 8) ? 64 : (E == 4) ? 32 : 8 * E);
    constexpr int LPB = BATCH / E;                        // loads per lane per batch
    constexpr int ISL = (BATCH + L - 1) / L;              // column indices held per lane
    const int lane = threadIdx.x & 31;
    const int gl = lane % L;
    const int gbase = lane - gl;
    const int64_t group = ((int64_t)blockIdx.x * kBlock + threadIdx.x) / L;
    const int64_t u = p.u_begin + group;
    // TMA ring: per group 2 buffers of BATCH/4 gather4 slots, slot = 4 rows rounded to 128 B
    extern __shared__ __align__(128) uint8_t tma_smem[];
    constexpr int GPC = kBlock / L;                      // groups per CTA
    const int row_bytes = p.nvec * 16;
    const int slot_bytes = (4 * row_bytes + 127) & ~127;
    const int buf_bytes = (BATCH / 4) * slot_bytes;
    const int gidx = threadIdx.x / L;
    uint8_t* gbuf = tma_smem + (size_t)gidx * 2 * buf_bytes;
    uint64_t* gbar = reinterpret_cast<uint64_t*>(tma_smem + (size_t)GPC * 2 * buf_bytes) + 2 * gidx;
    uint32_t ph0 = 0, ph1 = 0;
    const bool tma_group = (GATHER == 1) && ((gidx & 7) < p.tma_per8);
    const int fillv = tma_group ? (int)p.n : 0;
    if constexpr (GATHER == 1) {
        if (gl == 0) {
            ptx::mbar_init(&gbar[0], 1);
            ptx::mbar_init(&gbar[1], 1);
            ptx::fence_mbar_init();
        }
        __syncthreads();
    }
    if (u >= p.u_end) return;                           // group-uniform exit
    const unsigned gmask = (L == 32) ? 0xffffffffu : (((1u << L) - 1u) << gbase);
    const int VP = (E == 1) ? min(p.nvec, 32) : p.nvec;  // vectors per pass
    const int e_raw = gl / VP;
    const int c = gl - e_raw * VP;
    const bool active = e_raw < E;
    const int e = active ? e_raw : E - 1;                // idle lanes mirror a real lane's addresses
    const int32_t* __restrict__ colp = p.col;
    const uint32_t ld_in = (uint32_t)p.ld_in;

    const int r0 = p.unit_row[u], r1 = p.unit_row[u + 1];
    const int e0 = p.unit_e[u], e1 = p.unit_e[u + 1];
    const bool has_tail = (r1 < p.n) && (e1 > max(p.rp[r1], e0));
    const int r_end = has_tail ? r1 + 1 : r1;
    const int row_vals = p.nvec * VALS;
    const int npass = (p.nvec + VP - 1) / VP;

    const int r_stop = (int)min((int64_t)r_end, p.row_hi);
    for (int r = max((int64_t)r0, p.row_lo); r < r_stop; ++r) {
        // ---- tiny-row fast path: E consecutive rows with <= 8 arcs each, wholly inside this unit,
        // one row per edge slot.  With <= 8 arcs every reduction group holds at most one arc, so
        // acc_g = 0 + v_g and the in-lane tree ((v0+v1)+(v2+v3))+((v4+v5)+(v6+v7)) is exactly the
        // canonical butterfly: results are bitwise those of the general path.
        if (TINY && npass == 1 && r + E <= r1 && r + E <= r_stop) {
            const int my_r = r + e;
            const int trs = __ldg(p.rp + my_r), tre = __ldg(p.rp + my_r + 1);
            const int deg = tre - trs;
            const bool ok = deg <= 8 && !(my_r == r0 && trs < e0);
            if (__all_sync(gmask, ok)) {
                const bool cok = active && c < p.nvec;
                const int64_t voff = (int64_t)min(c, p.nvec - 1) * 16;
                const uint4 self_raw = ld_raw(p.S_in + (int64_t)my_r * p.ld_in + voff);
                const uint4 s0_raw = (p.alpha != 0.f) ? ld_raw(p.S0 + (int64_t)my_r * p.ld_s0 + voff)
                                                      : make_uint4(0u, 0u, 0u, 0u);
                const float ra = __ldg(p.rs + my_r), rb = __ldg(p.cs + my_r);
                int src[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) src[k] = (k < deg) ? __ldg(colp + trs + k) : 0;
                uint4 x8[8];
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    x8[k] = (k < deg) ? ld_raw(p.S_in + (int64_t)src[k] * p.ld_in + voff) : make_uint4(0u, 0u, 0u, 0u);
                float self[VALS], h[VALS], out[VALS];
#pragma unroll
                for (int i = 0; i < VALS; ++i) self[i] = h[i] = 0.f;
                V16<T>::add_raw(self, self_raw);
                V16<T>::add_raw(h, s0_raw);
                const float sig = (p.mode == 0) ? p.gamma * ra * rb : p.gamma * ra;
                const float beta = (p.mode == 0) ? p.alpha : p.alpha / rb;
#pragma unroll
                for (int i = 0; i < VALS; ++i) {
                    float g[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) g[k] = 0.f + V16<T>::elem(x8[k], i);   // acc_g = 0 + v_g
                    const float tot = ((g[0] + g[1]) + (g[2] + g[3])) + ((g[4] + g[5]) + (g[6] + g[7]));
                    out[i] = (p.alpha != 0.f) ? sig * (tot + self[i]) + beta * h[i] : sig * (tot + self[i]);
                }
                if (cok && e_raw < E) V16<T>::store(p.S_out + (int64_t)my_r * p.ld_out + voff, out);
                r += E - 1;
                continue;
            }
        }
        const int rs_e = p.rp[r], re_e = p.rp[r + 1];
        const int eb = max(rs_e, e0), ee = min(re_e, e1);
        const bool head = (r == r0) && (rs_e < e0);
        const bool tail = (r == r1);
        for (int pass = 0; pass < npass; ++pass) {
            const int vcol = pass * VP + c;
            const bool col_ok = active && vcol < p.nvec;
            const char* __restrict__ vbase = p.S_in + (int64_t)min(vcol, p.nvec - 1) * 16;
            // epilogue operands issued now so their latency hides behind the gather (short rows)
            const bool fin = !(head || tail) && e_raw == 0 && col_ok;
            uint4 self_raw = make_uint4(0u, 0u, 0u, 0u), s0_raw = make_uint4(0u, 0u, 0u, 0u);
            float ra = 0.f, rb = 0.f;
            if (fin) {
                self_raw = ld_raw(p.S_in + (int64_t)r * p.ld_in + (int64_t)vcol * 16);
                if (p.alpha != 0.f) s0_raw = ld_raw(p.S0 + (int64_t)r * p.ld_s0 + (int64_t)vcol * 16);
                ra = __ldg(p.rs + r);
                rb = __ldg(p.cs + r);
            }
            float acc[NACC][VALS];
#pragma unroll
            for (int k = 0; k < NACC; ++k)
#pragma unroll
                for (int i = 0; i < VALS; ++i) acc[k][i] = 0.f;
            // column indices of a batch: lane gl holds edges base + sl*L + gl (0 past the end)
            auto load_idx = [&](int base, int (&dst)[ISL]) {
#pragma unroll
                for (int sl = 0; sl < ISL; ++sl) {
                    const int j = base + sl * L + gl;
                    dst[sl] = (sl * L + gl < BATCH && j < ee) ? __ldg(colp + j) : fillv;
                }
            };
            // 16-byte loads of a batch; slots past the end read row 0 (never accumulated)
            auto load_data = [&](const int (&ix)[ISL], uint4 (&dst)[LPB]) {
#pragma unroll
                for (int t = 0; t < LPB; ++t) {
                    // edge t*E + e of the batch: held by lane (t*E % L) + e in slot (t*E)/L (E divides L)
                    const int src = __shfl_sync(gmask, ix[(t * E) / L], gbase + ((t * E) % L) + e);
                    dst[t] = ld_gather<POL>(vbase + (size_t)(uint32_t)src * ld_in);
                }
            };
            // edge base + t*E + e belongs to group (t*E + e) mod 8, i.e. acc[t % NACC]
            auto consume = [&](const uint4 (&v)[LPB], int base) {
                const int rem = ee - base;
                if (rem >= BATCH) {
#pragma unroll
                    for (int t = 0; t < LPB; ++t) V16<T>::add_raw(acc[t % NACC], v[t]);
                } else {
#pragma unroll
                    for (int t = 0; t < LPB; ++t)
                        if (t * E + e < rem) V16<T>::add_raw(acc[t % NACC], v[t]);
                }
            };
            if (!tma_group) {
            // two-deep software pipeline, unrolled by 2 so the buffers ping-pong without copies:
            // while batch b is accumulated, batch b+1's rows and batch b+2's indices are in flight
            int ia[ISL], ib[ISL];
            uint4 va[LPB], vb[LPB];
            load_idx(eb, ia);
            if (eb < ee) load_data(ia, va);
            load_idx(eb + BATCH, ib);
            for (int base = eb; base < ee;) {
                load_idx(base + 2 * BATCH, ia);
                if (base + BATCH < ee) load_data(ib, vb);
                consume(va, base);
                base += BATCH;
                if (base >= ee) break;
                load_idx(base + 2 * BATCH, ib);
                if (base + BATCH < ee) load_data(ia, va);
                consume(vb, base);
                base += BATCH;
            }
            } else {
            // TMA gather4 ring: batch b+1 in flight (buffer b+1 & 1) while batch b is read from smem
            auto issue = [&](int buf, const int (&ix)[ISL]) {
                if (gl == 0) ptx::mbar_expect_tx(&gbar[buf], BATCH * row_bytes);
                __syncwarp(gmask);
#pragma unroll
                for (int sl = 0; sl < ISL; ++sl) {
                    const int q1 = __shfl_sync(gmask, ix[sl], gbase + ((gl + 1) & (L - 1)));
                    const int q2 = __shfl_sync(gmask, ix[sl], gbase + ((gl + 2) & (L - 1)));
                    const int q3 = __shfl_sync(gmask, ix[sl], gbase + ((gl + 3) & (L - 1)));
                    const int jb = sl * L + gl;                       // first edge of this lane's gather
                    if ((gl & 3) == 0 && jb < BATCH)
                        ptx::tma_gather4(gbuf + buf * buf_bytes + (jb >> 2) * slot_bytes, &tmS, &gbar[buf], 0,
                                         ix[sl], q1, q2, q3);
                }
            };
            auto consume_smem = [&](int buf) {
                const uint8_t* b = gbuf + buf * buf_bytes + vcol * 16;
#pragma unroll
                for (int t = 0; t < LPB; ++t) {
                    const int jrel = t * E + e;
                    const uint4 x = *reinterpret_cast<const uint4*>(b + (jrel >> 2) * slot_bytes + (jrel & 3) * row_bytes);
                    V16<T>::add_raw(acc[t % NACC], x);                 // rows past the end are zero
                }
            };
            int ia[ISL], ib[ISL];
            load_idx(eb, ia);
            if (eb < ee) issue(0, ia);
            load_idx(eb + BATCH, ib);
            if (eb + BATCH < ee) issue(1, ib);
            for (int base = eb; base < ee;) {
                load_idx(base + 2 * BATCH, ia);
                ptx::mbar_wait(&gbar[0], ph0);
                ph0 ^= 1;
                consume_smem(0);
                __syncwarp(gmask);
                if (base + 2 * BATCH < ee) issue(0, ia);
                base += BATCH;
                if (base >= ee) break;
                load_idx(base + 2 * BATCH, ib);
                ptx::mbar_wait(&gbar[1], ph1);
                ph1 ^= 1;
                consume_smem(1);
                __syncwarp(gmask);
                if (base + 2 * BATCH < ee) issue(1, ib);
                base += BATCH;
            }
            }
            // fixed butterfly over the 8 reduction groups
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                if (b < LOG_E) {
                    const int partner = gbase + ((e ^ (1 << b)) * VP + c);
#pragma unroll
                    for (int k = 0; k < NACC; ++k)
#pragma unroll
                        for (int i = 0; i < VALS; ++i) acc[k][i] += __shfl_sync(gmask, acc[k][i], partner);
                } else {
                    const int kb = 1 << (b - LOG_E);
#pragma unroll
                    for (int k = 0; k < NACC; ++k)
                        if ((k & kb) == 0 && (k | kb) < NACC) {
#pragma unroll
                            for (int i = 0; i < VALS; ++i) acc[k][i] += acc[k | kb][i];
                        }
                }
            }
            if (e_raw != 0 || !col_ok) continue;
            if (head || tail) {
                float* dst = p.carry + ((u * 2 + (head ? 0 : 1)) * (int64_t)row_vals) + vcol * VALS;
#pragma unroll
                for (int i = 0; i < VALS; ++i) dst[i] = acc[0][i];
                continue;
            }
            const int64_t voff = (int64_t)vcol * 16;
            float self[VALS];
#pragma unroll
            for (int i = 0; i < VALS; ++i) self[i] = 0.f;
            V16<T>::add_raw(self, self_raw);
            const float a = ra;
            const float b = rb;
            const float sig = (p.mode == 0) ? p.gamma * a * b : p.gamma * a;
            float out[VALS];
            if (p.alpha != 0.f) {
                float h[VALS];
#pragma unroll
                for (int i = 0; i < VALS; ++i) h[i] = 0.f;
                V16<T>::add_raw(h, s0_raw);
                const float beta = (p.mode == 0) ? p.alpha : p.alpha / b;
#pragma unroll
                for (int i = 0; i < VALS; ++i) out[i] = sig * (acc[0][i] + self[i]) + beta * h[i];
            } else {
#pragma unroll
                for (int i = 0; i < VALS; ++i) out[i] = sig * (acc[0][i] + self[i]);
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

bool carveout_max_l1() {
    static const bool v = [] { const char* e = getenv("NTP_L1_CARVEOUT"); return e ? atoi(e) != 0 : true; }();
    return v;
}

template <typename T, int E, int L>
void launch_hop(const HopParams& p, cudaStream_t s) {
    static const int tma_env = [] { const char* v = getenv("NTP_SPMM_TMA"); return v ? atoi(v) : -1; }();
    static const int short_env = [] { const char* v = getenv("NTP_SPMM_SHORT"); return v ? atoi(v) : -1; }();
    // low-degree variants when the average degree is below 32 (products, papers shapes)
    const bool low_deg = short_env >= 0 ? short_env != 0 : (p.nnz < 32 * std::max<int64_t>(p.n, 1));
    // groups per 8 on the TMA path: measured sweet spots; NTP_SPMM_TMA overrides
    const int tma = tma_env >= 0 ? tma_env : 0;
    const int64_t groups = p.u_end - p.u_begin;
    const int64_t blocks = cdiv(groups * L, kBlock);
    CUtensorMap tm{};
    HopParams pp = p;
    pp.tma_per8 = std::min(tma, 8);
    const bool use_tma = tma > 0 && p.nvec <= 32 && (int64_t)p.nvec * 16 / (int64_t)sizeof(T) <= 256 && p.n > 0;
    if (use_tma) {
        constexpr int BATCH = (E == 8) ? 64 : (E == 4) ? 32 : 8 * E;
        const int row_bytes = p.nvec * 16;
        const int slot_bytes = (4 * row_bytes + 127) & ~127;
        const size_t smem = (size_t)(kBlock / L) * (2 * (BATCH / 4) * slot_bytes + 16) + 128;
        const cuuint64_t dims[2] = {(cuuint64_t)(row_bytes / sizeof(T)), (cuuint64_t)p.n};
        const cuuint64_t strides[1] = {(cuuint64_t)p.ld_in};
        const cuuint32_t box[2] = {(cuuint32_t)(row_bytes / sizeof(T)), 1};
        const cuuint32_t es[2] = {1, 1};
        CUresult r = tensor_map_encoder()(&tm, sizeof(T) == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                          2, const_cast<char*>(p.S_in), dims, strides, box, es,
                                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        NTP_CHECK(r == CUDA_SUCCESS, NTP_ERR_CUDA, "tensor map for the TMA gather failed (%d)", (int)r);
        static bool attr = false;
        if (!attr) {
            NTP_CUDA(cudaFuncSetAttribute(spmm_hop_kernel<T, E, L, 0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          200 * 1024));
            attr = true;
        }
        spmm_hop_kernel<T, E, L, 0, 1><<<(unsigned)blocks, kBlock, smem, s>>>(pp, tm);
    } else {
        // no shared memory on the LSU path: give the whole unified array to L1
        // low-degree mode: short batches where E >= 4, the tiny-row path where E >= 2
        constexpr int LOW = (E >= 4) ? 3 : (E >= 2) ? 2 : 0;
        static bool attr0 = false;
        if (!attr0 && carveout_max_l1()) {
            NTP_CUDA(cudaFuncSetAttribute(spmm_hop_kernel<T, E, L, 0, 0, 0>, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
            NTP_CUDA(cudaFuncSetAttribute(spmm_hop_kernel<T, E, L, 0, 0, LOW>, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
            attr0 = true;
        }
        if (low_deg) spmm_hop_kernel<T, E, L, 0, 0, LOW><<<(unsigned)blocks, kBlock, 0, s>>>(p, tm);
        else spmm_hop_kernel<T, E, L, 0, 0, 0><<<(unsigned)blocks, kBlock, 0, s>>>(p, tm);
    }
    NTP_LAUNCH_CHECK();
}

// (E, L) from the row width: E edge slots of nvec lanes each, E*nvec <= L.
template <typename T>
void dispatch_hop(const HopParams& p, int nvec, cudaStream_t s) {
    if (nvec == 1) launch_hop<T, 8, 8>(p, s);
    else if (nvec == 2) launch_hop<T, 8, 16>(p, s);
    else if (nvec <= 4) launch_hop<T, 8, 32>(p, s);
    else if (nvec <= 8) launch_hop<T, 4, 32>(p, s);
    else if (nvec <= 16) launch_hop<T, 2, 32>(p, s);
    else launch_hop<T, 1, 32>(p, s);
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
    p.nnz = g.nnz;

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
    if (dt == NTP_F32) dispatch_hop<float>(p, nvec, s);
    else dispatch_hop<__nv_bfloat16>(p, nvec, s);
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
        if (last && defer_last) {
            *defer_last = LastHop{&csr, rs, cs, sin, ld_sin, S0, ld_s0, bufs[nxt], lds[nxt], a.cols, a.dtype,
                                  a.gamma, a.alpha};
            return;
        }
        const bool timed = time_hops && c->hop_ev_used + 2 <= 256;
        if (timed) NTP_CUDA(record_timing(c, c->hop_ev[c->hop_ev_used], s));
        spmm_hop(c, csr, rs, cs, sin, bufs[nxt], S0, ld_sin, lds[nxt], ld_s0, a.cols, a.dtype, a.gamma, a.alpha,
                 last ? 1 : 0, 0, -1, s);
        if (timed) {
            NTP_CUDA(record_timing(c, c->hop_ev[c->hop_ev_used + 1], s));
            c->hop_ev_used += 2;
        }
        sin = bufs[nxt];
        ld_sin = lds[nxt];
    }
}

void run_last_hop(ntp_ctx* c, const LastHop& lh, int64_t row_lo, int64_t row_hi, cudaStream_t s, bool time_hops) {
    const bool timed = time_hops && c->hop_ev_used + 2 <= 256;
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
