// head.cu — fused classification head of the W1-after-propagation epoch (SURVEY §8(a) a5 unpack, a6,
// and the dW1 part of a10; reading R3: logits = (M·H1)·W1 = M·(H1·W1)).
//
// For this rank's vertex rows v (tiles of 128), with Z_v the gathered propagation output (bf16
// storage, blocked [P][V_p][d_s], P·d_s = 128 = the padded hidden width):
//   logits = Z_v · W1                          (tcgen05 kind::f16, W1 split into bf16 hi + lo)
//   loss   += log Σ_c exp(logits_c − m) + m − logits_y     (train rows; O7)
//   dl     = softmax(logits) − onehot(y)  (train rows, else 0; 1/N_train is folded into SGD, R12)
//   dW1   += Z_vᵀ · dl                      (accumulated in TMEM across the CTA's tiles)
//   dZ     = dl · W1ᵀ → out[q][v][j] = bf16(dZ[v][q·d_s + j] · gscale[row0 + v])   (the gradient
//            split's pack with the backward column-side pre-scale, a7)
// One pass over Z_v and one over the gradient slice; logits, dl and dZ never touch HBM.  The unfused
// path (unpack → GEMM → loss → 2 GEMMs → pack, model.cu) moved ~10× the compulsory bytes.
//
// Precision (bf16-storage runs, tolerance 2e-2, reading R10): Z is exactly bf16; W1 = hi + lo
// (2^-17 relative); dl is rounded to bf16 once (2^-9 relative, the same rounding the gradient slice
// gets when it is stored).  fp32 accumulation in TMEM.
//
// CTA: 16 warps, 1 CTA/SM, persistent over tiles (tile t → CTA t mod grid).
//   warp 0     : TMEM allocation (512 columns) + MMA issuer (one lane)
//   warps 1-3  : Z loader (16-byte global loads → 128B-swizzled K-major smem tile, double-buffered)
//   warps 4-11 : softmax epilogue, two warps per TMEM lane quarter (thread = tile row, each warp half
//                of the 32-column chunks; row max / sum combined through shared memory): loss, dl → smem
//   warps 12-15: dZ epilogue (tcgen05.ld dZ → scale, bf16 → gradient slice), final dW1 read-out
// MMA order per tile i: MMA1(i+1) is issued before MMA2(i)/MMA3(i), so the softmax of tile i+1 starts
// while the tensor core still works on tile i's gradients.
// TMEM columns: [0, 192) logits, [192, 320) dZ, [320, 512) dW1 (lanes = hidden index).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "ntp_internal.cuh"
#include "ptx.cuh"

namespace ntp {

namespace {

constexpr int kHeadThreads = 512;
constexpr int HP = 128;             // padded hidden width P·d_s (K of MMA1, N of MMA2, M of MMA3)
constexpr int kBox = 128 * 128;     // one 128-row × 128-byte swizzled box (64 bf16 columns)
constexpr uint32_t kColLogits = 0, kColDZ = 192, kColDW = 320;

struct HeadParams {
    const __nv_bfloat16* Z;     // gathered [P][V_p][d_s]
    int64_t V_p;
    int64_t v_lo, v_hi;         // this call's rows [v_lo, v_hi) of the V_p (row chunk of the a12 schedule)
    int d_s, P, lds;            // lds = log2(d_s) (d_s = 128 / P, P a power of two)
    int C, CB, n1, kc;          // classes, 64-class boxes, N of MMA1/3 (C rounded to 16), K steps of MMA2
    const __nv_bfloat16* W1s;   // [2][HP][CB*64] bf16: hi then lo, zero padded
    const int32_t* y;
    const uint8_t* mask;
    int64_t row0, n;
    const float* gscale;        // backward column side, original vertex order (len n)
    __nv_bfloat16* out;         // gradient slice [P][V_p][d_s] (or peer windows)
    void* const* peer;
    int rank;
    int hid;
    float* dW1part;             // [grid][hid][C]
    double* part;               // [grid]
    int64_t* cnt;               // [grid]
    int64_t tiles;
    uint32_t idesc1, idesc2, idesc3;
    const int32_t* out_perm;    // one GPU, reordered graph: gradient row of vertex v goes to slice row out_perm[v]
    int tma;                    // d_s >= 64: Z tiles by TMA (3-D map [P][V_p][d_s], 64-column boxes)
};

__device__ __forceinline__ uint32_t swz(int r, int col) {   // byte offset of (row, col) in a box set
    return (uint32_t)((col >> 6) * kBox + r * 128 + ((((col & 63) >> 3) ^ (r & 7)) << 4) + ((col & 7) << 1));
}

__device__ __forceinline__ uint64_t desc_k(uint32_t addr) {   // K-major SW128: 8-row atoms 1024 B apart
    return (uint64_t)((addr >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint64_t desc_mn(uint32_t addr) {  // MN-major SW128: 64-elem atoms a box apart
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)(kBox >> 4) << 16) | (64ull << 32) | (1ull << 46) |
           (2ull << 61);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     ptx::smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ float ex2(float x) {   // 2^x (MUFU.EX2; ex2(-inf) = 0)
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
}

__global__ void __launch_bounds__(kHeadThreads, 1) head_fused_kernel(const __grid_constant__ CUtensorMap tmZ,
                                                                     const HeadParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);   // stays a shared pointer
    uint8_t* sZ = smem;                              // [2][2 boxes]
    uint8_t* sDL = sZ + 4 * kBox;                    // [CB boxes]
    uint8_t* sW = sDL + p.CB * kBox;                 // [hi, lo][CB boxes]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sW + 2 * p.CB * kBox);
    uint64_t* zfull = bars;          // [2] loader → MMA
    uint64_t* zfree = bars + 2;      // [2] MMA (commit) → loader
    uint64_t* lfull = bars + 4;      // MMA1 done
    uint64_t* lfree = bars + 5;      // logits drained (128)
    uint64_t* dlfull = bars + 6;     // dl tile written (128)
    uint64_t* dlfree = bars + 7;     // MMA2/3 done reading dl (commit)
    uint64_t* dzfull = bars + 8;     // MMA2 done
    uint64_t* dzfree = bars + 9;     // dZ drained (128)
    uint64_t* dwfull = bars + 10;    // all MMA3 done
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 12);
    double* s_loss = reinterpret_cast<double*>(bars + 16);      // [128]
    int64_t* s_cnt = reinterpret_cast<int64_t*>(s_loss + 128);  // [128]
    float* s_stat = reinterpret_cast<float*>(s_cnt + 128);      // [tile parity][half][m, s, xy][128]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nloc = (int)((p.tiles - blockIdx.x + gridDim.x - 1) / gridDim.x);   // tiles of this CTA

    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&zfull[b], p.tma ? 1 : 96);
            ptx::mbar_init(&zfree[b], 1);
        }
        ptx::mbar_init(lfull, 1);
        ptx::mbar_init(lfree, 256);
        ptx::mbar_init(dlfull, 256);
        ptx::mbar_init(dlfree, 1);
        ptx::mbar_init(dzfull, 1);
        ptx::mbar_init(dzfree, 128);
        ptx::mbar_init(dwfull, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            ptx::smem_u32(tmem_holder)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // W1 hi/lo → swizzled smem [row = hidden index][col = class] (all threads)
    {
        const int cols = p.CB * 64;
        const int chunks = 2 * HP * cols / 8;
        for (int i = threadIdx.x; i < chunks; i += kHeadThreads) {
            const int e = i * 8;
            const int half = e / (HP * cols);
            const int rem = e - half * HP * cols;
            const int r = rem / cols, col = rem - r * cols;
            *reinterpret_cast<uint4*>(sW + half * p.CB * kBox + swz(r, col)) =
                *reinterpret_cast<const uint4*>(p.W1s + e);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_holder;

    if (warp == 0) {
        if (lane == 0 && nloc > 0) {
            // ------------------------------------------------ MMA issuer
            const uint32_t zb = ptx::smem_u32(sZ), dlb = ptx::smem_u32(sDL), wb = ptx::smem_u32(sW);
            // MMA1: logits[128 x n1] = Z[128 x 128] . W1[128 x n1]   (A K-major, B MN-major)
            auto mma1 = [&](int t) {
                const uint32_t za = zb + (t & 1) * 2 * kBox;
                ptx::mbar_wait(&zfull[t & 1], (t >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int k = 0; k < HP / 16; ++k)
                        mma_bf16(tmem + kColLogits, desc_k(za + (k >> 2) * kBox + (k & 3) * 32),
                                 desc_mn(wb + h * p.CB * kBox + k * 2048), p.idesc1, (h | k) ? 1u : 0u);
                commit(lfull);
            };
            mma1(0);
            for (int i = 0; i < nloc; ++i) {
                const uint32_t za = zb + (i & 1) * 2 * kBox;
                ptx::mbar_wait(lfree, i & 1);      // logits of tile i drained (softmax pass 2 done)
                ptx::mbar_wait(dlfull, i & 1);     // dl of tile i in shared memory
                if (i + 1 < nloc) mma1(i + 1);
                if (i > 0) ptx::mbar_wait(dzfree, (i - 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                // MMA2: dZ[128 x 128] = dl[128 x C] . W1^T   (A K-major dl, B K-major W1 rows)
                for (int h = 0; h < 2; ++h)
                    for (int k = 0; k < p.kc; ++k)
                        mma_bf16(tmem + kColDZ, desc_k(dlb + (k >> 2) * kBox + (k & 3) * 32),
                                 desc_k(wb + h * p.CB * kBox + (k >> 2) * kBox + (k & 3) * 32), p.idesc2,
                                 (h | k) ? 1u : 0u);
                commit(dzfull);
                // MMA3: dW1[128 x n1] += Z^T . dl   (A = Z MN-major, B = dl MN-major; K = tile rows)
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    mma_bf16(tmem + kColDW, desc_mn(za + k * 2048), desc_mn(dlb + k * 2048), p.idesc3,
                             (i > 0 || k > 0) ? 1u : 0u);
                commit(dlfree);
                commit(&zfree[i & 1]);
            }
            commit(dwfull);
        }
    } else if (warp < 4 && p.tma) {
        // ---------------------------------------------------- Z producer: TMA (one lane)
        if (warp == 1 && lane == 0) {
            for (int i = 0; i < nloc; ++i) {
                const int b = i & 1;
                if (i >= 2) ptx::mbar_wait(&zfree[b], ((i >> 1) - 1) & 1);
                const int v0 = (int)(p.v_lo + (blockIdx.x + (int64_t)i * gridDim.x) * 128);
                uint8_t* za = sZ + b * 2 * kBox;
                ptx::mbar_expect_tx(&zfull[b], 2 * kBox);
#pragma unroll
                for (int bx = 0; bx < 2; ++bx) {   // 64-column box bx = columns [64 bx, 64 bx + 64)
                    const int col = 64 * bx;
                    asm volatile(
                        "cp.async.bulk.tensor.3d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
                        "%5}], [%2];" ::"r"(ptx::smem_u32(za + bx * kBox)),
                        "l"(reinterpret_cast<uint64_t>(&tmZ)), "r"(ptx::smem_u32(&zfull[b])), "r"(col & (p.d_s - 1)),
                        "r"(v0), "r"(col >> p.lds)
                        : "memory");
                }
            }
        }
    } else if (warp < 4) {
        // ---------------------------------------------------- Z loader (d_s < 64: 16-byte loads)
        const int t = threadIdx.x - 32;
        const int lcpr = p.lds - 3;                // log2(16-byte chunks per row of a block)
        const int lpb = 7 + lcpr;                  // log2(chunks per 128-row block tile)
        for (int i = 0; i < nloc; ++i) {
            const int b = i & 1;
            if (i >= 2) ptx::mbar_wait(&zfree[b], ((i >> 1) - 1) & 1);
            const int64_t v0 = p.v_lo + (blockIdx.x + (int64_t)i * gridDim.x) * 128;
            uint8_t* za = sZ + b * 2 * kBox;
            constexpr int U = 22;                  // 2048 chunks / 96 threads: one round per tile
            for (int f0 = t; f0 < 2048; f0 += 96 * U) {
                uint4 x[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int f = f0 + u * 96;
                    x[u] = make_uint4(0, 0, 0, 0);
                    if (f < 2048) {
                        const int q = f >> lpb, rem = f & ((1 << lpb) - 1);
                        const int r = rem >> lcpr, jc = rem & ((1 << lcpr) - 1);
                        if (v0 + r < p.v_hi)
                            x[u] = __ldg(reinterpret_cast<const uint4*>(p.Z + ((int64_t)q * p.V_p + v0 + r) * p.d_s) + jc);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int f = f0 + u * 96;
                    if (f < 2048) {
                        const int q = f >> lpb, rem = f & ((1 << lpb) - 1);
                        const int r = rem >> lcpr, jc = rem & ((1 << lcpr) - 1);
                        *reinterpret_cast<uint4*>(za + swz(r, (q << p.lds) + jc * 8)) = x[u];
                    }
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            ptx::mbar_arrive(&zfull[b]);
        }
    } else if (warp < 12) {
        // ---------------------------------------------------- softmax epilogue (thread = row; two warps
        // per lane quarter, warp half hf takes the 32-column chunks cc with cc % 2 == hf)
        const int qd = warp & 3;
        const int hf = (warp - 4) >> 2;
        const int r = qd * 32 + lane;
        const uint32_t lrow = tmem + ((uint32_t)(qd * 32) << 16);
        constexpr float L2E = 1.4426950408889634f;
        double my_loss = 0.0;
        int64_t my_cnt = 0;
        const int nch = (p.C + 31) / 32;
        // mask and label of tile i+1 are loaded while tile i is processed (two independent loads, off
        // the per-tile critical path)
        auto row_of = [&](int t) { return p.v_lo + (blockIdx.x + (int64_t)t * gridDim.x) * 128 + r; };
        auto real_row = [&](int64_t v) { return v < p.v_hi && p.row0 + v < p.n; };
        uint8_t mk_n = 0;
        int y_n = 0;
        if (nloc > 0 && real_row(row_of(0))) {
            mk_n = __ldg(p.mask + row_of(0));
            y_n = __ldg(p.y + row_of(0));
        }
        for (int i = 0; i < nloc; ++i) {
            const int64_t v = row_of(i);
            const bool train = real_row(v) && mk_n != 0;
            const int yv = train ? y_n : -1;
            if (i + 1 < nloc && real_row(row_of(i + 1))) {
                mk_n = __ldg(p.mask + row_of(i + 1));
                y_n = __ldg(p.y + row_of(i + 1));
            }
            ptx::mbar_wait(lfull, i & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            // pass 1: online max / sum of exp over my chunks (masked columns are -inf: exp -> 0)
            float m = -INFINITY, sum = 0.f, xy = 0.f;
            for (int cc = hf; cc < nch; cc += 2) {
                uint32_t x[32];
                tmem_ld32(lrow + kColLogits + cc * 32, x);
                float f[32];
                float cm = -INFINITY;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const int col = cc * 32 + j;
                    f[j] = col < p.C ? __uint_as_float(x[j]) : -INFINITY;
                    cm = fmaxf(cm, f[j]);
                    xy = col == yv ? f[j] : xy;
                }
                const float mn = fmaxf(m, cm);
                const float mnl = mn * L2E;
                float add = 0.f;
#pragma unroll
                for (int j = 0; j < 32; ++j) add += ex2(fmaf(f[j], L2E, -mnl));
                sum = sum * ex2((m - mn) * L2E) + add;
                m = mn;
            }
            float* st = s_stat + (i & 1) * 768;
            st[hf * 384 + r] = m;
            st[hf * 384 + 128 + r] = sum;
            st[hf * 384 + 256 + r] = xy;
            asm volatile("bar.sync %0, 64;" ::"r"(1 + qd) : "memory");
            const float m0 = st[r], s0 = st[128 + r], m1 = st[384 + r], s1 = st[384 + 128 + r];
            const float mx = fmaxf(m0, m1);
            const float se = s0 * ex2((m0 - mx) * L2E) + s1 * ex2((m1 - mx) * L2E);   // same order in both halves
            if (hf == 0 && train) {
                const float ly = st[(((yv >> 5) & 1) ? 384 : 0) + 256 + r];
                my_loss += (double)(logf(se) + mx - ly);
                my_cnt += 1;
            }
            const float inv = 1.f / se;
            const float mxl = mx * L2E;
            if (i > 0) ptx::mbar_wait(dlfree, (i - 1) & 1);
            for (int cc = hf; cc < 2 * p.CB; cc += 2) {
                uint32_t x[32];
                if (cc < nch) tmem_ld32(lrow + kColLogits + cc * 32, x);
                uint32_t w[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    float g[2];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int col = cc * 32 + 2 * j + e;
                        const float pr = ex2(fmaf(__uint_as_float(x[2 * j + e]), L2E, -mxl)) * inv;
                        g[e] = (train && col < p.C) ? pr - (col == yv ? 1.f : 0.f) : 0.f;
                    }
                    w[j] = pack_bf16(g[0], g[1]);
                }
#pragma unroll
                for (int c4 = 0; c4 < 4; ++c4)
                    *reinterpret_cast<uint4*>(sDL + swz(r, cc * 32 + c4 * 8)) =
                        make_uint4(w[4 * c4], w[4 * c4 + 1], w[4 * c4 + 2], w[4 * c4 + 3]);
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            ptx::mbar_arrive(lfree);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            ptx::mbar_arrive(dlfull);
        }
        if (hf == 0) {
            s_loss[r] = my_loss;
            s_cnt[r] = my_cnt;
        }
    } else {
        // ---------------------------------------------------- dZ epilogue (thread = row, warps 12-15)
        const int qd = warp & 3;
        const int r = qd * 32 + lane;
        const uint32_t lrow = tmem + ((uint32_t)(qd * 32) << 16);
        auto scale_of = [&](int t) {
            const int64_t v = p.v_lo + (blockIdx.x + (int64_t)t * gridDim.x) * 128 + r;
            return (v < p.v_hi && p.row0 + v < p.n) ? __ldg(p.gscale + p.row0 + v) : 0.f;
        };
        float sc_n = nloc > 0 ? scale_of(0) : 0.f;
        for (int i = 0; i < nloc; ++i) {
            const int64_t v = p.v_lo + (blockIdx.x + (int64_t)i * gridDim.x) * 128 + r;
            const bool inb = v < p.v_hi;
            const float sc = sc_n;
            if (i + 1 < nloc) sc_n = scale_of(i + 1);
            ptx::mbar_wait(dzfull, i & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            for (int cc = 0; cc < HP / 32; ++cc) {
                uint32_t x[32];
                tmem_ld32(lrow + kColDZ + cc * 32, x);
                if (!inb) continue;
#pragma unroll
                for (int c8 = 0; c8 < 4; ++c8) {
                    const int col = cc * 32 + c8 * 8;
                    const int q = col >> p.lds, j = col & (p.d_s - 1);
                    uint4 o;
                    o.x = pack_bf16(__uint_as_float(x[c8 * 8 + 0]) * sc, __uint_as_float(x[c8 * 8 + 1]) * sc);
                    o.y = pack_bf16(__uint_as_float(x[c8 * 8 + 2]) * sc, __uint_as_float(x[c8 * 8 + 3]) * sc);
                    o.z = pack_bf16(__uint_as_float(x[c8 * 8 + 4]) * sc, __uint_as_float(x[c8 * 8 + 5]) * sc);
                    o.w = pack_bf16(__uint_as_float(x[c8 * 8 + 6]) * sc, __uint_as_float(x[c8 * 8 + 7]) * sc);
                    const int64_t ov = (p.out_perm && v < p.n) ? (int64_t)__ldg(p.out_perm + v) : v;   // padding rows stay
                    __nv_bfloat16* dst = p.peer ? static_cast<__nv_bfloat16*>(p.peer[q]) +
                                                      ((int64_t)p.rank * p.V_p + v) * p.d_s + j
                                                : p.out + ((int64_t)q * p.V_p + ov) * p.d_s + j;
                    *reinterpret_cast<uint4*>(dst) = o;
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            ptx::mbar_arrive(dzfree);
        }
        // dW1 partial of this CTA: TMEM lane = hidden index, column = class
        if (nloc > 0) {
            ptx::mbar_wait(dwfull, 0);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        float* dst = p.dW1part + (int64_t)blockIdx.x * p.hid * p.C + (int64_t)r * p.C;
        for (int cc = 0; cc < (p.n1 + 31) / 32; ++cc) {
            uint32_t x[32];
            if (nloc > 0) tmem_ld32(lrow + kColDW + cc * 32, x);
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int col = cc * 32 + j;
                if (r < p.hid && col < p.C) dst[col] = nloc > 0 ? __uint_as_float(x[j]) : 0.f;
            }
        }
#ifndef NTP_NO_P2P_FENCE
        if (p.peer) __threadfence_system();
#endif
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {   // fixed-order loss partial of this CTA
        double l = 0.0;
        int64_t k = 0;
        for (int i = 0; i < 128; ++i) {
            l += s_loss[i];
            k += s_cnt[i];
        }
        p.part[blockIdx.x] = l;
        p.cnt[blockIdx.x] = k;
    }
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

// W1 fp32 [hid x C] (ld) -> [2][HP][cols] bf16 (hi = rn(w), lo = rn(w - hi)), zero padded.
__global__ void head_w1_split_kernel(const float* __restrict__ W1, int64_t ld, int hid, int C, int cols,
                                     __nv_bfloat16* __restrict__ out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < HP * cols; i += gridDim.x * blockDim.x) {
        const int r = i / cols, c = i - r * cols;
        const float w = (r < hid && c < C) ? W1[(int64_t)r * ld + c] : 0.f;
        const __nv_bfloat16 hi = __float2bfloat16_rn(w);
        out[i] = hi;
        out[HP * cols + i] = __float2bfloat16_rn(w - __bfloat162float(hi));
    }
}

// dW1[h][c] = sum_b part[b][h][c] in CTA order (deterministic).
__global__ void head_dw1_reduce_kernel(const float* __restrict__ part, int nb, int64_t total, float* __restrict__ dW1) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        float a = 0.f;
        for (int b = 0; b < nb; ++b) a += part[b * total + i];
        dW1[i] = a;
    }
}

constexpr uint32_t idesc_bf16(int N, bool a_mn, bool b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

}  // namespace

bool head_fused_supported(int32_t P, int32_t d_s, int32_t hid, int32_t C, ntp_dtype dt) {
    const char* v = getenv("NTP_HEAD_FUSED");   // read per call (part of the epoch graph key)
    return !(v && atoi(v) == 0) && dt == NTP_BF16 && (int64_t)P * d_s == HP && hid <= HP && d_s >= 8 &&
           (d_s & (d_s - 1)) == 0 && C >= 1 && C <= 192;
}

int64_t head_fused(ntp_ctx* c, const void* gathered, int64_t V_p, int32_t d_s, int32_t P, int32_t hid, int32_t C,
                   const float* W1, int64_t ldw1, const int32_t* y, const uint8_t* mask, int64_t row0, int64_t n,
                   const float* gscale, void* out, void* const* peer, float* dW1, double* part, int64_t* cnt,
                   cudaStream_t s, int64_t v_lo, int64_t v_hi, const int32_t* out_perm) {
    if (v_hi < 0) v_hi = V_p;
    HeadParams p{};
    p.Z = static_cast<const __nv_bfloat16*>(gathered);
    p.V_p = V_p;
    p.v_lo = v_lo;
    p.v_hi = v_hi;
    p.out_perm = out_perm;
    p.d_s = d_s;
    p.P = P;
    p.lds = 0;
    while ((1 << p.lds) < d_s) ++p.lds;
    p.C = C;
    p.CB = (C + 63) / 64;
    p.n1 = (C + 15) / 16 * 16;
    p.kc = (C + 15) / 16;
    p.y = y;
    p.mask = mask;
    p.row0 = row0;
    p.n = n;
    p.gscale = gscale;
    p.out = static_cast<__nv_bfloat16*>(out);
    p.peer = peer;
    p.rank = c->rank;
    p.hid = hid;
    p.tiles = cdiv(v_hi - v_lo, 128);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(p.tiles, 148));
    const int cols = p.CB * 64;
    const size_t w_bytes = (size_t)2 * HP * cols * sizeof(__nv_bfloat16);
    const size_t dw_bytes = (size_t)grid * hid * C * sizeof(float);
    c->m_head.ensure(w_bytes + dw_bytes + 256);
    __nv_bfloat16* w1s = c->m_head.as<__nv_bfloat16>();
    float* dwp = reinterpret_cast<float*>(reinterpret_cast<char*>(c->m_head.p) + ((w_bytes + 255) / 256) * 256);
    p.W1s = w1s;
    p.dW1part = dwp;
    p.part = part;
    p.cnt = cnt;
    p.idesc1 = idesc_bf16(p.n1, false, true);
    p.idesc2 = idesc_bf16(HP, false, false);
    p.idesc3 = idesc_bf16(p.n1, true, true);
    const char* te = getenv("NTP_HEAD_TMA");   // 0: force the 16-byte-load Z loader (tests cover both paths)
    p.tma = (d_s >= 64 && !(te && atoi(te) == 0)) ? 1 : 0;
    CUtensorMap tmZ;
    std::memset(&tmZ, 0, sizeof(tmZ));
    if (p.tma) {
        const cuuint64_t dims[3] = {(cuuint64_t)d_s, (cuuint64_t)V_p, (cuuint64_t)P};
        const cuuint64_t strides[2] = {(cuuint64_t)d_s * 2, (cuuint64_t)V_p * d_s * 2};
        const cuuint32_t box[3] = {64, 128, 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        NTP_CHECK(((uintptr_t)gathered % 16) == 0, NTP_ERR_SHAPE, "fused head: gathered slice not 16-byte aligned");
        CUresult r = tensor_map_encoder()(&tmZ, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(gathered), dims,
                                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        NTP_CHECK(r == CUDA_SUCCESS, NTP_ERR_CUDA, "cuTensorMapEncodeTiled (head Z) failed (%d)", (int)r);
    }
    head_w1_split_kernel<<<(HP * cols + 255) / 256, 256, 0, s>>>(W1, ldw1, hid, C, cols, w1s);
    NTP_LAUNCH_CHECK();
    const size_t smem = 1024 + (size_t)(4 + 3 * p.CB) * kBox + 16 * 8 + 256 * 8 + 2 * 768 * 4 + 64;
    static bool attr = false;
    if (!attr) {
        NTP_CUDA(cudaFuncSetAttribute(head_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr = true;
    }
    NTP_CHECK(smem <= 227 * 1024, NTP_ERR_CONFIG, "fused head needs %zu B of shared memory", smem);
    head_fused_kernel<<<grid, kHeadThreads, smem, s>>>(tmZ, p);
    NTP_LAUNCH_CHECK();
    const int64_t total = (int64_t)hid * C;
    head_dw1_reduce_kernel<<<(unsigned)std::min<int64_t>(cdiv(total, 256), 148 * 4), 256, 0, s>>>(dwp, grid, total, dW1);
    NTP_LAUNCH_CHECK();
    count_launch(c, 3);
    return grid;
}

}  // namespace ntp
