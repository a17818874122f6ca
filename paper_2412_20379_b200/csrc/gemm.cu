// gemm.cu — tensor-core MLP GEMMs ("Tensor cores are used only for the
// small dense MLP GEMMs", BASELINE north_star) on 5th-generation tensor cores (tcgen05).
//
// C[M x N] = op(A)[M x K] . op(B)[K x N] in fp32 with fp32-level accuracy (reading R11):
// 3xTF32 split.  Every fp32 operand x is split into hi = rn_tf32(x) and lo = x - hi (exact in
// fp32); the product is accumulated in fp32 TMEM as hi_a*hi_b + hi_a*lo_b + lo_a*hi_b (the
// dropped lo*lo term is ~2^-22 relative), i.e. three kind::tf32 MMAs per K step.
//
// Structure (one 128 x BN output tile per CTA, optional split-K over grid.z):
//   warp 0   : TMEM allocation + TMA producer (one elected lane; 128-byte swizzled tiles)
//   warp 1   : MMA issuer (one lane: tcgen05.mma.cta_group::1.kind::tf32, tcgen05.commit)
//   warps 2-5: split workers (rn_tf32 in place + lo tile, fence.proxy.async) during the main
//              loop, then the epilogue (tcgen05.ld 32x32b -> registers -> global)
// Operands may be K-major (K contiguous) or MN-major (M/N contiguous); both are loaded by TMA
// with SWIZZLE_128B and described to the tensor core with the matching smem descriptor.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "ntp_internal.cuh"
#include "ptx.cuh"

namespace ntp {

namespace {

constexpr int BM = 128;
constexpr int BK = 32;                 // fp32 elements per 128-byte swizzle row
constexpr int kGemmThreads = 320;
constexpr int kTileA = BM * BK * 4;    // 16 KB
constexpr int kEpiStage = 4 * 32 * 32 * 4;   // epilogue transpose buffers: 4 warps x 32 x 32 fp32

struct GemmParams {
    int M, N, K;
    int k_tiles_total, k_tiles_per_split;
    int BN, bn_alloc, stages;
    uint32_t idesc;
    uint32_t tmem_cols;
    float* C;
    int64_t ldc;
    int64_t split_stride;               // elements between split-K partial outputs
    const float* aux;
    int64_t ldaux;
    int epi;                            // 0 store, 1 relu, 2 keep where aux > 0
    int vec;                            // C (and aux) rows 16-byte aligned: float4 epilogue
    int b_presplit;                     // B arrives as (hi, lo) pair: tmB = hi, tmBlo = lo (weights)
    uint32_t mn_lbo, mn_sbo;            // MN-major descriptor byte offsets (16-byte units)
    PackEpi pk;                         // epi 3: ReLU -> ReLU' bits + row-scaled bf16 feature-slice blocks
};

using ptx::smem_u32;
using ptx::mbar_init;
using ptx::mbar_wait;
using ptx::mbar_arrive;
using ptx::mbar_expect_tx;
using ptx::tma_load_2d;

// 128B-swizzled UMMA smem descriptors (sm_100 format: version 1, layout type 2 = SWIZZLE_128B).
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t addr) {
    // rows of 128 B, 8-row atoms 1024 B apart (SBO); LBO unused for swizzled K-major
    return (uint64_t)((addr >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    // MN-major tf32 needs layout type 1 = SWIZZLE_128B_BASE32B (32-byte swizzle atoms, 4 K-rows
    // of 128 B per atom): 32-element MN atoms `lbo` apart, 4-row K groups `sbo` apart (16-B units)
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)lbo << 16) | ((uint64_t)sbo << 32) | (1ull << 46) |
           (1ull << 61);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ float tf32_rn(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// Split of a staged fp32 tile.  The tensor core reads a kind::tf32 operand's 32-bit container and
// ignores the low 13 mantissa bits, so the raw tile IS the hi part, hi = trunc_tf32(x), and only
// lo = rn_tf32(x - trunc_tf32(x)) is written (x - trunc is exact in fp32): one smem write stream
// instead of two.  |x - hi| < 2^-10 |x|, so the dropped lo*lo term and the rounding of lo are
// ~2^-20 relative (reading R11).
__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
__device__ __forceinline__ void split_tile(const uint8_t* t, uint8_t* lo, int bytes, int tid, int nthreads) {
    for (int off = tid * 16; off < bytes; off += nthreads * 16) {
        const float4 x = *reinterpret_cast<const float4*>(t + off);
        const float4 l = make_float4(tf32_rn(x.x - tf32_trunc(x.x)), tf32_rn(x.y - tf32_trunc(x.y)),
                                     tf32_rn(x.z - tf32_trunc(x.z)), tf32_rn(x.w - tf32_trunc(x.w)));
        *reinterpret_cast<float4*>(lo + off) = l;
    }
}

// Persistent: grid = min(#tiles, #SMs); CTA b walks tiles b, b + grid, ... (tile = (m, n, split),
// m fastest so concurrent CTAs share the B operand in L2).  Pipeline stages and phases run on across
// tiles; the accumulator is double-buffered in TMEM (2 x BN columns) so the epilogue of tile i
// overlaps the MMAs of tile i+1.
//   warp 0   : TMEM alloc + TMA producer        warp 1   : MMA issuer
//   warps 2-5: split workers                    warps 6-9: epilogue (TMEM lane quarter = warp % 4)
template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const __grid_constant__ CUtensorMap tmBlo, const GemmParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = p.stages;
    const int tileB = p.bn_alloc * BK * 4;
    const int stage_bytes = 2 * kTileA + 2 * tileB;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
    uint64_t* full = bars;
    uint64_t* split = bars + S;
    uint64_t* empty = bars + 2 * S;
    uint64_t* tfull = bars + 3 * S;          // [2] accumulator ready
    uint64_t* tempty = bars + 3 * S + 2;     // [2] accumulator drained
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 3 * S + 4);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int m_tiles = (p.M + BM - 1) / BM;
    const int n_tiles = (p.N + p.BN - 1) / p.BN;
    const int splits = (p.k_tiles_total + p.k_tiles_per_split - 1) / p.k_tiles_per_split;
    const int num_tiles = m_tiles * n_tiles * splits;

    if (threadIdx.x == 0) {
        for (int st = 0; st < S; ++st) {
            mbar_init(&full[st], 1);
            mbar_init(&split[st], 128);
            mbar_init(&empty[st], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                     "r"(p.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_holder;

    auto decode = [&](int t, int& m0, int& n0, int& kt0, int& nk, int& z) {
        const int mt = t % m_tiles;
        const int rest = t / m_tiles;
        const int nt = rest % n_tiles;
        z = rest / n_tiles;
        m0 = mt * BM;
        n0 = nt * p.BN;
        kt0 = z * p.k_tiles_per_split;
        nk = min(p.k_tiles_per_split, p.k_tiles_total - kt0);
    };

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer
            int it = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
                int m0, n0, kt0, nk, z;
                decode(t, m0, n0, kt0, nk, z);
                for (int i = 0; i < nk; ++i, ++it) {
                    const int s = it % S;
                    if (it >= S) mbar_wait(&empty[s], ((it / S) - 1) & 1);
                    uint8_t* sa = smem + s * stage_bytes;
                    uint8_t* sb = sa + 2 * kTileA;
                    const int k0 = (kt0 + i) * BK;
                    mbar_expect_tx(&full[s], kTileA + (p.b_presplit ? 2 : 1) * tileB);
                    if (A_MN) {
                        for (int j = 0; j < BM / 32; ++j) tma_load_2d(sa + j * 4096, &tmA, &full[s], m0 + 32 * j, k0);
                    } else {
                        tma_load_2d(sa, &tmA, &full[s], k0, m0);
                    }
                    if (B_MN) {
                        for (int j = 0; j < p.bn_alloc / 32; ++j)
                            tma_load_2d(sb + j * 4096, &tmB, &full[s], n0 + 32 * j, k0);
                        if (p.b_presplit)
                            for (int j = 0; j < p.bn_alloc / 32; ++j)
                                tma_load_2d(sb + tileB + j * 4096, &tmBlo, &full[s], n0 + 32 * j, k0);
                    } else {
                        tma_load_2d(sb, &tmB, &full[s], k0, n0);
                        if (p.b_presplit) tma_load_2d(sb + tileB, &tmBlo, &full[s], k0, n0);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer
            int it = 0, tc = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++tc) {
                int m0, n0, kt0, nk, z;
                decode(t, m0, n0, kt0, nk, z);
                const int a = tc & 1;
                if (tc >= 2) mbar_wait(&tempty[a], ((tc >> 1) - 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t acc = tmem + (uint32_t)(a * p.BN);
                for (int i = 0; i < nk; ++i, ++it) {
                    const int s = it % S;
                    mbar_wait(&split[s], (it / S) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t sa = smem_u32(smem + s * stage_bytes);
                    const uint32_t salo = sa + kTileA;
                    const uint32_t sb = sa + 2 * kTileA;
                    const uint32_t sblo = sb + tileB;
#pragma unroll
                    for (int k = 0; k < BK / 8; ++k) {
                        const uint32_t ao = A_MN ? k * 1024 : k * 32;   // K step of 8 tf32
                        const uint32_t bo = B_MN ? k * 1024 : k * 32;
                        const uint64_t dA = A_MN ? desc_mnmajor(sa + ao, p.mn_lbo, p.mn_sbo) : desc_kmajor(sa + ao);
                        const uint64_t dAlo = A_MN ? desc_mnmajor(salo + ao, p.mn_lbo, p.mn_sbo) : desc_kmajor(salo + ao);
                        const uint64_t dB = B_MN ? desc_mnmajor(sb + bo, p.mn_lbo, p.mn_sbo) : desc_kmajor(sb + bo);
                        const uint64_t dBlo = B_MN ? desc_mnmajor(sblo + bo, p.mn_lbo, p.mn_sbo) : desc_kmajor(sblo + bo);
                        mma_tf32(acc, dA, dB, p.idesc, (i > 0 || k > 0) ? 1u : 0u);
                        mma_tf32(acc, dA, dBlo, p.idesc, 1u);
                        mma_tf32(acc, dAlo, dB, p.idesc, 1u);
                    }
                    mma_commit(&empty[s]);
                }
                mma_commit(&tfull[a]);
            }
        }
    } else if (warp < 6) {
        // ---------------- split workers
        const int tid = threadIdx.x - 64;
        int it = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            int m0, n0, kt0, nk, z;
            decode(t, m0, n0, kt0, nk, z);
            for (int i = 0; i < nk; ++i, ++it) {
                const int s = it % S;
                mbar_wait(&full[s], (it / S) & 1);
                uint8_t* sa = smem + s * stage_bytes;
                split_tile(sa, sa + kTileA, kTileA, tid, 128);
                uint8_t* sb = sa + 2 * kTileA;
                if (!p.b_presplit) split_tile(sb, sb + tileB, tileB, tid, 128);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(&split[s]);
            }
        }
    } else {
        // ---------------- epilogue: TMEM -> registers (thread = tile row) -> XOR-swizzled smem
        // transpose -> coalesced rows (a warp stores 4 rows x 128 B per instruction; the aux
        // mask is read the same way)
        const int q = warp & 3;                       // TMEM lane quarter of this warp
        float* stg = reinterpret_cast<float*>(smem + S * stage_bytes + 1024) + (warp - 6) * 1024;
        int tc = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++tc) {
            int m0, n0, kt0, nk, z;
            decode(t, m0, n0, kt0, nk, z);
            const int a = tc & 1;
            mbar_wait(&tfull[a], (tc >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            float* Cb = p.C + (int64_t)z * p.split_stride;
            for (int c0 = 0; c0 < p.BN; c0 += 32) {
                // epi 2: this lane's 8 mask quads of the chunk are loaded first, all in flight together,
                // before the TMEM read (one dependent load per quad had left the epilogue latency-bound:
                // the K = 41 dH1 GEMM of the Reddit shape took 516 us for ~0.5 GB of traffic)
                float4 mq[8];
                if (p.epi == 2 && p.vec) {
                    const int colq = n0 + c0 + 4 * (lane & 7);
#pragma unroll
                    for (int it = 0; it < 8; ++it) {
                        const int row = m0 + 32 * q + it * 4 + (lane >> 3);
                        mq[it] = (row < p.M && colq + 3 < p.N)
                                     ? __ldg(reinterpret_cast<const float4*>(p.aux + (int64_t)row * p.ldaux + colq))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                }
                uint32_t r[32];
                const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(a * p.BN + c0);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                      "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                      "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                      "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                      "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (n0 + c0 >= p.N) continue;         // warp-uniform
                if (p.epi == 3) {
                    // the split's pack fused in (a2 -> a3, W1 after propagation): thread = row, its 32 columns
                    // ReLU'd, their positivity as one mask word, scaled by the row's D~_out^{-1/2} (0 on padding
                    // rows) and stored as bf16 into block q = col / d_s of the blocked slice [P][V_p][d_s]
                    const int64_t row = m0 + 32 * q + lane;
                    if (row < p.M) {
                        const int64_t v = p.pk.roff + row;
                        const bool real = p.pk.row0 + v < p.pk.n;
                        const float sc = real ? __ldg(p.pk.scale + p.pk.row0 + v) : 0.f;
                        uint32_t word = 0;
                        float e[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            e[j] = real ? fmaxf(__uint_as_float(r[j]), 0.f) : 0.f;
                            word |= (e[j] > 0.f ? 1u : 0u) << j;
                        }
                        const int col0 = n0 + c0;
                        p.pk.bits[v * p.pk.nwb + (col0 >> 5)] = word;
                        // the row's destination, once per chunk (not per 16-byte piece: each lookup is a
                        // dependent global load ahead of the store)
                        const int64_t orow = (p.pk.perm && v < p.pk.n) ? (int64_t)__ldg(p.pk.perm + v) : v;   // padding rows stay
#pragma unroll
                        for (int g8 = 0; g8 < 4; ++g8) {
                            const int col = col0 + 8 * g8;
                            const int qb = col / p.pk.d_s, jj = col - qb * p.pk.d_s;
                            uint4 o;
                            uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const __nv_bfloat162 h2 =
                                    __floats2bfloat162_rn(e[8 * g8 + 2 * k] * sc, e[8 * g8 + 2 * k + 1] * sc);
                                ow[k] = *reinterpret_cast<const uint32_t*>(&h2);
                            }
                            *reinterpret_cast<uint4*>(p.pk.out + ((int64_t)qb * p.pk.V_p + orow) * p.pk.d_s + jj) = o;
                        }
                    }
                    continue;
                }
                // row `lane` of the 32 x 32 chunk: 16-byte piece j lands in slot j ^ (lane & 7)
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    *reinterpret_cast<float4*>(stg + lane * 32 + ((j ^ (lane & 7)) << 2)) =
                        make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                    __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
                __syncwarp();
                const int cj = lane & 7;
                const int col = n0 + c0 + 4 * cj;
#pragma unroll
                for (int it = 0; it < 8; ++it) {
                    const int rr = it * 4 + (lane >> 3);
                    const int row = m0 + 32 * q + rr;
                    float4 v = *reinterpret_cast<const float4*>(stg + rr * 32 + ((cj ^ (rr & 7)) << 2));
                    if (row >= p.M || col >= p.N) continue;
                    float e[4] = {v.x, v.y, v.z, v.w};
                    if (p.epi == 1) {
#pragma unroll
                        for (int i = 0; i < 4; ++i) e[i] = fmaxf(e[i], 0.f);
                    }
                    const float* ax = p.aux + (int64_t)row * p.ldaux + col;
                    float* dst = Cb + (int64_t)row * p.ldc + col;
                    if (p.vec && col + 3 < p.N) {
                        if (p.epi == 2) {
                            const float4 m = mq[it];
                            if (!(m.x > 0.f)) e[0] = 0.f;
                            if (!(m.y > 0.f)) e[1] = 0.f;
                            if (!(m.z > 0.f)) e[2] = 0.f;
                            if (!(m.w > 0.f)) e[3] = 0.f;
                        }
                        *reinterpret_cast<float4*>(dst) = make_float4(e[0], e[1], e[2], e[3]);
                    } else {
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            if (col + i < p.N) dst[i] = (p.epi == 2 && !(ax[i] > 0.f)) ? 0.f : e[i];
                    }
                }
                __syncwarp();
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            mbar_arrive(&tempty[a]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols));
    }
}

// out[m][n] = sum_z part[z][m][n] in split order (deterministic), then the epilogue.
__global__ void splitk_reduce_kernel(const float* __restrict__ part, int splits, int64_t split_stride, int M, int N,
                                     int64_t ldp, float* __restrict__ C, int64_t ldc, int epi,
                                     const float* __restrict__ aux, int64_t ldaux) {
    const int64_t total = (int64_t)M * N;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = i / N, n = i % N;
        float acc = 0.f;
        for (int z = 0; z < splits; ++z) acc += part[z * split_stride + m * ldp + n];
        if (epi == 1) acc = fmaxf(acc, 0.f);
        else if (epi == 2) acc = aux[m * ldaux + n] > 0.f ? acc : 0.f;
        C[m * ldc + n] = acc;
    }
}

}  // namespace

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    NTP_CHECK(fn != nullptr, NTP_ERR_CUDA, "cuTensorMapEncodeTiled not available");
    return fn;
}

namespace {

// 2-D fp32 tensor map over a row-major matrix with `rows` rows of `cols` elements (stride ld).
CUtensorMap make_map(const float* base, int64_t cols, int64_t rows, int64_t ld, int box_cols, int box_rows,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    NTP_CHECK(((uintptr_t)base % 16) == 0 && (ld * 4) % 16 == 0, NTP_ERR_SHAPE,
              "GEMM operand must be 16-byte aligned with ld %% 4 == 0 (ld=%lld)", (long long)ld);
    CUresult r = tensor_map_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    NTP_CHECK(r == CUDA_SUCCESS, NTP_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return m;
}

template <bool A_MN, bool B_MN>
void launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tblo, const GemmParams& p, dim3 grid,
                 size_t smem, cudaStream_t s) {
    static bool configured = false;
    if (!configured) {
        NTP_CUDA(cudaFuncSetAttribute(gemm_tf32x3_kernel<A_MN, B_MN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      227 * 1024));
        configured = true;
    }
    gemm_tf32x3_kernel<A_MN, B_MN><<<grid, kGemmThreads, smem, s>>>(ta, tb, tblo, p);
    NTP_LAUNCH_CHECK();
}

}  // namespace

// C[M x N] = op(A) op(B).  A: a_mn ? stored [K][M] (ld lda) : stored [M][K];
// B: b_mn ? stored [K][N] : stored [N][K].  epi: 0 store, 1 ReLU, 2 keep where aux > 0.
void gemm_tf32x3(ntp_ctx* c, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, bool a_mn, const float* B,
                 int64_t ldb, bool b_mn, float* C, int64_t ldc, int epi, const float* aux, int64_t ldaux,
                 cudaStream_t s, const float* B_lo) {
    if (M <= 0 || N <= 0) return;
    NTP_CHECK(K > 0, NTP_ERR_ARG, "GEMM with K == 0");
    GemmParams p{};
    p.M = (int)M;
    p.N = (int)N;
    p.K = (int)K;
    p.BN = (int)std::min<int64_t>(256, ((N + 15) / 16) * 16);
    p.bn_alloc = ((p.BN + 31) / 32) * 32;
    const int stage_bytes = 2 * kTileA + 2 * p.bn_alloc * BK * 4;
    p.stages = std::max(2, std::min(4, (225 * 1024 - 2048 - kEpiStage) / stage_bytes));
    p.tmem_cols = 32;
    while ((int)p.tmem_cols < 2 * p.BN) p.tmem_cols <<= 1;   // double-buffered accumulator
    p.idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
              ((uint32_t)(p.BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
    p.k_tiles_total = (int)cdiv(K, BK);
    const int m_tiles = (int)cdiv(M, BM);
    const int n_tiles = (int)cdiv(N, p.BN);
    int splits = 1;
    if ((int64_t)m_tiles * n_tiles < 148) {
        // split-K to (at most) one full wave: floor, so no CTA runs a second round of long tiles
        splits = (int)std::min<int64_t>(148 / ((int64_t)m_tiles * n_tiles), std::max(1, p.k_tiles_total / 4));
        splits = std::max(splits, 1);
    }
    if (epi == 3) splits = 1;              // the pack epilogue writes final values (no split-K partials)
    p.k_tiles_per_split = (int)cdiv(p.k_tiles_total, splits);
    splits = (int)cdiv(p.k_tiles_total, p.k_tiles_per_split);
    p.aux = aux;
    p.ldaux = ldaux;
    if (epi == 3) p.pk = c->pack_epi;
    p.mn_lbo = 4096 >> 4;
    p.mn_sbo = 512 >> 4;
    const CUtensorMapSwizzle mnswz = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
    CUtensorMap ta = a_mn ? make_map(A, M, K, lda, 32, 32, mnswz) : make_map(A, K, M, lda, 32, BM);
    CUtensorMap tb = b_mn ? make_map(B, N, K, ldb, 32, 32, mnswz) : make_map(B, K, N, ldb, 32, p.bn_alloc);
    CUtensorMap tblo = tb;
    p.b_presplit = B_lo != nullptr;
    if (B_lo) tblo = b_mn ? make_map(B_lo, N, K, ldb, 32, 32, mnswz) : make_map(B_lo, K, N, ldb, 32, p.bn_alloc);
    const size_t smem = (size_t)p.stages * stage_bytes + 1024 + 1024 + kEpiStage;   // align pad, barriers, staging
    const int64_t num_tiles = (int64_t)m_tiles * n_tiles * splits;
    dim3 grid((unsigned)std::min<int64_t>(num_tiles, 148));
    const int64_t ldp = (N + 3) / 4 * 4;      // split-K partials row pitch
    if (splits == 1) {
        p.C = C;
        p.ldc = ldc;
        p.epi = epi;
        p.split_stride = 0;
        p.vec = ((uintptr_t)C % 16) == 0 && ldc % 4 == 0 &&
                (epi != 2 || (((uintptr_t)aux % 16) == 0 && ldaux % 4 == 0));
    } else {
        c->m_gemm_part.ensure((size_t)splits * M * ldp * sizeof(float) + 16);
        p.C = c->m_gemm_part.as<float>();
        p.ldc = ldp;
        p.epi = 0;
        p.split_stride = M * ldp;
        p.vec = 1;
    }
    if (a_mn && b_mn) launch_gemm<true, true>(ta, tb, tblo, p, grid, smem, s);
    else if (a_mn) launch_gemm<true, false>(ta, tb, tblo, p, grid, smem, s);
    else if (b_mn) launch_gemm<false, true>(ta, tb, tblo, p, grid, smem, s);
    else launch_gemm<false, false>(ta, tb, tblo, p, grid, smem, s);
    count_launch(c);
    if (splits > 1) {
        const int64_t total = M * N;
        splitk_reduce_kernel<<<(unsigned)std::min<int64_t>(cdiv(total, 256), 148 * 8), 256, 0, s>>>(
            c->m_gemm_part.as<float>(), splits, M * ldp, (int)M, (int)N, ldp, C, ldc, epi, aux, ldaux);
        NTP_LAUNCH_CHECK();
        count_launch(c);
    }
}

// C = A B with the pack epilogue (epi 3): see PackEpi.  A [M x K] K-major, B [K x N] MN-major (weights,
// pre-split), N = P * d_s (no padding columns), N % 32 == 0, d_s % 8 == 0.
void gemm_tf32x3_pack(ntp_ctx* c, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B_hi,
                      const float* B_lo, int64_t ldb, const PackEpi& pk, cudaStream_t s) {
    NTP_CHECK(N % 32 == 0 && pk.d_s % 8 == 0, NTP_ERR_CONFIG, "pack epilogue needs N %% 32 == 0 and d_s %% 8 == 0");
    c->pack_epi = pk;
    gemm_tf32x3(c, M, N, K, A, lda, false, B_hi, ldb, true, nullptr, 0, 3, nullptr, 0, s, B_lo);
}

namespace {
__global__ void tf32_split_kernel(const float* __restrict__ src, int64_t rows, int32_t cols, int64_t ld,
                                  float* __restrict__ hi, float* __restrict__ lo) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * cols; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / cols, k = i - r * cols;
        const float x = src[r * ld + k];
        const float h = tf32_rn(x);
        hi[r * ld + k] = h;
        lo[r * ld + k] = tf32_rn(x - h);
    }
}
}  // namespace

// hi = rn_tf32(W), lo = rn_tf32(W - hi), same [rows x cols] / ld layout (pre-split GEMM operand).
void tf32_split(ntp_ctx* c, const float* src, int64_t rows, int64_t cols, int64_t ld, float* hi, float* lo,
                cudaStream_t s) {
    if (rows <= 0 || cols <= 0) return;
    tf32_split_kernel<<<(unsigned)std::min<int64_t>(cdiv(rows * cols, 256), 148 * 8), 256, 0, s>>>(src, rows, (int32_t)cols,
                                                                                                  ld, hi, lo);
    NTP_LAUNCH_CHECK();
    count_launch(c);
}

}  // namespace ntp
