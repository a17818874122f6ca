// wgrad.cu — dW0 = X_v^T (G .* [H1 > 0]) of the W1-after-propagation epoch (SURVEY §8(a) a9 unpack +
// a10) in one tcgen05 kernel, reading the gathered bf16 gradient slice directly.
//
// G (the backward propagation's output rows, bf16 storage) is exact in bf16, and every fp32 x splits
// exactly into three bf16 pieces x = b0 + b1 + b2 (b0 = rn(x), b1 = rn(x - b0), b2 = x - b0 - b1: 8 + 8 + 8
// mantissa bits), so three kind::f16 MMAs per K step give each product x*g exactly (8 x 8-bit
// mantissas fit fp32) with fp32 accumulation -- the fp32 GEMM's precision without the fp32 copy of
// G and without the separate unpack pass (which wrote and re-read 2x the slice's bytes in fp32).
//
// Tile: M = d_in (<= 128, TMEM lanes), N = hid = 128, K = 16 vertex rows per stage.  Each CTA owns a
// contiguous range of the chunk's rows (split-K; partials summed in CTA order afterwards).
//   warp 0    : TMA producer (X rows fp32 box [16 x d_in], no swizzle; G rows bf16 128B-swizzled boxes)
//   warp 1    : MMA issuer (3 x tcgen05.mma kind::f16 per stage), TMEM allocation
//   warps 2-5 : converters (X -> b0/b1/b2 tiles, MN-major SW128; ReLU' mask applied to G in place), then
//               the epilogue (TMEM -> fp32 partial rows)
#include <algorithm>
#include <cstring>

#include "ntp_internal.cuh"
#include "ptx.cuh"

namespace ntp {

namespace {

constexpr int kWgThreads = 192;
constexpr int kRows = 16;                       // K rows per stage
constexpr int kXStage = kRows * 128 * 4;        // fp32 X staging (d_in padded to 128 columns)
constexpr int kGStage = kRows * 128 * 2;        // bf16 G, two 64-column SW128 boxes of 16 rows
constexpr int kABox = kRows * 128;              // one 64-column bf16 box of 16 rows (2 KB)
constexpr int kATile = 2 * kABox;               // 4 KB per bf16 piece
constexpr int kBits = kRows * 16;               // ReLU' words of the stage's rows (nwb = 4 words per row)
constexpr int kStage = kXStage + kGStage + 3 * kATile + 1024;   // 25 KB: the mask words padded so every stage stays 1024-byte aligned (SW128 tiles)

struct WgParams {
    int64_t r_begin, r_end;   // this call's rows (absolute vertex rows of the rank)
    int64_t rows_per_cta;     // multiple of 16
    int d_in, hid, d_s, lds;  // d_s: slice width (>= 64), lds = log2(d_s)
    const uint32_t* bits;     // ReLU' words [V_p][nwb]
    int nwb;
    float* part;              // [grid][d_in][hid]
    int stages;
    uint32_t idesc;
};

__device__ __forceinline__ uint32_t swz(int r, int col) {   // (K row, 64-col box element) in SW128 boxes
    return (uint32_t)((col >> 6) * kABox + r * 128 + ((((col & 63) >> 3) ^ (r & 7)) << 4) + ((col & 7) << 1));
}
__device__ __forceinline__ uint64_t desc_mn(uint32_t addr) {   // MN-major SW128: 64-elem atoms a box apart
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)(kABox >> 4) << 16) | (64ull << 32) | (1ull << 46) |
           (2ull << 61);
}

__global__ void __launch_bounds__(kWgThreads, 1)
    wgrad_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmG,
                 const __grid_constant__ CUtensorMap tmB, const WgParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);   // stays a shared pointer
    const int S = p.stages;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * kStage);
    uint64_t* conv = full + S;
    uint64_t* empty = conv + S;
    uint64_t* done = empty + S;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(done + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t k0 = p.r_begin + (int64_t)blockIdx.x * p.rows_per_cta;
    const int64_t k1 = std::min<int64_t>(k0 + p.rows_per_cta, p.r_end);
    const int nsteps = k1 > k0 ? (int)((k1 - k0 + kRows - 1) / kRows) : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&conv[s], 128);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::mbar_init(done, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
            ptx::smem_u32(tmem_holder)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_holder;

    if (warp == 0) {
        if (lane == 0) {   // ---------------- TMA producer
            for (int j = 0; j < nsteps; ++j) {
                const int s = j % S;
                if (j >= S) ptx::mbar_wait(&empty[s], ((j / S) - 1) & 1);
                uint8_t* st = smem + (size_t)s * kStage;
                const int row = (int)(k0 + (int64_t)j * kRows);
                ptx::mbar_expect_tx(&full[s], kXStage + kGStage + kBits);
                ptx::tma_load_2d(st, &tmX, &full[s], 0, row);                       // X rows [16][128] fp32
                ptx::tma_load_2d(st + kXStage + kGStage + 3 * kATile, &tmB, &full[s], 0, row);   // mask words
#pragma unroll
                for (int bx = 0; bx < 2; ++bx) {                                    // G boxes [16][64] bf16
                    const int col = 64 * bx;
                    asm volatile(
                        "cp.async.bulk.tensor.3d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
                        "%5}], [%2];" ::"r"(ptx::smem_u32(st + kXStage + bx * kABox)),
                        "l"(reinterpret_cast<uint64_t>(&tmG)), "r"(ptx::smem_u32(&full[s])), "r"(col & (p.d_s - 1)),
                        "r"(row), "r"(col >> p.lds)
                        : "memory");
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {   // ---------------- MMA issuer
            for (int j = 0; j < nsteps; ++j) {
                const int s = j % S;
                ptx::mbar_wait(&conv[s], (j / S) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t st = ptx::smem_u32(smem + (size_t)s * kStage);
                const uint64_t bdesc = desc_mn(st + kXStage);
#pragma unroll
                for (int piece = 0; piece < 3; ++piece) {
                    const uint64_t adesc = desc_mn(st + kXStage + kGStage + piece * kATile);
                    const uint32_t acc = (j > 0 || piece > 0) ? 1u : 0u;
                    asm volatile(
                        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, q;\n\t}" ::"r"(tmem),
                        "l"(adesc), "l"(bdesc), "r"(p.idesc), "r"(acc));
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 ptx::smem_u32(&empty[s]))
                             : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             ptx::smem_u32(done))
                         : "memory");
        }
    } else {
        // ---------------- converters: warp cw takes rows 4cw .. 4cw+3, lane l columns 4l .. 4l+3 (16-byte
        // row segments: conflict-free reads of the fp32 staging, 8-byte stores into the swizzled tiles)
        const int cw = warp - 2;
        const int c4 = 4 * lane;
        for (int j = 0; j < nsteps; ++j) {
            const int s = j % S;
            ptx::mbar_wait(&full[s], (j / S) & 1);
            uint8_t* st = smem + (size_t)s * kStage;
            uint8_t* at = st + kXStage + kGStage;
            uint8_t* gt = st + kXStage;
            const uint32_t* bw = reinterpret_cast<const uint32_t*>(st + kXStage + kGStage + 3 * kATile);
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) {
                const int r = 4 * cw + rr;
                const int64_t row = k0 + (int64_t)j * kRows + r;
                const bool valid = row < k1;
                float4 x = *reinterpret_cast<const float4*>(st + r * 512 + c4 * 4);
                if (!valid) x = make_float4(0.f, 0.f, 0.f, 0.f);
                if (c4 >= p.d_in) x = make_float4(0.f, 0.f, 0.f, 0.f);
                else if (c4 + 3 >= p.d_in) {
                    if (c4 + 1 >= p.d_in) x.y = 0.f;
                    if (c4 + 2 >= p.d_in) x.z = 0.f;
                    x.w = 0.f;
                }
                // exact three-way split x = b0 + b1 + b2 (packed conversions, two values per instruction)
                const __nv_bfloat162 b0a = __floats2bfloat162_rn(x.x, x.y), b0b = __floats2bfloat162_rn(x.z, x.w);
                const float2 h0a = __bfloat1622float2(b0a), h0b = __bfloat1622float2(b0b);
                const float r0x = x.x - h0a.x, r0y = x.y - h0a.y, r0z = x.z - h0b.x, r0w = x.w - h0b.y;
                const __nv_bfloat162 b1a = __floats2bfloat162_rn(r0x, r0y), b1b = __floats2bfloat162_rn(r0z, r0w);
                const float2 h1a = __bfloat1622float2(b1a), h1b = __bfloat1622float2(b1b);
                const __nv_bfloat162 b2a = __floats2bfloat162_rn(r0x - h1a.x, r0y - h1a.y);
                const __nv_bfloat162 b2b = __floats2bfloat162_rn(r0z - h1b.x, r0w - h1b.y);
                const uint32_t off = swz(r, c4);   // 8-byte half of a 16-byte swizzle chunk
                *reinterpret_cast<uint2*>(at + off) =
                    make_uint2(*reinterpret_cast<const uint32_t*>(&b0a), *reinterpret_cast<const uint32_t*>(&b0b));
                *reinterpret_cast<uint2*>(at + kATile + off) =
                    make_uint2(*reinterpret_cast<const uint32_t*>(&b1a), *reinterpret_cast<const uint32_t*>(&b1b));
                *reinterpret_cast<uint2*>(at + 2 * kATile + off) =
                    make_uint2(*reinterpret_cast<const uint32_t*>(&b2a), *reinterpret_cast<const uint32_t*>(&b2b));
                // ReLU' mask on G (row r, columns c4 .. c4+3)
                const uint32_t word = valid ? (bw[r * 4 + (c4 >> 5)] >> (c4 & 31)) : 0u;
                uint2* q = reinterpret_cast<uint2*>(gt + off);
                uint2 v = *q;
                v.x &= ((word & 1u) ? 0x0000FFFFu : 0u) | ((word & 2u) ? 0xFFFF0000u : 0u);
                v.y &= ((word & 4u) ? 0x0000FFFFu : 0u) | ((word & 8u) ? 0xFFFF0000u : 0u);
                *q = v;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            ptx::mbar_arrive(&conv[s]);
        }
        // ---------------- epilogue: TMEM lane = input feature m, 32 columns at a time
        const int qd = warp & 3;
        const int m = qd * 32 + lane;
        if (nsteps > 0) {
            ptx::mbar_wait(done, 0);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        float* dst = p.part + (int64_t)blockIdx.x * p.d_in * p.hid + (int64_t)m * p.hid;
        for (int cc = 0; cc < p.hid; cc += 32) {
            uint32_t x[32];
            if (nsteps > 0) {
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7]),
                      "=r"(x[8]), "=r"(x[9]), "=r"(x[10]), "=r"(x[11]), "=r"(x[12]), "=r"(x[13]), "=r"(x[14]),
                      "=r"(x[15]), "=r"(x[16]), "=r"(x[17]), "=r"(x[18]), "=r"(x[19]), "=r"(x[20]), "=r"(x[21]),
                      "=r"(x[22]), "=r"(x[23]), "=r"(x[24]), "=r"(x[25]), "=r"(x[26]), "=r"(x[27]), "=r"(x[28]),
                      "=r"(x[29]), "=r"(x[30]), "=r"(x[31])
                    : "r"(tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)cc));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            }
            if (m < p.d_in)
#pragma unroll
                for (int k = 0; k < 32; ++k) dst[cc + k] = nsteps > 0 ? __uint_as_float(x[k]) : 0.f;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
    }
}

__global__ void wgrad_reduce_kernel(const float* __restrict__ part, int nb, int64_t total, float* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        float a = 0.f;
        for (int b = 0; b < nb; ++b) a += part[b * total + i];
        out[i] = a;
    }
}

}  // namespace

bool wgrad_fused_supported(int32_t P, int32_t d_s, int32_t d_in, int32_t hid, ntp_dtype dt) {
    const char* v = getenv("NTP_WGRAD_FUSED");
    return !(v && atoi(v) == 0) && dt == NTP_BF16 && hid == 128 && (int64_t)P * d_s == 128 && d_s >= 64 &&
           d_in >= 1 && d_in <= 128;   // hid = 128: 4 mask words per row (the TMA box of the mask)
}

void wgrad_fused(ntp_ctx* c, const float* X, int64_t ldx, int64_t V_p, int32_t d_in, const void* G, int32_t d_s,
                 int32_t P, int32_t hid, const uint32_t* bits, int32_t nwb, int64_t r_begin, int64_t r_end, float* dW0,
                 cudaStream_t s) {
    WgParams p{};
    p.r_begin = r_begin;
    p.r_end = r_end;
    p.d_in = d_in;
    p.hid = hid;
    p.d_s = d_s;
    p.lds = 0;
    while ((1 << p.lds) < d_s) ++p.lds;
    p.bits = bits;
    p.nwb = nwb;
    const int64_t rows = r_end - r_begin;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(148, cdiv(rows, 2048)));
    p.rows_per_cta = cdiv(cdiv(rows, grid), kRows) * kRows;
    p.stages = 8;
    p.idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(128 >> 3) << 17) |
              ((uint32_t)(128 >> 4) << 24);
    const size_t part_bytes = (size_t)grid * d_in * hid * sizeof(float);
    c->m_wgrad.ensure(part_bytes + 16);
    p.part = c->m_wgrad.as<float>();
    NTP_CHECK(((uintptr_t)X % 16) == 0 && (ldx * 4) % 16 == 0 && ((uintptr_t)G % 16) == 0, NTP_ERR_SHAPE,
              "fused dW0: operands must be 16-byte aligned");
    CUtensorMap tmX, tmG;
    {
        const cuuint64_t dims[2] = {(cuuint64_t)d_in, (cuuint64_t)V_p};
        const cuuint64_t strides[1] = {(cuuint64_t)ldx * 4};
        const cuuint32_t box[2] = {128, kRows};
        const cuuint32_t estr[2] = {1, 1};
        CUresult r = tensor_map_encoder()(&tmX, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(X), dims, strides,
                                          box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        NTP_CHECK(r == CUDA_SUCCESS, NTP_ERR_CUDA, "cuTensorMapEncodeTiled (dW0 X) failed (%d)", (int)r);
    }
    {
        const cuuint64_t dims[3] = {(cuuint64_t)d_s, (cuuint64_t)V_p, (cuuint64_t)P};
        const cuuint64_t strides[2] = {(cuuint64_t)d_s * 2, (cuuint64_t)V_p * d_s * 2};
        const cuuint32_t box[3] = {64, kRows, 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = tensor_map_encoder()(&tmG, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(G), dims, strides,
                                          box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        NTP_CHECK(r == CUDA_SUCCESS, NTP_ERR_CUDA, "cuTensorMapEncodeTiled (dW0 G) failed (%d)", (int)r);
    }
    CUtensorMap tmB;
    {
        const cuuint64_t dims[2] = {(cuuint64_t)nwb, (cuuint64_t)V_p};
        const cuuint64_t strides[1] = {(cuuint64_t)nwb * 4};
        const cuuint32_t box[2] = {4, kRows};
        const cuuint32_t estr[2] = {1, 1};
        CUresult r = tensor_map_encoder()(&tmB, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint32_t*>(bits), dims,
                                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        NTP_CHECK(r == CUDA_SUCCESS, NTP_ERR_CUDA, "cuTensorMapEncodeTiled (dW0 mask) failed (%d)", (int)r);
    }
    const size_t smem = 1024 + (size_t)p.stages * kStage + (3 * p.stages + 2) * 8 + 16;
    static bool attr = false;
    if (!attr) {
        NTP_CUDA(cudaFuncSetAttribute(wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr = true;
    }
    wgrad_kernel<<<grid, kWgThreads, smem, s>>>(tmX, tmG, tmB, p);
    NTP_LAUNCH_CHECK();
    const int64_t total = (int64_t)d_in * hid;
    wgrad_reduce_kernel<<<(unsigned)std::min<int64_t>(cdiv(total, 256), 148 * 4), 256, 0, s>>>(p.part, grid, total, dW0);
    NTP_LAUNCH_CHECK();
    count_launch(c, 2);
}

}  // namespace ntp
