// l2_probe.cu — measured L2 ceilings for the SpMM hop's roofline.
//
// The Reddit-shaped hop gathers rows of an L2-resident slice (41 MB at P = 1), so HBM does not
// bound it; these two kernels measure what the L2 path can deliver on this B200:
//   stream : coalesced 16-byte loads over an L2-resident buffer (every sector used once per pass)
//   gather : the hop's access pattern without its arithmetic -- for each of `m` random edge ids,
//            read one r-byte row of an [n][r] table (16-byte vectors, consecutive lanes per row),
//            sum into a register; indices streamed from HBM like col_idx
// Output: one JSON line per measurement (GB/s of sectors actually requested, and rows/s).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2_probe l2_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void stream_kernel(const uint4* __restrict__ buf, int64_t nvec, int passes, float* out) {
    float acc = 0.f;
    for (int p = 0; p < passes; ++p)
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec; i += (int64_t)gridDim.x * blockDim.x) {
            const uint4 v = __ldg(buf + i);
            acc += __uint_as_float(v.x) + __uint_as_float(v.w);
        }
    if (acc == 1234.5f) out[0] = acc;
}

// VP lanes per row (VP = r/16), 32/VP rows per warp instruction; ILP independent loads per lane.
template <int ILP>
__global__ void gather_kernel(const char* __restrict__ tab, const int32_t* __restrict__ idx, int64_t m, int vp,
                              int64_t ld, float* out) {
    const int lane = threadIdx.x & 31;
    const int rows_per_warp = 32 / vp;
    const int slot = lane / vp, c = lane % vp;
    const bool act = slot < rows_per_warp;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    float acc = 0.f;
    const int64_t step = (int64_t)rows_per_warp * ILP;
    for (int64_t base = warp * step; base < m; base += nwarps * step) {
        uint4 v[ILP];
#pragma unroll
        for (int k = 0; k < ILP; ++k) {
            const int64_t j = base + k * rows_per_warp + (act ? slot : 0);
            const int src = j < m ? __ldg(idx + j) : 0;
            v[k] = __ldg(reinterpret_cast<const uint4*>(tab + (int64_t)src * ld + c * 16));
        }
#pragma unroll
        for (int k = 0; k < ILP; ++k) acc += __uint_as_float(v[k].x) + __uint_as_float(v[k].w);
    }
    if (acc == 1234.5f) out[0] = acc;
}


// Shared-memory variant of the gather (what a source-blocked SpMM would pay per edge): each CTA
// holds a `tab_bytes` table in shared memory and gathers random r-byte rows of it.
template <int ILP>
__global__ void smem_gather_kernel(const int32_t* __restrict__ idx, int64_t m, int vp, int rows_in_smem, float* out) {
    extern __shared__ uint4 stab[];
    for (int i = threadIdx.x; i < rows_in_smem * vp; i += blockDim.x) stab[i] = make_uint4(i, 0, 0, i);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int rows_per_warp = 32 / vp;
    const int slot = lane / vp, c = lane % vp;
    const bool act = slot < rows_per_warp;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    float acc = 0.f;
    const int64_t step = (int64_t)rows_per_warp * ILP;
    for (int64_t base = warp * step; base < m; base += nwarps * step) {
        uint4 v[ILP];
#pragma unroll
        for (int k = 0; k < ILP; ++k) {
            const int64_t j = base + k * rows_per_warp + (act ? slot : 0);
            const int src = j < m ? (int)((uint32_t)__ldg(idx + j) % (uint32_t)rows_in_smem) : 0;
            v[k] = stab[src * vp + c];
        }
#pragma unroll
        for (int k = 0; k < ILP; ++k) acc += __uint_as_float(v[k].x) + __uint_as_float(v[k].w);
    }
    if (acc == 1234.5f) out[0] = acc;
}

static uint64_t splitmix(uint64_t& s) {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

int main(int argc, char** argv) {
    int dev = 0, nsm = 0;
    CK(cudaSetDevice(dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    float* out;
    CK(cudaMalloc(&out, 16));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    // ---- stream over sizes (L2-resident and not)
    for (int64_t mb : {16, 40, 64, 96, 2048}) {
        if (argc > 4) break;
        const int64_t bytes = mb << 20;
        void* buf;
        CK(cudaMalloc(&buf, bytes));
        CK(cudaMemset(buf, 0, bytes));
        const int passes = mb >= 1024 ? 2 : 40;
        float best = 1e30f;
        for (int it = 0; it < 5; ++it) {
            CK(cudaEventRecord(e0));
            stream_kernel<<<nsm * 8, 256>>>((const uint4*)buf, bytes / 16, passes, out);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (it > 0 && ms < best) best = ms;
        }
        printf("{\"probe\": \"stream\", \"MB\": %lld, \"GBps\": %.1f}\n", (long long)mb,
               (double)bytes * passes / (best * 1e-3) / 1e9);
        CK(cudaFree(buf));
    }
    // ---- random row gather: n rows of r bytes (Reddit: n = 232,965, r = 176 / 32 / 48 ...)
    const int64_t n = argc > 1 ? atoll(argv[1]) : 232965;
    const int64_t m = argc > 2 ? atoll(argv[2]) : 114082446;
    std::vector<int32_t> h(m);
    uint64_t s = 12345;
    for (int64_t i = 0; i < m; ++i) h[i] = (int32_t)(splitmix(s) % (uint64_t)n);
    int32_t* idx;
    CK(cudaMalloc(&idx, m * 4));
    CK(cudaMemcpy(idx, h.data(), m * 4, cudaMemcpyHostToDevice));
    const char* rl = argc > 3 ? argv[3] : "16,32,48,64,96,128,176,192,256";
    std::vector<int> rs;
    for (const char* q = rl; *q;) { rs.push_back(atoi(q)); while (*q && *q != ',') ++q; if (*q) ++q; }
    for (int r : rs) {
        const int vp = r / 16;
        const int64_t ld = r;
        char* tab;
        CK(cudaMalloc(&tab, n * ld + 64));
        CK(cudaMemset(tab, 0, n * ld + 64));
        const int rows_per_warp = 32 / vp;
        for (int ilp : {4, 8, 16}) {
            float best = 1e30f;
            for (int it = 0; it < 4; ++it) {
                CK(cudaEventRecord(e0));
                if (ilp == 4) gather_kernel<4><<<nsm * 8, 256>>>(tab, idx, m, vp, ld, out);
                else if (ilp == 8) gather_kernel<8><<<nsm * 8, 256>>>(tab, idx, m, vp, ld, out);
                else gather_kernel<16><<<nsm * 8, 256>>>(tab, idx, m, vp, ld, out);
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                if (it > 0 && ms < best) best = ms;
            }
            CK(cudaGetLastError());
            // sectors requested per row: rows start at multiples of r (16-byte aligned)
            double sec = 0;
            for (int k = 0; k < 32; ++k) { const int64_t a = (int64_t)k * r; sec += (double)((a + r + 31) / 32 - a / 32); }
            sec /= 32;
            printf("{\"probe\": \"gather\", \"n\": %lld, \"m\": %lld, \"row_bytes\": %d, \"ilp\": %d, \"table_MB\": %.1f, "
                   "\"ms\": %.4f, \"Grows_per_s\": %.1f, \"sector_GBps\": %.1f, \"rows_per_warp_instr\": %d}\n",
                   (long long)n, (long long)m, r, ilp, n * ld / 1e6, best, m / (best * 1e-3) / 1e9,
                   m * sec * 32 / (best * 1e-3) / 1e9, rows_per_warp);
            fflush(stdout);
        }
        if (argc <= 4) {   // shared-memory gather of the same rows (200 KB table per CTA)
            const int rows_in_smem = (200 * 1024) / r;
            const size_t sm_bytes = (size_t)rows_in_smem * r;
            CK(cudaFuncSetAttribute(smem_gather_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
            float best = 1e30f;
            for (int it = 0; it < 4; ++it) {
                CK(cudaEventRecord(e0));
                smem_gather_kernel<8><<<nsm, 1024, sm_bytes>>>(idx, m, vp, rows_in_smem, out);
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                if (it > 0 && ms < best) best = ms;
            }
            CK(cudaGetLastError());
            printf("{\"probe\": \"smem_gather\", \"m\": %lld, \"row_bytes\": %d, \"ms\": %.4f, \"Grows_per_s\": %.1f, "
                   "\"cycles_per_row_per_SM_at_1965MHz\": %.3f}\n", (long long)m, r, best, m / (best * 1e-3) / 1e9,
                   (best * 1e-3) * 1.965e9 * nsm / m);
            fflush(stdout);
        }
        CK(cudaFree(tab));
    }
    return 0;
}
