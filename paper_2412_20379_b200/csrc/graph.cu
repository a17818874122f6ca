// graph.cu — device-side graph setup (K13-K15).
//
//   R-MAT arcs (counter-based) -> 64-bit keys (dst<<32 | src),
//   invalid arcs (id >= n, self loop; R1) -> sentinel  ->  CUB radix sort ->
//   CUB unique (dedup, O1) -> in-CSR (row_ptr by binary search, col = low word)
//   -> transpose keys (src<<32 | dst) -> sort -> out-CSR  -> degrees,
//   D~^{-1/2} = (deg+1)^{-1/2}  -> merge-path work partition.
// Integer work is bit-exact against the oracle (tests/test_gpu_graph.py).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>

#include "ntp_internal.cuh"

namespace ntp {

// ------------------------------------------------------------------ hashing
__device__ __forceinline__ uint64_t splitmix_fin(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ void rmat_arc(int scale, uint32_t t0, uint32_t t1, uint32_t t2, uint64_t base,
                                         uint64_t i, uint64_t& s, uint64_t& d) {
    s = 0;
    d = 0;
    for (int l = 0; l < scale; ++l) {
        const uint32_t u = (uint32_t)(splitmix_fin(base + i * 64ull + (uint64_t)l) >> 32);
        const uint64_t sb = (u >= t1) ? 1u : 0u;                 // quadrants c, d
        const uint64_t db = (u >= t0 && u < t1) || (u >= t2) ? 1u : 0u;  // quadrants b, d
        s = (s << 1) | sb;
        d = (d << 1) | db;
    }
}

__global__ void rmat_raw_kernel(int scale, uint32_t t0, uint32_t t1, uint32_t t2, uint64_t base,
                                int64_t i0, int64_t count, int64_t* src, int64_t* dst) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count;
         k += (int64_t)gridDim.x * blockDim.x) {
        uint64_t s, d;
        rmat_arc(scale, t0, t1, t2, base, (uint64_t)(i0 + k), s, d);
        src[k] = (int64_t)s;
        dst[k] = (int64_t)d;
    }
}

__device__ __forceinline__ uint64_t arc_key(int64_t s, int64_t d, int64_t n, uint64_t sentinel) {
    const bool ok = s >= 0 && d >= 0 && s < n && d < n && s != d;
    return ok ? (((uint64_t)d << 32) | (uint64_t)s) : sentinel;
}

__global__ void rmat_keys_kernel(int scale, uint32_t t0, uint32_t t1, uint32_t t2, uint64_t base,
                                 int64_t i0, int64_t count, int64_t n, int sym, uint64_t sentinel,
                                 uint64_t* keys) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count;
         k += (int64_t)gridDim.x * blockDim.x) {
        uint64_t s, d;
        rmat_arc(scale, t0, t1, t2, base, (uint64_t)(i0 + k), s, d);
        keys[k] = arc_key((int64_t)s, (int64_t)d, n, sentinel);
        if (sym) keys[count + k] = arc_key((int64_t)d, (int64_t)s, n, sentinel);
    }
}

__global__ void arcs_to_keys_kernel(const int64_t* src, const int64_t* dst, int64_t m, int64_t n, int sym,
                                    uint64_t sentinel, uint64_t* keys) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
        keys[k] = arc_key(src[k], dst[k], n, sentinel);
        if (sym) keys[m + k] = arc_key(dst[k], src[k], n, sentinel);
    }
}

// in-CSR arrays -> keys (dst<<32 | src)
__global__ void csr_to_keys_kernel(const int64_t* row_ptr, const int32_t* col, int64_t n, int64_t n_arcs_unused,
                                   uint64_t sentinel, uint64_t* keys) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) keys[e] = arc_key(col[e], v, n, sentinel);
    }
}

// row_ptr[v] = lower_bound(keys, v << 32) for v in [0, n]; col[i] = low word
__global__ void keys_to_csr_kernel(const uint64_t* keys, int64_t nnz, int64_t n, int32_t* row_ptr, int32_t* col) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i < nnz; i += stride) col[i] = (int32_t)(keys[i] & 0xFFFFFFFFull);
    for (int64_t v = tid; v <= n; v += stride) {
        const uint64_t target = (uint64_t)v << 32;
        int64_t lo = 0, hi = nnz;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (keys[mid] < target) lo = mid + 1; else hi = mid;
        }
        row_ptr[v] = (int32_t)lo;
    }
}

__global__ void transpose_keys_kernel(const uint64_t* keys, int64_t nnz, uint64_t* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        out[i] = ((k & 0xFFFFFFFFull) << 32) | (k >> 32);
    }
}

__global__ void dinv_kernel(const int32_t* row_ptr, int64_t n, float* dinv) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const double deg = (double)(row_ptr[v + 1] - row_ptr[v]);
        dinv[v] = (float)(1.0 / sqrt(deg + 1.0));
    }
}

// Merge-path split of diagonal d: smallest r in [0, n] with r == n or row_ptr[r+1] + r >= d.
__global__ void merge_path_kernel(const int32_t* row_ptr, int64_t n, int64_t nnz, int64_t T, int64_t U,
                                  int32_t* unit_row, int32_t* unit_e) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u <= U; u += (int64_t)gridDim.x * blockDim.x) {
        const int64_t d = min(u * T, n + nnz);
        int64_t lo = max((int64_t)0, d - nnz), hi = min(d, n);
        while (lo < hi) {
            const int64_t r = (lo + hi) >> 1;
            if ((int64_t)row_ptr[r + 1] + r >= d) hi = r; else lo = r + 1;
        }
        unit_row[u] = (int32_t)lo;
        unit_e[u] = (int32_t)(d - lo);
    }
}

static int grid_for(int64_t work, int block = 256) {
    int64_t g = cdiv(std::max<int64_t>(work, 1), block);
    return (int)std::min<int64_t>(g, 148 * 32);
}

// ------------------------------------------------------------------ public pieces
void rmat_raw(ntp_ctx* c, int scale, const uint32_t thr[3], uint64_t seed, int64_t i0, int64_t count,
              int64_t* src, int64_t* dst, cudaStream_t s) {
    const uint64_t base = seed * 0x9E3779B97F4A7C15ULL;   // stream 0
    rmat_raw_kernel<<<grid_for(count), 256, 0, s>>>(scale, thr[0], thr[1], thr[2], base, i0, count, src, dst);
    NTP_LAUNCH_CHECK();
    count_launch(c);
}

static int key_bits(int64_t n) {       // 2^bits > n  (so the sentinel's dst field is never a vertex)
    int b = 1;
    while ((int64_t(1) << b) <= n) ++b;
    return b;
}
static uint64_t sentinel_for(int64_t n) {
    return (((uint64_t(1) << key_bits(n)) - 1) << 32) | 0xFFFFFFFFull;
}

void rmat_keys(ntp_ctx* c, int scale, const uint32_t thr[3], uint64_t seed, int64_t i0, int64_t count,
               int64_t n, bool symmetric, uint64_t* keys, cudaStream_t s) {
    const uint64_t base = seed * 0x9E3779B97F4A7C15ULL;
    rmat_keys_kernel<<<grid_for(count), 256, 0, s>>>(scale, thr[0], thr[1], thr[2], base, i0, count, n,
                                                     symmetric ? 1 : 0, sentinel_for(n), keys);
    NTP_LAUNCH_CHECK();
    count_launch(c);
}

void arcs_to_keys(ntp_ctx* c, const int64_t* src, const int64_t* dst, int64_t m, int64_t n, bool sym,
                  uint64_t* keys, cudaStream_t s) {
    arcs_to_keys_kernel<<<grid_for(m), 256, 0, s>>>(src, dst, m, n, sym ? 1 : 0, sentinel_for(n), keys);
    NTP_LAUNCH_CHECK();
    count_launch(c);
}

void csr_to_keys(ntp_ctx* c, const int64_t* row_ptr, const int32_t* col, int64_t n, uint64_t* keys,
                 cudaStream_t s) {
    csr_to_keys_kernel<<<grid_for(n), 256, 0, s>>>(row_ptr, col, n, 0, sentinel_for(n), keys);
    NTP_LAUNCH_CHECK();
    count_launch(c);
}

// Sort + dedup keys in place (keys/alt both hold >= m entries). Returns number of unique valid keys
// now at the front of *result.
static int64_t sort_unique(ntp_ctx* c, uint64_t* keys, uint64_t* alt, int64_t m, int64_t n, bool dedup,
                           uint64_t** result, cudaStream_t s) {
    const int end_bit = 32 + key_bits(n);
    cub::DoubleBuffer<uint64_t> db(keys, alt);
    size_t tmp_bytes = 0;
    NTP_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, db, (int64_t)m, 0, end_bit, s));
    DevBuf tmp;
    size_t tmp2 = 0;
    int64_t* d_count = nullptr;
    NTP_CUDA(cub::DeviceSelect::Unique(nullptr, tmp2, db.Current(), db.Alternate(), d_count, (int64_t)m, s));
    tmp.ensure(std::max(tmp_bytes, tmp2) + 256);
    NTP_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, db, (int64_t)m, 0, end_bit, s));
    count_launch(c, end_bit / 8 + 1);
    uint64_t* sorted = db.Current();
    uint64_t* other = db.Alternate();
    int64_t cnt = m;
    DevBuf dcount;
    dcount.ensure(sizeof(int64_t));
    if (dedup) {
        size_t tb = tmp.bytes - 256;
        NTP_CUDA(cub::DeviceSelect::Unique(tmp.p, tb, sorted, other, dcount.as<int64_t>(), (int64_t)m, s));
        count_launch(c, 2);
        NTP_CUDA(cudaMemcpyAsync(&cnt, dcount.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        NTP_CUDA(cudaStreamSynchronize(s));
        sorted = other;
    }
    // drop a trailing sentinel (the largest possible key)
    if (cnt > 0) {
        uint64_t last = 0;
        NTP_CUDA(cudaMemcpyAsync(&last, sorted + cnt - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        NTP_CUDA(cudaStreamSynchronize(s));
        if (last == sentinel_for(n)) {
            if (!dedup) {
                // count sentinels: they are all at the end
                int64_t lo = 0, hi = cnt;
                std::vector<uint64_t> probe(1);
                while (lo < hi) {   // host binary search with single-element reads (setup path only)
                    const int64_t mid = (lo + hi) / 2;
                    NTP_CUDA(cudaMemcpy(probe.data(), sorted + mid, 8, cudaMemcpyDeviceToHost));
                    if (probe[0] < sentinel_for(n)) lo = mid + 1; else hi = mid;
                }
                cnt = lo;
            } else {
                cnt -= 1;
            }
        }
    }
    *result = sorted;
    return cnt;
}

static void fill_csr(ntp_ctx* c, const uint64_t* keys, int64_t nnz, int64_t n, Csr& csr, cudaStream_t s) {
    csr.row_ptr.ensure((n + 1) * sizeof(int32_t));
    csr.col.ensure(std::max<int64_t>(nnz, 1) * sizeof(int32_t));
    keys_to_csr_kernel<<<grid_for(std::max(nnz, n + 1)), 256, 0, s>>>(keys, nnz, n, csr.row_ptr.as<int32_t>(),
                                                                       csr.col.as<int32_t>());
    NTP_LAUNCH_CHECK();
    count_launch(c);
}

static void make_partition(ntp_ctx* c, Csr& csr, int64_t n, int64_t nnz, int64_t T, cudaStream_t s) {
    const int64_t items = n + nnz;
    csr.U = std::max<int64_t>(1, cdiv(items, T));
    csr.unit_row.ensure((csr.U + 1) * sizeof(int32_t));
    csr.unit_e.ensure((csr.U + 1) * sizeof(int32_t));
    merge_path_kernel<<<grid_for(csr.U + 1), 256, 0, s>>>(csr.row_ptr.as<int32_t>(), n, nnz, T, csr.U,
                                                          csr.unit_row.as<int32_t>(), csr.unit_e.as<int32_t>());
    NTP_LAUNCH_CHECK();
    count_launch(c);
    csr.h_unit_row.resize(csr.U + 1);
    NTP_CUDA(cudaMemcpyAsync(csr.h_unit_row.data(), csr.unit_row.p, (csr.U + 1) * sizeof(int32_t),
                             cudaMemcpyDeviceToHost, s));
    NTP_CUDA(cudaStreamSynchronize(s));
}

// ---- degree-ordered internal vertex numbering (NTP_G_REORDER)
__global__ void key_degrees_kernel(const uint64_t* __restrict__ keys, int64_t nnz, int32_t* __restrict__ deg) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        atomicAdd(&deg[k >> 32], 1);                  // in-degree of the destination
        atomicAdd(&deg[k & 0xFFFFFFFFull], 1);        // out-degree of the source
    }
}
__global__ void order_keys_kernel(const int32_t* __restrict__ deg, int64_t n, uint64_t* __restrict__ keys, int mode) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t d = (uint32_t)deg[v] + 1u;
        uint32_t cls = d;                                        // mode 0: exact degree
        if (mode >= 1) {                                         // 1: octave, 2: quarter octave
            const int lz = 31 - __clz(d);
            cls = (uint32_t)lz << 2;
            if (mode == 2 && lz >= 2) cls |= (d >> (lz - 2)) & 3u;
        }
        keys[v] = ((uint64_t)(0xFFFFFFFFu - cls) << 32) | (uint64_t)v;   // stable within a class
    }
}
__global__ void order_maps_kernel(const uint64_t* __restrict__ sorted, int64_t n, int32_t* __restrict__ perm,
                                  int32_t* __restrict__ inv) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = (int32_t)(sorted[i] & 0xFFFFFFFFull);
        inv[i] = v;
        perm[v] = (int32_t)i;
    }
}
__global__ void relabel_keys_kernel(const uint64_t* __restrict__ in, int64_t nnz, const int32_t* __restrict__ map,
                                    uint64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = in[i];
        out[i] = ((uint64_t)(uint32_t)map[k >> 32] << 32) | (uint64_t)(uint32_t)map[k & 0xFFFFFFFFull];
    }
}

// Internal ids by descending total degree (in + out, ties by id): the rows the hops gather most
// often become contiguous, so their lines stay resident in L2/L1.  g.perm maps
// original -> internal, g.inv internal -> original.  `sorted` (nnz keys, original ids) is
// relabelled and re-sorted into `out_sorted` (alt buffer).
static uint64_t* reorder_vertices(ntp_ctx* c, uint64_t* sorted, uint64_t* spare, int64_t nnz, int64_t n, cudaStream_t s) {
    Graph& g = c->g;
    g.perm.ensure(std::max<int64_t>(n, 1) * sizeof(int32_t));
    g.inv.ensure(std::max<int64_t>(n, 1) * sizeof(int32_t));
    {
        DevBuf deg, ok, oalt, tmp;
        deg.ensure(std::max<int64_t>(n, 1) * sizeof(int32_t));
        ok.ensure(std::max<int64_t>(n, 1) * sizeof(uint64_t));
        oalt.ensure(std::max<int64_t>(n, 1) * sizeof(uint64_t));
        NTP_CUDA(cudaMemsetAsync(deg.p, 0, std::max<int64_t>(n, 1) * sizeof(int32_t), s));
        key_degrees_kernel<<<grid_for(nnz), 256, 0, s>>>(sorted, nnz, deg.as<int32_t>());
        static const int mode = [] { const char* e = getenv("NTP_REORDER_MODE"); return e ? atoi(e) : 1; }();
        order_keys_kernel<<<grid_for(n), 256, 0, s>>>(deg.as<int32_t>(), n, ok.as<uint64_t>(), mode);
        NTP_LAUNCH_CHECK();
        cub::DoubleBuffer<uint64_t> db(ok.as<uint64_t>(), oalt.as<uint64_t>());
        size_t tb = 0;
        NTP_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, (int64_t)n, 0, 64, s));
        tmp.ensure(tb + 256);
        NTP_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, db, (int64_t)n, 0, 64, s));
        order_maps_kernel<<<grid_for(n), 256, 0, s>>>(db.Current(), n, g.perm.as<int32_t>(), g.inv.as<int32_t>());
        NTP_LAUNCH_CHECK();
        count_launch(c, 12);
        NTP_CUDA(cudaStreamSynchronize(s));
    }
    relabel_keys_kernel<<<grid_for(nnz), 256, 0, s>>>(sorted, nnz, g.perm.as<int32_t>(), spare);
    NTP_LAUNCH_CHECK();
    count_launch(c);
    uint64_t* out = nullptr;
    sort_unique(c, spare, sorted, nnz, n, false, &out, s);   // a permutation: no duplicates appear
    g.reordered = true;
    return out;
}

__global__ void original_keys_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ col, int64_t n,
                                     const int32_t* __restrict__ inv, uint64_t* __restrict__ keys) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t hi = (uint64_t)(uint32_t)inv[r] << 32;
        for (int32_t e = rp[r]; e < rp[r + 1]; ++e) keys[e] = hi | (uint64_t)(uint32_t)inv[col[e]];
    }
}
__global__ void gather_f32_kernel(const float* __restrict__ src, const int32_t* __restrict__ idx, int64_t n,
                                  float* __restrict__ dst) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        dst[v] = src[idx[v]];
}

// keys: device buffer with m keys and room for an alternate buffer of m keys at keys + m_cap.
void build_graph_from_keys(ntp_ctx* c, uint64_t* keys, int64_t m, int64_t n, bool symmetric,
                           DevBuf& owner, bool reorder) {
    cudaStream_t s = c->s_comp;
    Graph& g = c->g;
    g.reset();   // drops the previous graph
    drop_epoch_graph(c);
    c->graph_warm = false;
    c->g_version++;
    // merge-path unit size T (a graph constant): measured per hop, T = 1024 vs 2048 -- Reddit d_s 44 / 24 / 8:
    // 2.28 / 1.36 / 0.78 vs 2.29 / 1.42 / 0.86 ms; products d_s 48 / 12: 2.65 / 1.06 vs 2.95 / 1.13; papers bf16
    // d_s 128 / 16: 107.1 / 24.3 vs 104.9 / 23.5 (more units = more carries on the 111M-vertex graph); 512 and
    // 256 were slower everywhere.  So 1024 below 10M vertices, 2048 above.
    g.unit_items = n < 10000000 ? 1024 : 2048;
    if (const char* t = getenv("NTP_UNIT_ITEMS")) g.unit_items = std::max(64, atoi(t));
    g.n = n;
    g.symmetric = symmetric;
    DevBuf alt;
    alt.ensure(std::max<int64_t>(m, 1) * sizeof(uint64_t));
    uint64_t* sorted = nullptr;
    const int64_t nnz = sort_unique(c, keys, alt.as<uint64_t>(), m, n, true, &sorted, s);
    NTP_CHECK(nnz < (int64_t(1) << 31), NTP_ERR_CONFIG, "nnz = %lld >= 2^31 is not supported", (long long)nnz);
    g.nnz = nnz;
    if (reorder && n > 0 && nnz > 0) sorted = reorder_vertices(c, sorted, (sorted == keys) ? alt.as<uint64_t>() : keys, nnz, n, s);
    fill_csr(c, sorted, nnz, n, g.in, s);
    make_partition(c, g.in, n, nnz, g.unit_items, s);
    g.dinv_in.ensure(std::max<int64_t>(n, 1) * sizeof(float));
    dinv_kernel<<<grid_for(n), 256, 0, s>>>(g.in.row_ptr.as<int32_t>(), n, g.dinv_in.as<float>());
    NTP_LAUNCH_CHECK();
    count_launch(c);
    if (!symmetric) {
        uint64_t* other = (sorted == keys) ? alt.as<uint64_t>() : keys;
        transpose_keys_kernel<<<grid_for(nnz), 256, 0, s>>>(sorted, nnz, other);
        NTP_LAUNCH_CHECK();
        count_launch(c);
        uint64_t* sorted_t = nullptr;
        uint64_t* spare = (other == keys) ? alt.as<uint64_t>() : keys;
        const int64_t nnz_t = sort_unique(c, other, spare, nnz, n, false, &sorted_t, s);
        NTP_CHECK(nnz_t == nnz, NTP_ERR_CUDA, "transpose lost arcs (%lld vs %lld)", (long long)nnz_t,
                  (long long)nnz);
        fill_csr(c, sorted_t, nnz, n, g.out, s);
        make_partition(c, g.out, n, nnz, g.unit_items, s);
        g.dinv_out.ensure(std::max<int64_t>(n, 1) * sizeof(float));
        dinv_kernel<<<grid_for(n), 256, 0, s>>>(g.out.row_ptr.as<int32_t>(), n, g.dinv_out.as<float>());
        NTP_LAUNCH_CHECK();
        count_launch(c);
    }
    if (g.reordered) {   // original-order copies of the scales for the layout kernels
        g.dinv_orig.ensure(2 * std::max<int64_t>(n, 1) * sizeof(float));
        gather_f32_kernel<<<grid_for(n), 256, 0, s>>>(g.dinv_in_p(), g.perm.as<int32_t>(), n, g.dinv_orig.as<float>());
        gather_f32_kernel<<<grid_for(n), 256, 0, s>>>(g.dinv_out_p(), g.perm.as<int32_t>(), n,
                                                      g.dinv_orig.as<float>() + n);
        NTP_LAUNCH_CHECK();
        count_launch(c, 2);
    }
    NTP_CUDA(cudaStreamSynchronize(s));
    g.loaded = true;
    (void)owner;
}

// The CSR `csr` of a reordered graph expressed in ORIGINAL ids (rows and columns), columns ascending
// per row, into `out` (row_ptr / col only): what ntp_copy_csr returns.
void export_original_csr(ntp_ctx* c, const Csr& csr, Csr& out) {
    const Graph& g = c->g;
    cudaStream_t s = c->s_comp;
    const int64_t n = g.n, nnz = g.nnz;
    DevBuf keys, alt;
    keys.ensure(std::max<int64_t>(nnz, 1) * sizeof(uint64_t));
    alt.ensure(std::max<int64_t>(nnz, 1) * sizeof(uint64_t));
    original_keys_kernel<<<grid_for(n), 256, 0, s>>>(csr.row_ptr.as<int32_t>(), csr.col.as<int32_t>(), n,
                                                     g.inv.as<int32_t>(), keys.as<uint64_t>());
    NTP_LAUNCH_CHECK();
    uint64_t* sorted = keys.as<uint64_t>();
    if (nnz) sort_unique(c, keys.as<uint64_t>(), alt.as<uint64_t>(), nnz, n, false, &sorted, s);
    fill_csr(c, sorted, nnz, n, out, s);
    NTP_CUDA(cudaStreamSynchronize(s));
}

}  // namespace ntp
