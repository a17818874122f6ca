// api.cu — the extern "C" boundary of libntp (include/ntp.h).
// Every entry point validates its arguments, runs inside a try/catch that maps
// internal failures to ntp_status, and records the message in the context.
#include <cstdarg>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <chrono>
#include <thread>
#include <memory>

#include "ntp_internal.cuh"

namespace ntp {

thread_local std::string g_last_global_error;

void fail(ntp_status st, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    throw Error{st, std::string(buf)};
}

// Bumped whenever any DevBuf is (re)allocated or freed: captured epoch graphs bake scratch pointers in,
// so a replay is only valid while no buffer has moved since the capture (EpochKey::alloc_gen).
static std::atomic<int64_t> g_alloc_gen{0};
int64_t alloc_generation() { return g_alloc_gen.load(); }

void DevBuf::ensure(size_t b) {
    if (b <= bytes && p) return;
    release();
    ++g_alloc_gen;
    if (b == 0) b = 16;
    cudaError_t e = cudaMalloc(&p, b);
    if (e != cudaSuccess) {
        p = nullptr;
        bytes = 0;
        cudaGetLastError();
        fail(NTP_ERR_OOM, "cudaMalloc(%zu) failed: %s", b, cudaGetErrorString(e));
    }
    bytes = b;
}

void DevBuf::release() {
    if (p) {
        cudaFree(p);
        ++g_alloc_gen;
    }
    p = nullptr;
    bytes = 0;
}

static bool valid_align(int a) { return a == 16 || a == 32 || a == 64 || a == 128; }

int32_t slice_width(int32_t w, int32_t P, ntp_dtype dt, int align) {
    const int32_t q = align / (int32_t)esize(dt);
    const int32_t base = (int32_t)cdiv(w, P);
    return (int32_t)(cdiv(base, q) * q);
}

void count_launch(ntp_ctx* c, int k) { c->launches += k; }

static void check_tensor(const ntp_tensor* t, const char* name, bool need_vec) {
    NTP_CHECK(t != nullptr, NTP_ERR_ARG, "%s is NULL", name);
    NTP_CHECK(t->data != nullptr || t->rows == 0, NTP_ERR_ARG, "%s->data is NULL", name);
    NTP_CHECK(t->dtype == NTP_F32 || t->dtype == NTP_BF16, NTP_ERR_SHAPE, "%s: bad dtype %d", name, (int)t->dtype);
    NTP_CHECK(t->rows >= 0 && t->cols >= 0 && t->ld >= t->cols, NTP_ERR_SHAPE,
              "%s: bad shape rows=%lld cols=%d ld=%lld", name, (long long)t->rows, t->cols, (long long)t->ld);
    if (need_vec) {
        const size_t es = esize(t->dtype);
        NTP_CHECK(((uintptr_t)t->data % 16) == 0, NTP_ERR_SHAPE, "%s: data not 16-byte aligned", name);
        NTP_CHECK((t->ld * es) % 16 == 0 && (t->cols * es) % 16 == 0, NTP_ERR_SHAPE,
                  "%s: cols*elem (%zu) and ld*elem (%zu) must be multiples of 16 bytes", name, t->cols * es,
                  (size_t)t->ld * es);
    }
}

static void need_graph(const ntp_ctx* c) {
    NTP_CHECK(c->g.loaded, NTP_ERR_STATE, "no graph loaded");
}

void need_comm(const ntp_ctx* c) {
    NTP_CHECK(!(c->world > 1 && (c->comm_aborted || !c->comm)), NTP_ERR_NCCL,
              "the NCCL communicator was aborted after an error or a timeout; destroy this context");
}

static void abort_comm(ntp_ctx* c) {
    if (c->comm) ncclCommAbort(c->comm);   // kernels of the aborted communicator return
    c->comm = nullptr;
    c->comm_aborted = true;
    drop_epoch_graph(c);                    // captured epochs hold its kernels
}

void wait_stream(ntp_ctx* c, cudaStream_t s) {
    if (!c->comm) {
        NTP_CUDA(cudaStreamSynchronize(s));
        return;
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (int spin = 0;; ++spin) {
        const cudaError_t e = cudaStreamQuery(s);
        if (e == cudaSuccess) return;
        if (e != cudaErrorNotReady) NTP_CUDA(e);
        ncclResult_t ar = ncclSuccess;
        if (ncclCommGetAsyncError(c->comm, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress) {
            abort_comm(c);
            cudaStreamSynchronize(s);
            fail(NTP_ERR_NCCL, "NCCL asynchronous error: %s (communicator aborted)", ncclGetErrorString(ar));
        }
        const int64_t ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
        if (c->timeout_ms > 0 && ms > c->timeout_ms) {
            abort_comm(c);
            cudaStreamSynchronize(s);
            cudaGetLastError();
            fail(NTP_ERR_TIMEOUT, "collective work did not complete within %lld ms (communicator aborted)",
                 (long long)c->timeout_ms);
        }
        if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
}

// P = world * vs feature slices: V_pad = P * ceil(n / P); this rank's vertex rows V_pad / world.
static int64_t pad_rows(const ntp_ctx* c, int64_t n) { return (int64_t)nslices(c) * cdiv(n, nslices(c)); }
static int64_t rank_rows(const ntp_ctx* c, int64_t n) { return pad_rows(c, n) / c->world; }

}  // namespace ntp

using namespace ntp;

#define NTP_API_BEGIN(ctx)                                                                  \
    if (!(ctx)) return NTP_ERR_ARG;                                                         \
    try {
#define NTP_API_END(ctx)                                                                    \
    }                                                                                       \
    catch (const ntp::Error& e) {                                                           \
        (ctx)->err = e.msg;                                                                 \
        return e.st;                                                                        \
    }                                                                                       \
    catch (const std::exception& e) {                                                       \
        (ctx)->err = e.what();                                                              \
        return NTP_ERR_CUDA;                                                                \
    }                                                                                       \
    catch (...) {                                                                           \
        (ctx)->err = "unknown internal error";                                              \
        return NTP_ERR_CUDA;                                                                \
    }                                                                                       \
    (ctx)->err.clear();                                                                     \
    return NTP_OK;

extern "C" {

int ntp_abi_version(void) { return NTP_ABI_VERSION; }

const char* ntp_status_string(ntp_status s) {
    switch (s) {
        case NTP_OK: return "NTP_OK";
        case NTP_ERR_ARG: return "NTP_ERR_ARG";
        case NTP_ERR_SHAPE: return "NTP_ERR_SHAPE";
        case NTP_ERR_CONFIG: return "NTP_ERR_CONFIG";
        case NTP_ERR_GRAPH: return "NTP_ERR_GRAPH";
        case NTP_ERR_STATE: return "NTP_ERR_STATE";
        case NTP_ERR_OOM: return "NTP_ERR_OOM";
        case NTP_ERR_CUDA: return "NTP_ERR_CUDA";
        case NTP_ERR_NCCL: return "NTP_ERR_NCCL";
        case NTP_ERR_TIMEOUT: return "NTP_ERR_TIMEOUT";
    }
    return "NTP_ERR_UNKNOWN";
}

const char* ntp_last_error(const ntp_ctx* ctx) {
    if (!ctx) return g_last_global_error.c_str();
    return ctx->err.c_str();
}

ntp_status ntp_get_unique_id(uint8_t id[128]) {
    if (!id) return NTP_ERR_ARG;
    ncclUniqueId u;
    ncclResult_t r = ncclGetUniqueId(&u);
    if (r != ncclSuccess) {
        g_last_global_error = ncclGetErrorString(r);
        return NTP_ERR_NCCL;
    }
    static_assert(sizeof(ncclUniqueId) == 128, "unexpected ncclUniqueId size");
    memcpy(id, &u, 128);
    return NTP_OK;
}

ntp_status ntp_create(ntp_ctx** out, int device, int rank, int world, const uint8_t id[128], int slice_align) {
    if (!out) return NTP_ERR_ARG;
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world || (world > 1 && !id) || !valid_align(slice_align)) {
        g_last_global_error = "ntp_create: bad rank/world/id/slice_align";
        return NTP_ERR_ARG;
    }
    std::unique_ptr<ntp_ctx> c(new ntp_ctx());
    c->device = device;
    c->rank = rank;
    c->world = world;
    c->slice_align = slice_align;
    try {
        NTP_CUDA(cudaSetDevice(device));
        NTP_CUDA(cudaStreamCreateWithFlags(&c->s_comp, cudaStreamNonBlocking));
        NTP_CUDA(cudaStreamCreateWithFlags(&c->s_comm, cudaStreamNonBlocking));
        NTP_CUDA(cudaStreamCreateWithFlags(&c->s_copy, cudaStreamNonBlocking));
        for (int i = 0; i < NTP_STAGE_SLOTS; ++i) {
            NTP_CUDA(cudaEventCreateWithFlags(&c->st_ready[i], cudaEventDisableTiming));
            NTP_CUDA(cudaEventCreateWithFlags(&c->st_free[i], cudaEventDisableTiming));
        }
        for (int i = 0; i < 2; ++i) {
            NTP_CUDA(cudaEventCreateWithFlags(&c->hs_ready[i], cudaEventDisableTiming));
            NTP_CUDA(cudaEventCreateWithFlags(&c->hs_free[i], cudaEventDisableTiming));
        }
        for (auto& e : c->ev) NTP_CUDA(cudaEventCreate(&e));
        for (auto& e : c->ov_ev) NTP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (auto& e : c->tr_ev) NTP_CUDA(cudaEventCreate(&e));
        for (auto& e : c->hop_ev) NTP_CUDA(cudaEventCreate(&e));
        if (world > 1) {
            ncclUniqueId u;
            memcpy(&u, id, 128);
            NTP_NCCL(ncclCommInitRank(&c->comm, world, u, rank));
        }
    } catch (const ntp::Error& e) {
        g_last_global_error = e.msg;
        ntp_destroy(c.release());
        return e.st;
    }
    *out = c.release();
    return NTP_OK;
}

void ntp_destroy(ntp_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    try {   // a hung collective (and a timeout set) aborts the communicator instead of blocking here
        if (c->s_comp) wait_stream(c, c->s_comp);
        if (c->s_comm) wait_stream(c, c->s_comm);
    } catch (...) {
    }
    drop_epoch_graph(c);
    p2p_shutdown(c);
    if (c->comm) ncclCommDestroy(c->comm);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : c->hop_ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : c->tr_ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : c->ov_ev)
        if (e) cudaEventDestroy(e);
    if (c->s_copy) cudaStreamSynchronize(c->s_copy);
    for (int i = 0; i < NTP_STAGE_SLOTS; ++i) {
        if (c->st_ready[i]) cudaEventDestroy(c->st_ready[i]);
        if (c->st_free[i]) cudaEventDestroy(c->st_free[i]);
    }
    for (int i = 0; i < 2; ++i) {
        if (c->hs_ready[i]) cudaEventDestroy(c->hs_ready[i]);
        if (c->hs_free[i]) cudaEventDestroy(c->hs_free[i]);
    }
    if (c->s_comp) cudaStreamDestroy(c->s_comp);
    if (c->s_comm) cudaStreamDestroy(c->s_comm);
    if (c->s_copy) cudaStreamDestroy(c->s_copy);
    delete c;   // DevBufs free themselves
}

// ------------------------------------------------------------------ graph
ntp_status ntp_load_graph(ntp_ctx* c, const int64_t* row_ptr, const int32_t* col_idx, int64_t n, int64_t nnz,
                          uint32_t flags) {
    NTP_API_BEGIN(c)
    NTP_CHECK(row_ptr && (col_idx || nnz == 0), NTP_ERR_ARG, "null CSR arrays");
    NTP_CHECK(n >= 0 && n < (int64_t(1) << 31) && nnz >= 0 && nnz < (int64_t(1) << 31), NTP_ERR_CONFIG,
              "n and nnz must be < 2^31 (n=%lld nnz=%lld)", (long long)n, (long long)nnz);
    if (flags & NTP_G_VALIDATE) {
        NTP_CHECK(row_ptr[0] == 0 && row_ptr[n] == nnz, NTP_ERR_GRAPH, "row_ptr[0] != 0 or row_ptr[n] != nnz");
        for (int64_t v = 0; v < n; ++v) {
            NTP_CHECK(row_ptr[v + 1] >= row_ptr[v], NTP_ERR_GRAPH, "row_ptr decreases at row %lld", (long long)v);
            for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) {
                NTP_CHECK(col_idx[e] >= 0 && col_idx[e] < n, NTP_ERR_GRAPH, "col out of range at %lld", (long long)e);
                NTP_CHECK(e == row_ptr[v] || col_idx[e] > col_idx[e - 1], NTP_ERR_GRAPH,
                          "row %lld not strictly ascending", (long long)v);
            }
        }
    }
    NTP_CUDA(cudaSetDevice(c->device));
    DevBuf drp, dcol, keys;
    drp.ensure((n + 1) * sizeof(int64_t));
    dcol.ensure(std::max<int64_t>(nnz, 1) * sizeof(int32_t));
    keys.ensure(std::max<int64_t>(nnz, 1) * sizeof(uint64_t));
    NTP_CUDA(cudaMemcpyAsync(drp.p, row_ptr, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, c->s_comp));
    if (nnz) NTP_CUDA(cudaMemcpyAsync(dcol.p, col_idx, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, c->s_comp));
    csr_to_keys(c, drp.as<int64_t>(), dcol.as<int32_t>(), n, keys.as<uint64_t>(), c->s_comp);
    drp.release();
    dcol.release();
    build_graph_from_keys(c, keys.as<uint64_t>(), nnz, n, (flags & NTP_G_SYMMETRIC) != 0, keys,
                          (flags & NTP_G_REORDER) != 0);
    NTP_API_END(c)
}

ntp_status ntp_build_graph(ntp_ctx* c, const int64_t* src, const int64_t* dst, int64_t m, int64_t n, uint32_t flags) {
    NTP_API_BEGIN(c)
    NTP_CHECK((src && dst) || m == 0, NTP_ERR_ARG, "null arc arrays");
    NTP_CHECK(m >= 0 && n >= 0 && n < (int64_t(1) << 31), NTP_ERR_CONFIG, "bad m/n");
    NTP_CUDA(cudaSetDevice(c->device));
    const bool sym = (flags & NTP_G_SYMMETRIC) != 0;
    const int64_t mk = sym ? 2 * m : m;
    DevBuf ds, dd, keys;
    ds.ensure(std::max<int64_t>(m, 1) * sizeof(int64_t));
    dd.ensure(std::max<int64_t>(m, 1) * sizeof(int64_t));
    keys.ensure(std::max<int64_t>(mk, 1) * sizeof(uint64_t));
    if (m) {
        NTP_CUDA(cudaMemcpyAsync(ds.p, src, m * sizeof(int64_t), cudaMemcpyHostToDevice, c->s_comp));
        NTP_CUDA(cudaMemcpyAsync(dd.p, dst, m * sizeof(int64_t), cudaMemcpyHostToDevice, c->s_comp));
        arcs_to_keys(c, ds.as<int64_t>(), dd.as<int64_t>(), m, n, sym, keys.as<uint64_t>(), c->s_comp);
    }
    NTP_CUDA(cudaStreamSynchronize(c->s_comp));
    ds.release();
    dd.release();
    build_graph_from_keys(c, keys.as<uint64_t>(), mk, n, sym, keys, (flags & NTP_G_REORDER) != 0);
    NTP_API_END(c)
}

ntp_status ntp_generate_rmat(ntp_ctx* c, int64_t n, int scale, int64_t m_raw, const uint32_t thr[3], uint64_t seed,
                             uint32_t flags) {
    NTP_API_BEGIN(c)
    NTP_CHECK(thr != nullptr, NTP_ERR_ARG, "thresholds NULL");
    NTP_CHECK(scale >= 1 && scale <= 31 && n >= 0 && n <= (int64_t(1) << scale) && m_raw >= 0, NTP_ERR_CONFIG,
              "bad scale/n/m_raw");
    NTP_CUDA(cudaSetDevice(c->device));
    const bool sym = (flags & NTP_G_SYMMETRIC) != 0;
    const int64_t mk = sym ? 2 * m_raw : m_raw;
    DevBuf keys;
    keys.ensure(std::max<int64_t>(mk, 1) * sizeof(uint64_t));
    if (m_raw) rmat_keys(c, scale, thr, seed, 0, m_raw, n, sym, keys.as<uint64_t>(), c->s_comp);
    build_graph_from_keys(c, keys.as<uint64_t>(), mk, n, sym, keys, (flags & NTP_G_REORDER) != 0);
    NTP_API_END(c)
}

ntp_status ntp_rmat_arcs(ntp_ctx* c, int scale, const uint32_t thr[3], uint64_t seed, int64_t i0, int64_t count,
                         int64_t* src_host, int64_t* dst_host) {
    NTP_API_BEGIN(c)
    NTP_CHECK(thr && src_host && dst_host && count >= 0 && i0 >= 0, NTP_ERR_ARG, "bad arguments");
    NTP_CHECK(scale >= 1 && scale <= 31, NTP_ERR_CONFIG, "bad scale");
    NTP_CUDA(cudaSetDevice(c->device));
    if (count) {
        DevBuf s, d;
        s.ensure(count * sizeof(int64_t));
        d.ensure(count * sizeof(int64_t));
        rmat_raw(c, scale, thr, seed, i0, count, s.as<int64_t>(), d.as<int64_t>(), c->s_comp);
        NTP_CUDA(cudaMemcpyAsync(src_host, s.p, count * sizeof(int64_t), cudaMemcpyDeviceToHost, c->s_comp));
        NTP_CUDA(cudaMemcpyAsync(dst_host, d.p, count * sizeof(int64_t), cudaMemcpyDeviceToHost, c->s_comp));
        NTP_CUDA(cudaStreamSynchronize(c->s_comp));
    }
    NTP_API_END(c)
}

ntp_status ntp_graph_info(const ntp_ctx* cc, int64_t* n, int64_t* nnz, int* symmetric) {
    ntp_ctx* c = const_cast<ntp_ctx*>(cc);
    NTP_API_BEGIN(c)
    need_graph(c);
    if (n) *n = c->g.n;
    if (nnz) *nnz = c->g.nnz;
    if (symmetric) *symmetric = c->g.symmetric ? 1 : 0;
    NTP_API_END(c)
}

ntp_status ntp_copy_csr(const ntp_ctx* cc, int transposed, int64_t* row_ptr, int32_t* col_idx, int32_t* deg) {
    ntp_ctx* c = const_cast<ntp_ctx*>(cc);
    NTP_API_BEGIN(c)
    need_graph(c);
    NTP_CUDA(cudaSetDevice(c->device));
    const Csr* csrp = transposed ? &c->g.bwd() : &c->g.fwd();
    Csr orig;
    if (c->g.reordered) {   // internal ids -> original ids, columns re-sorted
        export_original_csr(c, *csrp, orig);
        csrp = &orig;
    }
    const Csr& csr = *csrp;
    const int64_t n = c->g.n, nnz = c->g.nnz;
    std::vector<int32_t> rp(n + 1);
    NTP_CUDA(cudaMemcpy(rp.data(), csr.row_ptr.p, (n + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (row_ptr)
        for (int64_t i = 0; i <= n; ++i) row_ptr[i] = rp[i];
    if (deg)
        for (int64_t i = 0; i < n; ++i) deg[i] = rp[i + 1] - rp[i];
    if (col_idx && nnz) NTP_CUDA(cudaMemcpy(col_idx, csr.col.p, nnz * sizeof(int32_t), cudaMemcpyDeviceToHost));
    NTP_API_END(c)
}

ntp_status ntp_copy_dinv(const ntp_ctx* cc, float* dinv_in, float* dinv_out) {
    ntp_ctx* c = const_cast<ntp_ctx*>(cc);
    NTP_API_BEGIN(c)
    need_graph(c);
    NTP_CUDA(cudaSetDevice(c->device));
    const int64_t n = c->g.n;
    const float* di = c->g.dinv_in_orig();     // original vertex order either way
    const float* dout = c->g.dinv_out_orig();
    if (dinv_in && n) NTP_CUDA(cudaMemcpy(dinv_in, di, n * sizeof(float), cudaMemcpyDeviceToHost));
    if (dinv_out && n) NTP_CUDA(cudaMemcpy(dinv_out, dout, n * sizeof(float), cudaMemcpyDeviceToHost));
    NTP_API_END(c)
}

ntp_status ntp_set_slices(ntp_ctx* c, int32_t P) {
    NTP_API_BEGIN(c)
    need_comm(c);
    NTP_CHECK(P >= c->world && P % c->world == 0 && P <= 4096, NTP_ERR_ARG,
              "P = %d must be a multiple of world = %d (and <= 4096)", P, c->world);
    NTP_CUDA(cudaSetDevice(c->device));
    NTP_CUDA(cudaStreamSynchronize(c->s_comp));
    drop_epoch_graph(c);
    c->vs = P / c->world;
    NTP_API_END(c)
}

ntp_status ntp_set_timeout(ntp_ctx* c, int64_t ms) {
    NTP_API_BEGIN(c)
    NTP_CHECK(ms >= 0, NTP_ERR_ARG, "timeout must be >= 0 ms");
    c->timeout_ms = ms;
    NTP_API_END(c)
}

ntp_status ntp_abort(ntp_ctx* c) {
    NTP_API_BEGIN(c)
    NTP_CUDA(cudaSetDevice(c->device));
    abort_comm(c);
    NTP_API_END(c)
}

ntp_status ntp_sync(ntp_ctx* c, ntp_stream st) {
    NTP_API_BEGIN(c)
    NTP_CUDA(cudaSetDevice(c->device));
    wait_stream(c, (cudaStream_t)st);
    NTP_API_END(c)
}

ntp_status ntp_set_trace(ntp_ctx* c, int on) {
    NTP_API_BEGIN(c)
    c->trace_on = on != 0;
    c->tr_recs.clear();
    c->tr_used = 0;
    NTP_API_END(c)
}

ntp_status ntp_trace(ntp_ctx* c, ntp_trace_rec* out, int32_t max, int32_t* count) {
    NTP_API_BEGIN(c)
    NTP_CHECK(count && (out || max == 0) && max >= 0, NTP_ERR_ARG, "null output");
    NTP_CUDA(cudaSetDevice(c->device));
    *count = (int32_t)c->tr_recs.size();
    if (c->tr_used > 0) NTP_CUDA(cudaEventSynchronize(c->tr_ev[c->tr_used - 1]));
    for (int32_t i = 0; i < std::min<int32_t>(max, *count); ++i) {
        const auto& r = c->tr_recs[i];
        float b = 0.f, e = 0.f;
        NTP_CUDA(cudaEventElapsedTime(&b, c->ev[0], c->tr_ev[r.ev0]));
        NTP_CUDA(cudaEventElapsedTime(&e, c->ev[0], c->tr_ev[r.ev1]));
        out[i] = ntp_trace_rec{r.stream, r.phase, r.chunk, b, e};
    }
    NTP_API_END(c)
}

ntp_status ntp_hop_timing(ntp_ctx* c, double* ms, int32_t* launches) {
    NTP_API_BEGIN(c)
    NTP_CHECK(ms && launches, NTP_ERR_ARG, "null output");
    NTP_CUDA(cudaSetDevice(c->device));
    if (c->hop_ev_used > 0) NTP_CUDA(cudaEventSynchronize(c->hop_ev[c->hop_ev_used - 1]));
    int nh = 0;
    *ms = collect_hop_ms(c, &nh);
    *launches = nh;
    NTP_API_END(c)
}

// ------------------------------------------------------------------ partition maps
ntp_status ntp_partition(int64_t n, int32_t w, int32_t P, ntp_dtype dtype, int32_t chunks, int slice_align,
                         ntp_partition_info* out) {
    if (!out || n < 0 || w < 0 || P < 1 || chunks < 1 || (dtype != NTP_F32 && dtype != NTP_BF16) ||
        !valid_align(slice_align))
        return NTP_ERR_ARG;
    out->n = n;
    out->w = w;
    out->P = P;
    out->V_p = n > 0 ? cdiv(n, P) : 0;
    out->V_pad = out->V_p * P;
    out->elem_bytes = (int32_t)esize(dtype);
    out->d_s = slice_width(w, P, dtype, slice_align);
    out->w_pad = out->d_s * P;
    out->chunks = chunks;
    out->chunk = out->V_p > 0 ? cdiv(out->V_p, chunks) : 0;
    return NTP_OK;
}

// ------------------------------------------------------------------ features / layouts
ntp_status ntp_scatter_features(ntp_ctx* c, const void* X_host, ntp_dtype dtype, int64_t n, int32_t d,
                                ntp_layout layout, ntp_tensor* out) {
    NTP_API_BEGIN(c)
    NTP_CHECK(X_host != nullptr, NTP_ERR_ARG, "X_host NULL");
    check_tensor(out, "out", false);
    NTP_CHECK(out->dtype == dtype, NTP_ERR_SHAPE, "dtype mismatch");
    NTP_CUDA(cudaSetDevice(c->device));
    const size_t es = esize(dtype);
    const int64_t V_r = rank_rows(c, n), V_pad = pad_rows(c, n);
    if (layout == NTP_LAYOUT_VERTEX) {
        NTP_CHECK(out->rows >= V_r && out->cols >= d, NTP_ERR_SHAPE, "vertex tensor must be >= [V_p x d] = [%lld x %d]",
                  (long long)V_r, d);
        NTP_CUDA(cudaMemset2DAsync(out->data, out->ld * es, 0, out->cols * es, out->rows, c->s_comp));
        const int64_t r0 = (int64_t)c->rank * V_r;
        const int64_t nr = std::max<int64_t>(0, std::min<int64_t>(V_r, n - r0));
        if (nr > 0 && d > 0)
            NTP_CUDA(cudaMemcpy2DAsync(out->data, out->ld * es, static_cast<const char*>(X_host) + r0 * d * es, d * es,
                                       d * es, nr, cudaMemcpyHostToDevice, c->s_comp));
    } else {
        // this rank's vs slices stacked: slice j (global slice rank*vs + j) = rows [j*V_pad, (j+1)*V_pad)
        const int32_t d_s = slice_width(d, nslices(c), dtype, c->slice_align);
        NTP_CHECK(out->rows >= (int64_t)c->vs * V_pad && out->cols >= d_s, NTP_ERR_SHAPE,
                  "feature tensor must be >= [vs*V_pad x d_s] = [%lld x %d]", (long long)(c->vs * V_pad), d_s);
        NTP_CUDA(cudaMemset2DAsync(out->data, out->ld * es, 0, out->cols * es, out->rows, c->s_comp));
        for (int j = 0; j < c->vs; ++j) {
            const int32_t c0 = (c->rank * c->vs + j) * d_s;
            const int32_t nc = std::max(0, std::min(d_s, d - c0));
            if (nc > 0 && n > 0)
                NTP_CUDA(cudaMemcpy2DAsync(static_cast<char*>(out->data) + (size_t)j * V_pad * out->ld * es, out->ld * es,
                                           static_cast<const char*>(X_host) + c0 * es, d * es, nc * es, n,
                                           cudaMemcpyHostToDevice, c->s_comp));
        }
    }
    NTP_CUDA(cudaStreamSynchronize(c->s_comp));
    NTP_API_END(c)
}

ntp_status ntp_layout_v2f(ntp_ctx* c, const ntp_tensor* Hv, ntp_tensor* Hf, ntp_stream st) {
    NTP_API_BEGIN(c)
    need_comm(c);
    need_graph(c);
    check_tensor(Hv, "Hv", false);
    check_tensor(Hf, "Hf", true);
    NTP_CHECK(Hv->dtype == Hf->dtype, NTP_ERR_SHAPE, "dtype mismatch");
    const int32_t P = nslices(c);
    const int64_t V_p = rank_rows(c, c->g.n), V_pad = pad_rows(c, c->g.n);
    const int32_t d_s = slice_width(Hv->cols, P, Hv->dtype, c->slice_align);
    NTP_CHECK(Hv->rows >= V_p, NTP_ERR_SHAPE, "Hv rows %lld < V_p %lld", (long long)Hv->rows, (long long)V_p);
    NTP_CHECK(Hf->rows == (int64_t)c->vs * V_pad && Hf->cols == d_s && Hf->ld == d_s, NTP_ERR_SHAPE,
              "Hf must be dense [vs*V_pad x d_s] = [%lld x %d]", (long long)(c->vs * V_pad), d_s);
    cudaStream_t s = (cudaStream_t)st;
    const size_t es = esize(Hv->dtype);
    c->send.ensure((size_t)P * V_p * d_s * es + 16);
    pack_v2f(c, Hv->data, Hv->ld, Hv->cols, c->send.p, V_p, d_s, P, nullptr, (int64_t)c->rank * V_p, c->g.n,
             Hv->dtype, Hf->dtype, s);
    exchange_v2f(c, c->send.p, Hf->data, V_p * d_s, Hf->dtype, s);
    NTP_API_END(c)
}

ntp_status ntp_layout_f2v(ntp_ctx* c, const ntp_tensor* Hf, ntp_tensor* Hv, ntp_stream st) {
    NTP_API_BEGIN(c)
    need_comm(c);
    need_graph(c);
    check_tensor(Hf, "Hf", true);
    check_tensor(Hv, "Hv", false);
    NTP_CHECK(Hv->dtype == Hf->dtype, NTP_ERR_SHAPE, "dtype mismatch");
    const int32_t P = nslices(c);
    const int64_t V_p = rank_rows(c, c->g.n), V_pad = pad_rows(c, c->g.n);
    const int32_t d_s = slice_width(Hv->cols, P, Hv->dtype, c->slice_align);
    NTP_CHECK(Hv->rows >= V_p, NTP_ERR_SHAPE, "Hv rows < V_p");
    NTP_CHECK(Hf->rows == (int64_t)c->vs * V_pad && Hf->cols == d_s && Hf->ld == d_s, NTP_ERR_SHAPE,
              "Hf must be dense [vs*V_pad x d_s] = [%lld x %d]", (long long)(c->vs * V_pad), d_s);
    cudaStream_t s = (cudaStream_t)st;
    const size_t es = esize(Hv->dtype);
    c->recv.ensure((size_t)P * V_p * d_s * es + 16);
    exchange_f2v(c, Hf->data, c->recv.p, V_p * d_s, Hf->dtype, s);
    unpack_f2v(c, c->recv.p, V_p, d_s, P, Hv->data, Hv->ld, Hv->cols, Hf->dtype, Hv->dtype, s);
    NTP_API_END(c)
}

// ------------------------------------------------------------------ propagation
static ntp_status do_propagate(ntp_ctx* c, const ntp_tensor* H, ntp_tensor* Z, int K, float gamma, float alpha,
                               ntp_stream st, bool transposed) {
    NTP_API_BEGIN(c)
    need_graph(c);
    check_tensor(H, "H", true);
    check_tensor(Z, "Z", true);
    NTP_CHECK(H->dtype == Z->dtype && H->cols == Z->cols, NTP_ERR_SHAPE, "H/Z dtype or cols mismatch");
    NTP_CHECK(H->rows >= c->g.n && Z->rows >= c->g.n, NTP_ERR_SHAPE, "tensors need >= n rows");
    NTP_CHECK(H->data != Z->data, NTP_ERR_ARG, "Z must not alias H");
    NTP_CHECK(K >= 0, NTP_ERR_ARG, "K < 0");
    NTP_CHECK(gamma > 0.f && gamma <= 1.f, NTP_ERR_ARG, "gamma must be in (0, 1]");
    NTP_CHECK(alpha >= 0.f && alpha < 1.f, NTP_ERR_ARG, "alpha must be in [0, 1)");
    NTP_CUDA(cudaSetDevice(c->device));
    cudaStream_t s = (cudaStream_t)st;
    PropArgs a{};
    a.H = H->data;
    a.Z = Z->data;
    a.ld_h = H->ld;
    a.ld_z = Z->ld;
    a.cols = H->cols;
    a.dtype = H->dtype;
    a.K = K;
    a.gamma = gamma;
    a.alpha = alpha;
    a.transposed = transposed;
    const size_t es = esize(H->dtype);
    if (Z->rows > c->g.n)
        NTP_CUDA(cudaMemset2DAsync(static_cast<char*>(Z->data) + c->g.n * Z->ld * es, Z->ld * es, 0, Z->cols * es,
                                   Z->rows - c->g.n, s));
    c->hop_ev_used = 0;
    if (H->cols > 0) propagate(c, a, s, /*time_hops*/ true);
    NTP_API_END(c)
}

ntp_status ntp_propagate_fwd(ntp_ctx* c, const ntp_tensor* H, ntp_tensor* Z, int K, float gamma, float alpha,
                             ntp_stream s) {
    return do_propagate(c, H, Z, K, gamma, alpha, s, false);
}

ntp_status ntp_propagate_bwd(ntp_ctx* c, const ntp_tensor* G, ntp_tensor* dH, int K, float gamma, float alpha,
                             ntp_stream s) {
    return do_propagate(c, G, dH, K, gamma, alpha, s, true);
}

ntp_status ntp_propagate_pipeline(ntp_ctx* c, const ntp_tensor* Hv, ntp_tensor* Zv, int K, float gamma, float alpha,
                                  int transposed, ntp_dtype dt, int32_t chunks, uint32_t flags, ntp_stream st) {
    NTP_API_BEGIN(c)
    need_comm(c);
    need_graph(c);
    check_tensor(Hv, "Hv", false);
    check_tensor(Zv, "Zv", false);
    NTP_CHECK(Hv->dtype == NTP_F32 && Zv->dtype == NTP_F32, NTP_ERR_SHAPE, "Hv, Zv must be fp32");
    NTP_CHECK(dt == NTP_F32 || dt == NTP_BF16, NTP_ERR_ARG, "bad storage dtype");
    const int64_t V_p = rank_rows(c, c->g.n);
    NTP_CHECK(Hv->rows >= V_p && Zv->rows >= V_p && Hv->cols == Zv->cols && Hv->cols > 0, NTP_ERR_SHAPE,
              "Hv, Zv must be [>= V_p x w], same w");
    NTP_CHECK(Hv->data != Zv->data, NTP_ERR_ARG, "Zv must not alias Hv");
    NTP_CHECK(K >= 1, NTP_ERR_ARG, "K >= 1");
    NTP_CHECK(gamma > 0.f && gamma <= 1.f && alpha >= 0.f && alpha < 1.f, NTP_ERR_ARG, "gamma in (0,1], alpha in [0,1)");
    NTP_CHECK(chunks >= 1, NTP_ERR_ARG, "chunks >= 1");
    NTP_CUDA(cudaSetDevice(c->device));
    propagate_pipeline(c, Hv, Zv, K, gamma, alpha, transposed != 0, dt, chunks, (flags & NTP_M_OVERLAP) != 0,
                       (cudaStream_t)st);
    NTP_API_END(c)
}

// ------------------------------------------------------------------ MLP GEMM
ntp_status ntp_gemm_f32(ntp_ctx* c, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, int trans_a,
                        const float* B, int64_t ldb, int trans_b, float* C, int64_t ldc, int epilogue,
                        ntp_stream st) {
    NTP_API_BEGIN(c)
    NTP_CHECK(A && B && C, NTP_ERR_ARG, "null operand");
    NTP_CHECK(M >= 0 && N >= 0 && K > 0 && M < (int64_t(1) << 31) && N <= 65535 * 256, NTP_ERR_ARG, "bad sizes");
    NTP_CHECK(epilogue == 0 || epilogue == 1, NTP_ERR_ARG, "epilogue must be 0 or 1");
    NTP_CHECK(ldc >= N, NTP_ERR_SHAPE, "ldc < N");
    NTP_CUDA(cudaSetDevice(c->device));
    gemm_tf32x3(c, M, N, K, A, lda, trans_a != 0, B, ldb, trans_b == 0, C, ldc, epilogue, nullptr, 0,
                (cudaStream_t)st);
    NTP_API_END(c)
}

// ------------------------------------------------------------------ epoch
ntp_status ntp_train_epoch(ntp_ctx* c, const ntp_model* m, const ntp_tensor* X_v, const int32_t* labels_v,
                           const uint8_t* train_mask_v, ntp_tensor* W0, ntp_tensor* W1, ntp_epoch_report* rep,
                           ntp_stream st) {
    NTP_API_BEGIN(c)
    need_comm(c);
    need_graph(c);
    NTP_CHECK(m && X_v && labels_v && train_mask_v && W0 && W1, NTP_ERR_ARG, "null argument");
    NTP_CHECK(m->d_in > 0 && m->hid > 0 && m->C > 0 && m->K >= 1, NTP_ERR_ARG, "bad model dims / K");
    NTP_CHECK(m->gamma > 0.f && m->gamma <= 1.f && m->alpha >= 0.f && m->alpha < 1.f, NTP_ERR_ARG,
              "gamma in (0,1], alpha in [0,1)");
    NTP_CHECK(m->dtype == NTP_F32 || m->dtype == NTP_BF16, NTP_ERR_ARG, "bad dtype");
    NTP_CHECK(X_v->dtype == NTP_F32 && W0->dtype == NTP_F32 && W1->dtype == NTP_F32, NTP_ERR_SHAPE,
              "X_v, W0, W1 must be fp32");
    const int64_t V_p = rank_rows(c, c->g.n);
    NTP_CHECK(X_v->rows >= V_p && X_v->cols == m->d_in && X_v->ld >= m->d_in, NTP_ERR_SHAPE, "X_v must be [V_p x d_in]");
    NTP_CHECK(W0->rows == m->d_in && W0->cols == m->hid && W0->ld == m->hid, NTP_ERR_SHAPE,
              "W0 must be dense [d_in x hid]");
    NTP_CHECK(W1->rows == m->hid && W1->cols == m->C && W1->ld == m->C, NTP_ERR_SHAPE, "W1 must be dense [hid x C]");
    NTP_CHECK(m->C <= 256, NTP_ERR_CONFIG, "C = %d > 256 classes is not supported", m->C);
    if (m->flags & NTP_M_STAGED) {
        const int slot = (int)((m->flags >> NTP_M_SLOT_SHIFT) & NTP_M_SLOT_MASK);
        NTP_CHECK(slot < NTP_STAGE_SLOTS, NTP_ERR_ARG, "staging slot %d out of range (0..%d)", slot,
                  NTP_STAGE_SLOTS - 1);
        NTP_CHECK(c->st_rows[slot] == V_p && c->st_d_in[slot] == m->d_in, NTP_ERR_STATE,
                  "staging slot %d holds no inputs of shape [%lld x %d] (ntp_stage_inputs first)", slot, (long long)V_p,
                  m->d_in);
    }
    if (m->flags & NTP_M_HOST_STREAM)
        NTP_CHECK((m->flags & NTP_M_W1_AFTER_PROP) && !(m->flags & (NTP_M_STAGED | NTP_M_HOST_INPUTS | NTP_M_DATA_PARALLEL)),
                  NTP_ERR_CONFIG, "NTP_M_HOST_STREAM: W1-after-propagation epochs with device labels/mask only");
    if ((m->flags & NTP_M_OVERLAP) && (m->flags & NTP_M_W1_AFTER_PROP) && c->world > 1) {
        const int64_t nch = cdiv(V_p, epoch_row_chunk(m, V_p));   // 4 layout changes x 2 events per row chunk
        NTP_CHECK(8 * nch <= kOvEvents, NTP_ERR_CONFIG, "too many overlap chunks (%lld > %d)", (long long)nch,
                  kOvEvents / 8);
    }
    NTP_CUDA(cudaSetDevice(c->device));
    train_epoch(c, m, X_v, labels_v, train_mask_v, W0, W1, rep, (cudaStream_t)st);
    NTP_API_END(c)
}

ntp_status ntp_train_epoch_gat(ntp_ctx* c, const ntp_model* m, const ntp_tensor* X_v, const int32_t* labels_v,
                               const uint8_t* train_mask_v, ntp_tensor* W0, ntp_tensor* W1, ntp_tensor* att, float slope,
                               ntp_epoch_report* rep, ntp_stream st) {
    NTP_API_BEGIN(c)
    need_comm(c);
    need_graph(c);
    NTP_CHECK(m && X_v && labels_v && train_mask_v && W0 && W1 && att, NTP_ERR_ARG, "null argument");
    NTP_CHECK(m->d_in > 0 && m->hid > 0 && m->C > 0 && m->K >= 1, NTP_ERR_ARG, "bad model dims / K");
    NTP_CHECK(m->gamma > 0.f && m->gamma <= 1.f, NTP_ERR_ARG, "gamma in (0,1]");
    NTP_CHECK(m->alpha == 0.f, NTP_ERR_CONFIG, "the GAT epoch has no alpha mix (reading G3): alpha must be 0");
    NTP_CHECK(m->dtype == NTP_F32 || m->dtype == NTP_BF16, NTP_ERR_ARG, "bad dtype");
    NTP_CHECK(m->flags == 0, NTP_ERR_CONFIG, "the GAT epoch takes no epoch flags (device inputs, W1 before propagation)");
    NTP_CHECK(m->C <= 256, NTP_ERR_CONFIG, "C = %d > 256 classes is not supported", m->C);
    NTP_CHECK(slope >= 0.f && slope < 1.f, NTP_ERR_ARG, "LeakyReLU slope in [0, 1)");
    NTP_CHECK(X_v->dtype == NTP_F32 && W0->dtype == NTP_F32 && W1->dtype == NTP_F32 && att->dtype == NTP_F32,
              NTP_ERR_SHAPE, "X_v, W0, W1, att must be fp32");
    const int64_t V_p = rank_rows(c, c->g.n);
    NTP_CHECK(X_v->rows >= V_p && X_v->cols == m->d_in && X_v->ld >= m->d_in, NTP_ERR_SHAPE, "X_v must be [V_p x d_in]");
    NTP_CHECK(W0->rows == m->d_in && W0->cols == m->hid && W0->ld == m->hid, NTP_ERR_SHAPE, "W0 must be dense [d_in x hid]");
    NTP_CHECK(W1->rows == m->hid && W1->cols == m->C && W1->ld == m->C, NTP_ERR_SHAPE, "W1 must be dense [hid x C]");
    NTP_CHECK(att->rows == 2 && att->cols == m->C && att->ld == m->C, NTP_ERR_SHAPE, "att must be dense [2 x C]");
    NTP_CUDA(cudaSetDevice(c->device));
    train_epoch_gat(c, m, X_v, labels_v, train_mask_v, W0, W1, att, slope, rep, (cudaStream_t)st);
    NTP_API_END(c)
}

ntp_status ntp_stage_inputs(ntp_ctx* c, int slot, const float* X_host, int64_t rows, int32_t d_in, int64_t ldx,
                            const int32_t* labels_host, const uint8_t* train_mask_host) {
    NTP_API_BEGIN(c)
    need_graph(c);
    NTP_CHECK(X_host && labels_host && train_mask_host, NTP_ERR_ARG, "null argument");
    NTP_CHECK(slot >= 0 && slot < NTP_STAGE_SLOTS, NTP_ERR_ARG, "slot must be in 0..%d", NTP_STAGE_SLOTS - 1);
    NTP_CHECK(d_in > 0 && ldx >= d_in && rows == rank_rows(c, c->g.n), NTP_ERR_SHAPE, "X_host must be [V_p x d_in]");
    NTP_CUDA(cudaSetDevice(c->device));
    stage_inputs(c, slot, X_host, rows, d_in, ldx, labels_host, train_mask_host);
    NTP_API_END(c)
}

ntp_status ntp_train_epoch_coupled(ntp_ctx* c, const ntp_coupled_model* m, const ntp_tensor* X_v,
                                   const int32_t* labels_v, const uint8_t* train_mask_v, ntp_tensor* const* W,
                                   ntp_coupled_report* rep, ntp_stream st) {
    NTP_API_BEGIN(c)
    need_comm(c);
    need_graph(c);
    NTP_CHECK(m && X_v && labels_v && train_mask_v && W, NTP_ERR_ARG, "null argument");
    NTP_CHECK(m->L >= 1 && m->L <= NTP_MAX_LAYERS, NTP_ERR_ARG, "L must be in [1, %d]", NTP_MAX_LAYERS);
    for (int l = 0; l <= m->L; ++l) NTP_CHECK(m->widths[l] > 0, NTP_ERR_ARG, "widths must be positive");
    NTP_CHECK(m->widths[m->L] <= 256, NTP_ERR_CONFIG, "C > 256 classes is not supported");
    NTP_CHECK(m->dtype == NTP_F32 || m->dtype == NTP_BF16, NTP_ERR_ARG, "bad dtype");
    NTP_CHECK(c->vs == 1, NTP_ERR_CONFIG, "the coupled epoch runs one slice per rank (no virtual slices)");
    const int64_t V_p = cdiv(c->g.n, c->world);
    NTP_CHECK(X_v->dtype == NTP_F32 && X_v->rows >= V_p && X_v->cols == m->widths[0] && X_v->ld >= m->widths[0],
              NTP_ERR_SHAPE, "X_v must be fp32 [V_p x d_in]");
    for (int l = 0; l < m->L; ++l) {
        NTP_CHECK(W[l] != nullptr, NTP_ERR_ARG, "null weight");
        NTP_CHECK(W[l]->dtype == NTP_F32 && W[l]->rows == m->widths[l] && W[l]->cols == m->widths[l + 1] &&
                      W[l]->ld == m->widths[l + 1],
                  NTP_ERR_SHAPE, "W[%d] must be dense fp32 [%d x %d]", l, m->widths[l], m->widths[l + 1]);
    }
    NTP_CUDA(cudaSetDevice(c->device));
    train_epoch_coupled(c, m, X_v, labels_v, train_mask_v, W, rep, (cudaStream_t)st);
    NTP_API_END(c)
}

}  // extern "C"
