// ntp_internal.cuh — internal declarations of libntp (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <nccl.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "ntp.h"

namespace ntp {

// ---------------------------------------------------------------- errors
struct Error {
    ntp_status st;
    std::string msg;
};

[[noreturn]] void fail(ntp_status st, const char* fmt, ...);

#define NTP_CUDA(expr)                                                                     \
    do {                                                                                   \
        cudaError_t _e = (expr);                                                           \
        if (_e != cudaSuccess)                                                             \
            ::ntp::fail(_e == cudaErrorMemoryAllocation ? NTP_ERR_OOM : NTP_ERR_CUDA,      \
                        "%s:%d %s -> %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
    } while (0)

#define NTP_NCCL(expr)                                                                     \
    do {                                                                                   \
        ncclResult_t _r = (expr);                                                          \
        if (_r != ncclSuccess)                                                             \
            ::ntp::fail(NTP_ERR_NCCL, "%s:%d %s -> %s", __FILE__, __LINE__, #expr,         \
                        ncclGetErrorString(_r));                                           \
    } while (0)

#define NTP_CHECK(cond, st, ...)                                                           \
    do {                                                                                   \
        if (!(cond)) ::ntp::fail((st), __VA_ARGS__);                                       \
    } while (0)

#define NTP_LAUNCH_CHECK() NTP_CUDA(cudaGetLastError())

// ------------------------------------------------------------- device buffer
int64_t alloc_generation();        // bumped by every DevBuf (re)allocation / free

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void ensure(size_t b);          // grow-only (contents not preserved)
    void release();
    template <class T> T* as() const { return static_cast<T*>(p); }
    ~DevBuf() { release(); }
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

// ---------------------------------------------------------------- graph
// One CSR orientation plus its merge-path work partition.
// Merge path (rows + nnz items): unit u covers diagonals [u*T, (u+1)*T);
// unit_row[u] = row-ends consumed before the unit, unit_e[u] = edges consumed.
struct Csr {
    DevBuf row_ptr;                 // int32 [n+1]
    DevBuf col;                     // int32 [nnz]
    DevBuf unit_row;                // int32 [U+1]
    DevBuf unit_e;                  // int32 [U+1]
    std::vector<int32_t> h_unit_row; // host copy (row-range restriction of launches)
    int64_t U = 0;
    void reset() {
        row_ptr.release(); col.release(); unit_row.release(); unit_e.release();
        h_unit_row.clear(); U = 0;
    }
};

struct Graph {
    int64_t n = 0, nnz = 0;
    bool symmetric = false;
    bool loaded = false;
    int32_t unit_items = 2048;      // T, a graph-level constant (P-invariant schedule)
    Csr in;                         // rows = destinations (A^)
    Csr out;                        // rows = sources (A^T); unused if symmetric
    DevBuf dinv_in, dinv_out;       // fp32 [n]
    // NTP_G_REORDER: the CSRs and D~^{-1/2} use internal ids (descending total degree); slices
    // handed across the ABI stay in original vertex order (perm: original -> internal, inv:
    // internal -> original; the first hop gathers through inv, the last hop scatters through it).
    bool reordered = false;
    DevBuf perm, inv;               // int32 [n]
    DevBuf dinv_orig;               // fp32 [2n]: D~_in^{-1/2}, D~_out^{-1/2} in ORIGINAL order (reordered only)
    void reset() {
        n = nnz = 0; symmetric = false; loaded = false; unit_items = 2048; reordered = false;
        in.reset(); out.reset(); dinv_in.release(); dinv_out.release(); perm.release(); inv.release();
        dinv_orig.release();
    }
    const int32_t* inv_p() const { return reordered ? inv.as<int32_t>() : nullptr; }
    // per-vertex scales indexed by ORIGINAL vertex id (what the layout kernels use)
    const float* dinv_in_orig() const { return reordered ? dinv_orig.as<float>() : dinv_in_p(); }
    const float* dinv_out_orig() const { return reordered ? dinv_orig.as<float>() + n : dinv_out_p(); }
    const Csr& fwd() const { return in; }
    const Csr& bwd() const { return symmetric ? in : out; }
    const float* dinv_in_p() const { return dinv_in.as<float>(); }
    const float* dinv_out_p() const { return symmetric ? dinv_in.as<float>() : dinv_out.as<float>(); }
};

}  // namespace ntp

// Pack epilogue of the MLP forward GEMM (W1 after propagation): H1 = ReLU(X W0) never reaches HBM in fp32;
// its ReLU' mask words (bits[v][nwb]) and the row-scaled bf16 blocks of the split are written instead.
namespace ntp {
struct PackEpi {
    __nv_bfloat16* out;        // send buffer [P][V_p][d_s] (bf16)
    int64_t V_p;
    int d_s;
    const float* scale;        // D~_out^{-1/2}, original vertex order
    int64_t row0, n;           // this rank's first vertex, graph size
    uint32_t* bits;            // [V_p][nwb]
    int nwb;
    int64_t roff;              // GEMM row 0 = vertex row roff of this rank (row chunk)
    const int32_t* perm;       // one GPU, reordered graph: slice row of vertex v = perm[v] (internal order)
};
}  // namespace ntp
// ---------------------------------------------------------------- context
// Everything a captured epoch graph bakes in.
struct EpochKey {
    ntp_model m;
    const void* ptrs[5];
    int64_t ld;
    int64_t graph_version;
    int64_t head_chunk;     // NTP_HEAD_CHUNK (row chunk of the W1-after-propagation epoch)
    int64_t head_fused;     // NTP_HEAD_FUSED (fused tcgen05 head on/off)
    bool operator==(const EpochKey& o) const {
        return std::memcmp(&m, &o.m, sizeof(m)) == 0 && std::memcmp(ptrs, o.ptrs, sizeof(ptrs)) == 0 && ld == o.ld &&
               graph_version == o.graph_version && head_chunk == o.head_chunk && head_fused == o.head_fused;
    }
};

constexpr int kTrEvents = 1024;   // overlap trace events per epoch

struct ntp_ctx {
    int device = 0, rank = 0, world = 1, slice_align = 16;
    int vs = 1;                     // virtual feature slices per rank (ntp_set_slices): P = world * vs
    int64_t timeout_ms = 0;         // collective deadline of the synchronising calls (ntp_set_timeout), 0 = none
    uint32_t ce_seq = 0;            // epoch sequence number of the copy-engine layout flags
    bool comm_aborted = false;      // the communicator was aborted after an error or a timeout
    ncclComm_t comm = nullptr;
    cudaStream_t s_comp = nullptr, s_comm = nullptr;
    ntp::Graph g;
    // scratch
    ntp::DevBuf carry, carry2, prop_tmp, prop_s0, send, recv, xfer;
    // decoupled GAT (gat.cu): score halves, coefficients (+ out-CSR order), their gradients, level stack
    ntp::DevBuf gat_fg, gat_msum, gat_alpha, gat_alpha_t, gat_pspd, gat_perm, gat_Z, gat_X, gat_da, gat_big;
    int32_t gat_nbig[2] = {0, 0};   // hub rows (in-CSR, out-CSR) listed in gat_big
    int64_t gat_perm_version = -1, gat_big_version = -1;
    ntp::DevBuf m_A, m_H1, m_L, m_dL, m_dH1, m_dW, m_scal, m_part, m_Xs, m_lab, m_mask;
    ntp::DevBuf m_gemm_part, m_W0p, m_W1p, m_Xh, m_Wsplit, m_bits, m_dWp, m_head, m_wgrad;
    // coupled (naive TP) epoch: Z^l, H^l per layer, dA / dZ scratch, padded weights
    ntp::DevBuf cp_Z[NTP_MAX_LAYERS + 1], cp_H[NTP_MAX_LAYERS + 1], cp_A, cp_B, cp_W;
    // input staging slots (ntp_stage_inputs): X [V_p x round4(d_in)], raw host-pitch copy, labels, mask
    ntp::DevBuf st_X[NTP_STAGE_SLOTS], st_raw[NTP_STAGE_SLOTS], st_y[NTP_STAGE_SLOTS], st_m[NTP_STAGE_SLOTS];
    cudaStream_t s_copy = nullptr;
    cudaEvent_t st_ready[NTP_STAGE_SLOTS] = {}, st_free[NTP_STAGE_SLOTS] = {};
    // NTP_M_HOST_STREAM: X_v stays in (pinned) host memory; row chunks stream through a 2-slot device ring
    ntp::DevBuf hs_ring;
    cudaEvent_t hs_ready[2] = {}, hs_free[2] = {};
    bool hs_used[2] = {false, false};
    bool st_free_rec[NTP_STAGE_SLOTS] = {};
    int64_t st_rows[NTP_STAGE_SLOTS] = {}, st_ld[NTP_STAGE_SLOTS] = {};
    int32_t st_d_in[NTP_STAGE_SLOTS] = {};
    // peer-direct layouts (CUDA IPC windows over NVLink), see layout.cu
    int p2p_state = 0;                      // 0 not set up, 1 usable, -1 unavailable
    ntp::DevBuf p2p_split, p2p_gath;        // this rank's windows (zero-initialised)
    size_t p2p_split_bytes = 0, p2p_gath_bytes = 0;
    size_t p2p_used_sb = 0, p2p_used_gb = 0;   // layout the windows currently hold (cleared on change)
    std::vector<void*> p2p_peer_split, p2p_peer_gath;   // opened peer mappings (own entry = local)
    ntp::DevBuf p2p_tab;                    // device: [2][P] pointers (split windows, gather windows)
    ntp::DevBuf p2p_bar;                    // one int for the barrier allreduce
    cudaEvent_t ev[64] = {};
    cudaEvent_t ov_ev[256] = {};    // fork/join events of the chunked layout exchanges (a12)
    // overlap trace (ntp_set_trace): timed events at chunk begin / end on both streams
    bool trace_on = false;
    cudaEvent_t tr_ev[kTrEvents] = {};
    int tr_used = 0;
    struct TraceRec { int stream, phase, chunk, ev0, ev1; };
    std::vector<TraceRec> tr_recs;
    ntp::PackEpi pack_epi{};        // parameters of the next pack-epilogue GEMM launch
    cudaEvent_t hop_ev[512] = {};   // start/stop pairs around SpMM hop launches (timed epochs)
    int hop_ev_used = 0;
    int64_t launches = 0;
    std::string err;
    // captured epoch (CUDA graph)
    int64_t g_version = 0;          // bumped whenever the graph (CSR) is rebuilt
    EpochKey graph_key{};
    bool graph_warm = false, graph_valid = false;
    cudaGraphExec_t graph_exec = nullptr;
    // captured staged epochs, one per input slot (NTP_M_STAGED; the slot's buffers are baked in)
    EpochKey sg_key[NTP_STAGE_SLOTS]{};
    bool sg_warm[NTP_STAGE_SLOTS] = {}, sg_valid[NTP_STAGE_SLOTS] = {};
    cudaGraphExec_t sg_exec[NTP_STAGE_SLOTS] = {};
    int sg_hops[NTP_STAGE_SLOTS] = {};
    int64_t sg_launches[NTP_STAGE_SLOTS] = {};
    int64_t graph_gen = -1, sg_gen[NTP_STAGE_SLOTS] = {-1, -1, -1};   // alloc_generation() at capture
    int64_t graph_wire[8] = {}, sg_wire[NTP_STAGE_SLOTS][8] = {};  // wire bytes counted while recording (replays reuse them)
    // bytes handed to the transport (NCCL send/recv, all-gather, peer stores) per layout change of the
    // current epoch: 0 v2f fwd, 1 f2v fwd, 2 v2f bwd, 3 f2v bwd (wire_phase selects the entry)
    int64_t wire_sent[4] = {}, wire_recv[4] = {};
    int wire_phase = 0;
    bool capturing = false;         // timing events become external event nodes while capturing
    int graph_hops = 0;
    int64_t graph_launches = 0;
};

namespace ntp {

// -------------------------------------------------------------- internal API
void build_graph_from_keys(ntp_ctx* c, uint64_t* keys, int64_t m, int64_t n, bool symmetric,
                           DevBuf& keybuf_owner, bool reorder = false);
void export_original_csr(ntp_ctx* c, const Csr& csr, Csr& out);
void rmat_keys(ntp_ctx* c, int scale, const uint32_t thr[3], uint64_t seed, int64_t i0, int64_t count,
               int64_t n, bool symmetric, uint64_t* keys, cudaStream_t s);
void rmat_raw(ntp_ctx* c, int scale, const uint32_t thr[3], uint64_t seed, int64_t i0, int64_t count,
              int64_t* src, int64_t* dst, cudaStream_t s);

// Propagation on one feature slice (dtype-generic storage, fp32 accumulation).
// Peer-direct output of a layout-changing producer (P2P stores over NVLink into the peers' IPC
// windows): row v of the global order goes to rank q = v / V_p, into block `rank` of q's
// [P][V_p][d_s] window, i.e. element offset (rank * V_p + v - q * V_p) * ld.  tab == nullptr:
// ordinary local output.
struct PeerOut {
    void* const* tab = nullptr;   // device array [P] of window base pointers (own = local)
    int64_t V_p = 0;
    int rank = 0;
};
struct PropArgs {
    const void* H;          // [n x cols] original input (alpha term)
    void* Z;                // output
    int64_t ld_h, ld_z;     // elements
    int32_t cols;           // elements per row (cols*esize % 16 == 0)
    ntp_dtype dtype;
    int K;
    float gamma, alpha;
    bool transposed;        // backward (A^T)
    PeerOut po;             // last hop: write straight into the peers' gather windows (f2v fused)
};
// State needed to run the last hop later, chunk by chunk (overlap scheduler, a12).
struct LastHop {
    const Csr* csr;
    const float* rs;
    const float* cs;
    const void* sin;
    int64_t ld_sin;
    const void* S0;
    int64_t ld_s0;
    void* out;
    int64_t ld_out;
    int32_t cols;
    ntp_dtype dt;
    float gamma, alpha;
};
// time_hops: record an event pair around every hop launch into c->hop_ev (read after a
// sync with collect_hop_ms).  defer_last: run hops 1..K-1 only and describe hop K.
void propagate(ntp_ctx* c, const PropArgs& a, cudaStream_t s, bool time_hops = false,
               bool prescaled_input = false, LastHop* defer_last = nullptr);
void run_last_hop(ntp_ctx* c, const LastHop& lh, int64_t row_lo, int64_t row_hi, cudaStream_t s, bool time_hops);
// Pre-scaled input that may be consumed (alpha == 0: S^0 is dead after hop 1): the hops ping-pong
// between a.H and a.Z (same ld) with no scratch slice; returns the buffer holding Z^K (a.H or a.Z).
// alpha != 0 falls back to propagate() (S^0 must live through every hop) and returns a.Z.
// input_internal: a.H already holds S^0 in the graph's internal vertex order (the producer scattered it)
void* propagate_consume(ntp_ctx* c, const PropArgs& a, cudaStream_t s, bool time_hops, bool input_internal = false);
double collect_hop_ms(ntp_ctx* c, int* n_hops);
void propagate_pipeline(ntp_ctx* c, const ntp_tensor* Hv, ntp_tensor* Zv, int K, float gamma, float alpha,
                        bool transposed, ntp_dtype dt, int chunks, bool overlap, cudaStream_t user);
void train_epoch(ntp_ctx* c, const ntp_model* m, const ntp_tensor* X_v, const int32_t* labels_v,
                 const uint8_t* mask_v, ntp_tensor* W0, ntp_tensor* W1, ntp_epoch_report* rep, cudaStream_t user);
void drop_epoch_graph(ntp_ctx* c);
// Waits for stream s under the collective contract (the analogue of SPEC S:407's round
// timeout): polls the stream and ncclCommGetAsyncError; on an NCCL error or after c->timeout_ms it aborts
// the communicator (ncclCommAbort) and fails with NTP_ERR_NCCL / NTP_ERR_TIMEOUT.
void wait_stream(ntp_ctx* c, cudaStream_t s);
void need_comm(const ntp_ctx* c);   // NTP_ERR_NCCL once the communicator has been aborted
// epoch building blocks (model.cu), shared with the GAT epoch (gat.cu)
void epoch_phases(cudaEvent_t* E, double* ms);
void epoch_gemm(ntp_ctx* c, bool ta, bool tb, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                const float* B, int64_t ldb, float* C, int64_t ldc, cudaStream_t s, int epi, const float* aux,
                int64_t ldaux, const float* B_hi, const float* B_lo);
int64_t epoch_loss(ntp_ctx* c, const void* in, ntp_dtype tin, int in_blocked, int64_t V_p, int32_t d_s, int32_t C,
                   const int32_t* y, const uint8_t* mask, int64_t row0, int64_t n, void* out, ntp_dtype tout,
                   int out_blocked, const float* gscale, double* part, int64_t* cnt, int64_t ld_plain, cudaStream_t s);
void epoch_zero_pad_cols(ntp_ctx* c, void* buf, ntp_dtype dt, int64_t V_p, int32_t d_s, int32_t P, int32_t C,
                         cudaStream_t s);
void epoch_reduce_loss(ntp_ctx* c, const double* part, const int64_t* cnt, int64_t nb, double* scal, cudaStream_t s);
void epoch_sgd(ntp_ctx* c, float* W, int64_t n, const float* dW, const double* scal, float lr, cudaStream_t s);
void train_epoch_gat(ntp_ctx* c, const ntp_model* m, const ntp_tensor* X_v, const int32_t* labels_v,
                     const uint8_t* mask_v, ntp_tensor* W0, ntp_tensor* W1, ntp_tensor* att, float slope,
                     ntp_epoch_report* rep, cudaStream_t user);
int64_t epoch_row_chunk(const ntp_model* m, int64_t V_p);
constexpr int kMaxLayers = NTP_MAX_LAYERS;
constexpr int kOvEvents = 256;
constexpr int kHopEvents = 512;
void stage_inputs(ntp_ctx* c, int slot, const float* X, int64_t rows, int32_t d_in, int64_t ldx, const int32_t* y,
                  const uint8_t* m);
void train_epoch_coupled(ntp_ctx* c, const ntp_coupled_model* m, const ntp_tensor* X_v, const int32_t* labels_v,
                         const uint8_t* mask_v, ntp_tensor* const* W, ntp_coupled_report* rep, cudaStream_t user);
void arcs_to_keys(ntp_ctx* c, const int64_t* src, const int64_t* dst, int64_t m, int64_t n, bool sym,
                  uint64_t* keys, cudaStream_t s);
void csr_to_keys(ntp_ctx* c, const int64_t* row_ptr, const int32_t* col, int64_t n, uint64_t* keys,
                 cudaStream_t s);

// One hop over rows [row_lo, row_hi) (all rows if row_hi < 0).
// mode 0: intermediate (pre-scaled output), 1: last (unscaled output Z^K).
void spmm_hop(ntp_ctx* c, const Csr& csr, const float* rs, const float* cs, const void* S_in,
              void* S_out, const void* H, int64_t ld_in, int64_t ld_out, int64_t ld_h, int32_t cols,
              ntp_dtype dt, float gamma, float alpha, int mode, int64_t row_lo, int64_t row_hi,
              cudaStream_t s, const int32_t* out_rows = nullptr, const PeerOut* po = nullptr,
              const float* ew = nullptr, const float* sw = nullptr,    // weighted hop (GAT): arc / self coefficients
              void* S_out2 = nullptr, float slope2 = 0.f);             // dual weighted hop: second output (below)
// S[r] = scale[r] * H[src_rows ? src_rows[r] : r] (scale may be null: plain copy / permutation)
void prescale(ntp_ctx* c, const void* H, int64_t ld_h, void* S, int64_t ld_s, int32_t cols,
              const float* scale, int64_t rows, ntp_dtype dt, cudaStream_t s,
              const int32_t* src_rows = nullptr);

// layouts
void pack_v2f(ntp_ctx* c, const void* Hv, int64_t ld_v, int32_t w, void* send, int64_t V_p,
              int32_t d_s, int32_t P, const float* row_scale, int64_t row0, int64_t n,
              ntp_dtype dt_in, ntp_dtype dt_out, cudaStream_t s, void* const* peer_tab = nullptr,
              int64_t rows = -1, int64_t vofs = 0, uint32_t* bits = nullptr, int32_t nw = 0);
// Peer-direct layouts: IPC windows of this rank ([P][V_p][d_s] split target and gather target),
// exchanged once per size (collective); false when P2P is unavailable (NCCL all-to-all path).
bool p2p_ensure(ntp_ctx* c, size_t split_bytes, size_t gather_bytes, cudaStream_t s);
// Copy-engine layout changes (a12, W1 after propagation): completion flags at the tail of every gather
// window, kCeFlagBytes long: flag (phase, source rank, chunk) of rank q's window = q's inbox.
constexpr int kCeRanks = 64, kCeChunks = 64;
constexpr size_t kCeFlagBytes = (size_t)4 * kCeRanks * kCeChunks * sizeof(uint32_t);
inline size_t ce_flag_slot(int phase, int src, int ch) { return ((size_t)phase * kCeRanks + src) * kCeChunks + ch; }
uint32_t* ce_flags(ntp_ctx* c, int q);                 // rank q's inbox (own: local; else the opened IPC window)
void stream_write_u32(cudaStream_t s, void* addr, uint32_t v);     // cuStreamWriteValue32 (with its memory fence)
void stream_wait_u32_geq(cudaStream_t s, void* addr, uint32_t v);  // cuStreamWaitValue32, GEQ (+ remote-write flush)
void p2p_barrier(ntp_ctx* c, cudaStream_t s);   // stream-ordered all-rank barrier (tiny allreduce)
void p2p_shutdown(ntp_ctx* c);                  // closes the peer mappings (ntp_destroy)
void unpack_f2v(ntp_ctx* c, const void* recv, int64_t V_p, int32_t d_s, int32_t P, void* Hv,
                int64_t ld_v, int32_t w, ntp_dtype dt_in, ntp_dtype dt_out, cudaStream_t s,
                const float* keep = nullptr, int64_t ld_keep = 0, int64_t rows = -1, int64_t vofs = 0,
                const uint32_t* keep_bits = nullptr, int32_t nw = 0);
void alltoall_blocks(ntp_ctx* c, const void* send, void* recv, int64_t block_elems, ntp_dtype dt,
                     cudaStream_t s);
// Layout exchanges with P = world * vs feature slices (vs virtual slices per rank, processed in sequence).
// Blocks are blk = V_r * d_s elements (V_r = vs * V_p rows per rank).
//   split  (v2f): send [P][V_r][d_s] (block s = slice s of my rows)  ->  feature slices [vs][V_pad][d_s]
//                 (slice j, rows of rank q = block j*world + q)
//   gather (f2v): feature slices [vs][V_pad][d_s]  ->  recv [P][V_r][d_s] (block s = slice s of my rows)
// world == 1: both layouts coincide (identity; a copy only if the buffers differ).
void exchange_v2f(ntp_ctx* c, const void* send, void* feat, int64_t blk, ntp_dtype dt, cudaStream_t s);
void exchange_f2v(ntp_ctx* c, const void* feat, void* recv, int64_t blk, ntp_dtype dt, cudaStream_t s);
inline int32_t nslices(const ntp_ctx* c) { return c->world * c->vs; }

void gemm_tf32x3_pack(ntp_ctx* c, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B_hi,
                      const float* B_lo, int64_t ldb, const PackEpi& pk, cudaStream_t s);
// Tensor-core (tcgen05 kind::tf32, 3xTF32) GEMM, gemm.cu.  A stored [K][M] if a_mn else [M][K];
// B stored [K][N] if b_mn else [N][K]; lda/ldb multiples of 4.  epi: 0 store, 1 ReLU, 2 keep where aux > 0.
void gemm_tf32x3(ntp_ctx* c, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, bool a_mn,
                 const float* B, int64_t ldb, bool b_mn, float* C, int64_t ldc, int epi, const float* aux,
                 int64_t ldaux, cudaStream_t s, const float* B_lo = nullptr);
// B_lo != nullptr: B is already rn_tf32-rounded and B_lo holds the residual (tf32_split), e.g. weights.
void tf32_split(ntp_ctx* c, const float* src, int64_t rows, int64_t cols, int64_t ld, float* hi, float* lo,
                cudaStream_t s);

// dW0 = X^T (G .* ReLU') straight from the bf16 gradient slice (wgrad.cu): bf16 slices, hid = P*d_s = 128,
// d_s >= 64, d_in <= 128.
bool wgrad_fused_supported(int32_t P, int32_t d_s, int32_t d_in, int32_t hid, ntp_dtype dt);
void wgrad_fused(ntp_ctx* c, const float* X, int64_t ldx, int64_t V_p, int32_t d_in, const void* G, int32_t d_s,
                 int32_t P, int32_t hid, const uint32_t* bits, int32_t nwb, int64_t r_begin, int64_t r_end, float* dW0,
                 cudaStream_t s);
// Fused W1-after-propagation head (head.cu): bf16 gathered slice, P*d_s == 128, C <= 192.
bool head_fused_supported(int32_t P, int32_t d_s, int32_t hid, int32_t C, ntp_dtype dt);
int64_t head_fused(ntp_ctx* c, const void* gathered, int64_t V_p, int32_t d_s, int32_t P, int32_t hid, int32_t C,
                   const float* W1, int64_t ldw1, const int32_t* y, const uint8_t* mask, int64_t row0, int64_t n,
                   const float* gscale, void* out, void* const* peer, float* dW1, double* part, int64_t* cnt,
                   cudaStream_t s, int64_t v_lo = 0, int64_t v_hi = -1, const int32_t* out_perm = nullptr);

inline size_t esize(ntp_dtype d) { return d == NTP_BF16 ? 2 : 4; }
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
int32_t slice_width(int32_t w, int32_t P, ntp_dtype dt, int align);

void count_launch(ntp_ctx* c, int k = 1);
// Record a TIMING event (phase marks, SpMM hop pairs): external event node under graph capture.
// Layout-change traffic handed to the transport by this rank (see ntp_ctx::wire_sent).
inline void wire_add(ntp_ctx* c, int64_t sent, int64_t recv) {
    c->wire_sent[c->wire_phase & 3] += sent;
    c->wire_recv[c->wire_phase & 3] += recv;
}
inline void wire_reset(ntp_ctx* c) {
    for (int i = 0; i < 4; ++i) c->wire_sent[i] = c->wire_recv[i] = 0;
    c->wire_phase = 0;
}
inline cudaError_t record_timing(ntp_ctx* c, cudaEvent_t e, cudaStream_t s) {
    return cudaEventRecordWithFlags(e, s, c->capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
}

}  // namespace ntp
