/*
 * ntp.h — C ABI of libntp, a B200 (sm_100a) implementation of the data-parallel
 * hot path of NeutronTP (arXiv 2412.20379): feature-sliced ("GNN tensor
 * parallel") full-graph propagation for decoupled GNN training.
 *
 * Citation keys: P:n = PAPER.md line n, S:n = SPEC.md line n, SURVEY §x.
 *
 * Model:
 *   A^ = D~_in^{-1/2} (A + I) D~_out^{-1/2},   D~ = D + I       (reading R1)
 *   forward  Z^0 = H,  Z^k = gamma * A^   Z^{k-1} + alpha * H     (Eq. 9, reading R2)
 *   backward Y^0 = G,  Y^k = gamma * A^T  Y^{k-1} + alpha * G     (exact adjoint)
 *   epoch    Alg. 1: MLP on vertex rows -> split -> K hops on
 *            feature slices -> gather -> loss -> split -> K backward hops ->
 *            gather -> MLP backward -> allreduce(dW) -> SGD.
 *
 * Layouts (P = number of feature slices = world size, or world * vs after ntp_set_slices;
 * SURVEY §8(a) a1):
 *   V_p   = ceil(n / P),  V_pad = P * V_p
 *   d_s   = ceil(w / P) rounded up so d_s*elem_bytes % slice_align == 0 (16, 32, 64 or 128)
 *   VERTEX  layout on rank q: rows [q*V_p, (q+1)*V_p) of the padded matrix at width w
 *   FEATURE layout on rank q: all V_pad rows x columns [q*d_s, (q+1)*d_s), row-major,
 *           rows >= n and columns >= w are zero padding.
 *
 * Conventions (all entry points):
 *   - Every call returns ntp_status; no C++ exception, abort or exit crosses the ABI.
 *     On failure ntp_last_error(ctx) returns a context-owned message.
 *   - Arguments are validated before any device work.
 *   - Device pointers inside ntp_tensor are caller-owned (typically torch
 *     tensors); the library never frees them.  Graph arrays passed in are
 *     copied.  The library owns the device CSR (both orientations), D~^{-1/2},
 *     the NCCL communicator, its streams and scratch; ntp_destroy frees them.
 *   - Calls taking an ntp_stream (a cudaStream_t) only enqueue work on it;
 *     kernel errors surface at the next synchronising call.
 *   - Collective contract: every rank issues the same sequence of
 *     collective-bearing calls (layout changes, ntp_train_epoch).
 *   - One context per process/GPU; all calls on one host thread per context.
 */
#ifndef NTP_H
#define NTP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NTP_ABI_VERSION 1

typedef struct ntp_ctx ntp_ctx;
typedef void* ntp_stream;          /* a cudaStream_t; NULL = legacy default stream */

typedef enum {
    NTP_OK = 0,
    NTP_ERR_ARG = -1,       /* null pointer / out-of-range scalar            */
    NTP_ERR_SHAPE = -2,     /* tensor shape, dtype, layout or alignment       */
    NTP_ERR_CONFIG = -3,    /* unsupported configuration (e.g. nnz >= 2^31)   */
    NTP_ERR_GRAPH = -4,     /* NTP_G_VALIDATE failed                          */
    NTP_ERR_STATE = -5,     /* call out of order (e.g. no graph loaded)       */
    NTP_ERR_OOM = -6,       /* device allocation failed                       */
    NTP_ERR_CUDA = -7,      /* CUDA runtime / kernel error                    */
    NTP_ERR_NCCL = -8,      /* NCCL error (communicator aborted)              */
    NTP_ERR_TIMEOUT = -9    /* collective did not complete in time (aborted)  */
} ntp_status;

typedef enum { NTP_F32 = 0, NTP_BF16 = 1 } ntp_dtype;
typedef enum { NTP_LAYOUT_VERTEX = 0, NTP_LAYOUT_FEATURE = 1 } ntp_layout;

/* A strided row-major matrix in caller-owned memory (device unless a call says
 * otherwise).  Element (r, c) lives at data + (r*ld + c)*elem_bytes.
 * For propagation and layout calls: data 16-byte aligned, (ld*elem_bytes) % 16 == 0. */
typedef struct {
    void*      data;
    ntp_dtype  dtype;
    ntp_layout layout;
    int64_t    rows;
    int32_t    cols;
    int64_t    ld;
} ntp_tensor;

/* ---------------------------------------------------------------- context */

/* Rank 0 calls this and broadcasts the 128 bytes (e.g. torch.distributed). */
ntp_status ntp_get_unique_id(uint8_t id[128]);

/* Creates a context on CUDA `device`.  world == 1: no NCCL communicator is
 * created and `id` may be NULL.  world > 1: ncclCommInitRank with `id`.
 * slice_align: 16, 32, 64 or 128 (bytes; d_s rounding, see Layouts).  The padding columns are zero
 * and cost bytes; on an L2-resident slice a slice row of a power of two bytes can still be the faster
 * hop (16 fp32 columns hop faster than 12, 32 faster than 24 on the Reddit shape). */
ntp_status ntp_create(ntp_ctx** ctx, int device, int rank, int world,
                      const uint8_t id[128], int slice_align);
void        ntp_destroy(ntp_ctx* ctx);
const char* ntp_last_error(const ntp_ctx* ctx);
const char* ntp_status_string(ntp_status s);
int         ntp_abi_version(void);

/* Virtual slices (SURVEY §8(b) "P > world with P % world == 0"): from now on the context splits the
 * propagated width into P = world * vs feature slices, vs per rank, processed in sequence on this GPU
 * (every slice is aggregated independently; the paper's workers become virtual).  All
 * layout definitions below then use P: V_p = ceil(n / P), V_pad = P * V_p, d_s = slice width for P;
 * this rank's VERTEX rows are the vs*V_p rows from rank*vs*V_p, its FEATURE tensor stacks its vs slices
 * [vs*V_pad x d_s] (slice j = global slice rank*vs + j), and the layout changes exchange per (peer,
 * slice) blocks (world == 1: device-local, the exchange is the identity).  Collective: every rank calls it
 * with the same P.  NTP_ERR_ARG unless P >= world and P % world == 0.  Default P = world. */
ntp_status ntp_set_slices(ntp_ctx* ctx, int32_t P);

/* Collective deadline (SURVEY §8(b) "collective failures or timeouts abort the communicator"; the
 * analogue of SPEC S:407's round timeout).  Every call that waits for collective-bearing work
 * (ntp_train_epoch*, ntp_sync, ntp_destroy) polls the stream and ncclCommGetAsyncError; an NCCL error
 * aborts the communicator (ncclCommAbort) and returns NTP_ERR_NCCL, and work still pending after `ms`
 * milliseconds (e.g. ranks that issued different collective sequences) aborts it and returns
 * NTP_ERR_TIMEOUT.  After an abort every collective-bearing call returns NTP_ERR_NCCL; destroy the
 * context.  ms = 0 (default): wait without a deadline (errors are still detected). */
ntp_status ntp_set_timeout(ntp_ctx* ctx, int64_t ms);

/* Aborts this rank's communicator now (e.g. after a peer reported NTP_ERR_TIMEOUT), so that no call --
 * including ntp_destroy -- waits for peers any more.  Afterwards as above. */
ntp_status ntp_abort(ntp_ctx* ctx);

/* Waits for the work enqueued on `s` (e.g. layout changes, pipelines) under the contract above. */
ntp_status ntp_sync(ntp_ctx* ctx, ntp_stream s);

/* Overlap trace (per-stage begin/end with chunk ids, to verify the overlap).  With tracing on,
 * ntp_train_epoch records a timed CUDA event at the begin and end of every row chunk of the chunked
 * layout-change schedule (NTP_M_OVERLAP on W1-after-propagation epochs, NCCL or copy-engine transfers):
 * on the comm stream each chunk's exchange, on the compute stream each chunk's producer / consumer work
 * (MLP forward + pack, head, MLP backward) and the forward / backward hops as one interval each.  Traced
 * epochs run eagerly (no epoch graph).  ntp_trace copies up to `max` records of the last epoch (waiting
 * for it), times in ms from the epoch's start event; *count = records available.  Off by default. */
typedef struct {
    int32_t stream;    /* 0 compute, 1 comm */
    int32_t phase;     /* comm: 0 split, 1 gather, 2 gradient split, 3 gradient gather; compute: 0 MLP forward,
                          1 head, 3 MLP backward, 4 forward hops, 5 backward hops */
    int32_t chunk;     /* row chunk (-1: whole phase) */
    float begin_ms, end_ms;
} ntp_trace_rec;
ntp_status ntp_set_trace(ntp_ctx* ctx, int on);
ntp_status ntp_trace(ntp_ctx* ctx, ntp_trace_rec* out, int32_t max, int32_t* count);

/* CUDA-event duration (ms, summed) and count of the SpMM hop launches -- each spmm_hop_kernel with its
 * spmm_fixup_kernel -- enqueued by the last ntp_propagate_fwd / _bwd / _pipeline or ntp_train_epoch
 * call; waits for the last of them.  The events are recorded on the stream the hops run on. */
ntp_status ntp_hop_timing(ntp_ctx* ctx, double* ms, int32_t* launches);

/* -------------------------------------------------------------- graph (a0) */

#define NTP_G_SYMMETRIC 1u   /* graph is undirected: transpose == CSR (saves memory) */
#define NTP_G_VALIDATE  2u   /* check the input CSR: rp[0]=0, monotone,
                                rp[n]=nnz, 0<=col<n, strictly ascending per row     */
#define NTP_G_REORDER   4u   /* store the graph under an internal vertex numbering by
                                descending total degree (the hot rows of the gather
                                become contiguous).  Invisible at the ABI: slices,
                                ntp_copy_csr and ntp_copy_dinv stay in original ids.
                                Not combinable with the last-hop chunked gather of
                                NTP_M_OVERLAP (W1 before propagation) or with
                                ntp_propagate_pipeline's overlap (NTP_ERR_CONFIG); the
                                W1-after-propagation epoch overlaps its layout changes
                                by vertex-row chunk and accepts it. */

/* Loads an in-CSR from HOST arrays: row v = destination, columns = sources u
 * of arcs u->v ("N_in(v)", Eq. 1).  Explicit self loops are dropped
 * (A~ adds exactly one, reading R1).  Builds the out-CSR (transpose) on the
 * device unless NTP_G_SYMMETRIC, then degrees and D~^{-1/2}.
 * Requires n < 2^31 and nnz < 2^31 (NTP_ERR_CONFIG otherwise). */
ntp_status ntp_load_graph(ntp_ctx* ctx, const int64_t* row_ptr, const int32_t* col_idx,
                          int64_t n, int64_t nnz, uint32_t flags);

/* Builds the graph from a HOST arc list (src[i] -> dst[i]) on the device:
 * reject ids outside [0,n) and self loops, optionally append reverse arcs
 * (NTP_G_SYMMETRIC), sort by (dst, src), deduplicate (O1). */
ntp_status ntp_build_graph(ntp_ctx* ctx, const int64_t* src, const int64_t* dst, int64_t m,
                           int64_t n, uint32_t flags);

/* Generates m_raw R-MAT arcs on the device with the counter-based generator
 * of SURVEY §8(d) (h = SplitMix64 finaliser of seed*G + stream*D + i; level l
 * of arc i draws u = h(seed,0,i*64+l)>>32 against thresholds t[0..2]; MSB
 * first; ids < 2^scale), then builds the graph exactly as ntp_build_graph. */
ntp_status ntp_generate_rmat(ntp_ctx* ctx, int64_t n, int scale, int64_t m_raw,
                             const uint32_t thresholds[3], uint64_t seed, uint32_t flags);

/* Writes raw R-MAT arcs [i0, i0+count) to HOST arrays (generator parity tests). */
ntp_status ntp_rmat_arcs(ntp_ctx* ctx, int scale, const uint32_t thresholds[3], uint64_t seed,
                         int64_t i0, int64_t count, int64_t* src_host, int64_t* dst_host);

ntp_status ntp_graph_info(const ntp_ctx* ctx, int64_t* n, int64_t* nnz, int* symmetric);

/* Copies the device CSR to HOST arrays: transposed=0 -> in-CSR, 1 -> out-CSR.
 * row_ptr: n+1 entries, col_idx: nnz entries, deg: n entries (may be NULL). */
ntp_status ntp_copy_csr(const ntp_ctx* ctx, int transposed, int64_t* row_ptr,
                        int32_t* col_idx, int32_t* deg);

/* Copies D~_in^{-1/2} and D~_out^{-1/2} (fp32, n entries each) to HOST. */
ntp_status ntp_copy_dinv(const ntp_ctx* ctx, float* dinv_in, float* dinv_out);

/* ------------------------------------------------------ partition maps (a1) */

typedef struct {
    int64_t n, V_p, V_pad;
    int32_t w, P, d_s, w_pad, elem_bytes, chunks;
    int64_t chunk;              /* rows per chunk inside each owner block */
} ntp_partition_info;

/* Pure host computation of the maps above (no context needed). */
ntp_status ntp_partition(int64_t n, int32_t w, int32_t P, ntp_dtype dtype, int32_t chunks,
                         int slice_align, ntp_partition_info* out);

/* --------------------------------------------------- features and layouts */

/* Copies this rank's part of the HOST matrix X [n x d] (row-major, dtype) into
 * `out` (device): VERTEX -> rows R_rank at width d (out->cols >= d), FEATURE ->
 * all V_pad rows x columns [rank*d_s, (rank+1)*d_s); padding is zero-filled. */
ntp_status ntp_scatter_features(ntp_ctx* ctx, const void* X_host, ntp_dtype dtype,
                                int64_t n, int32_t d, ntp_layout layout, ntp_tensor* out);

/* "split": Hv = this rank's VERTEX rows [V_p x w] (w = Hv->cols) ->
 * Hf = this rank's FEATURE slice [V_pad x d_s] (ld == d_s).  One all-to-all.
 * "gather": the inverse.  Pure data movement: f2v(v2f(x)) == x bitwise. */
ntp_status ntp_layout_v2f(ntp_ctx* ctx, const ntp_tensor* Hv, ntp_tensor* Hf, ntp_stream s);
ntp_status ntp_layout_f2v(ntp_ctx* ctx, const ntp_tensor* Hf, ntp_tensor* Hv, ntp_stream s);

/* ------------------------------------------------ propagation (a4, a8) */

/* K hops on one feature slice (no communication).  H, Z: [rows >= n] x cols,
 * same dtype (fp32 or bf16 storage; fp32 accumulation).  Z must not alias H.
 * Rows [n, Z->rows) of Z are zero-filled.  K >= 0, gamma in (0,1], alpha in [0,1).
 * propagate_fwd uses the in-CSR (A^), propagate_bwd the out-CSR (A^T). */
ntp_status ntp_propagate_fwd(ntp_ctx* ctx, const ntp_tensor* H, ntp_tensor* Z, int K,
                             float gamma, float alpha, ntp_stream s);
ntp_status ntp_propagate_bwd(ntp_ctx* ctx, const ntp_tensor* G, ntp_tensor* dH, int K,
                             float gamma, float alpha, ntp_stream s);

/* Vertex-layout propagation pipeline (a3 -> a4 -> a5, or a7 -> a8 -> a9 when `transposed`;
 * Alg. 1 lines 9-12 / 22-25): this rank's rows Hv [V_p x w] (fp32,
 * DEVICE, caller-owned) are split into feature slices with the column-side D~^{-1/2}
 * pre-scale fused into the pack (one all-to-all), propagated K >= 1 hops in storage dtype
 * `dt` (fp32 accumulation), and gathered back into Zv [V_p x w] (fp32).  flags & NTP_M_OVERLAP:
 * the last hop runs per (peer block, sub-chunk) -- `chunks` sub-chunks per block -- and each
 * finished chunk is exchanged on the comm stream while the next computes (a12, P:855,
 * Fig. 7(c)); arithmetic is identical either way.  Collective-bearing: every rank calls
 * it with the same arguments.  NTP_ERR_CONFIG for NTP_M_OVERLAP on an NTP_G_REORDER graph. */
ntp_status ntp_propagate_pipeline(ntp_ctx* ctx, const ntp_tensor* Hv, ntp_tensor* Zv, int K,
                                  float gamma, float alpha, int transposed, ntp_dtype dt,
                                  int32_t chunks, uint32_t flags, ntp_stream s);

/* ------------------------------------------------------ MLP contraction (a2, a10) */

/* C[M x N] = op(A) op(B) on the tensor cores (tcgen05 kind::tf32, 3xTF32 split: fp32-level
 * accuracy, reading R11).  All matrices fp32, row-major, DEVICE memory, caller-owned.
 * op(A) = A (stored [M x K], lda) or A^T (trans_a: stored [K x M]); op(B) = B (stored [K x N])
 * or B^T (trans_b: stored [N x K]).  lda, ldb: multiples of 4, 16-byte aligned bases
 * (NTP_ERR_SHAPE otherwise).  epilogue: 0 plain, 1 ReLU (Eq. 4 sigma).  These are the
 * GEMMs of the MLP forward and backward inside ntp_train_epoch. */
ntp_status ntp_gemm_f32(ntp_ctx* ctx, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, int trans_a,
                        const float* B, int64_t ldb, int trans_b, float* C, int64_t ldc, int epilogue,
                        ntp_stream s);

/* ------------------------------------------------------ one epoch (Alg. 1) */

#define NTP_M_W1_AFTER_PROP 1u  /* propagate H1 (w = hid) and apply W1 after (reading R3) */
#define NTP_M_OVERLAP       2u  /* chunked last hop with the gather on a comm stream (a12) */
#define NTP_M_HOST_INPUTS   4u  /* X_v/labels_v/train_mask_v are HOST (pinned) pointers;
                                   copied to the device inside the call (e2e path)       */
#define NTP_M_STAGED       16u  /* inputs come from staging slot (flags >> 8) & 3 (< NTP_STAGE_SLOTS), filled by
                                   ntp_stage_inputs (its host->device copy may overlap the
                                   previous epoch); X_v / labels_v / train_mask_v are ignored
                                   except for X_v's shape.  Each slot's epoch is captured as
                                   its own CUDA graph (the slot's buffers are baked in; the copy
                                   stream's ready / free events become external event nodes).
                                   NTP_ERR_STATE if the slot was never staged with [V_p x d_in]. */
#define NTP_M_SLOT_SHIFT    8
#define NTP_M_SLOT_MASK     3u
#define NTP_STAGE_SLOTS     3   /* input staging slots: with three, a loop keeps two epochs' copies queued */
#define NTP_M_DATA_PARALLEL 32u /* NEXT-4 baseline: each rank aggregates its own vertex rows at
                                   full width after an all-gather of the state before every hop,
                                   instead of feature slices (same function; load follows the rows'
                                   degrees).  W1 before propagation, NCCL, no NTP_G_REORDER */
#define NTP_M_HOST_STREAM  64u  /* memory-efficient scheduling (NEXT-3): X_v is a HOST pointer (pinned
                                   for asynchronous copies, row pitch X_v->ld) that stays in host memory;
                                   every vertex-row chunk of it is copied into a 2-slot device ring on
                                   the copy stream right before the MLP forward / dW0 kernels that read
                                   it (the copy of chunk ch+1 overlaps chunk ch).  Labels and mask stay
                                   device pointers.  W1 after propagation only; eager (no epoch graph).
                                   Frees the V_p x d_in fp32 input from HBM (fp32 papers shape at P = 1) */
#define NTP_M_P2P_LAYOUTS   8u  /* P > 1: peer-direct layout changes instead of the NCCL block
                                   all-to-all: the producers (pack, last-hop epilogue, loss
                                   kernel) store into the owners' CUDA-IPC windows over
                                   NVLink and a barrier replaces each exchange; same bits.
                                   Opt-in: measured no faster than NCCL.
                                   With NTP_M_OVERLAP and NTP_M_W1_AFTER_PROP: the row-chunked
                                   overlap schedule with copy-engine transfers -- one
                                   cudaMemcpyAsync per peer and chunk into the owner's window,
                                   then a fenced flag write into its inbox that the consumer
                                   waits on (cuStreamWriteValue32 / cuStreamWaitValue32); eager */

typedef struct {
    int32_t   d_in, hid, C, K;
    float     gamma, alpha, lr;
    ntp_dtype dtype;            /* propagation storage dtype (fp32 accumulation always) */
    int32_t   chunks;           /* sub-chunks per owner block for the overlapped gather  */
    uint32_t  flags;
} ntp_model;

enum {  /* ntp_epoch_report.ms[] phases (CUDA-event times on the library's streams) */
    NTP_PH_MLP_FWD = 0, NTP_PH_V2F_FWD, NTP_PH_PROP_FWD, NTP_PH_F2V_FWD, NTP_PH_LOSS,
    NTP_PH_V2F_BWD, NTP_PH_PROP_BWD, NTP_PH_F2V_BWD, NTP_PH_MLP_BWD, NTP_PH_ALLREDUCE,
    NTP_PH_SGD, NTP_PH_TOTAL, NTP_PH_COUNT
};

typedef struct {
    double  loss;               /* global mean train loss, before this epoch's update */
    int64_t n_train;            /* global number of train vertices                    */
    double  ms[NTP_PH_COUNT];
    int64_t bytes_sent[4];      /* per layout change: v2f fwd, f2v fwd, v2f bwd, f2v bwd --   */
    int64_t bytes_recv[4];      /* counted where issued: NCCL send/recv / all-gather counts to
                                   and from peers, or the peer-store extents of the P2P path
                                   (NTP_M_DATA_PARALLEL: all its all-gathers in entry 0)      */
    int64_t collectives;        /* logical collective rounds issued (4 layout + allreduce) */
    int64_t kernel_launches;    /* libntp kernels launched in this call                 */
    double  spmm_ms;            /* summed duration of the SpMM hop kernels              */
    int32_t spmm_launches;
    int32_t pad_;
} ntp_epoch_report;

/* One training epoch.  The second call with the same model and pointers captures the enqueue
 * sequence into a CUDA graph; later calls replay it while no library buffer has been
 * (re)allocated or freed since the capture (any entry point that grows scratch invalidates it).
 * X_v [V_p x d_in] fp32 (this rank's VERTEX rows, rows
 * >= n zero), labels_v int32 [V_p], train_mask_v uint8 [V_p] (device unless
 * NTP_M_HOST_INPUTS).  The MLP GEMMs read X_v with TMA: pass ld % 4 == 0 and a 16-byte
 * aligned base, otherwise X_v is staged into a padded copy every epoch (561 MB on reddit).  W0 [d_in x hid], W1 [hid x C] fp32 device, replicated
 * on every rank, updated in place by SGD.  Synchronous: returns after
 * the epoch completed; `s` orders the call after prior work on that stream and
 * later work after it.  rep may be NULL. */
ntp_status ntp_train_epoch(ntp_ctx* ctx, const ntp_model* m, const ntp_tensor* X_v,
                           const int32_t* labels_v, const uint8_t* train_mask_v,
                           ntp_tensor* W0, ntp_tensor* W1, ntp_epoch_report* rep, ntp_stream s);

/* NEXT-2: one epoch of decoupled GAT (Eq. 5; §4.1.1: attention
 * "precomputed ... before the graph aggregation" and shared, then aggregation on feature slices):
 *   z = ReLU(X W0) W1 (w = C);  s_uv = a_src.z_u + a_dst.z_v over N_in(v) + {v} (A~ = A + I);
 *   alpha_uv = softmax_v(LeakyReLU(s_uv, slope));  Z^0 = z, Z^k = gamma A_att Z^{k-1};  softmax
 *   cross-entropy on Z^K;  gradients of W0, W1 and att by the chain rule (through the attention);
 *   SGD on all three.
 * att: [2 x C] fp32 device (row 0 a_src, row 1 a_dst), updated in place.  m->alpha must be 0, m->flags 0
 * (device inputs, W1 before propagation), C <= 256, graph without NTP_G_REORDER; virtual slices allowed.
 * slope: LeakyReLU slope in [0, 1) (NTP_ERR_ARG otherwise).
 * Per epoch: 4 layout changes, one all-gather of 2 floats per vertex (score halves: every rank then
 * evaluates every coefficient itself), one allreduce of 3n floats (the per-vertex contractions of the
 * attention gradient: the per-arc gradient is never formed, csrc/gat.cu), one of dW0|dW1|da.
 * Synchronous; eager (no epoch graph).  Errors as ntp_train_epoch. */
ntp_status ntp_train_epoch_gat(ntp_ctx* ctx, const ntp_model* m, const ntp_tensor* X_v, const int32_t* labels_v,
                               const uint8_t* train_mask_v, ntp_tensor* W0, ntp_tensor* W1, ntp_tensor* att,
                               float slope, ntp_epoch_report* rep, ntp_stream s);

/* Input staging for end-to-end training loops: enqueues the host->device copy of one epoch's
 * inputs (this rank's rows: X_host [V_p x d_in] fp32 with row pitch ldx elements, labels int32[V_p],
 * train mask uint8[V_p]; pinned host memory for a truly asynchronous copy) into library-owned slot
 * `slot` (0 .. NTP_STAGE_SLOTS-1) on the library's copy stream and returns at once.  The copy waits
 * until the last epoch that read the slot has finished with it, so a loop can stage epoch i+1's (and
 * i+2's) inputs while epoch i computes and then call ntp_train_epoch with
 * NTP_M_STAGED | (slot of that epoch) << NTP_M_SLOT_SHIFT.  Staging two epochs ahead over three slots
 * keeps the copy engine busy back to back: epoch i+2's copy no longer waits for epoch i's end, so a
 * loop whose copy and epoch take about as long runs at max(copy, epoch) instead of paying their jitter.
 * Host buffers must stay valid until that epoch returns.  NTP_ERR_ARG / NTP_ERR_STATE as usual. */
ntp_status ntp_stage_inputs(ntp_ctx* ctx, int slot, const float* X_host, int64_t rows, int32_t d_in, int64_t ldx,
                            const int32_t* labels_host, const uint8_t* train_mask_host);

/* NEXT-1: naive (coupled) GNN tensor parallelism, the paper's baseline for the
 * decoupled epoch ("twice per layer", Fig. 6).  One epoch of the L-layer GCN
 *   H^0 = X_v;  H^l = ReLU(A^ H^{l-1} W^l) (l < L);  logits = A^ H^{L-1} W^L
 * (Eq. 3-4, two-sided A^ of reading R1, no bias) with every aggregation on this rank's
 * feature slice: a split before and a gather after each layer's hop, forward and (layers 2..L)
 * backward -> 4L - 2 layout changes per epoch.  Loss / gradients / SGD as ntp_train_epoch
 * (O7-O9: softmax cross-entropy over the global train rows, ReLU'(0) = 0, W -= lr dW).
 *   m->widths[0..L]: d_in, hidden widths..., C (C <= 256); 1 <= L <= NTP_MAX_LAYERS; dtype = slice
 *   storage (fp32 accumulation).  X_v: this rank's rows [V_p x d_in] fp32 (device).  W[l]: dense
 *   [widths[l] x widths[l+1]] fp32 device tensors, updated in place.  Synchronous; eager (no graph).
 * Errors: NTP_ERR_ARG / NTP_ERR_SHAPE before any device work; NTP_ERR_STATE without a graph. */
#define NTP_MAX_LAYERS 8
typedef struct {
    int32_t L;
    int32_t widths[NTP_MAX_LAYERS + 1];
    float lr;
    ntp_dtype dtype;
    uint32_t flags;            /* reserved, 0 */
} ntp_coupled_model;
typedef struct {
    double loss;               /* pre-update loss of this epoch                              */
    int64_t n_train;
    int32_t layout_changes;    /* split / gather all-to-alls issued (4L - 2 when P > 1)      */
    int32_t hops;              /* SpMM hop launches                                          */
    int64_t bytes_sent, bytes_recv;   /* per rank, over all layout changes                   */
    double ms_total, ms_agg;   /* CUDA-event times: whole epoch, SpMM hops                    */
    int64_t kernel_launches;
} ntp_coupled_report;
ntp_status ntp_train_epoch_coupled(ntp_ctx* ctx, const ntp_coupled_model* m, const ntp_tensor* X_v,
                                   const int32_t* labels_v, const uint8_t* train_mask_v,
                                   ntp_tensor* const* W, ntp_coupled_report* rep, ntp_stream s);

/* ------------------------------------------------------ development switches
 * Environment variables read by the library (A/B measurement only; the defaults are the product):
 *   NTP_GRAPH=0          no CUDA-graph capture of epochs
 *   NTP_HEAD_CHUNK=r     rows per vertex-side chunk of the W1-after-propagation epoch
 *   NTP_HEAD_FUSED=0     unfused head (unpack -> GEMM -> loss -> GEMMs -> pack) instead of head.cu
 *   NTP_HEAD_TMA=0       head.cu loads Z with 16-byte loads instead of TMA
 *   NTP_PACK_FUSED=0     pack_v2f pass instead of the MLP GEMM's pack epilogue
 *   NTP_WGRAD_FUSED=0    unpack + 3xTF32 GEMM instead of wgrad.cu
 *   NTP_SPMM_VB=16|32    force the hop kernel's vector width; NTP_SPMM_SHORT=0|1 low-degree variants;
 *   NTP_SPMM_OCC=0|1|2   occupancy variant; NTP_UNIT_ITEMS=T merge-path unit size; NTP_L1_CARVEOUT=0
 *   NTP_SPMM_BULK=0|1    bulk-copy gather for wide rows off / forced (auto: rows of >= 1 KB)
 *   NTP_REORDER_MODE=m   degree-class granularity of NTP_G_REORDER; NTP_P2P=0 disables peer windows
 *   NTP_GAT_PERMUTE=1    GAT: permute the coefficients into out-CSR order instead of re-deriving them
 *   NTP_SPMM_INVARIANT=1 keep the slice-width-invariant reduction order at two edge slots on high-degree
 *                        graphs too (default there: one accumulator per lane slot at 4 CTAs/SM, faster;
 *                        results then differ between slice widths by rounding, within R10 of the oracle)
 * Every switch keeps the arithmetic of the reduction order except NTP_UNIT_ITEMS (it changes which
 * rows are cut across units) and NTP_SPMM_INVARIANT / NTP_SPMM_OCC on the two-slot high-degree path:
 * results stay within tolerance but not bitwise. */

#ifdef __cplusplus
}
#endif

#endif /* NTP_H */
