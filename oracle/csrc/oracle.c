/*
 * oracle.c — TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct CPU
 * reference for the NeutronTP hot path (arXiv 2412.20379).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may call it.  It shares no code, header or constant generator with the
 * CUDA library under paper_2412_20379_b200/.
 *
 * Precision: fp64 throughout.  Parallelism: OpenMP over output rows only; each
 * row's summation order is fixed (self term first, then ascending source id),
 * so results do not depend on the thread count.
 */
#include <stdint.h>
#include <stddef.h>
#include <math.h>

/* ------------------------------------------------------------------------ *
 * Counter-based R-MAT arc generator (SURVEY §8(d) "R-MAT"):
 *   h(seed, stream, i) = splitmix64_finaliser(seed*G + stream*D + i)
 *   for arc i, level l (MSB first): u = h(seed, 0, i*64 + l) >> 32
 *     u <  t0        -> quadrant a: (src bit 0, dst bit 0)
 *     u <  t1        -> quadrant b: (0, 1)
 *     u <  t2        -> quadrant c: (1, 0)
 *     otherwise      -> quadrant d: (1, 1)
 * Raw arcs only: rejection of ids >= n and self loops is done by the caller
 * (oracle/graph.py), following O1.
 * ------------------------------------------------------------------------ */
static uint64_t oracle_splitmix_fin(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t oracle_hash(uint64_t seed, uint64_t stream, uint64_t i) {
    return oracle_splitmix_fin(seed * 0x9E3779B97F4A7C15ULL + stream * 0xD1B54A32D192ED03ULL + i);
}

void oracle_rmat_arcs(int scale, uint32_t t0, uint32_t t1, uint32_t t2, uint64_t seed,
                      int64_t i0, int64_t count, int64_t* src, int64_t* dst) {
    #pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < count; ++k) {
        uint64_t i = (uint64_t)(i0 + k);
        int64_t s = 0, d = 0;
        for (int l = 0; l < scale; ++l) {
            uint32_t u = (uint32_t)(oracle_hash(seed, 0, i * 64u + (uint64_t)l) >> 32);
            int sb, db;
            if (u < t0)      { sb = 0; db = 0; }
            else if (u < t1) { sb = 0; db = 1; }
            else if (u < t2) { sb = 1; db = 0; }
            else             { sb = 1; db = 1; }
            s = (s << 1) | sb;
            d = (d << 1) | db;
        }
        src[k] = s;
        dst[k] = d;
    }
}

/* Full-scale sampled pin: regenerate ALL raw arcs [0, m_raw) and keep the valid ones (ids < n,
 * no self loop) whose destination (by_dst = 1) or source (by_dst = 0) is flagged in `bitmap`
 * (bit v of bitmap[v >> 6]); reverse arcs are included when `symmetric`.  Writes up to `cap`
 * (src, dst) pairs in unspecified order and returns how many matched (may exceed cap). */
int64_t oracle_rmat_filter(int scale, uint32_t t0, uint32_t t1, uint32_t t2, uint64_t seed, int64_t m_raw,
                           int64_t n, int symmetric, const uint64_t* bitmap, int by_dst,
                           int64_t* out_src, int64_t* out_dst, int64_t cap) {
    int64_t count = 0;
    #pragma omp parallel for schedule(static, 65536)
    for (int64_t k = 0; k < m_raw; ++k) {
        int64_t s = 0, d = 0;
        for (int l = 0; l < scale; ++l) {
            uint32_t u = (uint32_t)(oracle_hash(seed, 0, (uint64_t)k * 64u + (uint64_t)l) >> 32);
            int sb, db;
            if (u < t0)      { sb = 0; db = 0; }
            else if (u < t1) { sb = 0; db = 1; }
            else if (u < t2) { sb = 1; db = 0; }
            else             { sb = 1; db = 1; }
            s = (s << 1) | sb;
            d = (d << 1) | db;
        }
        if (s >= n || d >= n || s == d) continue;
        for (int rev = 0; rev <= (symmetric ? 1 : 0); ++rev) {
            const int64_t a = rev ? d : s, b = rev ? s : d;     /* arc a -> b */
            const int64_t key = by_dst ? b : a;
            if ((bitmap[key >> 6] >> (key & 63)) & 1ull) {
                int64_t slot;
                #pragma omp atomic capture
                slot = count++;
                if (slot < cap) { out_src[slot] = a; out_dst[slot] = b; }
            }
        }
    }
    return count;
}

/* ------------------------------------------------------------------------ *
 * K-hop propagation, O3 (fwd) / O4 (bwd), SURVEY §8(c):
 *   Z^0 = H
 *   Z^k[v,:] = gamma * ( c_vv Z^{k-1}[v,:] + sum_{u in N(v), ascending} c_uv Z^{k-1}[u,:] )
 *              + alpha * H[v,:]
 *   c_uv = rs[v] * cs[u]   (row-side and column-side D~^{-1/2}),  c_vv = rs[v]*cs[v]
 * Paper: Eq. 9 "Z^k = gamma A^ Z^{k-1}", A^ = D~^{-1/2}(A+I)D~^{-1/2}
 * (P:738-739), two-sided reading R1; alpha mix reading R2.
 * Forward: CSR = in-CSR (row v = destination), rs = dinv_in, cs = dinv_out.
 * Backward (adjoint, A^T): CSR = out-CSR (row u = source), rs = dinv_out,
 * cs = dinv_in  ("accumulate gradients along out-edges").
 * Layout: row-major [n x d] with leading dimension d.  tmp: n*d scratch.
 * ------------------------------------------------------------------------ */
void oracle_propagate(int64_t n, const int64_t* row_ptr, const int32_t* col,
                      const double* rs, const double* cs, int64_t d,
                      const double* H, double* Z, double* tmp,
                      int K, double gamma, double alpha) {
    /* Z^0 = H, kept in `cur`; ping-pong between Z and tmp, result lands in Z. */
    double* bufs[2] = { Z, tmp };
    int cur = (K % 2 == 0) ? 0 : 1;        /* so that after K hops the result is in bufs[0] = Z */
    for (int64_t i = 0; i < n * d; ++i) bufs[cur][i] = H[i];
    for (int k = 1; k <= K; ++k) {
        const double* zin = bufs[cur];
        double* zout = bufs[cur ^ 1];
        #pragma omp parallel for schedule(dynamic, 256)
        for (int64_t v = 0; v < n; ++v) {
            double* o = zout + v * d;
            const double cvv = rs[v] * cs[v];
            for (int64_t j = 0; j < d; ++j) o[j] = cvv * zin[v * d + j];          /* self term first */
            for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) {              /* ascending sources */
                const int64_t u = col[e];
                const double cuv = rs[v] * cs[u];
                for (int64_t j = 0; j < d; ++j) o[j] += cuv * zin[u * d + j];
            }
            for (int64_t j = 0; j < d; ++j) o[j] = gamma * o[j] + alpha * H[v * d + j];
        }
        cur ^= 1;
    }
}

/* Single hop applied to an explicit sample of output rows (full-scale spot
 * checks): out[s,:] = gamma*(c_vv zin[v] + sum c_uv zin[u]) + alpha*h[v] for
 * v = rows[s].  zin / h are full [n x d] arrays. */
void oracle_hop_rows(const int64_t* row_ptr, const int32_t* col,
                     const double* rs, const double* cs, int64_t d,
                     const double* zin, const double* h, double gamma, double alpha,
                     const int64_t* rows, int64_t nrows, double* out) {
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t s = 0; s < nrows; ++s) {
        const int64_t v = rows[s];
        double* o = out + s * d;
        const double cvv = rs[v] * cs[v];
        for (int64_t j = 0; j < d; ++j) o[j] = cvv * zin[v * d + j];
        for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) {
            const int64_t u = col[e];
            const double cuv = rs[v] * cs[u];
            for (int64_t j = 0; j < d; ++j) o[j] += cuv * zin[u * d + j];
        }
        for (int64_t j = 0; j < d; ++j) o[j] = gamma * o[j] + alpha * (h ? h[v * d + j] : 0.0);
    }
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Thread count of the OpenMP loops above (bench.py's single-thread baseline; results do not depend on it). */
void oracle_set_num_threads(int t) {
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    omp_set_num_threads(t);
#else
    (void)t;
#endif
}
