/*
 * skb.h — C ABI of the B200-native hot path of the sketched long-step IPM
 * (arXiv 2209.08722). The reference (`skipm`, pure Python) calls numpy /
 * scipy / LAPACK at each of the seams below; each entry point names the
 * reference call it replaces (paths relative to /root/reference/pkg/src/skipm).
 *
 * Conventions
 *  - All pointers are DEVICE pointers unless the name ends in _host.
 *  - `stream` is a cudaStream_t passed as void*; every call is asynchronous
 *    on it unless documented as synchronising.
 *  - Dense A is column-major: column j at A + j*lda, lda even, A 16-byte
 *    aligned (column blocks are contiguous for the TMA bulk engine).
 *  - Kernels never allocate: callers pass a device workspace (`workspace`,
 *    `ws_bytes`); see the *_workspace_bytes helpers.
 *  - Return value: 0 on success, negative SKB_ERR_* on argument / launch
 *    errors. Numerical outcomes (breakdown, rank loss) are reported through
 *    device status words with the SKB_ST_* bits, which the host maps onto the
 *    reference exception classes (errors.py).
 *  - No global mutable state: calls are reentrant per stream.
 */
#ifndef SKB_H_
#define SKB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SKB_OK 0
#define SKB_ERR_ARG (-1)
#define SKB_ERR_DIMS (-2)        /* errors.InvalidDims (sketching.py:100-103) */
#define SKB_ERR_WORKSPACE (-3)
#define SKB_ERR_CUDA (-4)
#define SKB_ERR_INTERNAL (-5)
#define SKB_ERR_UNSUPPORTED (-6)

#define SKB_ST_BREAKDOWN_CURV 1  /* errors.Breakdown (krylov_solvers.py:353-354) */
#define SKB_ST_BREAKDOWN_RZ 2    /* errors.Breakdown (krylov_solvers.py:341-342,360-361) */
#define SKB_ST_CHOL_FAIL 4       /* errors.RankDeficient (preconditioning.py:47-50) */
#define SKB_ST_NONPOSITIVE 8     /* errors.NonpositiveScaling / NonpositivePoint */

/* ----------------------------------------------------------- K1 hashes --
 * Replaces build_sparse_embedding (sketching.py:93-119): Generator(Philox(seed))
 * with key = SeedSequence(seed).generate_state(2, uint64) computed by the
 * caller. cols: n*s int32 row-major, vals: n*s doubles (+-1/sqrt(s)).
 * Bit-exact with numpy 2.3.5. Synchronises the stream (duplicate-redraw loop). */
int skb_sparse_embedding(uint64_t key0, uint64_t key1, int64_t n, int32_t w, int32_t s,
                         int32_t* cols, double* vals, uint64_t* words_used_host,
                         void* workspace, size_t ws_bytes, void* stream);

/* Raw bounded draws rng.integers(0, bound, count) continuing at 32-bit word
 * `word_offset` of the stream (numpy random_bounded_uint64_fill, bound <= 2^32).
 * Synchronises the stream. */
int skb_lemire_draw(uint64_t key0, uint64_t key1, uint64_t word_offset, uint32_t bound,
                    uint64_t count, uint32_t* out, uint64_t* words_used_host,
                    void* workspace, size_t ws_bytes, void* stream);

/* ------------------------------------------------- K4/K8 column streams --
 * Every call reads A once. m <= 2048 (dense). Outputs that are m-vectors are
 * summed over column blocks in a fixed order; `sub` (nullable) is subtracted
 * after the sum. Workspace: skb_stream_workspace_bytes(m). */
size_t skb_stream_workspace_bytes(int64_t m);

/* u = A (d2 .* (A' z)) [- sub]      NormalOperator.apply (krylov_solvers.py:46-47) */
int skb_normal_apply(const double* A, int64_t m, int64_t n, int64_t lda, const double* d2,
                     const double* z, double* u, const double* sub, void* workspace,
                     size_t ws_bytes, void* stream);

/* u = A x [- sub]                    lp.A @ x (ipm_core.py:99) */
int skb_gemv(const double* A, int64_t m, int64_t n, int64_t lda, const double* x, double* u,
             const double* sub, void* workspace, size_t ws_bytes, void* stream);

/* u = A (v ./ s) [- sub]             v-invariant recheck (ipm_core.py:502) */
int skb_gemv_ratio(const double* A, int64_t m, int64_t n, int64_t lda, const double* v,
                   const double* s, double* u, const double* sub, void* workspace,
                   size_t ws_bytes, void* stream);

/* p = A (x - sigma_mu ./ s [- (x ./ s) .* r_d]) [- r_p]   build_rhs (ipm_core.py:196-206);
 * r_d == NULL and r_p == NULL give the feasible form. */
int skb_rhs(const double* A, int64_t m, int64_t n, int64_t lda, const double* x,
            const double* s, const double* r_d, double sigma_mu, double* p, const double* r_p,
            void* workspace, size_t ws_bytes, void* stream);

/* t = (A' y [+ add]) [- sub]         lp.A.T @ y (+ s - c) (ipm_core.py:100) */
int skb_gemv_t(const double* A, int64_t m, int64_t n, int64_t lda, const double* y,
               const double* add, const double* sub, double* t, void* workspace,
               size_t ws_bytes, void* stream);

/* One pass of assemble_directions (ipm_core.py:218-223):
 * atdy = A' dy; ds = -atdy [- r_d]; dx = -x + sigma_mu/s - (x/s) ds - v/s; adx = A dx. */
int skb_directions(const double* A, int64_t m, int64_t n, int64_t lda, const double* dy,
                   const double* x, const double* s, const double* v, const double* r_d,
                   double sigma_mu, double* ds, double* dx, double* atdy, double* adx,
                   void* workspace, size_t ws_bytes, void* stream);

/* One pass of make_iterate (ipm_core.py:94-102) at x + alpha dx, y_new, s + alpha ds:
 * x_out, s_out (nullable), r_d = A' y_new + s_new - c, r_p = A x_new - b.
 * dx/ds may be NULL (alpha ignored). */
int skb_iterate(const double* A, int64_t m, int64_t n, int64_t lda, const double* x,
                const double* dx, const double* s, const double* ds, double alpha,
                const double* y_new, const double* b, const double* c, double* x_out,
                double* s_out, double* r_p, double* r_d, void* workspace, size_t ws_bytes,
                void* stream);

/* out = sum_b part[b*m:(b+1)*m] (fixed order) [- sub]. */
int skb_reduce_partials(const double* part, int32_t nparts, int64_t m, const double* sub,
                        double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SKB_H_ */
