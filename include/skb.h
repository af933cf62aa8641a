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

#define SKB_ST_BREAKDOWN_CURV 1  /* errors.Breakdown (krylov_solvers.py:89-90; chebyshev :191-192) */
#define SKB_ST_BREAKDOWN_RZ 2    /* errors.Breakdown (krylov_solvers.py:77-78,96-97) */
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
 * Every call reads A once. m <= 16384 (dense; per-warp TMA ring up to 1024,
 * CTA-cooperative blocks above). Outputs that are m-vectors are
 * summed over column blocks in a fixed order; `sub` (nullable) is subtracted
 * after the sum. Workspace: skb_stream_workspace_bytes(m). */
size_t skb_stream_workspace_bytes(int64_t m);

/* u = A (d2 .* (A' z)) [- sub]      NormalOperator.apply (krylov_solvers.py:46-47).
 * gate (nullable device int): when *gate != 0 the launches are no-ops (PCG stopped). */
int skb_normal_apply(const double* A, int64_t m, int64_t n, int64_t lda, const double* d2,
                     const double* z, double* u, const double* sub, const int* gate,
                     void* workspace, size_t ws_bytes, void* stream);

/* The streaming pass of skb_normal_apply alone: per-CTA partial m-vectors into
 * part (>= skb_stream_workspace_bytes(m)); *nparts_host receives their count.
 * Reduce with skb_reduce_partials. (Used for per-kernel roofline timing.) */
int skb_normal_apply_partials(const double* A, int64_t m, int64_t n, int64_t lda,
                              const double* d2, const double* z, double* part,
                              int32_t* nparts_host, void* stream);

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

/* skb_directions plus avs = A (v ./ s), the v-invariant recheck's product
 * (ipm_core.py:502), in the same pass over A; adx and avs are bitwise those of
 * skb_directions and skb_gemv_ratio. Dense m <= 1024 only (else
 * SKB_ERR_UNSUPPORTED: use the two separate passes). */
int skb_directions_v(const double* A, int64_t m, int64_t n, int64_t lda, const double* dy,
                     const double* x, const double* s, const double* v, const double* r_d,
                     double sigma_mu, double* ds, double* dx, double* atdy, double* adx,
                     double* avs, void* workspace, size_t ws_bytes, void* stream);

/* make_iterate's pass at a precomputed (x_new, s_new) fused with the next step's
 * build_rhs (ipm_core.py:94-102, :196-206): r_d = A' y_new + s_new - c,
 * r_p = A x_new - b (b nullable), p = A (x_new - smu/s_new [- (x_new/s_new) r_d])
 * [- r_p when p_sub_rp], smu = *smu_dev (skb_sigma_mu). r_d, r_p and p are bitwise
 * those of skb_iterate and skb_rhs. Dense m <= 2048 (else SKB_ERR_UNSUPPORTED). */
int skb_iterate_rhs(const double* A, int64_t m, int64_t n, int64_t lda, const double* xn,
                    const double* sn, const double* y_new, const double* c, const double* smu_dev,
                    int32_t infeasible, const double* b, double* r_p, double* r_d, double* p,
                    int32_t p_sub_rp, void* workspace, size_t ws_bytes, void* stream);

/* x_new = x + alpha dx, s_new = s + alpha ds (make_iterate's rounding, no FMA). */
int skb_step_xs(const double* x, const double* dx, const double* s, const double* ds,
                double alpha, double* xn, double* sn, int64_t n, void* stream);

/* out[0] = sigma * (sum[0] / n) on the device (the next step's sigma * mu). */
int skb_sigma_mu(const double* sum, double n, double sigma, double* out, void* stream);

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

/* ---------------------------------------------- sparse A (CSC), config c4 --
 * The same passes over A stored as CSC: colptr (int64, n+1), rowidx (int32),
 * vals (double); z and the CTA's m-vector partial in shared memory; partials
 * reduced in a fixed order. The passes that produce an m-vector take a plan
 (skb_csc_plan_build, once per matrix: whole columns cut into chunks that fit
 * a shared-memory stage, stored as vals | row u16 + row-sorted slot u16 |
 * column offsets u16, see csrc/skb_cscplan.cuh): the chunks stream through a
 * TMA bulk-copy ring and the scatter is a per-warp pass over row-disjoint
 * ranges of the row-sorted products -- no atomics, deterministic, 12 B/nnz
 * + 10 B/column per pass. plan == NULL (or m > 65535, a column too long for a
 * stage, z + partial too large for shared memory) runs the thread-per-column
 * kernel with shared atomics (m <= 14080). */
size_t skb_csc_plan_bytes(int64_t m, int64_t n, int64_t nnz, int64_t maxlen);
/* ELL head records (m <= 65535): one 64-byte record per column with its first
 * 5 rows (u16) and values; with them every pass (`ell`, nullable) reads a
 * column as one contiguous load instead of colptr -> rowidx -> vals. */
size_t skb_csc_ell_bytes(int64_t m, int64_t n);
int skb_csc_ell_build(const int64_t* colptr, const int32_t* rowidx, const double* vals,
                      int64_t m, int64_t n, void* ell, size_t ell_bytes, void* stream);
int skb_csc_plan_build(const int64_t* colptr, const int32_t* rowidx, const double* vals,
                       int64_t m, int64_t n, int64_t nnz, int64_t maxlen, void* plan,
                       size_t plan_bytes, int64_t* nchunks_out, void* stream);
int skb_csc_normal_apply(const int64_t* colptr, const int32_t* rowidx, const double* vals,
                         const void* plan, int64_t plan_chunks, const void* ell, int64_t m, int64_t n,
                         const double* d2, const double* z, double* u, const double* sub,
                         const int* gate, void* workspace, size_t ws_bytes, void* stream);
int skb_csc_gemv(const int64_t* colptr, const int32_t* rowidx, const double* vals,
                 const void* plan, int64_t plan_chunks, const void* ell, int64_t m, int64_t n, const double* x,
                 double* u, const double* sub, void* workspace, size_t ws_bytes, void* stream);
int skb_csc_gemv_ratio(const int64_t* colptr, const int32_t* rowidx, const double* vals,
                       const void* plan, int64_t plan_chunks, const void* ell, int64_t m, int64_t n,
                       const double* v, const double* s, double* u, const double* sub,
                       void* workspace, size_t ws_bytes, void* stream);
int skb_csc_rhs(const int64_t* colptr, const int32_t* rowidx, const double* vals,
                const void* plan, int64_t plan_chunks, const void* ell, int64_t m, int64_t n, const double* x,
                const double* s, const double* r_d, double sigma_mu, double* p,
                const double* r_p, void* workspace, size_t ws_bytes, void* stream);
int skb_csc_gemv_t(const int64_t* colptr, const int32_t* rowidx, const double* vals,
                   const void* plan, int64_t plan_chunks, const void* ell, int64_t m, int64_t n,
                   const double* y, const double* add, const double* sub, double* t,
                   void* workspace, size_t ws_bytes, void* stream);
int skb_csc_directions(const int64_t* colptr, const int32_t* rowidx, const double* vals,
                       const void* plan, int64_t plan_chunks, const void* ell, int64_t m, int64_t n,
                       const double* dy, const double* x, const double* s, const double* v,
                       const double* r_d, double sigma_mu, double* ds, double* dx, double* atdy,
                       double* adx, void* workspace, size_t ws_bytes, void* stream);
int skb_csc_iterate(const int64_t* colptr, const int32_t* rowidx, const double* vals,
                    const void* plan, int64_t plan_chunks, const void* ell, int64_t m, int64_t n, const double* x,
                    const double* dx, const double* s, const double* ds, double alpha,
                    const double* y_new, const double* b, const double* c, double* x_out,
                    double* s_out, double* r_p, double* r_d, void* workspace, size_t ws_bytes,
                    void* stream);
/* Bit-exact ADW for CSC A (ascending-j sums per (row, bucket), no FMA). With
 * the matrix's ELL records (`ell`, nullable; this call writes d into them) and
 * 2048 < m <= 65535: one CTA per bucket, records prefetched a batch ahead,
 * each batch's terms radix-sorted by (row, member) and applied run by run. */
int skb_csc_sketch_apply(const int64_t* colptr, const int32_t* rowidx, const double* av,
                         void* ell, int64_t m, int64_t n, const double* d, const int32_t* cols,
                         const double* vals, int32_t s, int32_t w, double* X, int64_t ldx,
                         void* workspace, size_t ws_bytes, void* stream);
/* Dense column-major copy (A zeroed by the caller). */
int skb_csc_to_dense(const int64_t* colptr, const int32_t* rowidx, const double* vals, int64_t n,
                     double* A, int64_t lda, void* stream);

/* ------------------------------------------------------------ K2 sketch --
 * X = (A diag(d) W)' for the sparse-sign W given by cols/vals (n x s), i.e.
 * X[b*ldx + i] = ADW[i, b] (bucket-major, w rows of length m). Bit-exact with
 * apply_sketch (sketching.py:142-161): per (i, b) the terms fl(fl(A_ij d_j) v)
 * are added in ascending j without FMA. m <= 2048, w*4 bytes <= 220 KB.
 * Workspace: skb_sketch_workspace_bytes(n, w, s). */
size_t skb_sketch_workspace_bytes(int64_t n, int32_t w, int32_t s);
int skb_sketch_apply(const double* A, int64_t m, int64_t n, int64_t lda, const double* d,
                     const int32_t* cols, const double* vals, int32_t s, int32_t w, double* X,
                     int64_t ldx, void* workspace, size_t ws_bytes, void* stream);

/* Identity sketch (w >= n, sketching.py:155-156): X[j*ldx + i] = A_ij * d_j. */
int skb_scale_columns(const double* A, int64_t m, int64_t n, int64_t lda, const double* d,
                      double* X, int64_t ldx, void* stream);

/* v_j = [sqrt(x_j s_j) *] sum_k vals[j,k] u[cols[j,k]]  (SketchOperator.matvec,
 * sketching.py:72-80; compute_v, correction.py:58). x == NULL: W u only. */
int skb_sketch_gather(const int32_t* cols, const double* vals, int32_t s, int64_t n,
                      const double* u, const double* x, const double* sv, double* v,
                      void* stream);

/* ------------------------------------------------------ K9 Gaussian sketch --
 * build_gaussian_sketch (sketching.py:131-139): W = standard_normal((n, w)) /
 * sqrt(w) from Generator(Philox(seed)), bit-exact with numpy's ziggurat
 * (tables taken from numpy's build). Writes draws [lo, count) (lo = 0,
 * count = n*w: the whole W). Synchronises the stream.
 * skb_gaussian_apply: X = (A diag(d) W)' (w x m) as one DMMA GEMM. */
size_t skb_gaussian_workspace_bytes(int64_t count);
/* Extra workspace (8 bytes per stream position) that lets the generator store
 * the fast draws' values in its classify pass instead of running Philox again
 * in the emit pass; optional (without it: the recompute path, same bits). */
size_t skb_gaussian_value_bytes(int64_t count);
int skb_gaussian_sketch(uint64_t key0, uint64_t key1, int64_t lo, int64_t count, int32_t w,
                        double* W, void* workspace, size_t ws_bytes, void* stream);

/* The draws whose ziggurat attempts START in stream positions [p0, p1)
 * (multiples of 4096), in order, / sqrt(w), into out[0, min(count, cap));
 * *count_host = count. Consecutive ranges partition the draw sequence
 * (a rank-parallel W: each rank generates one range, then exchanges by global
 * draw index). Synchronises the stream. Workspace: skb_gaussian_workspace_bytes. */
int skb_gaussian_range(uint64_t key0, uint64_t key1, uint64_t p0, uint64_t p1, int32_t w,
                       double* out, int64_t cap, uint64_t* count_host, void* workspace,
                       size_t ws_bytes, void* stream);
int skb_gaussian_apply(const double* A, int64_t m, int64_t n, int64_t lda, const double* d,
                       const double* W, int32_t w, double* X, int64_t ldx, void* workspace,
                       size_t ws_bytes, void* stream);
/* v = sqrt(x .* s) .* t (compute_v for a dense or identity W, correction.py:58). */
int skb_sqrt_xs_scale(const double* t, const double* x, const double* s, double* v, int64_t n,
                      void* stream);

/* ------------------------------------------------------- K3 factor (FP64) --
 * Replaces np.linalg.svd(ADW) (preconditioning.py:46). Factor matrices are
 * Mp x Mp row-major (Mp = skb_factor_padded_dim(m), identity-padded).
 * skb_factor_cholqr2: Q = X'X = L L' by CholeskyQR2 (shifted CholeskyQR3 when
 * the first Gram Cholesky breaks down). Outputs Linv = L^-1 (lower), LinvT
 * (upper), Lfac = L. stats_host[4] = {min|L_ii|, max|L_ii|, shifted, status}.
 * Synchronises the stream. Workspace: skb_factor_workspace_bytes(m, w). */
int32_t skb_factor_padded_dim(int32_t m);
size_t skb_factor_workspace_bytes(int32_t m, int32_t w);
int skb_factor_cholqr2(const double* X, int64_t ldx, int32_t w, int32_t m, double* Linv,
                       double* LinvT, double* Lfac, double* stats_host, void* workspace,
                       size_t ws_bytes, void* stream);

/* C = alpha op(A) op(B) + beta C (row-major, FP64 DMMA tensor cores, batched).
 * The GEMM-class work of the reference's LAPACK gesdd / numpy matmul
 * (preconditioning.py:46, sketching.py:158-159, krylov_solvers.py:50). */
int skb_gemm(int32_t ta, int32_t tb, int32_t M, int32_t N, int32_t K, double alpha,
             const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
             int64_t ldc, int32_t lower_only, int32_t batch, int64_t strideA, int64_t strideB,
             int64_t strideC, void* workspace, size_t ws_bytes, void* stream);

/* The same product emulated in FP64 on the INT8 tensor cores (CRT over 16
 * moduli, csrc/skb_ozaki.cu; the same reference seams as skb_gemm, results
 * within fp64 rounding of them); lower_only writes j <= i only. skb_gemm routes
 * large unbatched products here (SKB_GEMM_EMU=0 disables). Returns
 * SKB_ERR_UNSUPPORTED when cuBLASLt cannot be loaded or the workspace is short. */
int skb_gemm_ozaki(int32_t ta, int32_t tb, int32_t M, int32_t N, int32_t K, double alpha,
                   const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                   double* C, int64_t ldc, int32_t lower_only, void* workspace, size_t ws_bytes,
                   void* stream);
size_t skb_gemm_ozaki_workspace_bytes(int32_t M, int32_t N, int32_t K);
int64_t skb_gemm_ozaki_calls(void);

/* Batched INT8 x INT8 -> INT32 GEMM on the tcgen05 tensor cores (TMA-fed,
 * TMEM accumulators; csrc/skb_i8gemm.cu), the core of the FP64 emulation:
 * C_l[r][c] = sum_{k in [k0,k1)} A_l[ar0+r][k] B_l[br0+c][k] for l < n, with
 * K-major int8 slabs (Kp bytes per row, Ra / Rb rows, batch strides sa / sb),
 * int32 C (row stride ldc, batch stride sc). k0 % 128 == 0, cols % 16 == 0;
 * entries of [k0, k1) the caller does not want must be zero in the slabs.
 * tri = 1 computes only the 256 x 256 tiles meeting col <= row + tri_off. */
int skb_i8gemm_batched(const int8_t* A, int64_t Ra, int64_t sa, const int8_t* B, int64_t Rb,
                       int64_t sb, int64_t Kp, int32_t* C, int64_t ldc, int64_t sc, int32_t rows,
                       int32_t cols, int32_t ar0, int32_t br0, int32_t k0, int32_t k1, int32_t n,
                       int32_t tri, int32_t tri_off, void* stream);

/* skb_i8gemm_batched with a residue epilogue: each int32 product is stored as its
 * symmetric residue mod mod[l] in int8 (C8: row stride ldc8, batch stride sc8, in
 * bytes, multiples of 16; p = 256 ties as -128), which is all the FP64
 * emulation's CRT needs (preconditioning.py:46 / sketching.py:158-159 products).
 * Persistent 2-SM kernel; n <= 24. */
int skb_i8gemm_residues(const int8_t* A, int64_t Ra, int64_t sa, const int8_t* B, int64_t Rb,
                        int64_t sb, int64_t Kp, int8_t* C8, int64_t ldc8, int64_t sc8,
                        int32_t rows, int32_t cols, int32_t ar0, int32_t br0, int32_t k0,
                        int32_t k1, int32_t n, int32_t tri, int32_t tri_off, const double* mod,
                        void* stream);

/* One-shot all-reduce of an m-vector over NVLink peer memory (csrc/skb_p2p.cu):
 * the exchange SURVEY.md §8(e) puts after every sharded A-pass that yields an
 * m-vector (reference: the single-process sums of krylov_solvers.py:46-47,
 * ipm_core.py:196-242). Peers' symmetric buffers ([2][ld] doubles) and flag
 * words (>= skb_p2p_max_blocks(m) u64) are opened with skb_ipc_open; mode 0 =
 * publish + gather, 1 / 2 = one half (single-process tests). A peer whose flag
 * is not seen within timeout_cycles (SM clock) sets *err = 1 (sticky) and the
 * result is NaN; the caller reads err with its per-step scalars and raises. */
int skb_p2p_alloc(int64_t bytes, uint64_t* dev_ptr_out);
int skb_p2p_free(uint64_t dev_ptr);
int skb_ipc_handle(void* dev_ptr, void* handle_out);
int skb_ipc_open(const void* handle, uint64_t* dev_ptr_out);
int skb_ipc_close(uint64_t dev_ptr);
int32_t skb_p2p_can_access(int32_t device, int32_t peer);
int32_t skb_p2p_max_blocks(int64_t m);
int skb_p2p_allreduce(const double* local, double* out, int64_t m, int64_t ld, int32_t rank,
                      int32_t world, const uint64_t* data_ptrs, const uint64_t* flag_ptrs,
                      uint64_t epoch, int32_t mode, int64_t timeout_cycles, int* err,
                      void* stream);

/* Blocked Cholesky (lower, in place) and triangular inverse; Mp % 64 == 0.
 * status: device int, SKB_ST_CHOL_FAIL on a nonpositive pivot. */
int skb_potrf(double* G, int64_t ld, int32_t Mp, int* status, void* workspace, size_t ws_bytes,
              void* stream);
int skb_trtri(const double* L, double* Li, int64_t ld, int32_t Mp, void* workspace,
              size_t ws_bytes, void* stream);

/* y = M x, M row-major rows x cols; tri 0 full, 1 lower (k <= i), 2 upper (k >= i).
 * apply_inv = two calls (Linv then LinvT); apply_pinv_adw = one full call on X. */
int skb_rowdot_gemv(const double* M, int64_t ld, int32_t rows, int32_t cols, int32_t tri,
                    const double* x, double* y, const int* gate, void* stream);

/* ------------------------------------------------------------- K6 PCG --
 * pcg (krylov_solvers.py:65-105) with M^-1 = Linv' Linv. state: device buffer
 * of skb_pcg_state_bytes(); trace: device (t_max+1) doubles. The step kernels
 * are gated on the state so a fixed launch sequence can run after convergence
 * (multi-GPU drivers interleave NCCL allreduces between them). */
size_t skb_pcg_state_bytes(void);
int skb_pcg_init(const double* p, double* r, double* dy, int64_t m, void* state, void* stream);
int skb_pcg_init2(const double* r, const double* z, double* q, int64_t m, double tol, void* state,
                  double* trace, void* stream);
int skb_pcg_step_a(const double* q, const double* Aq, double* dy, double* r, int64_t m,
                   void* state, void* stream);
int skb_pcg_step_b(const double* r, const double* z, double* q, int64_t m, int32_t t_max,
                   void* state, double* trace, void* stream);

/* Chebyshev iteration (krylov_solvers.py:108-153) on the same state: after
 * skb_pcg_init and z = Q^-1 r, skb_cheb_init (tol < 0: run the full schedule);
 * per step k: skb_cheb_step_q (q = z | z + beta q; dy += alpha q), the normal
 * apply Aq = A D^2 A' q, skb_cheb_step_r (r -= alpha Aq), z = Q^-1 r,
 * skb_cheb_trace. alpha_k, beta_k come from the fixed band (host scalars). */
int skb_cheb_init(const double* r, const double* z, int64_t m, double tol, void* state,
                  double* trace, void* stream);
int skb_cheb_step_q(const double* z, double* q, double* dy, int64_t m, double alpha, double beta,
                    int32_t first, void* state, void* stream);
int skb_cheb_step_r(double* r, const double* Aq, int64_t m, double alpha, void* state,
                    void* stream);
int skb_cheb_trace(const double* r, const double* z, int64_t m, int32_t t_max, void* state,
                   double* trace, void* stream);

/* Direct solver pieces (krylov_solvers.py:156-171): G = A diag(w) A' (lower
 * tiles, DMMA), transpose, identity padding of a factor matrix. */
int skb_weighted_gram(const double* A, int64_t m, int64_t n, int64_t lda, const double* wts,
                      double* G, int64_t ldg, void* workspace, size_t ws_bytes, void* stream);
int skb_transpose(const double* S, double* D, int64_t ld, int32_t n, void* stream);
int skb_set_identity_pad(double* G, int64_t ld, int32_t m, int32_t Mp, void* stream);

/* Whole single-device PCG, one synchronisation. vec: 5*ldv doubles scratch.
 * out_host = {iterations, converged, status bits}; trace_host: iterations+1. */
int skb_pcg_solve(const double* A, int64_t m, int64_t n, int64_t lda, const double* d2,
                  const double* Linv, const double* LinvT, int64_t ld, const double* p,
                  double* dy, double* vec, int64_t ldv, int32_t t_max, double tol, void* state,
                  double* trace, double* trace_host, int32_t* out_host, void* workspace,
                  size_t ws_bytes, void* stream);

/* ------------------------------------------------- K8 step reductions --
 * Deterministic fused elementwise + reduction passes (one launch each; the
 * results land in the device array `out`). The reduction workspace
 * (skb_reduce_workspace_bytes) holds a ticket word that must start at zero
 * (skb_reduce_workspace_init) and must not be shared with other scratch. */
size_t skb_reduce_workspace_bytes(void);
int skb_reduce_workspace_init(void* workspace, void* stream);

/* d = sqrt(clip(x/s, 1e-32, 1e32)), d2 = d*d (ipm_core.py:415-421, krylov_solvers.py:40);
 * out = {clip_count, min x, min s}. */
int skb_step_prep(const double* x, const double* s, int64_t n, double* d, double* d2,
                  double* out, void* workspace, size_t ws_bytes, void* stream);

/* out = {sum x.s, min x.s, min x, min s, ||r_d||^2}  (duality_measure / in_neighborhood). */
int skb_iter_stats(const double* x, const double* s, const double* r_d, int64_t n, double* out,
                   void* workspace, size_t ws_bytes, void* stream);

/* out = {max|comp|, max|x s|, max|x ds|, max|s dx|, dx'ds, ||dx||^2, sum(x ds + s dx),
 *        x'ds, s'dx, sum v} with comp = x ds + s dx + x s - sigma_mu + v
 * (assemble_directions ipm_core.py:237-242, max_alpha :286-289, argmin :328, v_bar :524). */
int skb_dir_stats(const double* x, const double* s, const double* dx, const double* ds,
                  const double* v, double sigma_mu, int64_t n, double* out, void* workspace,
                  size_t ws_bytes, void* stream);

/* Vectorised _first_crossing (ipm_core.py:245-275) for max_alpha's proximity
 * quadratics: a = dx ds - g1a, b = x ds + s dx - g1b, c = x s - g1mu.
 * out = {min c, max|c|, crossing with c clamped at 0 (inf if none)}. */
int skb_crossing(const double* x, const double* s, const double* dx, const double* ds, double g1a,
                 double g1b, double g1mu, int64_t n, double* out, void* workspace,
                 size_t ws_bytes, void* stream);

/* out = {sum t^2, sum t, max|t|, min t} for t = a [- sub]. */
int skb_vec_stats(const double* a, const double* sub, int64_t n, double* out, void* workspace,
                  size_t ws_bytes, void* stream);

/* feasible_start pieces (ipm_core.py:814-969):
 * skb_ratio_min: out = {min over dv<0 of -v/dv, min over dw<0 of -w/dw} (inf if none);
 * skb_centering_grid: for 8 step lengths alphas[k], prod = (x + a dx)(s + a ds),
 *   out[3k..3k+2] = {min prod, sum prod, count(prod <= 0)};
 * skb_zero_col_fill: x[j] = 1 for every all-zero column of A. */
int skb_ratio_min(const double* v, const double* dv, const double* w, const double* dw,
                  int64_t n, double* out, void* workspace, size_t ws_bytes, void* stream);
int skb_centering_grid(const double* x, const double* s, const double* dx, const double* ds,
                       const double* alphas, int64_t n, double* out, void* workspace,
                       size_t ws_bytes, void* stream);
int skb_zero_col_fill(const double* A, int64_t m, int64_t n, int64_t lda, double* x,
                      void* stream);

/* y = x + alpha d;  out = a - b. */
int skb_axpy(const double* x, double alpha, const double* d, double* y, int64_t n, void* stream);
int skb_sub(const double* a, const double* b, double* out, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SKB_H_ */
