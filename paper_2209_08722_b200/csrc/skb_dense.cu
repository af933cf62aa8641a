// K3/K5/K7: the sketched preconditioner on device, FP64 throughout.
//
// Replaces build_preconditioner's thin SVD (reference preconditioning.py:38-51,
// LAPACK gesdd) and its applications apply_inv / apply_pinv_adw (:59-66).
// With X = (ADW)' (w x m, stored bucket-major by skb_sketch_apply):
//   CholeskyQR2   G1 = X'X = L1 L1',  Y = X L1^-T,  G2 = Y'Y = L2 L2',
//                 L = L1 L2  (so Q = ADW ADW' = X'X = L L'),  Linv = L2^-1 L1^-1
//   Q^-1 r      = Linv' (Linv r)                      two triangular gemvs
//   (ADW)^+ r   = ADW' Q^-1 r = X Q^-1 r              (full row rank)
// CholeskyQR2 recovers R to QR accuracy where one Gram Cholesky squares the
// conditioning. A failed first Cholesky (kappa(ADW) ~> 1e8)
// is retried with the shifted CholeskyQR3 of Fukaya et al.
//
// GEMM-class work runs on the FP64 tensor pipe through warp-level
// mma.sync.aligned.m8n8k4 f64 (SASS DMMA): sm_100a has no tcgen05 kind for
// FP64. Everything else here is latency- or HBM-bound.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "skb_common.cuh"
#include "skb_internal.h"

namespace skb {

// ------------------------------------------------------------------ DMMA GEMM
// C[M][N] = alpha * sum_k opA(i,k) opB(k,j) + beta * C, all row-major.
// opA(i,k) = TA ? A[k*lda+i] : A[i*lda+k];  opB(k,j) = TB ? B[j*ldb+k] : B[k*ldb+j].
// Tile 64x64x16, 4 warps (2x2), warp tile 32x32 = 4x4 m8n8k4 fragments.
// lower_only: skip tiles strictly above the diagonal (symmetric / triangular C).
// Split-K: blockIdx.z = batch * splits + split; split partials go to `part`
// and are summed in split order by gemm_splitk_reduce (deterministic).
constexpr int GBM = 64, GBN = 64, GBK = 16, GPAD = 8;

struct GemmArgs {
  const double* A;
  const double* B;
  double* C;
  double* part;  // split-K partial buffer (nullptr when splits == 1)
  int64_t lda, ldb, ldc;
  int64_t sA, sB, sC;  // batch strides
  int M, N, K;
  int splits, kchunk;
  double alpha, beta;
  int ta, tb, lower_only;
  const double* kscale;  // optional: opA(i,k) *= kscale[k] (weighted SYRK A diag(w) A')
  // Triangular operands (zeros outside are skipped, not multiplied): tri_a 1 =
  // opA lower (k <= i), 2 = upper (k >= i); tri_b 1 = opB lower (k >= j),
  // 2 = upper (k <= j). Each tile trims its k range accordingly.
  int tri_a, tri_b;
};

// The k range [kb, ke) a (i0, j0, bm x bn) tile needs under the tri flags.
SKB_DEV void tri_krange(const GemmArgs& g, int i0, int j0, int bm, int bn, int& kb, int& ke) {
  if (g.tri_a == 1) ke = min(ke, i0 + bm);
  else if (g.tri_a == 2) kb = max(kb, i0);
  if (g.tri_b == 1) kb = max(kb, j0);
  else if (g.tri_b == 2) ke = min(ke, j0 + bn);
}

SKB_DEV void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(128) dgemm_kernel(GemmArgs g) {
  __shared__ double As[2][GBK][GBM + GPAD];
  __shared__ double Bs[2][GBK][GBN + GPAD];
  const int batch = blockIdx.z / g.splits, split = blockIdx.z % g.splits;
  const int bm = blockIdx.y, bn = blockIdx.x;
  if (g.lower_only && bn * GBN > bm * GBM + GBM - 1) return;
  const int i0 = bm * GBM, j0 = bn * GBN;
  const double* A = g.A + (int64_t)batch * g.sA;
  const double* B = g.B + (int64_t)batch * g.sB;
  int k_begin = split * g.kchunk, k_end = min(g.K, k_begin + g.kchunk);
  tri_krange(g, i0, j0, GBM, GBN, k_begin, k_end);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int gq = lane >> 2, tq = lane & 3;

  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  double ra[8], rb[8];
  // element e of this thread's tile load: tile index t = tid + 128*e in [0, 1024)
  auto load_tiles = [&](int k0) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int t = tid + 128 * e;
      int kk, ii;
      if (g.ta) {
        kk = t >> 6;
        ii = t & 63;
      } else {
        ii = t >> 4;
        kk = t & 15;
      }
      const int gi = i0 + ii, gk = k0 + kk;
      double v = 0.0;
      if (gi < g.M && gk < k_end) {
        v = g.ta ? A[(int64_t)gk * g.lda + gi] : A[(int64_t)gi * g.lda + gk];
        if (g.kscale) v *= g.kscale[gk];
      }
      ra[e] = v;
      int kb, jj;
      if (g.tb) {
        jj = t >> 4;
        kb = t & 15;
      } else {
        kb = t >> 6;
        jj = t & 63;
      }
      const int gj = j0 + jj, gk2 = k0 + kb;
      double u = 0.0;
      if (gj < g.N && gk2 < k_end)
        u = g.tb ? B[(int64_t)gj * g.ldb + gk2] : B[(int64_t)gk2 * g.ldb + gj];
      rb[e] = u;
    }
  };
  auto store_tiles = [&](int buf) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int t = tid + 128 * e;
      if (g.ta)
        As[buf][t >> 6][t & 63] = ra[e];
      else
        As[buf][t & 15][t >> 4] = ra[e];
      if (g.tb)
        Bs[buf][t & 15][t >> 4] = rb[e];
      else
        Bs[buf][t >> 6][t & 63] = rb[e];
    }
  };

  int buf = 0;
  if (k_begin < k_end) {
    load_tiles(k_begin);
    store_tiles(0);
  }
  __syncthreads();
  for (int k0 = k_begin; k0 < k_end; k0 += GBK) {
    const bool more = k0 + GBK < k_end;
    if (more) load_tiles(k0 + GBK);
#pragma unroll
    for (int kk = 0; kk < GBK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) af[a] = As[buf][kk + tq][wm + a * 8 + gq];
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = Bs[buf][kk + tq][wn + b * 8 + gq];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma(acc[a][b], af[a], bf[b]);
    }
    if (more) {
      store_tiles(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }

  // epilogue
  const bool direct = g.splits == 1;
  double* C = direct ? g.C + (int64_t)batch * g.sC
                     : g.part + ((int64_t)blockIdx.z) * (int64_t)g.M * g.N;
  const int64_t ldc = direct ? g.ldc : g.N;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int i = i0 + wm + a * 8 + gq, j = j0 + wn + b * 8 + tq * 2 + q;
        if (i < g.M && j < g.N) {
          double* dst = C + (int64_t)i * ldc + j;
          if (direct) {
            double v = g.alpha * acc[a][b][q];
            if (g.beta != 0.0) v = fma(g.beta, *dst, v);
            *dst = v;
          } else {
            *dst = acc[a][b][q];
          }
        }
      }
}

// Pipelined variant for 16-byte-aligned operands (even leading dims and batch
// strides, 16 B base pointers): CTA tile 128 x 64 x BK, 8 warps (4 x 2) of
// 32 x 32, an ST-stage cp.async ring (zero-filled at the M/N/K edges) so the
// global loads never pass through registers. Shared tiles keep the global
// orientation with row strides = 4 (mod 16) doubles, which makes every
// fragment read conflict-free in both 16-lane phases. Same k order and the
// same products as dgemm_kernel (kscale is applied to the A fragment).
constexpr int PBM = 128, PBN = 64;

template <int TA, int BK>
struct PTileA {  // TA=1: [k][i] (BK x 128), TA=0: [i][k] (128 x BK)
  static constexpr int kStride = TA ? PBM + 4 : BK + 4;
  static constexpr int kSize = TA ? BK * kStride : PBM * kStride;
};
template <int TB, int BK>
struct PTileB {  // TB=0: [k][j] (BK x 64), TB=1: [j][k] (64 x BK)
  static constexpr int kStride = TB ? BK + 4 : PBN + 4;
  static constexpr int kSize = TB ? PBN * kStride : BK * kStride;
};

SKB_DEV void cp_async16(double* smem, const double* gmem, int bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes)
               : "memory");
}
SKB_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
SKB_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <int TA, int TB, int PBK, int PST>
__global__ void __launch_bounds__(256, 2) dgemm_pipe_kernel(GemmArgs g) {
  extern __shared__ __align__(16) double psm[];
  using TAt = PTileA<TA, PBK>;
  using TBt = PTileB<TB, PBK>;
  constexpr int kStage = TAt::kSize + TBt::kSize + PBK;  // + the k-tile's kscale
  constexpr int kHalf = PBK / 2;                         // 16-byte chunks per k-row
  const int batch = blockIdx.z / g.splits, split = blockIdx.z % g.splits;
  const int bm = blockIdx.y, bn = blockIdx.x;
  if (g.lower_only && bn * PBN > bm * PBM + PBM - 1) return;
  const int i0 = bm * PBM, j0 = bn * PBN;
  const double* A = g.A + (int64_t)batch * g.sA;
  const double* B = g.B + (int64_t)batch * g.sB;
  int k_begin = split * g.kchunk, k_end = min(g.K, k_begin + g.kchunk);
  tri_krange(g, i0, j0, PBM, PBN, k_begin, k_end);
  const int nk = k_end > k_begin ? (k_end - k_begin + PBK - 1) / PBK : 0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int gq = lane >> 2, tq = lane & 3;

  auto load_stage = [&](int t, int stage) {
    double* As = psm + stage * kStage;
    double* Bs = As + TAt::kSize;
    const int k0 = k_begin + t * PBK;
#pragma unroll
    for (int e = 0; e < PBK / 4; ++e) {  // A: 128 * PBK / 2 16-byte chunks
      const int c = tid + 256 * e;
      int kk, ii, bytes;
      const double* src;
      double* dst;
      if (TA) {
        kk = c >> 6;
        ii = (c & 63) * 2;
        const int gi = i0 + ii, gk = k0 + kk;
        bytes = gk < k_end ? max(0, min(16, (g.M - gi) * 8)) : 0;
        src = bytes ? A + (int64_t)gk * g.lda + gi : A;
        dst = As + kk * TAt::kStride + ii;
      } else {
        ii = c / kHalf;
        kk = (c % kHalf) * 2;
        const int gi = i0 + ii, gk = k0 + kk;
        bytes = gi < g.M ? max(0, min(16, (k_end - gk) * 8)) : 0;
        src = bytes ? A + (int64_t)gi * g.lda + gk : A;
        dst = As + ii * TAt::kStride + kk;
      }
      cp_async16(dst, src, bytes);
    }
#pragma unroll
    for (int e = 0; e < PBK / 8; ++e) {  // B: 64 * PBK / 2 chunks
      const int c = tid + 256 * e;
      int kk, jj, bytes;
      const double* src;
      double* dst;
      if (TB) {
        jj = c / kHalf;
        kk = (c % kHalf) * 2;
        const int gj = j0 + jj, gk = k0 + kk;
        bytes = gj < g.N ? max(0, min(16, (k_end - gk) * 8)) : 0;
        src = bytes ? B + (int64_t)gj * g.ldb + gk : B;
        dst = Bs + jj * TBt::kStride + kk;
      } else {
        kk = c >> 5;
        jj = (c & 31) * 2;
        const int gj = j0 + jj, gk = k0 + kk;
        bytes = gk < k_end ? max(0, min(16, (g.N - gj) * 8)) : 0;
        src = bytes ? B + (int64_t)gk * g.ldb + gj : B;
        dst = Bs + kk * TBt::kStride + jj;
      }
      cp_async16(dst, src, bytes);
    }
    if (g.kscale && tid < kHalf) {  // the k-tile's PBK scale factors ride along
      const int gk = k0 + 2 * tid;
      const int bytes = max(0, min(16, (k_end - gk) * 8));
      cp_async16(Bs + TBt::kSize + 2 * tid, bytes ? g.kscale + gk : g.kscale, bytes);
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
  for (int s = 0; s < PST - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_async_commit();
  }
  for (int t = 0; t < nk; ++t) {
    cp_async_wait<PST - 2>();
    __syncthreads();
    if (t + PST - 1 < nk) load_stage(t + PST - 1, (t + PST - 1) % PST);
    cp_async_commit();
    const double* As = psm + (t % PST) * kStage;
    const double* Bs = As + TAt::kSize;
#pragma unroll
    for (int kk = 0; kk < PBK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
        af[a] = TA ? As[(kk + tq) * TAt::kStride + wm + a * 8 + gq]
                   : As[(wm + a * 8 + gq) * TAt::kStride + kk + tq];
#pragma unroll
      for (int b = 0; b < 4; ++b)
        bf[b] = TB ? Bs[(wn + b * 8 + gq) * TBt::kStride + kk + tq]
                   : Bs[(kk + tq) * TBt::kStride + wn + b * 8 + gq];
      if (g.kscale) {
        const double sc = Bs[TBt::kSize + kk + tq];  // zero-filled past k_end
#pragma unroll
        for (int a = 0; a < 4; ++a) af[a] *= sc;
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma(acc[a][b], af[a], bf[b]);
    }
  }
  cp_async_wait<0>();

  const bool direct = g.splits == 1;
  double* C = direct ? g.C + (int64_t)batch * g.sC
                     : g.part + ((int64_t)blockIdx.z) * (int64_t)g.M * g.N;
  const int64_t ldc = direct ? g.ldc : g.N;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int i = i0 + wm + a * 8 + gq, j = j0 + wn + b * 8 + tq * 2 + q;
        if (i < g.M && j < g.N) {
          double* dst = C + (int64_t)i * ldc + j;
          if (direct) {
            double v = g.alpha * acc[a][b][q];
            if (g.beta != 0.0) v = fma(g.beta, *dst, v);
            *dst = v;
          } else {
            *dst = acc[a][b][q];
          }
        }
      }
}

template <int TA, int TB, int BK, int ST>
static size_t pipe_smem_bytes() {
  return (size_t)ST * (PTileA<TA, BK>::kSize + PTileB<TB, BK>::kSize + BK) * sizeof(double);
}

template <int TA, int TB, int BK, int ST>
static void launch_pipe_cfg(const GemmArgs& g, dim3 grid, cudaStream_t st) {
  static bool configured = false;  // one per template instantiation
  const size_t smem = pipe_smem_bytes<TA, TB, BK, ST>();
  if (!configured) {
    cudaFuncSetAttribute(dgemm_pipe_kernel<TA, TB, BK, ST>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  dgemm_pipe_kernel<TA, TB, BK, ST><<<grid, 256, smem, st>>>(g);
}

// k-tile 32 with a 2-stage ring (one barrier per 32 k) measured 3-8% faster
// than 16 x 3 stages across the factor / Gaussian shapes; both fit 2 CTAs/SM.
template <int TA, int TB>
static void launch_pipe(const GemmArgs& g, dim3 grid, cudaStream_t st) {
  static const bool k16 = getenv("SKB_GEMM_K16") != nullptr;
  if (k16)
    launch_pipe_cfg<TA, TB, 16, 3>(g, grid, st);
  else
    launch_pipe_cfg<TA, TB, 32, 2>(g, grid, st);
}

static bool pipe_ok(const GemmArgs& g) {
  if (getenv("SKB_GEMM_NOPIPE")) return false;
  auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  return al(g.A) && al(g.B) && (g.lda % 2 == 0) && (g.ldb % 2 == 0) && (g.sA % 2 == 0) &&
         (g.sB % 2 == 0) && (!g.kscale || al(g.kscale));
}

__global__ void gemm_splitk_reduce_kernel(GemmArgs g, int nbatch) {
  const int64_t MN = (int64_t)g.M * g.N;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= MN * nbatch) return;
  const int batch = (int)(idx / MN);
  const int64_t r = idx - (int64_t)batch * MN;
  const int i = (int)(r / g.N), j = (int)(r - (int64_t)i * g.N);
  if (g.lower_only && j > i) return;
  double s = 0.0;
  for (int q = 0; q < g.splits; ++q) s += g.part[((int64_t)batch * g.splits + q) * MN + r];
  double* dst = g.C + (int64_t)batch * g.sC + (int64_t)i * g.ldc + j;
  double v = g.alpha * s;
  if (g.beta != 0.0) v = fma(g.beta, *dst, v);
  *dst = v;
}

// ----------------------------------------------------------------- Cholesky
constexpr int NB = 64;

// The 64 x 64 diagonal block at (k0, k0): Cholesky in place (lower) plus its
// inverse Dinv = L11^-1 (64 x 64, row-major), which turns the panel TRSM into a
// GEMM. 256 threads; thread t owns row i = t / 4, columns q4 + 4 j (q4 = t % 4,
// j < 16) in registers. Column c is published through a double-buffered
// shared vector, so each of the 64 right-looking steps costs ONE barrier,
// one rsqrt (computed redundantly by every thread) and <= 16 independent
// FMAs per thread; the inverse runs the same way over rows of L^-1. Loops
// are runtime loops over groups of 4 columns with the register row ROTATED
// by one group each time, so indices stay static and the code stays small
// (straight-line versions were instruction-fetch bound).
constexpr int LDP = NB + 1;
constexpr int kLeafThreads = 256;

// X = L^-1 for the lower 64 x 64 L in Lsm (rinv[q] = 1 / L_qq) into out (ld).
SKB_DEV void leaf_inverse(const double (*Lsm)[LDP], const double* rinv, double* out, int64_t ld) {
  // thread j < 64: column j of L^-1 by right-looking forward substitution, no
  // barriers; x is rotated every 8 rows (static register indices in a runtime
  // loop); rows q < j stay zero. out[q * ld + j] stores are coalesced over j.
  const int j = threadIdx.x;
  if (j >= NB) return;
  constexpr int R = 8;
  double x[NB + R];
#pragma unroll
  for (int k = 0; k < NB; ++k) x[k] = (k == j) ? 1.0 : 0.0;
#pragma unroll
  for (int k = NB; k < NB + R; ++k) x[k] = 0.0;
  for (int q0 = 0; q0 < NB; q0 += R) {
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int q = q0 + u;
      const double xq = x[u] * rinv[q];
      out[(int64_t)q * ld + j] = xq;
      // rows past 63 wrap onto real rows: they only feed discarded entries
#pragma unroll
      for (int k = u + 1; k < NB + u; ++k) x[k] = fma(-Lsm[(q0 + k) & (NB - 1)][q], xq, x[k]);
    }
#pragma unroll
    for (int k = 0; k < NB; ++k) x[k] = x[k + R];
#pragma unroll
    for (int k = NB; k < NB + R; ++k) x[k] = 0.0;
  }
}

// The 64 x 64 diagonal factor (+ inverse Dinv = L^-1, 64 x 64 row-major) of
// the tile at src (ld), L written to dst (ld_dst; may alias src).
SKB_DEV void diag_factor(const double* src, int64_t ld, double* dst, int64_t ld_dst, int* status,
                         double* Dinv) {
  __shared__ double Lsm[NB][LDP];
  __shared__ double colc[2][NB];
  __shared__ double rinv[NB];
  __shared__ int bad_s;
  const int t = threadIdx.x, i = t >> 2, q4 = t & 3;
  const double* B = src;
  double r[16];  // r[j] = A[i][q4 + 4 (j + g)] in column group g
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int k = q4 + 4 * j;
    r[j] = k <= i ? B[(int64_t)i * ld + k] : 0.0;
    Lsm[i][k] = 0.0;
  }
  if (t == 0) bad_s = 0;
  for (int c0 = 0; c0 < NB; c0 += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c0 + u, buf = u & 1;
      if (q4 == u && i >= c) colc[buf][i] = r[0];
      __syncthreads();
      const double piv = colc[buf][c];
      const double rs = rsqrt(piv);
      if (t == 0) {
        if (!(piv > 0.0)) bad_s = 1;
        rinv[c] = rs;
      }
      const double ai = colc[buf][i];
      if (q4 == u && i >= c) Lsm[i][c] = i == c ? piv * rs : ai * rs;
      if (i > c) {
        const double air = ai * (rs * rs);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int k = q4 + 4 * j + c0;  // column of r[j]
          if (k > c && k <= i) r[j] = fma(-air, colc[buf][k], r[j]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 15; ++j) r[j] = r[j + 1];
    r[15] = 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int k = q4 + 4 * j;
    dst[(int64_t)i * ld_dst + k] = Lsm[i][k];
  }
  if (bad_s) {
    if (t == 0) atomicOr(status, ST_CHOL_FAIL);
    return;
  }
  if (!Dinv) return;
  leaf_inverse(Lsm, rinv, Dinv, NB);
}


__global__ void __launch_bounds__(kLeafThreads) potrf_diag_kernel(double* G, int64_t ld, int k0,
                                                                   int nb, int* status,
                                                                   double* Dinv) {
  double* B = G + (int64_t)k0 * ld + k0;
  diag_factor(B, ld, B, ld, status, Dinv);
}

// ---- fused right-looking step (one launch per 64-wide panel, nb <= kStepMax)
// Step k runs one CTA per lower tile pair (i, j), k < j <= i < T: it forms the
// panel tiles L_ik = A_ik Dinv_k' and L_jk (64^3 DMMA products from shared
// memory), updates A_ij -= L_ik L_jk', CTA (i, k + 1) stores L_ik, and CTA
// (k + 1, k + 1) -- the only one updating the next diagonal tile -- factors
// that tile and inverts it for step k + 1 (Dinv ping-pongs between two
// buffers). One launch per panel instead of three, and the next diagonal
// factor overlaps the rest of the trailing update. Every product runs the
// same DMMA k sequence (0, 4, ..., 60 from zero) and the same epilogue
// rounding as the GEMM-based loop, so L is bitwise identical to it. L goes to
// a separate buffer Lo (the panel's A tiles are still being read during the
// step) and is copied back at the end.
constexpr int kSLD = NB + 4;  // row stride = 4 (mod 16) doubles: conflict-free fragment reads

SKB_DEV void tile_load(double* s, const double* g, int64_t ld) {
  for (int e = threadIdx.x; e < NB * NB / 2; e += kLeafThreads) {
    const int r = e >> 5, c = (e & 31) * 2;
    *reinterpret_cast<double2*>(s + r * kSLD + c) =
        *reinterpret_cast<const double2*>(g + (int64_t)r * ld + c);
  }
}

// acc[a][b] (warp tile 32 x 16 at (wr * 32, wc * 16)) = sum_q sA[row][q] sB[col][q]
SKB_DEV void tile_mm_nt(const double* sA, const double* sB, double (&acc)[4][2][2]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = warp >> 2, wc = warp & 3, gq = lane >> 2, tq = lane & 3;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll 4
  for (int kk = 0; kk < NB; kk += 4) {
    double af[4], bf[2];
#pragma unroll
    for (int a = 0; a < 4; ++a) af[a] = sA[(wr * 32 + a * 8 + gq) * kSLD + kk + tq];
#pragma unroll
    for (int b = 0; b < 2; ++b) bf[b] = sB[(wc * 16 + b * 8 + gq) * kSLD + kk + tq];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) dmma(acc[a][b], af[a], bf[b]);
  }
}

SKB_DEV void tile_store_acc(double* s, const double (&acc)[4][2][2]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = warp >> 2, wc = warp & 3, gq = lane >> 2, tq = lane & 3;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
      *reinterpret_cast<double2*>(s + (wr * 32 + a * 8 + gq) * kSLD + wc * 16 + b * 8 + tq * 2) =
          make_double2(acc[a][b][0], acc[a][b][1]);
}

// mode 0: the fused step above. Steps with more lower tile pairs than the GPU
// has SMs run it as two launches instead (the pair CTAs otherwise recompute
// both panel tiles, 3 GEMMs each, over several waves): mode 1, one CTA per
// tile row i, L_ik = A_ik Dinv_k' straight into Lo; mode 2, one CTA per pair,
// A_ij -= L_ik L_jk' from Lo (+ the next diagonal factor). Same products in the
// same order: bitwise identical.
__global__ void __launch_bounds__(kLeafThreads) potrf_step_kernel(double* G, int64_t ld,
                                                                   double* Lo, int64_t ldo, int k,
                                                                   double* Dbuf, int* status,
                                                                   int mode) {
  extern __shared__ __align__(16) double psm[];
  double* sAi = psm;
  double* sAj = sAi + NB * kSLD;
  double* sD = sAj + NB * kSLD;
  int i = 0, j = 0;
  if (mode == 1) {  // panel: tile row i = k + 1 + blockIdx.x
    i = k + 1 + blockIdx.x;
    tile_load(sAi, G + (int64_t)i * NB * ld + (int64_t)k * NB, ld);
    tile_load(sD, Dbuf + (k & 1) * NB * NB, NB);
    __syncthreads();
    double acc[4][2][2];
    tile_mm_nt(sAi, sD, acc);
    __syncthreads();
    tile_store_acc(sAi, acc);
    __syncthreads();
    double* o = Lo + (int64_t)i * NB * ldo + (int64_t)k * NB;
    for (int e = threadIdx.x; e < NB * NB / 2; e += kLeafThreads) {
      const int r = e >> 5, c = (e & 31) * 2;
      *reinterpret_cast<double2*>(o + (int64_t)r * ldo + c) =
          *reinterpret_cast<const double2*>(sAi + r * kSLD + c);
    }
    return;
  }
  if (k >= 0 && mode == 2) {
    const int p = blockIdx.x;
    int ii = (int)((sqrt(8.0 * p + 1.0) - 1.0) * 0.5);
    while ((ii + 1) * (ii + 2) / 2 <= p) ++ii;
    while (ii * (ii + 1) / 2 > p) --ii;
    i = k + 1 + ii;
    j = k + 1 + (p - ii * (ii + 1) / 2);
    tile_load(sAi, Lo + (int64_t)i * NB * ldo + (int64_t)k * NB, ldo);
    if (j != i) tile_load(sAj, Lo + (int64_t)j * NB * ldo + (int64_t)k * NB, ldo);
    __syncthreads();
    double acc[4][2][2];
    tile_mm_nt(sAi, j != i ? sAj : sAi, acc);  // L_ik L_jk'
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wr = warp >> 2, wc = warp & 3, gq = lane >> 2, tq = lane & 3;
    double* C = G + (int64_t)i * NB * ld + (int64_t)j * NB;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int r = wr * 32 + a * 8 + gq, c = wc * 16 + b * 8 + tq * 2 + q;
          if (i != j || c <= r) {
            double* dst = C + (int64_t)r * ld + c;
            *dst = fma(1.0, *dst, -acc[a][b][q]);
          }
        }
  } else if (k >= 0) {
    const int p = blockIdx.x;
    int ii = (int)((sqrt(8.0 * p + 1.0) - 1.0) * 0.5);
    while ((ii + 1) * (ii + 2) / 2 <= p) ++ii;
    while (ii * (ii + 1) / 2 > p) --ii;
    i = k + 1 + ii;
    j = k + 1 + (p - ii * (ii + 1) / 2);
    const double* Dk = Dbuf + (k & 1) * NB * NB;
    tile_load(sAi, G + (int64_t)i * NB * ld + (int64_t)k * NB, ld);
    if (j != i) tile_load(sAj, G + (int64_t)j * NB * ld + (int64_t)k * NB, ld);
    tile_load(sD, Dk, NB);
    __syncthreads();
    double acc[4][2][2], acc2[4][2][2];
    tile_mm_nt(sAi, sD, acc);                      // L_ik = A_ik Dinv_k'
    if (j != i) tile_mm_nt(sAj, sD, acc2);         // L_jk
    __syncthreads();
    tile_store_acc(sAi, acc);
    if (j != i) tile_store_acc(sAj, acc2);
    __syncthreads();
    const double* sLj = j != i ? sAj : sAi;
    if (j == k + 1) {  // the unique CTA of tile row i that stores L_ik
      double* o = Lo + (int64_t)i * NB * ldo + (int64_t)k * NB;
      for (int e = threadIdx.x; e < NB * NB / 2; e += kLeafThreads) {
        const int r = e >> 5, c = (e & 31) * 2;
        *reinterpret_cast<double2*>(o + (int64_t)r * ldo + c) =
            *reinterpret_cast<const double2*>(sAi + r * kSLD + c);
      }
    }
    tile_mm_nt(sAi, sLj, acc);                     // L_ik L_jk'
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wr = warp >> 2, wc = warp & 3, gq = lane >> 2, tq = lane & 3;
    double* C = G + (int64_t)i * NB * ld + (int64_t)j * NB;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int r = wr * 32 + a * 8 + gq, c = wc * 16 + b * 8 + tq * 2 + q;
          if (i != j || c <= r) {  // diagonal tiles: lower part only (upper stays zero)
            double* dst = C + (int64_t)r * ld + c;
            *dst = fma(1.0, *dst, -acc[a][b][q]);
          }
        }
  }
  if (i == k + 1 && j == k + 1) {  // the next diagonal tile: factor + invert it
    __syncthreads();                 // this CTA's global writes are visible to it
    const double* src = G + (int64_t)i * NB * ld + (int64_t)i * NB;
    diag_factor(src, ld, Lo + (int64_t)i * NB * ldo + (int64_t)i * NB, ldo, status,
                Dbuf + ((k + 1) & 1) * NB * NB);
  }
}

// G[lower tiles] <- Lo (the strict upper part of the diagonal tiles is zero in Lo).
__global__ void copy_lower_tiles_kernel(double* G, int64_t ld, const double* Lo, int64_t ldo,
                                        int nb) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t half = (int64_t)nb * nb / 2;
  if (idx >= half) return;
  const int r = (int)(idx / (nb / 2)), c = (int)(idx % (nb / 2)) * 2;
  if (c / NB > r / NB) return;
  *reinterpret_cast<double2*>(G + (int64_t)r * ld + c) =
      *reinterpret_cast<const double2*>(Lo + (int64_t)r * ldo + c);
}

constexpr size_t kStepSmem = (size_t)3 * NB * kSLD * sizeof(double);

// Inverses of the 64 x 64 diagonal blocks of a lower-triangular L (one CTA
// per block), with the row-parallel scheme of potrf_diag_kernel.
__global__ void __launch_bounds__(kLeafThreads) trtri_diag_kernel(const double* L, double* Li,
                                                                   int64_t ld) {
  __shared__ double Lsm[NB][LDP];
  __shared__ double rinv[NB];
  const int t = threadIdx.x, i = t >> 2, q4 = t & 3;
  const int64_t b0 = (int64_t)blockIdx.x * NB;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int k = q4 + 4 * j;
    Lsm[i][k] = k <= i ? L[(b0 + i) * ld + b0 + k] : 0.0;
  }
  __syncthreads();
  if (t < NB) rinv[t] = 1.0 / Lsm[t][t];
  __syncthreads();
  leaf_inverse(Lsm, rinv, Li + b0 * ld + b0, ld);
}

__global__ void set_identity_pad_kernel(double* G, int64_t ld, int m, int Mp) {
  // zero rows/cols >= m, unit diagonal there
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)Mp * Mp) return;
  const int i = (int)(idx / Mp), j = (int)(idx % Mp);
  if (i >= m || j >= m) G[(int64_t)i * ld + j] = (i == j) ? 1.0 : 0.0;
}

__global__ void zero_upper_kernel(double* G, int64_t ld, int Mp) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)Mp * Mp) return;
  const int i = (int)(idx / Mp), j = (int)(idx % Mp);
  if (j > i) G[(int64_t)i * ld + j] = 0.0;
}

__global__ void transpose_kernel(const double* __restrict__ S, double* __restrict__ D, int64_t ld,
                                 int n) {
  __shared__ double t[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = by + r, j = bx + threadIdx.x;
    if (i < n && j < n) t[r][threadIdx.x] = S[(int64_t)i * ld + j];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = bx + r, j = by + threadIdx.x;
    if (i < n && j < n) D[(int64_t)i * ld + j] = t[threadIdx.x][r];
  }
}

__global__ void add_diag_kernel(double* G, int64_t ld, int m, double shift) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) G[(int64_t)i * ld + i] += shift;
}

// stats[0] = trace(G) (= ||X||_F^2), stats[1] = min |L_ii|, stats[2] = max |L_ii|
__global__ void diag_stats_kernel(const double* G, int64_t ld, int m, double* out, int which) {
  __shared__ double buf[32];
  double s = 0.0, mn = INFINITY, mx = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double v = G[(int64_t)i * ld + i];
    s += v;
    mn = fmin(mn, fabs(v));
    mx = fmax(mx, fabs(v));
  }
  const double ts = block_sum(s, buf);
  mn = warp_min(mn);
  mx = warp_max(mx);
  __shared__ double smn[32], smx[32];
  if ((threadIdx.x & 31) == 0) {
    smn[threadIdx.x >> 5] = mn;
    smx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      mn = fmin(mn, smn[w]);
      mx = fmax(mx, smx[w]);
    }
    if (which == 0)
      out[0] = ts;
    else {
      out[1] = mn;
      out[2] = mx;
    }
  }
}

// dprod[i] = |L_ii| (init) or dprod[i] * |L_ii|: diag of a product of triangular factors.
__global__ void diag_accum_kernel(const double* L, int64_t ld, int m, double* dprod, int init) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const double v = fabs(L[(int64_t)i * ld + i]);
  dprod[i] = init ? v : dprod[i] * v;
}

// out[1] = min v, out[2] = max v (single CTA).
__global__ void vec_minmax_kernel(const double* v, int m, double* out) {
  __shared__ double smn[32], smx[32];
  double mn = INFINITY, mx = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    mn = fmin(mn, v[i]);
    mx = fmax(mx, v[i]);
  }
  mn = warp_min(mn);
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) {
    smn[threadIdx.x >> 5] = mn;
    smx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      mn = fmin(mn, smn[w]);
      mx = fmax(mx, smx[w]);
    }
    out[1] = mn;
    out[2] = mx;
  }
}

// ------------------------------------------------------------ row-dot gemv
// y[i] = sum_k M[i][k] x[k] over k in [lo(i), hi(i)); tri = 0 full, 1 lower (k<=i), 2 upper (k>=i).
// Warp per row. Optional: y = alpha*y... kept plain; scal (nullable) divides by scal[i].
__global__ void __launch_bounds__(256) rowdot_gemv_kernel(const double* __restrict__ Mx,
                                                          int64_t ld, int rows, int cols, int tri,
                                                          const double* __restrict__ x,
                                                          double* __restrict__ y,
                                                          const int* __restrict__ gate) {
  if (gate && *gate) return;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const int i = warp;
  const int lo = tri == 2 ? i : 0, hi = tri == 1 ? min(i + 1, cols) : cols;
  const double* row = Mx + (int64_t)i * ld;
  // 8 independent 256-byte loads in flight per warp (latency-bound at m ~ 1e3)
  double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  int k = lo + lane;
  for (; k + 7 * 32 < hi; k += 8 * 32) {
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = fma(__ldg(&row[k + 32 * u]), __ldg(&x[k + 32 * u]), acc[u]);
  }
#pragma unroll
  for (int u = 0; u < 8; ++u)
    if (k + 32 * u < hi) acc[u] = fma(__ldg(&row[k + 32 * u]), __ldg(&x[k + 32 * u]), acc[u]);
  const double s = warp_sum(((acc[0] + acc[1]) + (acc[2] + acc[3])) +
                            ((acc[4] + acc[5]) + (acc[6] + acc[7])));
  if (lane == 0) y[i] = s;
}

}  // namespace skb

using namespace skb;

// ----------------------------------------------------------------- host API

// Large unbatched products go to the INT8-tensor-core FP64 emulation
// (skb_ozaki.cu) when its cost model beats DMMA: 16 INT8 GEMMs at ~2.4 POP/s
// plus the HBM passes of the residue split and the CRT, against DMMA at
// ~30 TFLOP/s on the (triangle-trimmed) flops. SKB_GEMM_EMU=0 disables it,
// SKB_GEMM_EMU=2 forces it for every eligible shape (tests).
static int emulate_one(const GemmArgs& g, skb_ws* ws, cudaStream_t st);

static int try_emulated(const GemmArgs& g, int nbatch, skb_ws* ws, cudaStream_t st) {
  const char* env = getenv("SKB_GEMM_EMU");
  const int mode = env ? atoi(env) : 1;
  if (!mode || g.K < 256) return 1;
  const double M = g.M, N = g.N, K = g.K;
  double dm = 2.0 * M * N * K;
  if (g.lower_only) dm *= 0.5;
  if (g.tri_a || g.tri_b) dm *= 0.5;
  const double t_dmma = dm / 30e12;
  // triangles are exploited by 1280-wide slabs (~1/(2s) waste) in the emulation
  const double t_emu = 16.0 * 1.1 * dm / 2.4e15 + ((M + N) * K * 26.0 + M * N * 80.0) / 5e12 +
                       60e-6;
  if (mode == 1 && !(t_emu < 0.8 * t_dmma)) return 1;
  // batched (the triangular-inverse levels): one emulated product per item
  for (int bi = 0; bi < nbatch; ++bi) {
    GemmArgs gb = g;
    gb.A = g.A + (int64_t)bi * g.sA;
    gb.B = g.B + (int64_t)bi * g.sB;
    gb.C = g.C + (int64_t)bi * g.sC;
    const int rc = emulate_one(gb, ws, st);
    if (rc) return bi == 0 ? rc : (rc == 1 ? SKB_ERR_WORKSPACE : rc);
  }
  return 0;
}

static int emulate_one(const GemmArgs& g, skb_ws* ws, cudaStream_t st) {
  skb_oz_args o{};
  o.a = g.ta ? skb_oz_operand{g.A, 1, g.lda} : skb_oz_operand{g.A, g.lda, 1};
  o.b = g.tb ? skb_oz_operand{g.B, g.ldb, 1} : skb_oz_operand{g.B, 1, g.ldb};
  o.kscale = g.kscale;
  o.C = g.C;
  o.ldc = g.ldc;
  o.M = g.M;
  o.N = g.N;
  o.K = g.K;
  o.alpha = g.alpha;
  o.beta = g.beta;
  o.lower_only = g.lower_only;
  o.tri_a = g.tri_a;
  o.tri_b = g.tri_b;
  return skb_oz_gemm(o, ws, st);
}

static int gemm_launch(const GemmArgs& base, int nbatch, skb_ws* ws, cudaStream_t st) {
  GemmArgs g = base;
  if (g.M <= 0 || g.N <= 0) return 0;
  {
    const int rc = try_emulated(g, nbatch, ws, st);
    if (rc <= 0) return rc;
  }
  const bool pipe = pipe_ok(g);
  const int bmt = pipe ? PBM : GBM, bnt = pipe ? PBN : GBN;
  const int tm = (g.M + bmt - 1) / bmt, tn = (g.N + bnt - 1) / bnt;
  int tiles = tm * tn * nbatch;
  if (g.lower_only) tiles = (tiles + 1) / 2;
  const int target = 2 * skb_num_sms();
  int splits = 1;
  if (g.K > 256 && tiles < target) {
    splits = std::min((target + tiles - 1) / tiles, std::max(1, g.K / 256));
    splits = std::max(1, std::min(splits, 64));
    // bound the partial buffer by the remaining workspace
    const size_t per = (size_t)nbatch * g.M * g.N * 8;
    const size_t avail = ws->cap > ws->off + 512 ? ws->cap - ws->off - 512 : 0;
    while (splits > 1 && per * splits > avail) --splits;
  } else if (g.K >= 4096 && !g.lower_only) {
    // many tiles but a long K: split to fill the last wave (e.g. 512 tiles on
    // 296 slots run at 86%; 4 splits at 99%)
    const auto eff = [&](int sp) {
      const long c = (long)tiles * sp, w = (c + target - 1) / target;
      return (double)c / (double)(w * target);
    };
    const size_t per = (size_t)nbatch * g.M * g.N * 8;
    const size_t avail = ws->cap > ws->off + 512 ? ws->cap - ws->off - 512 : 0;
    double best = eff(1);
    for (int sp = 2; sp <= 8 && g.K / sp >= 512; ++sp)
      if (eff(sp) > best + 0.05 && per * sp <= avail) {
        best = eff(sp);
        splits = sp;
      }
  }
  g.splits = splits;
  g.kchunk = (((g.K + splits - 1) / splits) + GBK - 1) / GBK * GBK;
  g.splits = (g.K + g.kchunk - 1) / g.kchunk;
  if (g.splits < 1) g.splits = 1;
  g.part = nullptr;
  const size_t mark = ws->off;
  if (g.splits > 1) {
    g.part = (double*)skb_ws_take(ws, (size_t)nbatch * g.splits * g.M * g.N * 8);
    if (!g.part) {  // fall back to no split
      g.splits = 1;
      g.kchunk = std::max(g.K, 1);
    }
  }
  if (g.K <= 0) g.kchunk = 1;
  dim3 grid(tn, tm, nbatch * g.splits);
  if (!pipe)
    dgemm_kernel<<<grid, 128, 0, st>>>(g);
  else if (g.ta && g.tb)
    launch_pipe<1, 1>(g, grid, st);
  else if (g.ta)
    launch_pipe<1, 0>(g, grid, st);
  else if (g.tb)
    launch_pipe<0, 1>(g, grid, st);
  else
    launch_pipe<0, 0>(g, grid, st);
  if (g.splits > 1) {
    const int64_t tot = (int64_t)g.M * g.N * nbatch;
    gemm_splitk_reduce_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(g, nbatch);
  }
  ws->off = mark;
  return skb_launch_status(__func__);
}

static GemmArgs gemm_args(const double* A, int64_t lda, int ta, const double* B, int64_t ldb,
                          int tb, double* C, int64_t ldc, int M, int N, int K, double alpha,
                          double beta, int lower_only) {
  GemmArgs g{};
  g.A = A;
  g.B = B;
  g.C = C;
  g.lda = lda;
  g.ldb = ldb;
  g.ldc = ldc;
  g.M = M;
  g.N = N;
  g.K = K;
  g.alpha = alpha;
  g.beta = beta;
  g.ta = ta;
  g.tb = tb;
  g.lower_only = lower_only;
  g.splits = 1;
  return g;
}

extern "C" int skb_gemm(int32_t ta, int32_t tb, int32_t M, int32_t N, int32_t K, double alpha,
                        const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                        double* C, int64_t ldc, int32_t lower_only, int32_t batch, int64_t strideA,
                        int64_t strideB, int64_t strideC, void* workspace, size_t ws_bytes,
                        void* stream) {
  skb_ws ws = skb_ws_make(workspace, ws_bytes);
  GemmArgs g = gemm_args(A, lda, ta, B, ldb, tb, C, ldc, M, N, K, alpha, beta, lower_only);
  g.sA = strideA;
  g.sB = strideB;
  g.sC = strideC;
  return gemm_launch(g, std::max(1, batch), &ws, (cudaStream_t)stream);
}

// G = A diag(w) A' (lower tiles) for column-major A (n columns of lda): the
// normal matrix of the direct solver (krylov_solvers.py:50, NormalOperator.dense).
extern "C" int skb_weighted_gram(const double* A, int64_t m, int64_t n, int64_t lda,
                                 const double* wts, double* G, int64_t ldg, void* workspace,
                                 size_t ws_bytes, void* stream) {
  skb_ws ws = skb_ws_make(workspace, ws_bytes);
  GemmArgs g = gemm_args(A, lda, 1, A, lda, 0, G, ldg, (int)m, (int)m, (int)n, 1.0, 0.0, 1);
  g.kscale = wts;
  return gemm_launch(g, 1, &ws, (cudaStream_t)stream);
}

// X = (A diag(d) W)' for a dense Gaussian W (n x w row-major): X[b][i] =
// sum_j W[j][b] d_j A[i][j] as one DMMA GEMM (M = w, N = m, K = n) with the
// column scaling fused into the operand load (sketching.py:158-159, K9).
extern "C" int skb_gaussian_apply(const double* A, int64_t m, int64_t n, int64_t lda,
                                  const double* d, const double* W, int32_t w, double* X,
                                  int64_t ldx, void* workspace, size_t ws_bytes, void* stream) {
  skb_ws ws = skb_ws_make(workspace, ws_bytes);
  GemmArgs g = gemm_args(W, w, 1, A, lda, 0, X, ldx, w, (int)m, (int)n, 1.0, 0.0, 0);
  g.kscale = d;
  return gemm_launch(g, 1, &ws, (cudaStream_t)stream);
}

extern "C" int skb_transpose(const double* S, double* D, int64_t ld, int32_t n, void* stream) {
  dim3 tg((n + 31) / 32, (n + 31) / 32);
  transpose_kernel<<<tg, dim3(32, 8), 0, (cudaStream_t)stream>>>(S, D, ld, n);
  return skb_launch_status(__func__);
}

extern "C" int skb_set_identity_pad(double* G, int64_t ld, int32_t m, int32_t Mp, void* stream) {
  set_identity_pad_kernel<<<(unsigned)(((int64_t)Mp * Mp + 255) / 256), 256, 0,
                            (cudaStream_t)stream>>>(G, ld, m, Mp);
  return skb_launch_status(__func__);
}

static int round_pad(int m) { return std::max(NB, (m + NB - 1) / NB * NB); }

extern "C" int32_t skb_factor_padded_dim(int32_t m) { return round_pad(m); }

// Blocked right-looking Cholesky of the (Mp x Mp, ld) lower part in place.
// Per 64-wide panel: diagonal factor + its inverse (one CTA), panel
// L21 = A21 L11^-T as a DMMA GEMM (in place: each CTA owns whole rows),
// trailing update A22 -= L21 L21' on the lower tiles.
static int potrf_fused(double* G, int64_t ld, int Mp, int* status, skb_ws* ws, cudaStream_t st) {
  const size_t mark = ws->off;
  double* Dbuf = (double*)skb_ws_take(ws, (size_t)2 * NB * NB * 8);
  double* Lo = (double*)skb_ws_take(ws, (size_t)Mp * Mp * 8);
  if (!Dbuf || !Lo) {
    ws->off = mark;
    return 1;
  }
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(potrf_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kStepSmem);
    configured = true;
  }
  const int T = Mp / NB;
  potrf_step_kernel<<<1, kLeafThreads, kStepSmem, st>>>(G, ld, Lo, Mp, -1, Dbuf, status, 0);
  const char* se = getenv("SKB_POTRF_SPLIT");  // pairs above which a step is split (dev)
  const int split_above = se ? atoi(se) : skb_num_sms();
  for (int k = 0; k + 1 < T; ++k) {
    const int tp = T - 1 - k, pairs = tp * (tp + 1) / 2;
    if (split_above <= 0 || pairs <= split_above) {
      potrf_step_kernel<<<pairs, kLeafThreads, kStepSmem, st>>>(G, ld, Lo, Mp, k, Dbuf, status,
                                                                0);
    } else {
      potrf_step_kernel<<<tp, kLeafThreads, kStepSmem, st>>>(G, ld, Lo, Mp, k, Dbuf, status, 1);
      potrf_step_kernel<<<pairs, kLeafThreads, kStepSmem, st>>>(G, ld, Lo, Mp, k, Dbuf, status,
                                                                2);
    }
  }
  const int64_t half = (int64_t)Mp * Mp / 2;
  copy_lower_tiles_kernel<<<(unsigned)((half + 255) / 256), 256, 0, st>>>(G, ld, Lo, Mp, Mp);
  ws->off = mark;
  return skb_launch_status(__func__);
}

static int potrf(double* G, int64_t ld, int Mp, int* status, skb_ws* ws, cudaStream_t st) {
  const char* loop = getenv("SKB_POTRF_LOOP");  // per call: the tests compare both
  if (!loop || !atoi(loop)) {
    const int rc = potrf_fused(G, ld, Mp, status, ws, st);
    if (rc <= 0) return rc;
  }
  const size_t mark = ws->off;
  double* Dinv = (double*)skb_ws_take(ws, (size_t)NB * NB * 8);
  if (!Dinv) return SKB_ERR_WORKSPACE;
  for (int k0 = 0; k0 < Mp; k0 += NB) {
    potrf_diag_kernel<<<1, kLeafThreads, 0, st>>>(G, ld, k0, NB, status, Dinv);
    const int rest = Mp - k0 - NB;
    if (rest <= 0) break;
    double* P = G + (int64_t)(k0 + NB) * ld + k0;
    double* T = G + (int64_t)(k0 + NB) * ld + k0 + NB;
    GemmArgs gp = gemm_args(P, ld, 0, Dinv, NB, 1, P, ld, rest, NB, NB, 1.0, 0.0, 0);
    gp.tri_b = 2;  // opB = Dinv' (upper)
    int rc = gemm_launch(gp, 1, ws, st);
    if (rc) return rc;
    GemmArgs g = gemm_args(P, ld, 0, P, ld, 1, T, ld, rest, rest, NB, -1.0, 1.0, 1);
    rc = gemm_launch(g, 1, ws, st);
    if (rc) return rc;
  }
  ws->off = mark;
  return 0;
}

static int trtri(const double* L, double* Li, int64_t ld, int Mp, skb_ws* ws, cudaStream_t st);

// Large Mp: two-level blocking. NBO-wide outer panels: the diagonal block is
// factored by potrf (64-wide panels) and
// inverted by trtri, the panel L21 = A21 L11^-T is ONE NBO-deep GEMM into a
// scratch block, and the trailing update A22 -= L21 L21' ONE lower-tile SYRK.
// A few large GEMMs per NBO columns instead of NBO/64 small ones; from
// NBO = 1024 they are long enough for the INT8 emulation's cost model.
// (measured at Mp = 2048..10048: the plain 64-panel loop wins below ~6000,
// 2048-wide outer blocks above)
constexpr int kNBO = 2048, kPotrfBigMin = 6144;

static int potrf_big(double* G, int64_t ld, int Mp, int* status, skb_ws* ws, cudaStream_t st) {
  if (Mp < kPotrfBigMin) return potrf(G, ld, Mp, status, ws, st);
  const int NBO = kNBO;
  const size_t mark = ws->off;
  double* Lc = (double*)skb_ws_take(ws, (size_t)NBO * NBO * 8);
  double* Lci = (double*)skb_ws_take(ws, (size_t)NBO * NBO * 8);
  double* Pb = (double*)skb_ws_take(ws, (size_t)Mp * NBO * 8);
  if (!Lc || !Lci || !Pb) return SKB_ERR_WORKSPACE;
  for (int k0 = 0; k0 < Mp; k0 += NBO) {
    const int nb = std::min(NBO, Mp - k0);
    double* D = G + (int64_t)k0 * ld + k0;
    int rc = potrf(D, ld, nb, status, ws, st);
    if (rc) return rc;
    const int rest = Mp - k0 - nb;
    if (rest <= 0) break;
    cudaMemcpy2DAsync(Lc, (size_t)nb * 8, D, (size_t)ld * 8, (size_t)nb * 8, nb,
                      cudaMemcpyDeviceToDevice, st);
    if ((rc = trtri(Lc, Lci, nb, nb, ws, st))) return rc;
    double* A21 = G + (int64_t)(k0 + nb) * ld + k0;
    GemmArgs gp = gemm_args(A21, ld, 0, Lci, nb, 1, Pb, nb, rest, nb, nb, 1.0, 0.0, 0);
    gp.tri_b = 2;  // opB = L11^-T (upper)
    if ((rc = gemm_launch(gp, 1, ws, st))) return rc;
    cudaMemcpy2DAsync(A21, (size_t)ld * 8, Pb, (size_t)nb * 8, (size_t)nb * 8, rest,
                      cudaMemcpyDeviceToDevice, st);
    double* T = G + (int64_t)(k0 + nb) * ld + k0 + nb;
    GemmArgs g = gemm_args(Pb, nb, 0, Pb, nb, 1, T, ld, rest, rest, nb, -1.0, 1.0, 1);
    if ((rc = gemm_launch(g, 1, ws, st))) return rc;
  }
  ws->off = mark;
  return 0;
}

extern "C" int skb_potrf(double* G, int64_t ld, int32_t Mp, int* status, void* workspace,
                         size_t ws_bytes, void* stream) {
  if (Mp % NB) return SKB_ERR_ARG;
  skb_ws ws = skb_ws_make(workspace, ws_bytes);
  cudaStream_t st = (cudaStream_t)stream;
  int rc = potrf_big(G, ld, Mp, status, &ws, st);
  if (rc) return rc;
  zero_upper_kernel<<<(unsigned)(((int64_t)Mp * Mp + 255) / 256), 256, 0, st>>>(G, ld, Mp);
  return skb_launch_status(__func__);
}

// Li = L^-1 for lower-triangular L (Mp = 64 q, ld), by recursive doubling:
// inv([A 0; B C]) = [A^-1 0; -C^-1 B A^-1  C^-1]. Level h merges aligned
// pairs of h-blocks (all full pairs of a level batched); a trailing partial
// block (Mp not a multiple of 2h) is merged with its left neighbour on its
// own. Triangular operands trim each tile's k range (about half the flops).
static int trtri(const double* L, double* Li, int64_t ld, int Mp, skb_ws* ws, cudaStream_t st) {
  cudaMemsetAsync(Li, 0, (size_t)Mp * ld * 8, st);
  trtri_diag_kernel<<<Mp / NB, kLeafThreads, 0, st>>>(L, Li, ld);
  const size_t mark = ws->off;
  double* T = (double*)skb_ws_take(ws, (size_t)Mp * Mp / 2 * 8 + 64);
  if (!T) return SKB_ERR_WORKSPACE;
  for (int h = NB; h < Mp; h <<= 1) {
    const int pairs = Mp / (2 * h);
    const int rem = Mp - pairs * 2 * h;
    const int h2 = rem > h ? rem - h : 0;  // size of a trailing partial right block
    const int64_t s = (int64_t)2 * h * (ld + 1);  // diagonal stride between pairs
    int rc;
    if (pairs) {
      // T_p = L21_p * Li11_p  (h x h each), T stored contiguous h x h per pair
      GemmArgs g1 = gemm_args(L + (int64_t)h * ld, ld, 0, Li, ld, 0, T, h, h, h, h, 1.0, 0.0, 0);
      g1.sA = s;
      g1.sB = s;
      g1.sC = (int64_t)h * h;
      g1.tri_b = 1;
      if ((rc = gemm_launch(g1, pairs, ws, st))) return rc;
      // Li21_p = -Li22_p * T_p
      GemmArgs g2 = gemm_args(Li + (int64_t)h * ld + h, ld, 0, T, h, 0, Li + (int64_t)h * ld, ld,
                              h, h, h, -1.0, 0.0, 0);
      g2.sA = s;
      g2.sB = (int64_t)h * h;
      g2.sC = s;
      g2.tri_a = 1;
      if ((rc = gemm_launch(g2, pairs, ws, st))) return rc;
    }
    if (h2) {
      const int64_t o = (int64_t)pairs * 2 * h;
      double* T2 = T + (size_t)pairs * h * h;
      GemmArgs g1 = gemm_args(L + (o + h) * ld + o, ld, 0, Li + o * ld + o, ld, 0, T2, h, h2, h, h,
                              1.0, 0.0, 0);
      g1.tri_b = 1;
      if ((rc = gemm_launch(g1, 1, ws, st))) return rc;
      GemmArgs g2 = gemm_args(Li + (o + h) * ld + o + h, ld, 0, T2, h, 0, Li + (o + h) * ld + o, ld,
                              h2, h, h2, -1.0, 0.0, 0);
      g2.tri_a = 1;
      if ((rc = gemm_launch(g2, 1, ws, st))) return rc;
    }
  }
  ws->off = mark;
  return skb_launch_status(__func__);
}

extern "C" int skb_trtri(const double* L, double* Li, int64_t ld, int32_t Mp, void* workspace,
                         size_t ws_bytes, void* stream) {
  if (Mp % NB || Mp <= 0) return SKB_ERR_ARG;
  skb_ws ws = skb_ws_make(workspace, ws_bytes);
  return trtri(L, Li, ld, Mp, &ws, (cudaStream_t)stream);
}

extern "C" size_t skb_factor_workspace_bytes(int32_t m, int32_t w) {
  const size_t Mp = (size_t)round_pad(m);
  const size_t ldx = (size_t)(m + (m & 1));
  // G, L1inv, L2inv, Y + trtri temp, then room for one GEMM's scratch: DMMA
  // split-K partials or the INT8 emulation's residues + INT32 slab (Gram: one
  // shared residue set over K = w; Y = X L1^-T: both over K = m).
  const size_t split = 4 * Mp * Mp * 8;
  const size_t emu = std::max(skb_oz_bytes(m, m, w, true), skb_oz_bytes(w, m, m, false));
  return 3 * Mp * Mp * 8 + (size_t)w * ldx * 8 + Mp * Mp * 4 + std::max(split, emu) + 16 * 256;
}

// CholeskyQR2 of X' (X: w x m bucket-major, ldx). Outputs (Mp x Mp, ld = Mp):
// Linv (lower, = L^-1), LinvT (upper, its transpose), Lfac (lower L = L1 L2).
// stats_host[0..3]: min|L_ii|, max|L_ii| (of L), shifted (0/1), chol status.
// Synchronises the stream once (to test the first Cholesky).
extern "C" int skb_factor_cholqr2(const double* X, int64_t ldx, int32_t w, int32_t m,
                                  double* Linv, double* LinvT, double* Lfac, double* stats_host,
                                  void* workspace, size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (m < 1 || w < m) return SKB_ERR_ARG;
  skb_ws ws = skb_ws_make(workspace, ws_bytes);
  const int Mp = round_pad(m);
  const int64_t ld = Mp;
  const size_t MM = (size_t)Mp * Mp;
  double* G = (double*)skb_ws_take(&ws, MM * 8);
  double* L1i = (double*)skb_ws_take(&ws, MM * 8);
  double* L2i = (double*)skb_ws_take(&ws, MM * 8);
  double* Y = (double*)skb_ws_take(&ws, (size_t)w * ldx * 8);
  int* status = (int*)skb_ws_take(&ws, 64);
  double* dstat = (double*)skb_ws_take(&ws, 64);
  double* dprod = (double*)skb_ws_take(&ws, (size_t)Mp * 8);
  if (!G || !L1i || !L2i || !Y || !status || !dstat || !dprod) return SKB_ERR_WORKSPACE;
  const unsigned eb = (unsigned)((MM + 255) / 256);
  int rc;
  double hstat[4];
  int hst = 0;
  bool shifted = false;

  auto gram = [&](const double* Z) -> int {  // G = Z'Z (lower tiles), identity padding
    cudaMemsetAsync(G, 0, MM * 8, st);
    GemmArgs g = gemm_args(Z, ldx, 1, Z, ldx, 0, G, ld, m, m, w, 1.0, 0.0, 1);
    int r = gemm_launch(g, 1, &ws, st);
    set_identity_pad_kernel<<<eb, 256, 0, st>>>(G, ld, m, Mp);
    return r;
  };
  // ---- pass 1 (optionally shifted)
  cudaMemsetAsync(status, 0, 64, st);
  if ((rc = gram(X))) return rc;
  diag_stats_kernel<<<1, 1024, 0, st>>>(G, ld, m, dstat, 0);
  if ((rc = potrf_big(G, ld, Mp, status, &ws, st))) return rc;
  {
    skb_readback rb(st);
    rb.add(&hst, status, 4);
    rb.add(hstat, dstat, 8);
    if (rb.sync() != cudaSuccess) return SKB_ERR_CUDA;
  }
  if (hst & ST_CHOL_FAIL) {
    // shifted CholeskyQR: s = 11 (m w + m (m + 1)) u ||X||_F^2
    shifted = true;
    const double u = 1.1102230246251565e-16;
    const double shift = 11.0 * ((double)m * w + (double)m * (m + 1)) * u * hstat[0];
    cudaMemsetAsync(status, 0, 64, st);
    if ((rc = gram(X))) return rc;
    add_diag_kernel<<<(m + 255) / 256, 256, 0, st>>>(G, ld, m, shift);
    if ((rc = potrf_big(G, ld, Mp, status, &ws, st))) return rc;
  }
  // potrf leaves the strict upper part zero (G was cleared before the lower-tile
  // Gram, diagonal blocks are rewritten, trailing updates stay on lower tiles).
  if ((rc = trtri(G, L1i, ld, Mp, &ws, st))) return rc;
  diag_accum_kernel<<<(m + 255) / 256, 256, 0, st>>>(G, ld, m, dprod, 1);  // |diag L| = |diag L1|

  const int passes = shifted ? 2 : 1;
  const double* Z = X;
  for (int p = 0; p < passes; ++p) {
    // Y = Z * L1i'  (w x m)
    GemmArgs gy = gemm_args(Z, ldx, 0, L1i, ld, 1, Y, ldx, w, m, m, 1.0, 0.0, 0);
    gy.tri_b = 2;  // opB = L1i' (upper)
    if ((rc = gemm_launch(gy, 1, &ws, st))) return rc;
    Z = Y;
    if ((rc = gram(Y))) return rc;
    if ((rc = potrf_big(G, ld, Mp, status, &ws, st))) return rc;
    if ((rc = trtri(G, L2i, ld, Mp, &ws, st))) return rc;
    diag_accum_kernel<<<(m + 255) / 256, 256, 0, st>>>(G, ld, m, dprod, 0);  // diag(L1 L2)
    // Linv = L2i * L1i (lower x lower; tiles above the diagonal are skipped -> clear first)
    cudaMemsetAsync(Linv, 0, MM * 8, st);
    GemmArgs gi = gemm_args(L2i, ld, 0, L1i, ld, 0, Linv, ld, Mp, Mp, Mp, 1.0, 0.0, 1);
    gi.tri_a = 1;  // lower x lower
    gi.tri_b = 1;
    if ((rc = gemm_launch(gi, 1, &ws, st))) return rc;
    if (p + 1 < passes) {
      // next pass factors X again: L1i <- Linv (cumulative inverse), Y = X Linv'
      cudaMemcpyAsync(L1i, Linv, MM * 8, cudaMemcpyDeviceToDevice, st);
      Z = X;
    }
  }
  dim3 tg((Mp + 31) / 32, (Mp + 31) / 32);
  transpose_kernel<<<tg, dim3(32, 8), 0, st>>>(Linv, LinvT, ld, Mp);
  if (Lfac) {  // L = Linv^-1 is not needed by the solver; only materialised on request
    if ((rc = trtri(Linv, Lfac, ld, Mp, &ws, st))) return rc;
  }
  vec_minmax_kernel<<<1, 1024, 0, st>>>(dprod, m, dstat);
  {
    skb_readback rb(st);
    rb.add(hstat, dstat, 24);
    rb.add(&hst, status, 4);
    if (rb.sync() != cudaSuccess) return SKB_ERR_CUDA;
  }
  if (stats_host) {
    stats_host[0] = hstat[1];
    stats_host[1] = hstat[2];
    stats_host[2] = shifted ? 1.0 : 0.0;
    stats_host[3] = (double)hst;
  }
  return 0;
}

// y = M x with M row-major (rows x cols, ld); tri 0 full, 1 lower, 2 upper.
extern "C" int skb_rowdot_gemv(const double* Mx, int64_t ld, int32_t rows, int32_t cols,
                               int32_t tri, const double* x, double* y, const int* gate,
                               void* stream) {
  if (rows <= 0) return 0;
  const int64_t threads = (int64_t)rows * 32;
  rowdot_gemv_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      Mx, ld, rows, cols, tri, x, y, gate);
  return skb_launch_status(__func__);
}
