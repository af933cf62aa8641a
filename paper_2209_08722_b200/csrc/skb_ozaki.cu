// FP64 GEMM emulated on the INT8 tensor cores (CRT / Ozaki scheme II).
//
// The sketched factor's large GEMMs (CholeskyQR2 Grams and Y = X L^-T at
// m ~ 1e4, w ~ 4e4; the Gaussian sketch AD W at n ~ 2e6) are FP64 in the
// reference (LAPACK gesdd / numpy matmul, preconditioning.py:38-51,
// sketching.py:158-159). sm_100a has no FP64 tcgen05 kind: the DMMA pipe tops
// out near 37 TFLOP/s, while the INT8 kind delivers ~2.5 POP/s. So:
//
//   1. per row r of each operand, scale by a power of two so the row maximum
//      sits just below 2^53, and round: a'(r,k) = rint(a(r,k) 2^sigma_r)
//      (integers, |a'| <= 2^53; the truncation is at fp64's own relative
//      precision with respect to the row maximum);
//   2. reduce a' modulo n small pairwise-coprime moduli p_l <= 256 (symmetric
//      residues fit int8) — n = 16 covers 2 * 53 + log2 K + 2 bits;
//   3. n exact INT8 x INT8 -> INT32 GEMMs (one batched launch of the
//      hand-written tcgen05 kernel, skb_i8gemm.cu);
//   4. per output element, residues of the exact integer product C' and the
//      Chinese remainder theorem in split-double arithmetic give C' to fp64
//      accuracy; C = alpha 2^-(sigma_i + tau_j) C' + beta C.
//
// Integer products are exact, so the result is deterministic and independent
// of the tiling. Error: fp64-level relative to rowmax_i * colmax_j per term
// (the same order as a DMMA GEMM's K u sum|a||b| bound). K <= 131071 per INT32
// accumulation; longer K runs in chunks accumulated in fp64.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <atomic>
#include <mutex>

#include <cublasLt.h>

#include "skb_common.cuh"
#include "skb_internal.h"
#include "skb_ozaki_tables.h"

namespace skb {
namespace oz {

constexpr int kBeta = 53;           // bits kept per row (rowmax < 2^kBeta)
constexpr int kMaxK = 131071;       // |sum r_a r_b| < K 2^14 < 2^31
constexpr int kPadR = 16, kPadK = 32;
constexpr int kMaxMod = SKB_OZ_MAX_MOD;

struct Table {
  int n, s2;
  double p2s2;  // 2^s2
  double p[kMaxMod], pinv[kMaxMod], yp[kMaxMod], c26[kMaxMod];  // c26 = 2^26 mod p
  double w1[kMaxMod + 1], w2[kMaxMod + 1], w3[kMaxMod + 1];  // [n] = P's split
};

static Table make_table(int n) {
  Table t{};
  const int idx = n - SKB_OZ_MIN_MOD;
  t.n = n;
  t.s2 = kOzS2[idx];
  t.p2s2 = std::ldexp(1.0, t.s2);
  for (int l = 0; l <= n; ++l) {
    const double* r = kOzRows[idx][l];
    if (l < n) {
      t.p[l] = r[0];
      t.pinv[l] = r[1];
      t.yp[l] = r[2];
      t.c26[l] = (double)((1u << 26) % (unsigned)r[0]);
    }
    t.w1[l] = r[3];
    t.w2[l] = r[4];
    t.w3[l] = r[5];
  }
  return t;
}

// Smallest modulus count whose product exceeds 4 |C'| <= 4 K 2^(2 kBeta).
static int moduli_for(int K) {
  const double need = 2.0 * kBeta + std::log2((double)std::max(K, 2)) + 2.0;
  for (int n = SKB_OZ_MIN_MOD; n <= SKB_OZ_MAX_MOD; ++n)
    if (kOzBits[n - SKB_OZ_MIN_MOD] >= need) return n;
  return -1;
}

// -------------------------------------------------------------- row maxima
// amax[r] = max_k |x(r,k) ks[k]| as the bit pattern of a nonnegative double
// (monotone in the value, NaN above +inf), by atomicMax. x(r,k) = p[r sr + k sk].
// Block 32 x 8: the 32-wide index runs along the contiguous dimension.
__global__ void __launch_bounds__(256) rowmax_kernel(const double* __restrict__ p, int64_t sr,
                                                     int64_t sk, int R, int K,
                                                     const double* __restrict__ ks, int kchunk,
                                                     int tri, int kg0,
                                                     unsigned long long* __restrict__ amax) {
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int k0 = blockIdx.y * kchunk, k1 = min(K, k0 + kchunk);
  __shared__ double red[8][33];
  if (sk == 1) {  // rows contiguous along k: warp ty owns row, lanes stride k
    const int r = blockIdx.x * 8 + ty;
    double m = 0.0;
    if (r < R) {
      const double* row = p + (int64_t)r * sr;
      int ka = k0, kz = k1;  // triangle: 1 keeps kg0 + k <= r, 2 keeps kg0 + k >= r
      if (tri == 1) kz = min(kz, r - kg0 + 1);
      if (tri == 2) ka = max(ka, r - kg0);
      for (int k = ka + tx; k < kz; k += 32) {
        double v = fabs(__ldg(&row[k]));
        if (ks) v *= fabs(__ldg(&ks[k]));
        m = (v > m || v != v) ? v : m;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double u = __shfl_xor_sync(0xffffffffu, m, o);
      m = (u > m || u != u) ? u : m;
    }
    if (tx == 0 && r < R && m != 0.0) atomicMax(&amax[r], (unsigned long long)__double_as_longlong(m));
  } else {  // rows contiguous across r: lane tx owns row blockIdx.x*32+tx, ty strides k
    const int r = blockIdx.x * 32 + tx;
    double m = 0.0;
    if (r < R) {
      int ka = k0, kz = k1;
      if (tri == 1) kz = min(kz, r - kg0 + 1);
      if (tri == 2) ka = max(ka, r - kg0);
      for (int k = ka + ty; k < kz; k += 8) {
        double v = fabs(__ldg(&p[(int64_t)k * sk + r]));
        if (ks) v *= fabs(__ldg(&ks[k]));
        m = (v > m || v != v) ? v : m;
      }
    }
    red[ty][tx] = m;
    __syncthreads();
    if (ty == 0) {
#pragma unroll
      for (int u = 1; u < 8; ++u) {
        const double v = red[u][tx];
        m = (v > m || v != v) ? v : m;
      }
      if (r < R && m != 0.0) atomicMax(&amax[r], (unsigned long long)__double_as_longlong(m));
    }
  }
}

// Row r's scaling: a' = a 2^sigma with sigma = kBeta - e, rowmax < 2^e, kept
// as two in-range factors (m1, m2) plus inv = 2^-sigma for the reconstruction.
// Zero rows get (0, 0, 0); rows holding inf/NaN get inv = NaN.
__global__ void scales_kernel(const unsigned long long* __restrict__ amax, int R, int Rp,
                              double2* __restrict__ mul, double* __restrict__ inv) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= Rp) return;
  const unsigned long long bits = r < R ? amax[r] : 0ull;
  const double mx = __longlong_as_double((long long)bits);
  if (bits == 0ull) {
    mul[r] = make_double2(0.0, 0.0);
    inv[r] = 0.0;
  } else if (!(mx <= 1.7976931348623157e308)) {
    mul[r] = make_double2(0.0, 0.0);
    inv[r] = __longlong_as_double(0x7ff8000000000000ll);
  } else {
    const int e = ilogb(mx) + 1;
    const int sg = kBeta - e, h = sg / 2;
    mul[r] = make_double2(ldexp(1.0, h), ldexp(1.0, sg - h));
    inv[r] = ldexp(1.0, -sg);
  }
}

// 1.5 * 2^52: x + kMagic rounds x to an integer (|x| < 2^51) and leaves it,
// two's complement, in the low word of the result.
constexpr double kMagic = 6755399441055744.0;

// ---------------------------------------------------------------- residues
// out[l][r][k] (int8, row stride Kp, modulus stride Rp*Kp) = symmetric residue
// of rint(x(r,k) ks[k] 2^sigma_r) mod p_l. 64 x 64 tiles staged in smem so the
// fp64 reads are coalesced along whichever dimension is contiguous; each
// thread then packs 4 consecutive k into one 32-bit store per modulus. Per
// modulus: q = rint(a / p) by the magic-constant FMA, r = a - q p exactly,
// the (rare) off-by-one of q fixed in integer arithmetic.
constexpr int kST = 64;

template <int NM>
__global__ void __launch_bounds__(256) split_kernel(const double* __restrict__ p, int64_t sr,
                                                    int64_t sk, int R, int K, int Rp, int Kp,
                                                    const double* __restrict__ ks, int tri,
                                                    int kg0, const double2* __restrict__ mul,
                                                    const Table tab, int8_t* __restrict__ out) {
  __shared__ double tile[kST][kST + 1];  // [r][k]
  const int t = threadIdx.x;
  const int r0 = blockIdx.y * kST, k0 = blockIdx.x * kST;
  if (sk == 1) {
    for (int e = t; e < kST * kST; e += 256) {
      const int rr = e >> 6, kk = e & 63, r = r0 + rr, k = k0 + kk;
      const bool in = r < R && k < K && (tri == 0 || (tri == 1 ? kg0 + k <= r : kg0 + k >= r));
      tile[rr][kk] = in ? __ldg(&p[(int64_t)r * sr + k]) : 0.0;
    }
  } else {
    for (int e = t; e < kST * kST; e += 256) {
      const int kk = e >> 6, rr = e & 63, r = r0 + rr, k = k0 + kk;
      const bool in = r < R && k < K && (tri == 0 || (tri == 1 ? kg0 + k <= r : kg0 + k >= r));
      tile[rr][kk] = in ? __ldg(&p[(int64_t)k * sk + r]) : 0.0;
    }
  }
  __syncthreads();
  const int kq = (t & 15) * 4;
  if (k0 + kq >= Kp) return;
  double ksv[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int k = k0 + kq + u;
    ksv[u] = (ks && k < K) ? __ldg(&ks[k]) : 1.0;
  }
  const int64_t lstride = (int64_t)Rp * Kp;
  for (int rr = t >> 4; rr < kST; rr += 16) {
    const int r = r0 + rr;
    if (r >= Rp) break;
    const double2 m = __ldg(&mul[r]);
    // a = ah 2^26 + al with al in [0, 2^26): v = ah (2^26 mod p) + al < 2^35,
    // whose quotient by p rounds exactly (1/(2p) >> 2^35 2^-53 / p)
    double ah[4], al[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double a = rint((tile[rr][kq + u] * ksv[u]) * m.x * m.y);
      ah[u] = floor(a * 1.4901161193847656e-08);  // 2^-26
      al[u] = fma(-ah[u], 67108864.0, a);         // exact
    }
    int8_t* o = out + (int64_t)r * Kp + k0 + kq;
#pragma unroll
    for (int l = 0; l < NM; ++l) {
      const double pl = tab.p[l], pi = tab.pinv[l], c26 = tab.c26[l];
      uint32_t ri[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double v = fma(ah[u], c26, al[u]);
        const double q = fma(v, pi, kMagic) - kMagic;
        ri[u] = (uint32_t)__double2loint(fma(-q, pl, v) + kMagic);  // low byte = residue
      }
      // 4 low bytes -> one word: 3 byte permutes
      const uint32_t pack = __byte_perm(__byte_perm(ri[0], ri[1], 0x0040),
                                        __byte_perm(ri[2], ri[3], 0x0040), 0x5410);
      *reinterpret_cast<uint32_t*>(o) = pack;
      o += lstride;
    }
  }
}

// ---------------------------------------------------------- reconstruction
// C[i][j] (i in [r0, r0+rows), j < N) from the n INT32 products
// c_l = sum_k a'_l b'_l (slab-local, row stride ldc32, modulus stride mstride).
// Residues r_l = c_l - rint(c_l / p_l) p_l in [-p/2, p/2] (exact: c/p's
// rounding error < 2^-30 cannot cross a half-integer whose denominator is p).
template <int NM>
__global__ void __launch_bounds__(256) crt_kernel(const int32_t* __restrict__ c32, int64_t ldc32,
                                                  int64_t mstride, int r0, int rows, int c0,
                                                  int cols, int lower_only, const Table tab,
                                                  const double* __restrict__ invA,
                                                  const double* __restrict__ invB,
                                                  double alpha, double beta, double* __restrict__ C,
                                                  int64_t ldc) {
  const int jj = blockIdx.x * 128 + (threadIdx.x & 127);
  const int ii = blockIdx.y * 2 + (threadIdx.x >> 7);
  if (ii >= rows || jj >= cols) return;
  const int i = r0 + ii, j = c0 + jj;
  if (lower_only && j > i) return;
  const int32_t* src = c32 + (int64_t)ii * ldc32 + jj;
  int c[NM];
#pragma unroll
  for (int l = 0; l < NM; ++l) {  // all loads in flight
    c[l] = __ldg(src);
    src += mstride;
  }
  constexpr double kI2D = 4503601774854144.0;  // 2^52 + 2^31
  double q = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
#pragma unroll
  for (int l = 0; l < NM; ++l) {
    const double d = __hiloint2double(0x43300000, c[l] ^ 0x80000000) - kI2D;  // exact
    const double qq = fma(d, tab.pinv[l], kMagic) - kMagic;
    const double r = fma(-qq, tab.p[l], d);
    q = fma(r, tab.yp[l], q);
    t1 = fma(r, tab.w1[l], t1);
    t2 = fma(r, tab.w2[l], t2);
    t3 = fma(r, tab.w3[l], t3);
  }
  q = rint(q);
  t1 = fma(-q, tab.w1[NM], t1);
  t2 = fma(-q, tab.w2[NM], t2);
  t3 = fma(-q, tab.w3[NM], t3);
  const double v = fma(t1, 1099511627776.0, t2) + t3;  // 2^40
  const double ia = __ldg(&invA[i]), ib = __ldg(&invB[j]);
  double val = (v * (ia * tab.p2s2)) * ib;
  if (ia == 0.0 || ib == 0.0) val = 0.0;
  double* cp = C + (int64_t)i * ldc + j;
  *cp = beta == 0.0 ? alpha * val : fma(alpha, val, beta * *cp);
}

// As crt_kernel, from the int8 residues the INT8 kernel's residue epilogue
// stored (skb_i8gemm_residues): one byte per product instead of four, the
// per-modulus reduction already done.
template <int NM>
__global__ void __launch_bounds__(256) crt8_kernel(const int8_t* __restrict__ r8, int64_t ldr,
                                                   int64_t mstride, int r0, int rows, int c0,
                                                   int cols, int lower_only, const Table tab,
                                                   const double* __restrict__ invA,
                                                   const double* __restrict__ invB,
                                                   double alpha, double beta,
                                                   double* __restrict__ C, int64_t ldc) {
  const int jj = blockIdx.x * 128 + (threadIdx.x & 127);
  const int ii = blockIdx.y * 2 + (threadIdx.x >> 7);
  if (ii >= rows || jj >= cols) return;
  const int i = r0 + ii, j = c0 + jj;
  if (lower_only && j > i) return;
  const int8_t* src = r8 + (int64_t)ii * ldr + jj;
  int rr[NM];
#pragma unroll
  for (int l = 0; l < NM; ++l) {  // all loads in flight
    rr[l] = __ldg(src);
    src += mstride;
  }
  double q = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
#pragma unroll
  for (int l = 0; l < NM; ++l) {
    const double r = (double)rr[l];
    q = fma(r, tab.yp[l], q);
    t1 = fma(r, tab.w1[l], t1);
    t2 = fma(r, tab.w2[l], t2);
    t3 = fma(r, tab.w3[l], t3);
  }
  q = rint(q);
  t1 = fma(-q, tab.w1[NM], t1);
  t2 = fma(-q, tab.w2[NM], t2);
  t3 = fma(-q, tab.w3[NM], t3);
  const double v = fma(t1, 1099511627776.0, t2) + t3;  // 2^40
  const double ia = __ldg(&invA[i]), ib = __ldg(&invB[j]);
  double val = (v * (ia * tab.p2s2)) * ib;
  if (ia == 0.0 || ib == 0.0) val = 0.0;
  double* cp = C + (int64_t)i * ldc + j;
  *cp = beta == 0.0 ? alpha * val : fma(alpha, val, beta * *cp);
}

// Launch K<NM> for the table's modulus count (12..20).
#define SKB_OZ_DISPATCH(n, KERNEL, GRID, ARGS)                                          \
  switch (n) {                                                                          \
    case 12: KERNEL<12><<<GRID, 256, 0, st>>> ARGS; break;                              \
    case 13: KERNEL<13><<<GRID, 256, 0, st>>> ARGS; break;                              \
    case 14: KERNEL<14><<<GRID, 256, 0, st>>> ARGS; break;                              \
    case 15: KERNEL<15><<<GRID, 256, 0, st>>> ARGS; break;                              \
    case 16: KERNEL<16><<<GRID, 256, 0, st>>> ARGS; break;                              \
    case 17: KERNEL<17><<<GRID, 256, 0, st>>> ARGS; break;                              \
    case 18: KERNEL<18><<<GRID, 256, 0, st>>> ARGS; break;                              \
    case 19: KERNEL<19><<<GRID, 256, 0, st>>> ARGS; break;                              \
    default: KERNEL<20><<<GRID, 256, 0, st>>> ARGS; break;                              \
  }

// ------------------------------------------------------------- cuBLASLt
// Loaded at run time (libcublasLt.so.12: torch's copy when torch is loaded,
// else the toolkit's), so libskb.so keeps no link-time dependency on it.
struct Lt {
  bool ok = false;
  cublasLtHandle_t h = nullptr;
  decltype(&cublasLtCreate) create;
  decltype(&cublasLtMatmulDescCreate) descCreate;
  decltype(&cublasLtMatmulDescDestroy) descDestroy;
  decltype(&cublasLtMatmulDescSetAttribute) descSet;
  decltype(&cublasLtMatrixLayoutCreate) layCreate;
  decltype(&cublasLtMatrixLayoutDestroy) layDestroy;
  decltype(&cublasLtMatrixLayoutSetAttribute) laySet;
  decltype(&cublasLtMatmulPreferenceCreate) prefCreate;
  decltype(&cublasLtMatmulPreferenceDestroy) prefDestroy;
  decltype(&cublasLtMatmulPreferenceSetAttribute) prefSet;
  decltype(&cublasLtMatmulAlgoGetHeuristic) heur;
  decltype(&cublasLtMatmul) matmul;
};

static Lt& lt() {
  static Lt L;
  static std::once_flag once;
  std::call_once(once, [] {
    void* so = dlopen("libcublasLt.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (!so) so = dlopen("/usr/local/cuda/lib64/libcublasLt.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (!so) return;
#define SKB_LT(f, n) L.f = (decltype(L.f))dlsym(so, n); if (!L.f) return;
    SKB_LT(create, "cublasLtCreate")
    SKB_LT(descCreate, "cublasLtMatmulDescCreate")
    SKB_LT(descDestroy, "cublasLtMatmulDescDestroy")
    SKB_LT(descSet, "cublasLtMatmulDescSetAttribute")
    SKB_LT(layCreate, "cublasLtMatrixLayoutCreate")
    SKB_LT(layDestroy, "cublasLtMatrixLayoutDestroy")
    SKB_LT(laySet, "cublasLtMatrixLayoutSetAttribute")
    SKB_LT(prefCreate, "cublasLtMatmulPreferenceCreate")
    SKB_LT(prefDestroy, "cublasLtMatmulPreferenceDestroy")
    SKB_LT(prefSet, "cublasLtMatmulPreferenceSetAttribute")
    SKB_LT(heur, "cublasLtMatmulAlgoGetHeuristic")
    SKB_LT(matmul, "cublasLtMatmul")
#undef SKB_LT
    if (L.create(&L.h) != CUBLAS_STATUS_SUCCESS) return;
    L.ok = true;
  });
  return L;
}

constexpr size_t kLtWs = 32u << 20;

// The INT8 products run on the hand-written tcgen05 kernel; SKB_OZ_CUBLASLT=1
// routes them to cuBLASLt instead (A/B comparisons in development and tests).
static bool use_cublaslt() {
  const char* e = getenv("SKB_OZ_CUBLASLT");
  return e && e[0] == '1';
}

// c32[l] (rows x cols, row stride ldc) = a8[l] (rows x Kk) * b8[l] (cols x Kk)'
// for l < n; a8/b8 row stride ld, modulus strides sa / sb, c32 stride sc.
static int int8_gemm_batched(const int8_t* a8, int64_t sa, const int8_t* b8, int64_t sb,
                             int32_t* c32, int64_t ldc, int64_t sc, int rows, int cols, int Kk,
                             int64_t ld, int n, void* lws, cudaStream_t st) {
  Lt& L = lt();
  if (!L.ok) return 1;
  cublasLtMatmulDesc_t desc = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
  cublasLtMatmulPreference_t pref = nullptr;
  int rc = 1;
  const cublasOperation_t opT = CUBLAS_OP_T, opN = CUBLAS_OP_N;
  const int32_t one = 1, zero = 0;
  const size_t wsb = kLtWs;
  // column-major view: C' (cols x rows) = B8 (Kp x cols)^T * A8 (Kp x rows)
  if (L.descCreate(&desc, CUBLAS_COMPUTE_32I, CUDA_R_32I) != CUBLAS_STATUS_SUCCESS) goto done;
  L.descSet(desc, CUBLASLT_MATMUL_DESC_TRANSA, &opT, sizeof(opT));
  L.descSet(desc, CUBLASLT_MATMUL_DESC_TRANSB, &opN, sizeof(opN));
  if (L.layCreate(&la, CUDA_R_8I, Kk, cols, ld) != CUBLAS_STATUS_SUCCESS) goto done;
  if (L.layCreate(&lb, CUDA_R_8I, Kk, rows, ld) != CUBLAS_STATUS_SUCCESS) goto done;
  if (L.layCreate(&lc, CUDA_R_32I, cols, rows, ldc) != CUBLAS_STATUS_SUCCESS) goto done;
  {
    const int32_t bc = n;
    L.laySet(la, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &bc, sizeof(bc));
    L.laySet(lb, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &bc, sizeof(bc));
    L.laySet(lc, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &bc, sizeof(bc));
    L.laySet(la, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sb, sizeof(sb));
    L.laySet(lb, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sa, sizeof(sa));
    L.laySet(lc, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sc, sizeof(sc));
  }
  if (L.prefCreate(&pref) != CUBLAS_STATUS_SUCCESS) goto done;
  L.prefSet(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsb, sizeof(wsb));
  {
    cublasLtMatmulHeuristicResult_t res{};
    int nres = 0;
    if (L.heur(L.h, desc, la, lb, lc, lc, pref, 1, &res, &nres) != CUBLAS_STATUS_SUCCESS ||
        nres < 1)
      goto done;
    if (L.matmul(L.h, desc, &one, b8, la, a8, lb, &zero, c32, lc, c32, lc, &res.algo, lws, wsb,
                 st) != CUBLAS_STATUS_SUCCESS) {
      rc = SKB_ERR_CUDA;
      goto done;
    }
    rc = 0;
  }
done:
  if (pref) L.prefDestroy(pref);
  if (lc) L.layDestroy(lc);
  if (lb) L.layDestroy(lb);
  if (la) L.layDestroy(la);
  if (desc) L.descDestroy(desc);
  return rc;
}

static inline int64_t up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

// Output tiling. Triangular structure is exploited by slabs: lower_only and
// tri_a slab the rows (a row slab [r0, r1) needs columns < r1 / k < r1 or
// k >= r0), tri_b slabs the columns (k >= c0 or k < c1). Slabs of 1280 rows
// (5 tiles of the 256-wide INT8 kernel) keep the wasted triangle ~1/(2s).
constexpr int kSlab = 1280;

static int chunk(const skb_oz_args& g, int k0, int Kc, double beta, skb_ws* ws, cudaStream_t st) {
  const int n = moduli_for(Kc);
  if (n < 0) return 1;
  const int Kp = (int)up(Kc, kPadK);
  const int Mp = (int)up(g.M, kPadR), Np = (int)up(g.N, kPadR);
  const bool share = g.a.p == g.b.p && g.a.sr == g.b.sr && g.a.sk == g.b.sk && !g.kscale &&
                     g.M == g.N && g.tri_a == 0 && g.tri_b == 0;
  const bool rslab = g.lower_only || g.tri_a, cslab = g.tri_b != 0;
  int wc = cslab && g.N > 2 * kSlab ? kSlab : Np;
  // the tcgen05 kernel skips tiles above the diagonal itself: lower_only needs no
  // row slabs (only triangular operands, whose K ranges shrink per slab, do)
  const bool tile_tri = g.lower_only && !g.tri_a && !use_cublaslt();
  int h = rslab && !tile_tri && g.M > 2 * kSlab ? kSlab : Mp;
  const size_t mark = ws->off;
  auto* amA = (unsigned long long*)skb_ws_take(ws, (size_t)Mp * 8);
  auto* amB = share ? amA : (unsigned long long*)skb_ws_take(ws, (size_t)Np * 8);
  auto* mulA = (double2*)skb_ws_take(ws, (size_t)Mp * 16);
  auto* mulB = share ? mulA : (double2*)skb_ws_take(ws, (size_t)Np * 16);
  auto* invA = (double*)skb_ws_take(ws, (size_t)Mp * 8);
  auto* invB = share ? invA : (double*)skb_ws_take(ws, (size_t)Np * 8);
  auto* a8 = (int8_t*)skb_ws_take(ws, (size_t)n * Mp * Kp);
  auto* b8 = share ? a8 : (int8_t*)skb_ws_take(ws, (size_t)n * Np * Kp);
  void* lws = skb_ws_take(ws, kLtWs);
  if (!amA || !amB || !mulA || !mulB || !invA || !invB || !a8 || !b8 || !lws) {
    ws->off = mark;
    return 1;
  }
  // residue mode (default with the tcgen05 kernel): the INT8 GEMM stores int8
  // residues, the CRT reads 1 byte per product (SKB_OZ_CRT32=1: int32 products)
  const char* c32e = getenv("SKB_OZ_CRT32");
  const bool r8mode = !use_cublaslt() && !(c32e && c32e[0] == '1');
  // product tile buffer: shrink the tile height (then width) to the workspace left
  const size_t left = ws->cap > ws->off + 1024 ? ws->cap - ws->off - 1024 : 0;
  const size_t per_elem = (size_t)n * (r8mode ? 1 : 4);
  if ((size_t)h * up(wc, kPadR) * per_elem > left) {
    h = (int)std::min<int64_t>(h, (int64_t)(left / (per_elem * up(wc, kPadR))) / 256 * 256);
    if (h < 128) {
      h = std::min(Mp, 128);
      wc = (int)std::min<int64_t>(wc, (int64_t)(left / (per_elem * h)) / 256 * 256);
    }
  }
  if (h < std::min(Mp, 128) || wc < std::min(Np, 256)) {
    ws->off = mark;
    return 1;
  }
  const int64_t ldt = up(wc, kPadR), mstr = (int64_t)h * ldt;
  auto* c32 = (int32_t*)skb_ws_take(ws, (size_t)mstr * per_elem);
  auto* c8 = reinterpret_cast<int8_t*>(c32);
  if (!c32) {
    ws->off = mark;
    return 1;
  }
  const Table tab = make_table(n);
  const double* pa = g.a.p + (int64_t)k0 * g.a.sk;
  const double* pb = g.b.p + (int64_t)k0 * g.b.sk;
  const double* ks = g.kscale ? g.kscale + k0 : nullptr;
  // row maxima and residues of both operands (kscale folded into b); entries
  // outside a triangular operand's triangle read as zero
  auto prep = [&](const double* p0, int64_t sr, int64_t sk, int R, int Rp, const double* kk,
                  int tri, unsigned long long* am, double2* mul, double* inv, int8_t* o) {
    cudaMemsetAsync(am, 0, (size_t)Rp * 8, st);
    // k split so the grid covers the GPU ~4x (row blocks alone are too few at m ~ 2e3)
    const int rb = sk == 1 ? (R + 7) / 8 : (R + 31) / 32;
    const int want = std::max(1, (4 * skb_num_sms() + rb - 1) / rb);
    const int kchunk = std::min(4096, std::max(256, (int)up((Kc + want - 1) / want, 256)));
    dim3 gm(rb, (Kc + kchunk - 1) / kchunk);
    rowmax_kernel<<<gm, 256, 0, st>>>(p0, sr, sk, R, Kc, kk, kchunk, tri, k0, am);
    scales_kernel<<<(Rp + 255) / 256, 256, 0, st>>>(am, R, Rp, mul, inv);
    dim3 gs((unsigned)((Kp + kST - 1) / kST), (unsigned)((Rp + kST - 1) / kST));
    SKB_OZ_DISPATCH(n, split_kernel, gs, (p0, sr, sk, R, Kc, Rp, Kp, kk, tri, k0, mul, tab, o))
  };
  // operand-relative triangles: 1 keeps k <= r, 2 keeps k >= r
  const int tria = g.tri_a == 1 ? 1 : (g.tri_a == 2 ? 2 : 0);
  const int trib = g.tri_b == 1 ? 2 : (g.tri_b == 2 ? 1 : 0);
  prep(pa, g.a.sr, g.a.sk, g.M, Mp, nullptr, tria, amA, mulA, invA, a8);
  if (!share) prep(pb, g.b.sr, g.b.sk, g.N, Np, ks, trib, amB, mulB, invB, b8);
  int rc = skb_launch_status("ozaki split");
  for (int c0 = 0; !rc && c0 < g.N; c0 += wc) {
    for (int r0 = 0; !rc && r0 < g.M; r0 += h) {
      const int r1 = std::min(g.M, r0 + h);
      int c1 = std::min(g.N, c0 + wc);
      if (g.lower_only) c1 = std::min(c1, r1);
      if (c1 <= c0) continue;
      // k range of this tile (chunk-local), widened to the 32-byte residue grid
      int kb = 0, ke = Kc;
      if (g.tri_a == 1) ke = std::min(ke, r1 - k0);
      if (g.tri_a == 2) kb = std::max(kb, r0 - k0);
      if (g.tri_b == 1) kb = std::max(kb, c0 - k0);
      if (g.tri_b == 2) ke = std::min(ke, c1 - k0);
      kb = std::max(0, kb) / kPadK * kPadK;
      ke = (int)std::min<int64_t>(Kp, up(std::max(0, std::min(ke, Kc)), kPadK));
      const int rows = r1 - r0, cols = c1 - c0;
      const int rows_p = (int)up(rows, kPadR), cols_p = (int)up(cols, kPadR);
      if (ke > kb) {
        if (use_cublaslt()) {  // development A/B only (SKB_OZ_CUBLASLT=1)
          rc = int8_gemm_batched(a8 + (int64_t)r0 * Kp + kb, (int64_t)Mp * Kp,
                                 b8 + (int64_t)c0 * Kp + kb, (int64_t)Np * Kp, c32, ldt, mstr,
                                 rows_p, cols_p, ke - kb, Kp, n, lws, st);
          if (rc == 1) rc = SKB_ERR_UNSUPPORTED;  // never fall back after tiles were written
        } else {
          // the tcgen05 kernel (skb_i8gemm.cu); its K range starts on a 128-byte box:
          // entries in [kb128, kb) of these rows are outside the operand's triangle, zero
          if (r8mode)
            rc = skb_i8gemm_residues(a8, Mp, (int64_t)Mp * Kp, b8, Np, (int64_t)Np * Kp, Kp, c8,
                                     ldt, mstr, rows_p, cols_p, r0, c0, kb / 128 * 128, ke, n,
                                     g.lower_only ? 1 : 0, r0 - c0, tab.p, st);
          else
            rc = skb_i8gemm_batched(a8, Mp, (int64_t)Mp * Kp, b8, Np, (int64_t)Np * Kp, Kp,
                                    c32, ldt, mstr, rows_p, cols_p, r0, c0, kb / 128 * 128, ke,
                                    n, g.lower_only ? 1 : 0, r0 - c0, st);
        }
      } else {
        cudaMemsetAsync(c32, 0, (size_t)mstr * per_elem, st);
      }
      if (rc) break;
      dim3 gc((unsigned)((cols + 127) / 128), (unsigned)((rows + 1) / 2));
      if (r8mode)
        SKB_OZ_DISPATCH(n, crt8_kernel, gc,
                        (c8, ldt, mstr, r0, rows, c0, cols, g.lower_only, tab, invA, invB,
                         g.alpha, beta, g.C, g.ldc))
      else
        SKB_OZ_DISPATCH(n, crt_kernel, gc,
                        (c32, ldt, mstr, r0, rows, c0, cols, g.lower_only, tab, invA, invB,
                         g.alpha, beta, g.C, g.ldc))
      rc = skb_launch_status("ozaki crt");
    }
  }
  ws->off = mark;
  return rc;
}

}  // namespace oz
}  // namespace skb

using namespace skb;

size_t skb_oz_bytes(int M, int N, int K, bool share) {
  const int Kc = std::min(K, oz::kMaxK);
  const int n = oz::moduli_for(Kc);
  if (n < 0) return 0;
  const size_t Kp = (size_t)oz::up(Kc, oz::kPadK), Mp = (size_t)oz::up(M, oz::kPadR),
               Np = (size_t)oz::up(N, oz::kPadR);
  return 8192 + 8192 + (Mp + Np) * 32 + oz::kLtWs + (size_t)n * Kp * (Mp + (share ? 0 : Np)) +
         (size_t)n * std::min<size_t>(Mp, 4096) * Np * 4;
}

static std::atomic<long long> g_calls{0};

// K = 0: C = beta C (the empty product), on the written part only.
__global__ void scale_c_kernel(double* C, int64_t ldc, int M, int N, int lower_only, double beta) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)M * N) return;
  const int i = (int)(e / N), j = (int)(e % N);
  if (lower_only && j > i) return;
  double* p = C + (int64_t)i * ldc + j;
  *p = beta == 0.0 ? 0.0 : beta * *p;
}

int skb_oz_gemm(const skb_oz_args& g, skb_ws* ws, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0) return 0;
  if (g.K <= 0) {
    const int64_t tot = (int64_t)g.M * g.N;
    scale_c_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(g.C, g.ldc, g.M, g.N,
                                                                 g.lower_only, g.beta);
    return skb_launch_status("ozaki k=0");
  }
  if (oz::use_cublaslt() && !oz::lt().ok) return 1;
  // K chunk: <= kMaxK (exact INT32 sums) and small enough that both residue
  // sets plus a 1024-row INT32 slab fit the workspace; chunks accumulate in fp64.
  const size_t avail = ws->cap > ws->off + 8192 ? ws->cap - ws->off - 8192 : 0;
  const int n = oz::moduli_for(std::min(g.K, oz::kMaxK));
  if (n < 0) return 1;
  const int64_t Mp = oz::up(g.M, oz::kPadR), Np = oz::up(g.N, oz::kPadR);
  const bool share = g.a.p == g.b.p && g.a.sr == g.b.sr && g.a.sk == g.b.sk && !g.kscale &&
                     g.M == g.N;
  const size_t fixed = oz::kLtWs + (size_t)(Mp + Np) * 32 + 8192 +
                       (size_t)n * std::min<int64_t>(Mp, 1024) * Np * 4;
  if (avail <= fixed) return 1;
  const size_t per_k = (size_t)n * (Mp + (share ? 0 : Np));
  int64_t kmax = (int64_t)((avail - fixed) / per_k) / oz::kPadK * oz::kPadK;
  kmax = std::min<int64_t>(kmax, oz::kMaxK / oz::kPadK * oz::kPadK);
  if (kmax < std::min(g.K, 1024)) return 1;
  const int nch = (int)((g.K + kmax - 1) / kmax);
  const int kc = (int)oz::up((g.K + nch - 1) / nch, oz::kPadK);
  for (int c = 0; c * kc < g.K; ++c) {
    const int k0 = c * kc, k1 = std::min(g.K, k0 + kc);
    const int rc = oz::chunk(g, k0, k1 - k0, c == 0 ? g.beta : 1.0, ws, st);
    if (rc) return c == 0 ? rc : (rc == 1 ? SKB_ERR_WORKSPACE : rc);
  }
  g_calls.fetch_add(1, std::memory_order_relaxed);
  return 0;
}

// Number of products the emulation has completed in this process (tests, bench).
extern "C" int64_t skb_gemm_ozaki_calls(void) { return (int64_t)g_calls.load(); }

extern "C" int skb_gemm_ozaki(int32_t ta, int32_t tb, int32_t M, int32_t N, int32_t K,
                              double alpha, const double* A, int64_t lda, const double* B,
                              int64_t ldb, double beta, double* C, int64_t ldc,
                              int32_t lower_only, void* workspace, size_t ws_bytes, void* stream) {
  skb_ws ws = skb_ws_make(workspace, ws_bytes);
  skb_oz_args g{};
  g.a = ta ? skb_oz_operand{A, 1, lda} : skb_oz_operand{A, lda, 1};
  g.b = tb ? skb_oz_operand{B, ldb, 1} : skb_oz_operand{B, 1, ldb};
  g.C = C;
  g.ldc = ldc;
  g.M = M;
  g.N = N;
  g.K = K;
  g.alpha = alpha;
  g.beta = beta;
  g.lower_only = lower_only;
  const int rc = skb_oz_gemm(g, &ws, (cudaStream_t)stream);
  return rc == 1 ? SKB_ERR_UNSUPPORTED : rc;
}

extern "C" size_t skb_gemm_ozaki_workspace_bytes(int32_t M, int32_t N, int32_t K) {
  return skb_oz_bytes(M, N, K, false);
}
