// K4/K8: single-pass column-streaming kernels over a dense column-major A.
//
// One template covers every A-pass of the hot path:
//   normal    u = A (d2 .* (A' z))                 krylov_solvers.py:46-47
//   gemv      u = A coef,  coef_j from n-vectors    ipm_core.py:99,204-206,502,223
//   gemv_t    t = A' y (+ add - sub)                 ipm_core.py:100,218
//   dir       A' dy -> ds, dx (elementwise) -> A dx  ipm_core.py:218-223 (one pass)
//   iter      x+a dx, s+a ds, A' y_new + s_new - c, A x_new   ipm_core.py:94-102,308
//
// Layout: column j of A is A[j*lda .. j*lda+m) (lda even, 16-byte aligned), so a
// group of cb consecutive columns is one contiguous range. Each warp owns a
// private ring of `stages` shared-memory buffers filled by the TMA engine
// (cp.async.bulk, L2 evict-first) and consumes one group per stage: lane l
// holds rows 64k+2l, 64k+2l+1 in registers, the column dot is a warp
// butterfly, and the rank-1 update accumulates into per-lane registers. A is
// read from HBM exactly once per pass. Per-warp partial m-vectors are summed
// in a fixed order per CTA, then across CTAs by skb_reduce_partials: the
// result is deterministic run to run.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include <cub/block/block_radix_sort.cuh>

#include "skb_common.cuh"
#include "skb_internal.h"

namespace skb {

struct Pre {
  double v[6];
};

SKB_DEV double dmul(double a, double b) { return __dmul_rn(a, b); }
SKB_DEV double dadd(double a, double b) { return __dadd_rn(a, b); }
SKB_DEV double dsub(double a, double b) { return __dsub_rn(a, b); }
SKB_DEV double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// ------------------------------------------------------------------- ops
// Elementwise formulas use explicit round-to-nearest intrinsics in numpy's
// evaluation order, so given equal inputs they are bit-identical to numpy.

struct OpNormal {  // u += (d2_j * <a_j, z>) a_j
  static constexpr bool kDot = true, kAxpy = true;
  static constexpr int kPre = 1;
  const double* d2;
  SKB_DEV void load(int64_t j, Pre& p) const { p.v[0] = d2[j]; }
  SKB_DEV const double* src(int) const { return d2; }
  SKB_DEV double coef(int64_t, const Pre& p, double dot) const { return dmul(p.v[0], dot); }
  SKB_DEV void emit(int64_t, const Pre&, double, double) const {}
};

struct OpGemvX {  // u += x_j a_j
  static constexpr bool kDot = false, kAxpy = true;
  static constexpr int kPre = 1;
  const double* x;
  SKB_DEV void load(int64_t j, Pre& p) const { p.v[0] = x[j]; }
  SKB_DEV const double* src(int) const { return x; }
  SKB_DEV double coef(int64_t, const Pre& p, double) const { return p.v[0]; }
  SKB_DEV void emit(int64_t, const Pre&, double, double) const {}
};

struct OpGemvRatio {  // u += (v_j / s_j) a_j          (ipm_core.py:502)
  static constexpr bool kDot = false, kAxpy = true;
  static constexpr int kPre = 2;
  const double* v;
  const double* s;
  SKB_DEV void load(int64_t j, Pre& p) const {
    p.v[0] = v[j];
    p.v[1] = s[j];
  }
  SKB_DEV const double* src(int q) const { return q == 0 ? v : s; }
  SKB_DEV double coef(int64_t, const Pre& p, double) const { return ddiv(p.v[0], p.v[1]); }
  SKB_DEV void emit(int64_t, const Pre&, double, double) const {}
};

struct OpRhs {  // u_j = x - smu/s [- (x/s) r_d]       (ipm_core.py:202-206)
  static constexpr bool kDot = false, kAxpy = true;
  static constexpr int kPre = 3;
  const double *x, *s, *rd;  // rd == nullptr: feasible mode
  double smu;
  SKB_DEV void load(int64_t j, Pre& p) const {
    p.v[0] = x[j];
    p.v[1] = s[j];
    p.v[2] = rd ? rd[j] : 0.0;
  }
  SKB_DEV const double* src(int q) const { return q == 0 ? x : (q == 1 ? s : rd); }
  SKB_DEV double coef(int64_t, const Pre& p, double) const {
    double u = dsub(p.v[0], ddiv(smu, p.v[1]));
    if (rd) u = dsub(u, dmul(ddiv(p.v[0], p.v[1]), p.v[2]));
    return u;
  }
  SKB_DEV void emit(int64_t, const Pre&, double, double) const {}
};

struct OpGemvT {  // out_j = (<a_j, y> + add_j) - sub_j
  static constexpr bool kDot = true, kAxpy = false;
  static constexpr int kPre = 2;
  const double *add, *sub;
  double* out;
  SKB_DEV void load(int64_t j, Pre& p) const {
    p.v[0] = add ? add[j] : 0.0;
    p.v[1] = sub ? sub[j] : 0.0;
  }
  SKB_DEV const double* src(int q) const { return q == 0 ? add : sub; }
  SKB_DEV double coef(int64_t, const Pre&, double) const { return 0.0; }
  SKB_DEV void emit(int64_t j, const Pre& p, double dot, double) const {
    double t = dot;
    if (add) t = dadd(t, p.v[0]);
    if (sub) t = dsub(t, p.v[1]);
    out[j] = t;
  }
};

struct OpDir {  // assemble_directions in one pass (ipm_core.py:218-223)
  static constexpr bool kDot = true, kAxpy = true;
  static constexpr int kPre = 4;
  const double *x, *s, *v, *rd;  // rd == nullptr: feasible mode
  double smu;
  double *ds_out, *dx_out, *atdy_out;
  SKB_DEV void load(int64_t j, Pre& p) const {
    p.v[0] = x[j];
    p.v[1] = s[j];
    p.v[2] = v[j];
    p.v[3] = rd ? rd[j] : 0.0;
  }
  SKB_DEV const double* src(int q) const { return q == 0 ? x : (q == 1 ? s : (q == 2 ? v : rd)); }
  SKB_DEV double ds_of(const Pre& p, double atdy) const {
    return rd ? dsub(-p.v[3], atdy) : -atdy;
  }
  SKB_DEV double coef(int64_t, const Pre& p, double dot) const {
    const double ds = ds_of(p, dot);
    const double xs = ddiv(p.v[0], p.v[1]);
    double dx = dadd(-p.v[0], ddiv(smu, p.v[1]));
    dx = dsub(dx, dmul(xs, ds));
    return dsub(dx, ddiv(p.v[2], p.v[1]));
  }
  SKB_DEV void emit(int64_t j, const Pre& p, double dot, double dx) const {
    ds_out[j] = ds_of(p, dot);
    dx_out[j] = dx;
    if (atdy_out) atdy_out[j] = dot;
  }
};

struct OpIter {  // make_iterate at x + a dx, y_new (=z), s + a ds (ipm_core.py:94-102)
  static constexpr bool kDot = true, kAxpy = true;
  static constexpr int kPre = 5;
  const double *x, *dx, *s, *ds, *c;
  double alpha;
  double *x_out, *s_out, *rd_out;
  SKB_DEV void load(int64_t j, Pre& p) const {
    p.v[0] = x[j];
    p.v[1] = dx ? dx[j] : 0.0;
    p.v[2] = s[j];
    p.v[3] = ds ? ds[j] : 0.0;
    p.v[4] = c[j];
  }
  SKB_DEV const double* src(int q) const {
    return q == 0 ? x : (q == 1 ? dx : (q == 2 ? s : (q == 3 ? ds : c)));
  }
  SKB_DEV double xnew(const Pre& p) const { return dx ? dadd(p.v[0], dmul(alpha, p.v[1])) : p.v[0]; }
  SKB_DEV double snew(const Pre& p) const { return ds ? dadd(p.v[2], dmul(alpha, p.v[3])) : p.v[2]; }
  SKB_DEV double coef(int64_t, const Pre& p, double) const { return xnew(p); }
  SKB_DEV void emit(int64_t j, const Pre& p, double dot, double xn) const {
    const double sn = snew(p);
    if (x_out) x_out[j] = xn;
    if (s_out) s_out[j] = sn;
    rd_out[j] = dsub(dadd(dot, sn), p.v[4]);
  }
};

// assemble_directions plus the v-invariant recheck's A (v ./ s) in the same
// pass (ipm_core.py:218-223 and :502): a second accumulator with coefficient
// v_j / s_j. Per lane and column the two accumulations are exactly those of
// OpDir and OpGemvRatio, so adx and A (v ./ s) are bitwise the separate passes'.
struct OpDirV : OpDir {
  static constexpr bool kAxpy2 = true;
  SKB_DEV double coef2(const Pre& p, double) const { return ddiv(p.v[2], p.v[1]); }
};

// make_iterate's pass at a precomputed (x_new, s_new) plus the NEXT step's
// build_rhs in the same pass (ipm_core.py:94-102 and :196-206): r_d = A'y_new +
// s_new - c from the column dot, r_p from the first accumulator (coefficient
// x_new), and p = A (x_new - smu/s_new [- (x_new/s_new) r_d]) from the second,
// smu = sigma mu_new read from the device (computed from the same x_new, s_new
// before the pass). Per element and per lane the same operations in the same
// order as OpIter's and OpRhs's passes: r_d, r_p and p are bitwise theirs.
struct OpIterP {
  static constexpr bool kDot = true, kAxpy = true, kAxpy2 = true;
  static constexpr int kPre = 3;
  const double *xn, *sn, *c;
  const double* smu_dev;
  int infeasible;
  double* rd_out;
  SKB_DEV void load(int64_t j, Pre& p) const {
    p.v[0] = xn[j];
    p.v[1] = sn[j];
    p.v[2] = c[j];
  }
  SKB_DEV const double* src(int q) const { return q == 0 ? xn : (q == 1 ? sn : c); }
  SKB_DEV double rd_of(const Pre& p, double dot) const { return dsub(dadd(dot, p.v[1]), p.v[2]); }
  SKB_DEV double coef(int64_t, const Pre& p, double) const { return p.v[0]; }
  SKB_DEV void emit(int64_t j, const Pre& p, double dot, double) const { rd_out[j] = rd_of(p, dot); }
  SKB_DEV double coef2(const Pre& p, double dot) const {  // OpRhs::coef at (x_new, s_new, r_d)
    const double smu = *smu_dev;
    double u = dsub(p.v[0], ddiv(smu, p.v[1]));
    if (infeasible) u = dsub(u, dmul(ddiv(p.v[0], p.v[1]), rd_of(p, dot)));
    return u;
  }
};

template <class Op, class = void>
struct Axpy2 {
  static constexpr bool value = false;
};
template <class Op>
struct Axpy2<Op, std::void_t<decltype(Op::kAxpy2)>> {
  static constexpr bool value = Op::kAxpy2;
};
template <class Op>
SKB_DEV double coef2_of(const Op& op, const Pre& p, double dot) {
  if constexpr (Axpy2<Op>::value) return op.coef2(p, dot);
  else return 0.0;
}

// --------------------------------------------------------------- kernel

template <int R2, bool ZREG, class Op>
__global__ void __launch_bounds__(256, 1)
    colstream_kernel(const double* __restrict__ A, int64_t lda, int m, int64_t n, int cb,
                     int stages, int64_t ngroups, const double* __restrict__ z,
                     double* __restrict__ part, Op op, const int* __restrict__ gate) {
  if (gate && *gate) return;  // gated off (e.g. PCG already stopped)
  extern __shared__ __align__(128) unsigned char smem[];
  const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t col_bytes = (size_t)lda * 8, stage_bytes = (size_t)cb * col_bytes;
  double* zs = reinterpret_cast<double*>(smem);
  size_t off = (((size_t)m * 8) + 127) & ~(size_t)127;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + off);
  off += (((size_t)nw * 4 * 8) + 127) & ~(size_t)127;
  unsigned char* bufs = smem + off;

  if (Op::kDot && !ZREG)
    for (int i = threadIdx.x; i < m; i += blockDim.x) zs[i] = z[i];
  uint64_t* mybar = bars + warp * 4;
  unsigned char* mybuf = bufs + (size_t)warp * stages * stage_bytes;
  if (lane == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&mybar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  constexpr bool A2 = Axpy2<Op>::value;
  double zr[ZREG ? 2 * R2 : 1];
  double acc[Op::kAxpy ? 2 * R2 : 1];
  double acc2[A2 ? 2 * R2 : 1];
#pragma unroll
  for (int k = 0; k < R2; ++k) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int r = 64 * k + 2 * lane + e;
      if (ZREG && Op::kDot) zr[2 * k + e] = r < m ? z[r] : 0.0;
      if (Op::kAxpy) acc[2 * k + e] = 0.0;
      if (A2) acc2[2 * k + e] = 0.0;
    }
  }

  const int64_t gw = (int64_t)blockIdx.x * nw + warp, GW = (int64_t)gridDim.x * nw;
  const int64_t my = gw < ngroups ? (ngroups - 1 - gw) / GW + 1 : 0;
  const uint64_t pol = l2_evict_first_policy();

  auto issue = [&](int64_t i, int st) {
    const int64_t c0 = (gw + i * GW) * cb;
    const int cnt = (int)min((int64_t)cb, n - c0);
    const uint32_t bytes = (uint32_t)(cnt * col_bytes);
    mbar_arrive_expect_tx(&mybar[st], bytes);
    bulk_g2s(mybuf + st * stage_bytes, A + c0 * lda, bytes, &mybar[st], pol);
  };
  if (lane == 0)
    for (int64_t i = 0; i < min((int64_t)stages, my); ++i) issue(i, (int)i);

  for (int64_t i = 0; i < my; ++i) {
    const int st = (int)(i % stages);
    const uint32_t ph = (uint32_t)((i / stages) & 1);
    const int64_t c0 = (gw + i * GW) * cb;
    const int cnt = (int)min((int64_t)cb, n - c0);
    Pre pre;
#pragma unroll
    for (int q = 0; q < 6; ++q) pre.v[q] = 0.0;
    if (lane < cnt) op.load(c0 + lane, pre);
    mbar_wait(&mybar[st], ph);
    const double* buf = reinterpret_cast<const double*>(mybuf + st * stage_bytes);
    for (int c = 0; c < cnt; ++c) {
      const double* col = buf + (size_t)c * lda;
      if constexpr (!ZREG && !A2) {
        // large m: stream the column from shared memory twice (dot, then axpy)
        double dot = 0.0;
        if (Op::kDot) {
          double d0 = 0.0, d1 = 0.0;
#pragma unroll
          for (int k = 0; k < R2; ++k) {
            const int r = 64 * k + 2 * lane;
            if (r < m) {
              const double2 t = *reinterpret_cast<const double2*>(col + r);
              const double2 zz = *reinterpret_cast<const double2*>(zs + r);  // one LDS.128
              d0 = fma(t.x, zz.x, d0);
              if (r + 1 < m) d1 = fma(t.y, zz.y, d1);
            }
          }
          dot = warp_sum(d0 + d1);
        }
        Pre pc;
#pragma unroll
        for (int q = 0; q < Op::kPre; ++q) pc.v[q] = __shfl_sync(0xffffffffu, pre.v[q], c);
        const double cf = op.coef(c0 + c, pc, dot);
        const double cf2 = coef2_of(op, pc, dot);
        if (lane == 0) op.emit(c0 + c, pc, dot, cf);
        if (Op::kAxpy) {
#pragma unroll
          for (int k = 0; k < R2; ++k) {
            const int r = 64 * k + 2 * lane;
            double2 t = make_double2(0.0, 0.0);
            if (r < m) {
              t = *reinterpret_cast<const double2*>(col + r);
              if (r + 1 >= m) t.y = 0.0;
            }
            acc[2 * k] = fma(cf, t.x, acc[2 * k]);
            acc[2 * k + 1] = fma(cf, t.y, acc[2 * k + 1]);
            if constexpr (A2) {
              acc2[2 * k] = fma(cf2, t.x, acc2[2 * k]);
              acc2[2 * k + 1] = fma(cf2, t.y, acc2[2 * k + 1]);
            }
          }
        }
        continue;
      }
      double2 a[R2];
#pragma unroll
      for (int k = 0; k < R2; ++k) {
        const int r = 64 * k + 2 * lane;
        double2 t = make_double2(0.0, 0.0);
        if (r < m) {
          t = *reinterpret_cast<const double2*>(col + r);
          if (r + 1 >= m) t.y = 0.0;
        }
        a[k] = t;
      }
      double dot = 0.0;
      if (Op::kDot) {
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int k = 0; k < R2; ++k) {
          const int r = 64 * k + 2 * lane;
          double z0, z1;
          if constexpr (ZREG) {
            z0 = zr[2 * k];
            z1 = zr[2 * k + 1];
          } else {  // one LDS.128 (zs has room past m: rows >= m are masked here)
            const double2 zz = *reinterpret_cast<const double2*>(zs + r);
            z0 = r < m ? zz.x : 0.0;
            z1 = r + 1 < m ? zz.y : 0.0;
          }
          d0 = fma(a[k].x, z0, d0);
          d1 = fma(a[k].y, z1, d1);
        }
        dot = warp_sum(d0 + d1);
      }
      Pre pc;
#pragma unroll
      for (int q = 0; q < Op::kPre; ++q) pc.v[q] = __shfl_sync(0xffffffffu, pre.v[q], c);
      const double cf = op.coef(c0 + c, pc, dot);
      if (lane == 0) op.emit(c0 + c, pc, dot, cf);
      if (Op::kAxpy) {
        const double cf2 = coef2_of(op, pc, dot);  // OpDirV (z from shared memory frees the room)
#pragma unroll
        for (int k = 0; k < R2; ++k) {
          acc[2 * k] = fma(cf, a[k].x, acc[2 * k]);
          acc[2 * k + 1] = fma(cf, a[k].y, acc[2 * k + 1]);
          if constexpr (A2) {
            acc2[2 * k] = fma(cf2, a[k].x, acc2[2 * k]);
            acc2[2 * k + 1] = fma(cf2, a[k].y, acc2[2 * k + 1]);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0 && i + stages < my) issue(i + stages, st);
  }

  if (!Op::kAxpy) return;
  __syncthreads();  // every warp is done with its stage buffers
  double* red = reinterpret_cast<double*>(bufs);
#pragma unroll
  for (int k = 0; k < R2; ++k) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int r = 64 * k + 2 * lane + e;
      if (r < m) red[(size_t)warp * m + r] = acc[2 * k + e];
    }
  }
  __syncthreads();
  for (int r = threadIdx.x; r < m; r += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += red[(size_t)w * m + r];
    part[(size_t)blockIdx.x * m + r] = s;
  }
  if constexpr (A2) {  // second m-vector: partials after the first block of partials
    __syncthreads();
#pragma unroll
    for (int k = 0; k < R2; ++k) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = 64 * k + 2 * lane + e;
        if (r < m) red[(size_t)warp * m + r] = acc2[2 * k + e];
      }
    }
    __syncthreads();
    double* part2 = part + (size_t)gridDim.x * m;
    for (int r = threadIdx.x; r < m; r += blockDim.x) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += red[(size_t)w * m + r];
      part2[(size_t)blockIdx.x * m + r] = s;
    }
  }
}

// ----------------------------------------------------- CTA-cooperative variant
// For m > 1024 (c3: m = 2000; any m up to 16384): the 256 threads of a CTA
// split the ROWS of every column (thread t owns row pairs t + 256k), so
// per-thread state stays small at any m. A stage holds cb consecutive
// columns, filled by one cp.async.bulk issued by thread 0; the column dots
// are reduced across the CTA through shared memory (fixed order), then every
// thread applies the rank-cb update to its rows. Two barriers per stage.
constexpr int kCoopThreads = 256;
constexpr int kCoopMaxCb = 8;

template <int KP, class Op>
__global__ void __launch_bounds__(kCoopThreads, KP <= 8 ? 2 : 1)
    colcoop_kernel(const double* __restrict__ A, int64_t lda, int m, int64_t n, int cb,
                   int stages, int64_t ngroups, const double* __restrict__ z,
                   double* __restrict__ part, Op op, const int* __restrict__ gate) {
  if (gate && *gate) return;
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int NW = kCoopThreads / 32;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  double* red = reinterpret_cast<double*>(smem + 256);         // [NW][kCoopMaxCb]
  double* prev = red + NW * kCoopMaxCb;                        // [kCoopMaxCb][6]
  unsigned char* bufs = smem + 256 + 8 * (NW * kCoopMaxCb + kCoopMaxCb * 6);
  bufs = reinterpret_cast<unsigned char*>(((uintptr_t)bufs + 127) & ~(uintptr_t)127);
  const size_t col_bytes = (size_t)lda * 8, stage_bytes = (size_t)cb * col_bytes;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  double zr[2 * KP], acc[2 * KP];
#pragma unroll
  for (int k = 0; k < KP; ++k) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int r = 512 * k + 2 * tid + e;
      zr[2 * k + e] = (Op::kDot && r < m) ? z[r] : 0.0;
      acc[2 * k + e] = 0.0;
    }
  }
  __syncthreads();
  const int64_t G = gridDim.x;
  const int64_t my = (int64_t)blockIdx.x < ngroups ? (ngroups - 1 - blockIdx.x) / G + 1 : 0;
  const uint64_t pol = l2_evict_first_policy();
  auto issue = [&](int64_t i, int st) {
    const int64_t c0 = ((int64_t)blockIdx.x + i * G) * cb;
    const int cnt = (int)min((int64_t)cb, n - c0);
    const uint32_t bytes = (uint32_t)(cnt * col_bytes);
    mbar_arrive_expect_tx(&full[st], bytes);
    bulk_g2s(bufs + st * stage_bytes, A + c0 * lda, bytes, &full[st], pol);
  };
  if (tid == 0)
    for (int64_t i = 0; i < min((int64_t)stages, my); ++i) issue(i, (int)i);
  for (int64_t i = 0; i < my; ++i) {
    const int st = (int)(i % stages);
    const uint32_t ph = (uint32_t)((i / stages) & 1);
    const int64_t c0 = ((int64_t)blockIdx.x + i * G) * cb;
    const int cnt = (int)min((int64_t)cb, n - c0);
    if (tid < cnt) {
      Pre p;
#pragma unroll
      for (int q = 0; q < 6; ++q) p.v[q] = 0.0;
      op.load(c0 + tid, p);
#pragma unroll
      for (int q = 0; q < 6; ++q) prev[tid * 6 + q] = p.v[q];
    }
    mbar_wait(&full[st], ph);
    const double* buf = reinterpret_cast<const double*>(bufs + st * stage_bytes);
    if (Op::kDot) {
      for (int c = 0; c < cnt; ++c) {
        const double* col = buf + (size_t)c * lda;
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          const int r = 512 * k + 2 * tid;
          if (r < m) {
            const double2 a = *reinterpret_cast<const double2*>(col + r);
            d0 = fma(a.x, zr[2 * k], d0);
            d1 = fma(r + 1 < m ? a.y : 0.0, zr[2 * k + 1], d1);
          }
        }
        const double s = warp_sum(d0 + d1);
        if (lane == 0) red[warp * kCoopMaxCb + c] = s;
      }
    }
    __syncthreads();
    for (int c = 0; c < cnt; ++c) {
      double dot = 0.0;
      if (Op::kDot) {
#pragma unroll
        for (int w = 0; w < NW; ++w) dot += red[w * kCoopMaxCb + c];
      }
      Pre pc;
#pragma unroll
      for (int q = 0; q < 6; ++q) pc.v[q] = prev[c * 6 + q];
      const double cf = op.coef(c0 + c, pc, dot);
      if (tid == c) op.emit(c0 + c, pc, dot, cf);
      if (Op::kAxpy) {
        const double* col = buf + (size_t)c * lda;
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          const int r = 512 * k + 2 * tid;
          if (r < m) {
            const double2 a = *reinterpret_cast<const double2*>(col + r);
            acc[2 * k] = fma(cf, a.x, acc[2 * k]);
            acc[2 * k + 1] = fma(cf, r + 1 < m ? a.y : 0.0, acc[2 * k + 1]);
          }
        }
      }
    }
    __syncthreads();  // stage, red and prev are free
    if (tid == 0 && i + stages < my) issue(i + stages, st);
  }
  if (!Op::kAxpy) return;
#pragma unroll
  for (int k = 0; k < KP; ++k) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int r = 512 * k + 2 * tid + e;
      if (r < m) part[(size_t)blockIdx.x * m + r] = acc[2 * k + e];
    }
  }
}

// ------------------------------------------------------ warp-pair variant
// For 1024 < m <= 2048 (c3: m = 2000): two warps stream the SAME column, each
// owning half of its rows (1024 rows = 16 row pairs per lane, z and the
// m-vector partial in registers as in colstream_kernel). A pair has its own
// TMA ring (one column per stage, one cp.async.bulk); the two half-dots meet
// in shared memory behind a 64-thread named barrier, then both warps re-read
// their half from the stage for the rank-1 update. 4 pairs per CTA, one CTA
// per SM: only pair-local barriers, unlike the CTA-wide lockstep of
// colcoop_kernel.
constexpr int kPairR2 = 16;
constexpr int kPairHalf = 64 * kPairR2;  // rows per warp

SKB_DEV void pair_bar(int id) { asm volatile("bar.sync %0, 64;\n" ::"r"(id) : "memory"); }

// The column's per-column operands (x_j, s_j, d2_j, ...) ride the same ring:
// the producer issues 8-byte cp.async copies into the stage's slot and an
// arrive.noinc on the stage barrier, so they land with the column instead of
// being loaded (latency exposed) when the column is consumed.
SKB_DEV void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
SKB_DEV void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// Only where it measured faster (m = 2000: directions 6.05 -> 4.86 ms,
// iterate 6.06 -> 5.27, rhs 4.85 -> 4.65); the one-operand passes keep the
// direct load.
template <class Op> struct PreRing { static constexpr bool value = false; };
template <> struct PreRing<OpDir> { static constexpr bool value = true; };
template <> struct PreRing<OpIter> { static constexpr bool value = true; };
template <> struct PreRing<OpRhs> { static constexpr bool value = true; };
template <> struct PreRing<OpDirV> { static constexpr bool value = true; };
template <> struct PreRing<OpIterP> { static constexpr bool value = true; };

template <class Op>
SKB_DEV void prefetch_pre(const Op& op, int64_t j, double* dst) {
#pragma unroll
  for (int q = 0; q < Op::kPre; ++q) {
    const double* src = op.src(q);
    if (src)
      cp_async8(dst + q, src + j);
    else
      dst[q] = 0.0;
  }
}
constexpr int kPairPreBytes = 2048;  // [4 pairs][<= 8 stages][8 doubles]

template <class Op>
__global__ void __launch_bounds__(256, 1)
    colpair_kernel(const double* __restrict__ A, int64_t lda, int m, int64_t n, int stages,
                   int half, const double* __restrict__ z, double* __restrict__ part, Op op,
                   const int* __restrict__ gate) {
  if (gate && *gate) return;
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int pair = warp >> 1, h = warp & 1;
  const size_t col_bytes = (size_t)lda * 8;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);               // [4][stages]
  double* dots = reinterpret_cast<double*>(smem + 8 * 4 * 8);         // [4][2]
  double* pres = reinterpret_cast<double*>(smem + 512);               // [4][stages][8]
  unsigned char* bufs = smem + 512 + kPairPreBytes;
  unsigned char* mybuf = bufs + (size_t)pair * stages * col_bytes;
  uint64_t* mybar = full + pair * stages;
  if (tid == 0) {
    for (int q = 0; q < 4 * stages; ++q) mbar_init(&full[q], 2);  // column tx + operand copies
    fence_mbar_init();
  }
  double* mypre = pres + pair * stages * 8;
  // two accumulators (OpDirV): z from shared memory, after the stage buffers
  constexpr bool A2 = Axpy2<Op>::value;
  double* zs = reinterpret_cast<double*>(
      bufs + max((size_t)4 * stages * col_bytes, (size_t)4 * m * 8));
  if (A2)
    for (int r = tid; r < m; r += blockDim.x) zs[r] = z[r];
  double zr[A2 ? 1 : 2 * kPairR2], acc[2 * kPairR2], acc2[A2 ? 2 * kPairR2 : 1];
  // warp h owns rows [h * half, min(m, (h + 1) * half)), half = ceil(m / 2) rounded to 64
  const int rbase = h * half + 2 * lane;
  const int rend = min(m, (h + 1) * half);
#pragma unroll
  for (int k = 0; k < kPairR2; ++k) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int r = rbase + 64 * k + e;
      if constexpr (!A2) zr[2 * k + e] = (Op::kDot && r < rend) ? z[r] : 0.0;
      acc[2 * k + e] = 0.0;
      if constexpr (A2) acc2[2 * k + e] = 0.0;
    }
  }
  __syncthreads();
  const int64_t gp = (int64_t)blockIdx.x * 4 + pair, GP = (int64_t)gridDim.x * 4;
  const int64_t my = gp < n ? (n - 1 - gp) / GP + 1 : 0;
  const uint64_t pol = l2_evict_first_policy();
  const bool producer = h == 0 && lane == 0;
  auto issue = [&](int64_t i, int st) {
    const int64_t j = gp + i * GP;
    mbar_arrive_expect_tx(&mybar[st], (uint32_t)col_bytes);
    bulk_g2s(mybuf + st * col_bytes, A + j * lda, (uint32_t)col_bytes, &mybar[st], pol);
    if (PreRing<Op>::value) prefetch_pre(op, j, mypre + st * 8);
    cp_async_arrive_noinc(&mybar[st]);  // (no copies pending: arrives at once)
  };
  if (producer)
    for (int64_t i = 0; i < min((int64_t)stages, my); ++i) issue(i, (int)i);
  const int bar_id = 1 + pair;
  for (int64_t i = 0; i < my; ++i) {
    const int st = (int)(i % stages);
    const uint32_t ph = (uint32_t)((i / stages) & 1);
    const int64_t j = gp + i * GP;
    Pre pre;
#pragma unroll
    for (int q = 0; q < 6; ++q) pre.v[q] = 0.0;
    if (!PreRing<Op>::value) op.load(j, pre);
    mbar_wait(&mybar[st], ph);
    if (PreRing<Op>::value) {
#pragma unroll
      for (int q = 0; q < Op::kPre; ++q) pre.v[q] = mypre[st * 8 + q];
    }
    const double* col = reinterpret_cast<const double*>(mybuf + st * col_bytes);
    double dot = 0.0;
    if (Op::kDot) {
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int k = 0; k < kPairR2; ++k) {
        const int r = rbase + 64 * k;
        if (r < rend) {
          const double2 a = *reinterpret_cast<const double2*>(col + r);
          double z0, z1;
          if constexpr (A2) {
            const double2 zz = *reinterpret_cast<const double2*>(zs + r);  // one LDS.128
            z0 = zz.x;
            z1 = r + 1 < rend ? zz.y : 0.0;
          } else {
            z0 = zr[2 * k];
            z1 = zr[2 * k + 1];
          }
          d0 = fma(a.x, z0, d0);
          d1 = fma(r + 1 < rend ? a.y : 0.0, z1, d1);
        }
      }
      const double sh = warp_sum(d0 + d1);
      if (lane == 0) dots[pair * 2 + h] = sh;
      pair_bar(bar_id);
      dot = dots[pair * 2] + dots[pair * 2 + 1];
    }
    const double cf = op.coef(j, pre, dot);
    const double cf2 = coef2_of(op, pre, dot);
    if (producer) op.emit(j, pre, dot, cf);
    if (Op::kAxpy) {
#pragma unroll
      for (int k = 0; k < kPairR2; ++k) {
        const int r = rbase + 64 * k;
        if (r < rend) {
          const double2 a = *reinterpret_cast<const double2*>(col + r);
          acc[2 * k] = fma(cf, a.x, acc[2 * k]);
          acc[2 * k + 1] = fma(cf, r + 1 < rend ? a.y : 0.0, acc[2 * k + 1]);
          if constexpr (A2) {
            acc2[2 * k] = fma(cf2, a.x, acc2[2 * k]);
            acc2[2 * k + 1] = fma(cf2, r + 1 < rend ? a.y : 0.0, acc2[2 * k + 1]);
          }
        }
      }
    }
    pair_bar(bar_id);  // both halves done with the stage (and with dots)
    if (producer && i + stages < my) issue(i + stages, st);
  }
  if (!Op::kAxpy) return;
  __syncthreads();
  double* red = reinterpret_cast<double*>(bufs);  // [4][m]
#pragma unroll
  for (int k = 0; k < kPairR2; ++k) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int r = rbase + 64 * k + e;
      if (r < rend) red[(size_t)pair * m + r] = acc[2 * k + e];
    }
  }
  __syncthreads();
  for (int r = tid; r < m; r += blockDim.x)
    part[(size_t)blockIdx.x * m + r] =
        (red[r] + red[(size_t)m + r]) + (red[2 * (size_t)m + r] + red[3 * (size_t)m + r]);
  if constexpr (A2) {  // second m-vector: partials after the first block of partials
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPairR2; ++k) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = rbase + 64 * k + e;
        if (r < rend) red[(size_t)pair * m + r] = acc2[2 * k + e];
      }
    }
    __syncthreads();
    double* part2 = part + (size_t)gridDim.x * m;
    for (int r = tid; r < m; r += blockDim.x)
      part2[(size_t)blockIdx.x * m + r] =
          (red[r] + red[(size_t)m + r]) + (red[2 * (size_t)m + r] + red[3 * (size_t)m + r]);
  }
}

// out[i] = sum_b part[b][i] (fixed order: 8 interleaved slices, combined in order) - sub[i]
__global__ void reduce_partials_kernel(const double* __restrict__ part, int nb, int m,
                                       const double* __restrict__ sub, double* __restrict__ out,
                                       const int* __restrict__ gate) {
  if (gate && *gate) return;
  __shared__ double sm[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int r = blockIdx.x * 32 + tx;
  double s = 0.0;
  if (r < m)
    for (int b = ty; b < nb; b += 8) s += part[(size_t)b * m + r];
  sm[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && r < m) {
    double t = ((sm[0][tx] + sm[1][tx]) + (sm[2][tx] + sm[3][tx])) +
               ((sm[4][tx] + sm[5][tx]) + (sm[6][tx] + sm[7][tx]));
    out[r] = sub ? __dsub_rn(t, sub[r]) : t;
  }
}

// ------------------------------------------------------------- launching

struct StreamCfg {
  int nw, stages, cb, grid;
  size_t smem;
  int64_t ngroups;
};

static StreamCfg stream_cfg(int m, int64_t n, int64_t lda) {
  StreamCfg c;
  const size_t col_bytes = (size_t)lda * 8;
  c.cb = (int)std::max<size_t>(1, std::min<size_t>(32, 8192 / col_bytes));
  const size_t stage_bytes = (size_t)c.cb * col_bytes;
  const size_t zb = (((size_t)m * 8) + 127) & ~(size_t)127;
  const size_t budget = 220 * 1024 - zb - 256;
  c.nw = 8;
  while (c.nw > 1 && (size_t)c.nw * 2 * stage_bytes > budget) c.nw >>= 1;
  c.stages = (int)std::min<size_t>(4, budget / ((size_t)c.nw * stage_bytes));
  size_t bufb = (size_t)c.nw * c.stages * stage_bytes;
  bufb = std::max(bufb, (size_t)c.nw * m * 8);  // epilogue reuse
  c.smem = zb + 256 + bufb;
  c.ngroups = (n + c.cb - 1) / c.cb;
  const int64_t need = (c.ngroups + c.nw - 1) / c.nw;
  c.grid = (int)std::max<int64_t>(1, std::min<int64_t>(skb_num_sms(), need));
  return c;
}

constexpr int kCoopMaxM = 16384;

static StreamCfg coop_cfg(int m, int64_t n, int64_t lda) {
  StreamCfg c;
  const size_t col_bytes = (size_t)lda * 8;
  c.cb = (int)std::max<size_t>(1, std::min<size_t>(kCoopMaxCb, 32768 / col_bytes));
  const size_t stage_bytes = (size_t)c.cb * col_bytes;
  const size_t head = 256 + 8 * (8 * kCoopMaxCb + kCoopMaxCb * 6) + 128;
  // CTAs per SM: the CTA runs its stages in lockstep, so a second resident CTA
  // overlaps one CTA's reduction latency with the other's streaming.
  static const int cps_env = getenv("SKB_COOP_CPS") ? atoi(getenv("SKB_COOP_CPS")) : 2;
  const int cps = m > 4096 ? 1 : cps_env;  // KP > 8 instantiations are 1 CTA/SM
  const size_t budget = (size_t)(200 * 1024) / (size_t)std::max(1, cps);
  c.stages = (int)std::max<size_t>(2, std::min<size_t>(8, budget / stage_bytes));
  while (c.stages > 2 && head + c.stages * stage_bytes > 225 * 1024) --c.stages;
  c.nw = kCoopThreads / 32;
  c.smem = head + (size_t)c.stages * stage_bytes;
  c.ngroups = (n + c.cb - 1) / c.cb;
  c.grid = (int)std::max<int64_t>(
      1, std::min<int64_t>((int64_t)skb_num_sms() * std::max(1, cps), c.ngroups));
  return c;
}

template <int KP, class Op>
static int launch_coop(const StreamCfg& c, const double* A, int64_t lda, int m, int64_t n,
                       const double* z, double* part, const Op& op, cudaStream_t st,
                       const int* gate) {
  auto kern = colcoop_kernel<KP, Op>;
  static size_t configured = 0;
  if (c.smem > configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem) !=
        cudaSuccess)
      return SKB_ERR_CUDA;
    configured = c.smem;
  }
  kern<<<c.grid, kCoopThreads, c.smem, st>>>(A, lda, m, n, c.cb, c.stages, c.ngroups, z, part, op,
                                             gate);
  return 0;
}

template <int R2, bool ZREG, class Op>
static int launch_r2(const StreamCfg& c, const double* A, int64_t lda, int m, int64_t n,
                     const double* z, double* part, const Op& op, cudaStream_t st,
                     const int* gate) {
  auto kern = colstream_kernel<R2, ZREG, Op>;
  static size_t configured = 0;
  if (c.smem > configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem) !=
        cudaSuccess)
      return SKB_ERR_CUDA;
    configured = c.smem;
  }
  kern<<<c.grid, c.nw * 32, c.smem, st>>>(A, lda, m, n, c.cb, c.stages, c.ngroups, z, part, op,
                                          gate);
  return 0;
}

// Runs the streaming pass. With part_ext != nullptr the per-CTA partials are
// written there (nparts_out receives their count) and the final reduction is
// left to the caller (skb_reduce_partials); otherwise out = sum - sub.
// ---- Dense passes past the staged kernels' shared-memory ceiling (two columns
// of m doubles per ring no longer fit: m > ~13,900). Two passes over A: (1) one
// warp per column forms the dot with z (read through L1/L2), the coefficient and
// the per-column outputs, and keeps the coefficient; (2) CTAs over (row block x
// column chunk) accumulate cf_j A[:, j] for their rows in registers (coalesced
// along the column) into per-chunk partials, which the usual fixed-order reduce
// sums. Deterministic; a robustness path, not a configuration's hot path.
template <class Op>
__global__ void __launch_bounds__(256)
    colwarp_dot_kernel(const double* __restrict__ A, int64_t lda, int m, int64_t n,
                       const double* __restrict__ z, double* __restrict__ cfo, Op op,
                       const int* __restrict__ gate) {
  if (gate && *gate) return;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t j = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); j < n; j += nw) {
    Pre p;
#pragma unroll
    for (int q = 0; q < 6; ++q) p.v[q] = 0.0;
    op.load(j, p);
    double dot = 0.0;
    if (Op::kDot) {
      const double* col = A + j * lda;
      for (int r = 2 * lane; r < m; r += 64) {
        const double2 a = *reinterpret_cast<const double2*>(col + r);
        dot = fma(a.x, __ldg(&z[r]), dot);
        if (r + 1 < m) dot = fma(a.y, __ldg(&z[r + 1]), dot);
      }
      dot = warp_sum(dot);
    }
    const double cf = op.coef(j, p, dot);
    if (lane == 0) {
      op.emit(j, p, dot, cf);
      if (Op::kAxpy) cfo[j] = cf;
    }
  }
}

constexpr int kBlkRows = 4096, kBlkPer = kBlkRows / 256;  // rows per CTA, per thread

__global__ void __launch_bounds__(256)
    colblk_axpy_kernel(const double* __restrict__ A, int64_t lda, int m, int64_t n,
                       const double* __restrict__ cf, int64_t chunk, double* __restrict__ part,
                       const int* __restrict__ gate) {
  if (gate && *gate) return;
  const int r0 = blockIdx.y * kBlkRows;
  const int64_t j0 = (int64_t)blockIdx.x * chunk, j1 = min(n, j0 + chunk);
  double acc[kBlkPer];
#pragma unroll
  for (int k = 0; k < kBlkPer; ++k) acc[k] = 0.0;
  for (int64_t j = j0; j < j1; ++j) {
    const double c = __ldg(&cf[j]);
    const double* col = A + j * lda;
#pragma unroll
    for (int k = 0; k < kBlkPer; ++k) {
      const int r = r0 + threadIdx.x + 256 * k;
      if (r < m) acc[k] = fma(c, col[r], acc[k]);
    }
  }
  double* o = part + (int64_t)blockIdx.x * m;
#pragma unroll
  for (int k = 0; k < kBlkPer; ++k) {
    const int r = r0 + threadIdx.x + 256 * k;
    if (r < m) o[r] = acc[k];
  }
}

template <class Op>
static int run_stream_global(const double* A, int64_t lda, int m, int64_t n, const double* z,
                             double* out, const double* sub, const Op& op, skb_ws* ws,
                             cudaStream_t st, const int* gate, double* part_ext,
                             int* nparts_out) {
  const int rb = (m + kBlkRows - 1) / kBlkRows;
  int64_t chunks = std::max<int64_t>(1, std::min<int64_t>(4 * skb_num_sms() / rb, n));
  double* cf = nullptr;
  if (Op::kAxpy) {
    cf = (double*)skb_ws_take(ws, (size_t)n * 8);
    if (!cf) return SKB_ERR_WORKSPACE;
  }
  if (n > 0)
    colwarp_dot_kernel<Op><<<(unsigned)std::min<int64_t>(8 * skb_num_sms(), (n + 7) / 8), 256, 0,
                             st>>>(A, lda, m, n, z, cf, op, gate);
  if (!Op::kAxpy) return skb_launch_status(__func__);
  double* part = part_ext;
  if (!part) {
    part = (double*)skb_ws_take(ws, (size_t)chunks * m * 8);
    if (!part) return SKB_ERR_WORKSPACE;
  }
  const int64_t chunk = (n + chunks - 1) / chunks;
  chunks = n > 0 ? (n + chunk - 1) / chunk : 0;
  if (nparts_out) *nparts_out = (int)chunks;
  if (chunks > 0)
    colblk_axpy_kernel<<<dim3((unsigned)chunks, (unsigned)rb), 256, 0, st>>>(A, lda, m, n, cf,
                                                                            chunk, part, gate);
  if (!part_ext)
    reduce_partials_kernel<<<(m + 31) / 32, 256, 0, st>>>(part, (int)chunks, m, sub, out, gate);
  return skb_launch_status(__func__);
}

template <class Op>
static int run_stream(const double* A, int64_t lda, int m, int64_t n, const double* z,
                      double* out, const double* sub, const Op& op, skb_ws* ws,
                      cudaStream_t st, const int* gate = nullptr, double* part_ext = nullptr,
                      int* nparts_out = nullptr) {
  if (m < 1 || n < 0 || lda < m || (lda & 1) || ((uintptr_t)A & 15)) return SKB_ERR_ARG;
  if (m > 1024 && (m > kCoopMaxM || coop_cfg(m, n, lda).smem > 225 * 1024))
    return run_stream_global(A, lda, m, n, z, out, sub, op, ws, st, gate, part_ext, nparts_out);
  if (n == 0) {
    if (nparts_out) *nparts_out = 0;
    if (Op::kAxpy && !part_ext) {
      if (sub) {
        reduce_partials_kernel<<<(m + 31) / 32, 256, 0, st>>>(nullptr, 0, m, sub, out, gate);
      } else {
        cudaMemsetAsync(out, 0, (size_t)m * 8, st);
      }
    }
    return 0;
  }
  static const bool no_pair = getenv("SKB_NO_PAIR") != nullptr;
  if (m > 1024 && m <= 2 * kPairHalf && !no_pair) {
    const size_t col_bytes = (size_t)lda * 8;
    int stages = (int)std::min<size_t>(6, (218 * 1024 - 512 - kPairPreBytes) / (4 * col_bytes));
    if (stages >= 2) {
      const size_t smem =
          512 + kPairPreBytes + std::max((size_t)4 * stages * col_bytes, (size_t)4 * m * 8);
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(skb_num_sms(), (n + 3) / 4));
      double* part = part_ext;
      if (Op::kAxpy && !part) {
        part = (double*)skb_ws_take(ws, (size_t)grid * m * 8);
        if (!part) return SKB_ERR_WORKSPACE;
      }
      if (nparts_out) *nparts_out = grid;
      auto kern = colpair_kernel<Op>;
      static size_t configured = 0;
      if (smem > configured) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) != cudaSuccess)
          return SKB_ERR_CUDA;
        configured = smem;
      }
      const int half = ((m + 1) / 2 + 63) / 64 * 64;
      kern<<<grid, 256, smem, st>>>(A, lda, m, n, stages, half, z, part, op, gate);
      if (Op::kAxpy && !part_ext)
        reduce_partials_kernel<<<(m + 31) / 32, 256, 0, st>>>(part, grid, m, sub, out, gate);
      return skb_launch_status(__func__);
    }
  }
  const StreamCfg c = m > 1024 ? coop_cfg(m, n, lda) : stream_cfg(m, n, lda);
  double* part = part_ext;
  if (Op::kAxpy && !part) {
    part = (double*)skb_ws_take(ws, (size_t)c.grid * m * 8);
    if (!part) return SKB_ERR_WORKSPACE;
  }
  if (nparts_out) *nparts_out = c.grid;
  int rc;
  if (m > 1024) {
    if (m <= 2048)
      rc = launch_coop<4>(c, A, lda, m, n, z, part, op, st, gate);
    else if (m <= 4096)
      rc = launch_coop<8>(c, A, lda, m, n, z, part, op, st, gate);
    else if (m <= 8192)
      rc = launch_coop<16>(c, A, lda, m, n, z, part, op, st, gate);
    else
      rc = launch_coop<32>(c, A, lda, m, n, z, part, op, st, gate);
  } else if (m <= 64)
    rc = launch_r2<1, true>(c, A, lda, m, n, z, part, op, st, gate);
  else if (m <= 128)
    rc = launch_r2<2, true>(c, A, lda, m, n, z, part, op, st, gate);
  else if (m <= 256)
    rc = launch_r2<4, true>(c, A, lda, m, n, z, part, op, st, gate);
  else if (m <= 512)
    rc = launch_r2<8, true>(c, A, lda, m, n, z, part, op, st, gate);
  else
    rc = launch_r2<16, true>(c, A, lda, m, n, z, part, op, st, gate);
  if (rc) return rc;
  if (Op::kAxpy && !part_ext)
    reduce_partials_kernel<<<(m + 31) / 32, 256, 0, st>>>(part, c.grid, m, sub, out, gate);
  return skb_launch_status(__func__);
}

}  // namespace skb

using namespace skb;

#define SKB_WS skb_ws ws = skb_ws_make(workspace, ws_bytes)

extern "C" int skb_normal_apply(const double* A, int64_t m, int64_t n, int64_t lda,
                                const double* d2, const double* z, double* u, const double* sub,
                                const int* gate, void* workspace, size_t ws_bytes, void* stream) {
  SKB_WS;
  OpNormal op{d2};
  return run_stream(A, lda, (int)m, n, z, u, sub, op, &ws, (cudaStream_t)stream, gate);
}

extern "C" int skb_normal_apply_partials(const double* A, int64_t m, int64_t n, int64_t lda,
                                         const double* d2, const double* z, double* part,
                                         int32_t* nparts_host, void* stream) {
  OpNormal op{d2};
  int np = 0;
  int rc = run_stream(A, lda, (int)m, n, z, nullptr, nullptr, op, nullptr,
                      (cudaStream_t)stream, nullptr, part, &np);
  if (nparts_host) *nparts_host = np;
  return rc;
}

extern "C" int skb_gemv(const double* A, int64_t m, int64_t n, int64_t lda, const double* x,
                        double* u, const double* sub, void* workspace, size_t ws_bytes,
                        void* stream) {
  SKB_WS;
  OpGemvX op{x};
  return run_stream(A, lda, (int)m, n, nullptr, u, sub, op, &ws, (cudaStream_t)stream);
}

extern "C" int skb_gemv_ratio(const double* A, int64_t m, int64_t n, int64_t lda,
                              const double* v, const double* s, double* u, const double* sub,
                              void* workspace, size_t ws_bytes, void* stream) {
  SKB_WS;
  OpGemvRatio op{v, s};
  return run_stream(A, lda, (int)m, n, nullptr, u, sub, op, &ws, (cudaStream_t)stream);
}

extern "C" int skb_rhs(const double* A, int64_t m, int64_t n, int64_t lda, const double* x,
                       const double* s, const double* r_d, double sigma_mu, double* p,
                       const double* r_p, void* workspace, size_t ws_bytes, void* stream) {
  SKB_WS;
  OpRhs op{x, s, r_d, sigma_mu};
  return run_stream(A, lda, (int)m, n, nullptr, p, r_p, op, &ws, (cudaStream_t)stream);
}

extern "C" int skb_gemv_t(const double* A, int64_t m, int64_t n, int64_t lda, const double* y,
                          const double* add, const double* sub, double* t, void* workspace,
                          size_t ws_bytes, void* stream) {
  SKB_WS;
  OpGemvT op{add, sub, t};
  return run_stream(A, lda, (int)m, n, y, nullptr, nullptr, op, &ws, (cudaStream_t)stream);
}

extern "C" int skb_directions(const double* A, int64_t m, int64_t n, int64_t lda,
                              const double* dy, const double* x, const double* s,
                              const double* v, const double* r_d, double sigma_mu, double* ds,
                              double* dx, double* atdy, double* adx, void* workspace,
                              size_t ws_bytes, void* stream) {
  SKB_WS;
  OpDir op{x, s, v, r_d, sigma_mu, ds, dx, atdy};
  return run_stream(A, lda, (int)m, n, dy, adx, nullptr, op, &ws, (cudaStream_t)stream);
}

// Two-accumulator passes (OpDirV, OpIterP): dense, m <= 2048 (column stream with
// z from shared memory, or the warp pair); out1 = sum1 - sub1, out2 = sum2 - sub2
// (sub2 is applied after out1 is written, so it may be out1). Returns
// SKB_ERR_UNSUPPORTED where the fused pass does not apply (the caller then runs
// the two single passes).
template <class Op>
static int run_stream2(const double* A, int64_t lda, int64_t m, int64_t n, const double* z,
                       double* out1, const double* sub1, double* out2, const double* sub2,
                       const Op& op, skb_ws* ws, cudaStream_t st) {
  if (m < 1 || m > 2 * kPairHalf || n < 1 || lda < m || (lda & 1) || ((uintptr_t)A & 15))
    return SKB_ERR_UNSUPPORTED;
  int grid;
  double* part;
  if (m > 1024) {
    static const bool no_pair = getenv("SKB_NO_PAIR") != nullptr;
    if (no_pair) return SKB_ERR_UNSUPPORTED;
    const size_t col_bytes = (size_t)lda * 8;
    const size_t zb = (size_t)m * 8;
    int stages = (int)std::min<size_t>(6, (218 * 1024 - 512 - kPairPreBytes - zb) /
                                              (4 * col_bytes));
    if (stages < 2) return SKB_ERR_UNSUPPORTED;
    const size_t smem = 512 + kPairPreBytes +
                        std::max((size_t)4 * stages * col_bytes, (size_t)4 * m * 8) + zb;
    grid = (int)std::max<int64_t>(1, std::min<int64_t>(skb_num_sms(), (n + 3) / 4));
    part = (double*)skb_ws_take(ws, (size_t)2 * grid * m * 8);
    if (!part) return SKB_ERR_WORKSPACE;
    auto kern = colpair_kernel<Op>;
    static size_t configured = 0;
    if (smem > configured) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
          cudaSuccess)
        return SKB_ERR_CUDA;
      configured = smem;
    }
    const int half = (((int)m + 1) / 2 + 63) / 64 * 64;
    kern<<<grid, 256, smem, st>>>(A, lda, (int)m, n, stages, half, z, part, op, nullptr);
  } else {
    // the column stays in registers, z comes from shared memory (z in registers
    // too spills at m = 1000: 2.71 ms against 1.34 ms for OpDirV at c2)
    const StreamCfg c = stream_cfg((int)m, n, lda);
    grid = c.grid;
    part = (double*)skb_ws_take(ws, (size_t)2 * c.grid * m * 8);
    if (!part) return SKB_ERR_WORKSPACE;
    int rc;
    if (m <= 64)
      rc = launch_r2<1, false>(c, A, lda, (int)m, n, z, part, op, st, nullptr);
    else if (m <= 128)
      rc = launch_r2<2, false>(c, A, lda, (int)m, n, z, part, op, st, nullptr);
    else if (m <= 256)
      rc = launch_r2<4, false>(c, A, lda, (int)m, n, z, part, op, st, nullptr);
    else if (m <= 512)
      rc = launch_r2<8, false>(c, A, lda, (int)m, n, z, part, op, st, nullptr);
    else
      rc = launch_r2<16, false>(c, A, lda, (int)m, n, z, part, op, st, nullptr);
    if (rc) return rc;
  }
  reduce_partials_kernel<<<(unsigned)((m + 31) / 32), 256, 0, st>>>(part, grid, (int)m, sub1,
                                                                    out1, nullptr);
  reduce_partials_kernel<<<(unsigned)((m + 31) / 32), 256, 0, st>>>(
      part + (size_t)grid * m, grid, (int)m, sub2, out2, nullptr);
  return skb_launch_status("skb_stream2");
}

extern "C" int skb_directions_v(const double* A, int64_t m, int64_t n, int64_t lda,
                                const double* dy, const double* x, const double* s,
                                const double* v, const double* r_d, double sigma_mu, double* ds,
                                double* dx, double* atdy, double* adx, double* avs,
                                void* workspace, size_t ws_bytes, void* stream) {
  SKB_WS;
  OpDirV op;
  static_cast<OpDir&>(op) = OpDir{x, s, v, r_d, sigma_mu, ds, dx, atdy};
  return run_stream2(A, lda, m, n, dy, adx, nullptr, avs, nullptr, op, &ws,
                     (cudaStream_t)stream);
}

extern "C" int skb_iterate_rhs(const double* A, int64_t m, int64_t n, int64_t lda,
                               const double* xn, const double* sn, const double* y_new,
                               const double* c, const double* smu_dev, int32_t infeasible,
                               const double* b, double* r_p, double* r_d, double* p,
                               int32_t p_sub_rp, void* workspace, size_t ws_bytes, void* stream) {
  SKB_WS;
  OpIterP op{xn, sn, c, smu_dev, infeasible, r_d};
  return run_stream2(A, lda, m, n, y_new, r_p, b, p, p_sub_rp ? r_p : nullptr, op, &ws,
                     (cudaStream_t)stream);
}

extern "C" int skb_iterate(const double* A, int64_t m, int64_t n, int64_t lda, const double* x,
                           const double* dx, const double* s, const double* ds, double alpha,
                           const double* y_new, const double* b, const double* c,
                           double* x_out, double* s_out, double* r_p, double* r_d,
                           void* workspace, size_t ws_bytes, void* stream) {
  SKB_WS;
  OpIter op{x, dx, s, ds, c, alpha, x_out, s_out, r_d};
  return run_stream(A, lda, (int)m, n, y_new, r_p, b, op, &ws, (cudaStream_t)stream);
}

extern "C" int skb_reduce_partials(const double* part, int32_t nparts, int64_t m,
                                   const double* sub, double* out, void* stream) {
  reduce_partials_kernel<<<(unsigned)((m + 31) / 32), 256, 0, (cudaStream_t)stream>>>(
      part, nparts, (int)m, sub, out, nullptr);
  return skb_launch_status(__func__);
}

extern "C" size_t skb_stream_workspace_bytes(int64_t m) {
  return (size_t)4 * skb_num_sms() * (size_t)m * 8 + 256;  // up to 4 partials per SM
}

// ===================================================== sparse A (CSC), c4
// The same Op family over a CSC matrix (colptr int64 n+1, rowidx int32, vals):
// one thread per column (coalesced colptr/pre loads), z and the CTA's partial
// m-vector in shared memory; the column dot gathers z, the update scatters
// into the partial with shared-memory atomics. Per-CTA partials are reduced in
// a fixed order as for the dense path; the order of additions inside a CTA
// follows the hardware's atomic arbitration (tolerance parity, not bitwise).
namespace skb {

// 1024 threads (32 warps) hide the dependent colptr -> rowidx -> z loads of the
// one-CTA-per-SM normal apply (0.62 -> 0.48 ms at c4); the axpy-only passes run
// two 512-thread CTAs per SM (their single m-vector leaves room for two).
// (Gathering z through L1 to fit two 1024-thread CTAs doubled the time.)
constexpr int kCscThreads = 1024;

// ELL head records (skb_csc_ell_build, once per matrix): 64 bytes per column
// holding its first kEll rows (u16) and values, the count in byte 10 (255:
// longer column, read from the CSC arrays). Thread j's record is one
// contiguous 64-byte load independent of colptr: the dependent
// colptr -> rowidx -> z chain of the plain CSC walk disappears.
constexpr int kEll = 5;
struct __align__(16) EllRec {
  uint16_t row[kEll];
  uint8_t cnt, pad[5];
  double val[kEll];
  int64_t spare;
};
static_assert(sizeof(EllRec) == 64, "ELL record");

template <class Op, bool ELL>
__global__ void __launch_bounds__(kCscThreads)
    csc_kernel(const int64_t* __restrict__ colptr, const int32_t* __restrict__ rowidx,
               const double* __restrict__ vals, const EllRec* __restrict__ ell, int m, int64_t n,
               const double* __restrict__ z, double* __restrict__ part, Op op,
               const int* __restrict__ gate) {
  if (gate && *gate) return;
  extern __shared__ __align__(16) double csm[];
  double* zs = csm;
  double* us = csm + (Op::kDot ? m : 0);
  if (Op::kDot)
    for (int i = threadIdx.x; i < m; i += blockDim.x) zs[i] = z[i];
  if (Op::kAxpy)
    for (int i = threadIdx.x; i < m; i += blockDim.x) us[i] = 0.0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ELL) {  // two records per thread in flight: the loads' latency, not the
              // shared-memory work, bounded the one-at-a-time loop (ncu: long_scoreboard 65 %)
    for (; j + stride < n; j += 2 * stride) {
      Pre p[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int q = 0; q < 6; ++q) p[h].v[q] = 0.0;
        op.load(j + h * stride, p[h]);
      }
      const EllRec r2[2] = {ell[j], ell[j + stride]};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const EllRec& r = r2[h];
        const int64_t jj = j + h * stride;
        if (r.cnt <= kEll) {
          double dot = 0.0;
          if (Op::kDot) {
#pragma unroll
            for (int q = 0; q < kEll; ++q)
              if (q < r.cnt) dot = fma(r.val[q], zs[r.row[q]], dot);
          }
          const double cf = op.coef(jj, p[h], dot);
          op.emit(jj, p[h], dot, cf);
          if (Op::kAxpy) {
#pragma unroll
            for (int q = 0; q < kEll; ++q)
              if (q < r.cnt) atomicAdd(&us[r.row[q]], cf * r.val[q]);
          }
        } else {
          const int64_t e0 = colptr[jj], e1 = colptr[jj + 1];
          double dot = 0.0;
          if (Op::kDot)
            for (int64_t e = e0; e < e1; ++e) dot = fma(vals[e], zs[rowidx[e]], dot);
          const double cf = op.coef(jj, p[h], dot);
          op.emit(jj, p[h], dot, cf);
          if (Op::kAxpy)
            for (int64_t e = e0; e < e1; ++e) atomicAdd(&us[rowidx[e]], cf * vals[e]);
        }
      }
    }
  }
  for (; j < n; j += stride) {
    Pre p;
#pragma unroll
    for (int q = 0; q < 6; ++q) p.v[q] = 0.0;
    op.load(j, p);
    if (ELL) {
      const EllRec r = ell[j];
      if (r.cnt <= kEll) {
        double dot = 0.0;
        if (Op::kDot) {
#pragma unroll
          for (int q = 0; q < kEll; ++q)
            if (q < r.cnt) dot = fma(r.val[q], zs[r.row[q]], dot);
        }
        const double cf = op.coef(j, p, dot);
        op.emit(j, p, dot, cf);
        if (Op::kAxpy) {
#pragma unroll
          for (int q = 0; q < kEll; ++q)
            if (q < r.cnt) atomicAdd(&us[r.row[q]], cf * r.val[q]);
        }
        continue;
      }
    }
    const int64_t e0 = colptr[j], e1 = colptr[j + 1];
    double dot = 0.0;
    if (Op::kDot)
      for (int64_t e = e0; e < e1; ++e) dot = fma(vals[e], zs[rowidx[e]], dot);
    const double cf = op.coef(j, p, dot);
    op.emit(j, p, dot, cf);
    if (Op::kAxpy)
      for (int64_t e = e0; e < e1; ++e) atomicAdd(&us[rowidx[e]], cf * vals[e]);
  }
  if (!Op::kAxpy) return;
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) part[(size_t)blockIdx.x * m + i] = us[i];
}

// CSC pass for m past the shared-memory kernels' ceiling (z and the partial
// m-vector no longer fit next to each other): z read through L1/L2, the products
// added straight into one global m-vector with fp64 RED (arbitration order, as
// the shared atomics above), then the same reduce / subtract epilogue.
template <class Op>
__global__ void __launch_bounds__(256)
    csc_global_kernel(const int64_t* __restrict__ colptr, const int32_t* __restrict__ rowidx,
                      const double* __restrict__ vals, int64_t n, const double* __restrict__ z,
                      double* __restrict__ acc, Op op, const int* __restrict__ gate) {
  if (gate && *gate) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    Pre p;
#pragma unroll
    for (int q = 0; q < 6; ++q) p.v[q] = 0.0;
    op.load(j, p);
    const int64_t e0 = colptr[j], e1 = colptr[j + 1];
    double dot = 0.0;
    if (Op::kDot)
      for (int64_t e = e0; e < e1; ++e) dot = fma(vals[e], __ldg(&z[rowidx[e]]), dot);
    const double cf = op.coef(j, p, dot);
    op.emit(j, p, dot, cf);
    if (Op::kAxpy)
      for (int64_t e = e0; e < e1; ++e) atomicAdd(&acc[rowidx[e]], cf * vals[e]);
  }
}

template <class Op>
static int run_csc(const int64_t* colptr, const int32_t* rowidx, const double* vals, int m,
                   int64_t n, const double* z, double* out, const double* sub, const Op& op,
                   skb_ws* ws, cudaStream_t st, const int* gate = nullptr,
                   const void* ell = nullptr) {
  if (m < 1 || n < 0) return SKB_ERR_ARG;
  const size_t smem = (size_t)((Op::kDot ? m : 0) + (Op::kAxpy ? m : 0)) * 8;
  if (smem > 220 * 1024) {  // m > 14080 with both vectors (28160 with one)
    double* acc = nullptr;
    if (Op::kAxpy) {
      acc = (double*)skb_ws_take(ws, (size_t)m * 8);
      if (!acc) return SKB_ERR_WORKSPACE;
      cudaMemsetAsync(acc, 0, (size_t)m * 8, st);
    }
    if (n > 0) {
      const int grid = (int)std::max<int64_t>(
          1, std::min<int64_t>((int64_t)skb_num_sms() * 8, (n + 255) / 256));
      csc_global_kernel<Op><<<grid, 256, 0, st>>>(colptr, rowidx, vals, n, z, acc, op, gate);
    }
    if (Op::kAxpy)
      reduce_partials_kernel<<<(m + 31) / 32, 256, 0, st>>>(acc, n > 0 ? 1 : 0, m, sub, out,
                                                            gate);
    return skb_launch_status(__func__);
  }
  const int per_sm = smem <= 100 * 1024 ? 2 : 1;
  int grid = skb_num_sms() * per_sm;
  const int thr = (Op::kDot || !Op::kAxpy) ? kCscThreads : 512;
  const int64_t need = (n + thr - 1) / thr;
  if (need < grid) grid = (int)std::max<int64_t>(1, need);
  double* part = nullptr;
  if (Op::kAxpy) {
    part = (double*)skb_ws_take(ws, (size_t)grid * m * 8);
    if (!part) return SKB_ERR_WORKSPACE;
  }
  auto kern = ell ? csc_kernel<Op, true> : csc_kernel<Op, false>;
  static size_t configured[2] = {0, 0};
  if (smem > 48 * 1024 && smem > configured[ell ? 1 : 0]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return SKB_ERR_CUDA;
    configured[ell ? 1 : 0] = smem;
  }
  if (n > 0)
    kern<<<grid, thr, smem, st>>>(colptr, rowidx, vals, (const EllRec*)ell, m, n, z, part, op,
                                  gate);
  if (Op::kAxpy)
    reduce_partials_kernel<<<(m + 31) / 32, 256, 0, st>>>(part, n > 0 ? grid : 0, m, sub, out,
                                                          gate);
  return skb_launch_status(__func__);
}

}  // namespace skb

#include "skb_cscplan.cuh"


namespace skb {
__global__ void csc_to_dense_kernel(const int64_t* __restrict__ colptr,
                                    const int32_t* __restrict__ rowidx,
                                    const double* __restrict__ vals, int64_t n, double* A,
                                    int64_t lda) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  for (int64_t e = colptr[j]; e < colptr[j + 1]; ++e) A[j * lda + rowidx[e]] = vals[e];
}
}  // namespace skb

// Dense column-major copy of a CSC matrix (A pre-zeroed, lda >= m): lets the
// dense-only paths (direct solver, phase 1) run on sparse inputs.
extern "C" int skb_csc_to_dense(const int64_t* colptr, const int32_t* rowidx, const double* vals,
                                int64_t n, double* A, int64_t lda, void* stream) {
  if (n <= 0) return 0;
  csc_to_dense_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      colptr, rowidx, vals, n, A, lda);
  return skb_launch_status(__func__);
}

#define SKB_CSC const int64_t *colptr, const int32_t *rowidx, const double *vals, int64_t m, \
                int64_t n
#define SKB_CSCP const int64_t *colptr, const int32_t *rowidx, const double *vals, \
                 const void *plan, int64_t plan_chunks, const void *ell, int64_t m, int64_t n
// the planned kernel when a plan is given (and applies), else the thread-per-column one
#define SKB_CSC_RUN(Z, OUT, SUB, GATE)                                                      \
  do {                                                                                      \
    CscPlanView pv;                                                                         \
    if (cscp_view(plan, plan_chunks, m, &pv))                                               \
      return run_cscp(pv, (int)m, Z, OUT, SUB, op, &ws, (cudaStream_t)stream, GATE);        \
    return run_csc(colptr, rowidx, vals, (int)m, n, Z, OUT, SUB, op, &ws,                   \
                   (cudaStream_t)stream, GATE, ell);                                        \
  } while (0)

extern "C" int skb_csc_normal_apply(SKB_CSCP, const double* d2, const double* z, double* u,
                                    const double* sub, const int* gate, void* workspace,
                                    size_t ws_bytes, void* stream) {
  SKB_WS;
  OpNormal op{d2};
  SKB_CSC_RUN(z, u, sub, gate);
}

extern "C" int skb_csc_gemv(SKB_CSCP, const double* x, double* u, const double* sub,
                            void* workspace, size_t ws_bytes, void* stream) {
  SKB_WS;
  OpGemvX op{x};
  SKB_CSC_RUN(nullptr, u, sub, nullptr);
}

extern "C" int skb_csc_gemv_ratio(SKB_CSCP, const double* v, const double* s, double* u,
                                  const double* sub, void* workspace, size_t ws_bytes,
                                  void* stream) {
  SKB_WS;
  OpGemvRatio op{v, s};
  SKB_CSC_RUN(nullptr, u, sub, nullptr);
}

extern "C" int skb_csc_rhs(SKB_CSCP, const double* x, const double* s, const double* r_d,
                           double sigma_mu, double* p, const double* r_p, void* workspace,
                           size_t ws_bytes, void* stream) {
  SKB_WS;
  OpRhs op{x, s, r_d, sigma_mu};
  SKB_CSC_RUN(nullptr, p, r_p, nullptr);
}

extern "C" int skb_csc_gemv_t(SKB_CSCP, const double* y, const double* add, const double* sub,
                              double* t, void* workspace, size_t ws_bytes, void* stream) {
  SKB_WS;
  (void)plan;
  (void)plan_chunks;
  OpGemvT op{add, sub, t};
  return run_csc(colptr, rowidx, vals, (int)m, n, y, nullptr, nullptr, op, &ws,
                 (cudaStream_t)stream, nullptr, ell);
}

namespace skb {
__global__ void ell_build_kernel(const int64_t* __restrict__ colptr,
                                 const int32_t* __restrict__ rowidx,
                                 const double* __restrict__ vals, int64_t n,
                                 EllRec* __restrict__ ell) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t e0 = colptr[j], e1 = colptr[j + 1];
  EllRec r{};
  const int64_t len = e1 - e0;
  r.cnt = len <= kEll ? (uint8_t)len : (uint8_t)255;
  for (int q = 0; q < kEll && q < len; ++q) {
    r.row[q] = (uint16_t)rowidx[e0 + q];
    r.val[q] = vals[e0 + q];
  }
  r.spare = e0;
  ell[j] = r;
}
}  // namespace skb

// ELL head records of a CSC matrix (m <= 65535): 64 bytes per column, built
// once per matrix; passed as `ell` to the CSC passes. 0 when not applicable.
extern "C" size_t skb_csc_ell_bytes(int64_t m, int64_t n) {
  return (m >= 1 && m <= 65535 && n >= 1) ? (size_t)n * sizeof(skb::EllRec) : 0;
}

extern "C" int skb_csc_ell_build(const int64_t* colptr, const int32_t* rowidx, const double* vals,
                                 int64_t m, int64_t n, void* ell, size_t ell_bytes,
                                 void* stream) {
  const size_t need = skb_csc_ell_bytes(m, n);
  if (!need) return SKB_ERR_UNSUPPORTED;
  if (!ell || ell_bytes < need || ((uintptr_t)ell & 15)) return SKB_ERR_ARG;
  skb::ell_build_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      colptr, rowidx, vals, n, (skb::EllRec*)ell);
  return skb_launch_status(__func__);
}

extern "C" int skb_csc_directions(SKB_CSCP, const double* dy, const double* x, const double* s,
                                  const double* v, const double* r_d, double sigma_mu, double* ds,
                                  double* dx, double* atdy, double* adx, void* workspace,
                                  size_t ws_bytes, void* stream) {
  SKB_WS;
  OpDir op{x, s, v, r_d, sigma_mu, ds, dx, atdy};
  SKB_CSC_RUN(dy, adx, nullptr, nullptr);
}

extern "C" int skb_csc_iterate(SKB_CSCP, const double* x, const double* dx, const double* s,
                               const double* ds, double alpha, const double* y_new,
                               const double* b, const double* c, double* x_out, double* s_out,
                               double* r_p, double* r_d, void* workspace, size_t ws_bytes,
                               void* stream) {
  SKB_WS;
  OpIter op{x, dx, s, ds, c, alpha, x_out, s_out, r_d};
  SKB_CSC_RUN(y_new, r_p, b, nullptr);
}
