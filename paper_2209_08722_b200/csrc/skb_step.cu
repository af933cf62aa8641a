// K8: fused elementwise + reduction kernels over the n-vectors of an IPM step.
//
// Compiled with -fmad=false: every formula is evaluated in numpy's order with
// one rounding per operation, so on equal inputs the elementwise values are
// bit-identical to the reference's numpy expressions. Reductions are
// deterministic: a fixed grid, fixed per-thread striding, fixed-order block
// trees, and a last-block fixed-order combine of the per-block partials (one
// launch per kernel, no atomics on data).
//
//   skb_step_prep      ipm_core.py:415-421, krylov_solvers.py:40   d, d2, clip count
//   skb_iter_stats     ipm_core.py:88-91,116-124                   mu, min x.s, norms
//   skb_dir_stats      ipm_core.py:237-242,286-289,328,524         comp check, cross, lin
//   skb_crossing       ipm_core.py:245-275 (vectorised part)       first crossing
//   skb_vec_stats      np.linalg.norm / sum / max|.|
#include <math.h>

#include "skb_common.cuh"
#include "skb_internal.h"

namespace skb {

enum RedOp { R_SUM = 0, R_MAX = 1, R_MIN = 2 };

SKB_DEV double red_init(int op) { return op == R_SUM ? 0.0 : (op == R_MAX ? -INFINITY : INFINITY); }
SKB_DEV double red_comb(int op, double a, double b) {
  return op == R_SUM ? a + b : (op == R_MAX ? fmax(a, b) : fmin(a, b));
}

constexpr int kRedThreads = 256;

// Block-reduce K values (ops[k]) and finish the grid reduction in the last block.
template <int K>
SKB_DEV void grid_reduce(double (&v)[K], const int (&ops)[K], double* part, unsigned* ticket,
                         double* out) {
  __shared__ double sm[kRedThreads / 32][K];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double x = v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = red_comb(ops[k], x, __shfl_xor_sync(0xffffffffu, x, o));
    if (lane == 0) sm[wid][k] = x;
  }
  __syncthreads();
  if (threadIdx.x < K) {
    const int k = threadIdx.x;
    double x = sm[0][k];
    for (int w = 1; w < kRedThreads / 32; ++w) x = red_comb(ops[k], x, sm[w][k]);
    part[(size_t)blockIdx.x * K + k] = x;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();  // (also orders the sm[] reuse below)
  if (!last) return;
  __threadfence();
  // last block: every thread folds a fixed strided subset of the partials,
  // then a block reduction (deterministic for a given grid size)
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double x = red_init(ops[k]);
    for (unsigned b = threadIdx.x; b < gridDim.x; b += kRedThreads)
      x = red_comb(ops[k], x, __ldcg(&part[(size_t)b * K + k]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = red_comb(ops[k], x, __shfl_xor_sync(0xffffffffu, x, o));
    if (lane == 0) sm[wid][k] = x;
  }
  __syncthreads();
  if (threadIdx.x < K) {
    const int k = threadIdx.x;
    double x = sm[0][k];
    for (int w = 1; w < kRedThreads / 32; ++w) x = red_comb(ops[k], x, sm[w][k]);
    out[k] = x;
  }
  if (threadIdx.x == 0) *ticket = 0;  // reusable
}

SKB_DEV int64_t gstride() { return (int64_t)gridDim.x * blockDim.x; }
SKB_DEV int64_t gtid() { return (int64_t)blockIdx.x * blockDim.x + threadIdx.x; }

// out: [clip_count, min x, min s]
__global__ void __launch_bounds__(kRedThreads)
    step_prep_kernel(const double* __restrict__ x, const double* __restrict__ s, int64_t n,
                     double* __restrict__ d, double* __restrict__ d2, double* part,
                     unsigned* ticket, double* out) {
  double v[3] = {0.0, INFINITY, INFINITY};
  const int ops[3] = {R_SUM, R_MIN, R_MIN};
  for (int64_t j = gtid(); j < n; j += gstride()) {
    const double xj = x[j], sj = s[j];
    const double ratio = xj / sj;
    const double cl = fmin(fmax(ratio, 1e-32), 1e32);
    v[0] += (cl != ratio) ? 1.0 : 0.0;
    v[1] = fmin(v[1], xj);
    v[2] = fmin(v[2], sj);
    const double dj = sqrt(cl);
    d[j] = dj;
    d2[j] = dj * dj;
  }
  grid_reduce<3>(v, ops, part, ticket, out);
}

// out: [sum x s, min x s, min x, min s, sum r_d^2]
__global__ void __launch_bounds__(kRedThreads)
    iter_stats_kernel(const double* __restrict__ x, const double* __restrict__ s,
                      const double* __restrict__ rd, int64_t n, double* part, unsigned* ticket,
                      double* out) {
  double v[5] = {0.0, INFINITY, INFINITY, INFINITY, 0.0};
  const int ops[5] = {R_SUM, R_MIN, R_MIN, R_MIN, R_SUM};
  for (int64_t j = gtid(); j < n; j += gstride()) {
    const double xs = x[j] * s[j];
    v[0] += xs;
    v[1] = fmin(v[1], xs);
    v[2] = fmin(v[2], x[j]);
    v[3] = fmin(v[3], s[j]);
    if (rd) v[4] += rd[j] * rd[j];
  }
  grid_reduce<5>(v, ops, part, ticket, out);
}

// out: [max|comp|, max|x s|, max|x ds|, max|s dx|, sum dx ds, sum dx^2,
//       sum (x ds + s dx), sum x ds, sum s dx, sum v]
__global__ void __launch_bounds__(kRedThreads)
    dir_stats_kernel(const double* __restrict__ x, const double* __restrict__ s,
                     const double* __restrict__ dx, const double* __restrict__ ds,
                     const double* __restrict__ vv, double smu, int64_t n, double* part,
                     unsigned* ticket, double* out) {
  double v[10] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  const int ops[10] = {R_MAX, R_MAX, R_MAX, R_MAX, R_SUM, R_SUM, R_SUM, R_SUM, R_SUM, R_SUM};
  for (int64_t j = gtid(); j < n; j += gstride()) {
    const double xj = x[j], sj = s[j], dxj = dx[j], dsj = ds[j], vj = vv ? vv[j] : 0.0;
    const double xds = xj * dsj, sdx = sj * dxj, xs = xj * sj;
    const double comp = (((xds + sdx) + xs) - smu) + vj;
    v[0] = fmax(v[0], fabs(comp));
    v[1] = fmax(v[1], fabs(xs));
    v[2] = fmax(v[2], fabs(xds));
    v[3] = fmax(v[3], fabs(sdx));
    v[4] += dxj * dsj;
    v[5] += dxj * dxj;
    v[6] += xds + sdx;
    v[7] += xds;
    v[8] += sdx;
    v[9] += vj;
  }
  grid_reduce<10>(v, ops, part, ticket, out);
}

// Smallest alpha > 0 where a_i t^2 + b_i t + c_i turns negative, with
// a = dx ds - g1a, b = (x ds + s dx) - g1b, c = max(x s - g1mu, 0).
// out: [min c (unclamped), max|c|, crossing (inf if none)]
__global__ void __launch_bounds__(kRedThreads)
    crossing_kernel(const double* __restrict__ x, const double* __restrict__ s,
                    const double* __restrict__ dx, const double* __restrict__ ds, double g1a,
                    double g1b, double g1mu, int64_t n, double* part, unsigned* ticket,
                    double* out) {
  double v[3] = {INFINITY, 0.0, INFINITY};
  const int ops[3] = {R_MIN, R_MAX, R_MIN};
  for (int64_t j = gtid(); j < n; j += gstride()) {
    const double xj = x[j], sj = s[j], dxj = dx[j], dsj = ds[j];
    const double a = dxj * dsj - g1a;
    const double b = (xj * dsj + sj * dxj) - g1b;
    const double c0 = xj * sj - g1mu;
    v[0] = fmin(v[0], c0);
    v[1] = fmax(v[1], fabs(c0));
    const double c = c0 < 0.0 ? fmax(c0, 0.0) : c0;
    const double disc = b * b - (4.0 * a) * c;
    const bool real = disc >= 0.0;
    const double sq = sqrt(real ? disc : 0.0);
    const double sgn = b >= 0.0 ? 1.0 : -1.0;
    const double qq = -0.5 * (b + sgn * sq);
    double r1 = (a != 0.0 && real) ? qq / a : INFINITY;
    double r2 = (qq != 0.0 && real) ? c / qq : INFINITY;
    double r3 = (a == 0.0 && b < 0.0) ? (-c) / b : INFINITY;
    r1 = (r1 > 0.0 && isfinite(r1)) ? r1 : INFINITY;
    r2 = (r2 > 0.0 && isfinite(r2)) ? r2 : INFINITY;
    r3 = (r3 > 0.0 && isfinite(r3)) ? r3 : INFINITY;
    const double cand = fmin(fmin(r1, r2), r3);
    if (isfinite(cand)) {
      const double h = 0.5 * cand;
      const double val = (a * (h * h) + b * h) + c;
      v[2] = fmin(v[2], val < 0.0 ? 0.0 : cand);
    }
  }
  grid_reduce<3>(v, ops, part, ticket, out);
}

// out: [sum a^2, sum a, max|a|, min a]   (a - sub if sub)
__global__ void __launch_bounds__(kRedThreads)
    vec_stats_kernel(const double* __restrict__ a, const double* __restrict__ sub, int64_t n,
                     double* part, unsigned* ticket, double* out) {
  double v[4] = {0.0, 0.0, 0.0, INFINITY};
  const int ops[4] = {R_SUM, R_SUM, R_MAX, R_MIN};
  for (int64_t j = gtid(); j < n; j += gstride()) {
    const double t = sub ? a[j] - sub[j] : a[j];
    v[0] += t * t;
    v[1] += t;
    v[2] = fmax(v[2], fabs(t));
    v[3] = fmin(v[3], t);
  }
  grid_reduce<4>(v, ops, part, ticket, out);
}

// ---- feasible_start centering step (ipm_core.py:914-969)

// out = {min over dv<0 of (-v)/dv (inf if none), min over dw<0 of (-w)/dw}
__global__ void __launch_bounds__(kRedThreads)
    ratio_min_kernel(const double* __restrict__ v, const double* __restrict__ dv,
                     const double* __restrict__ w, const double* __restrict__ dw, int64_t n,
                     double* part, unsigned* ticket, double* out) {
  double r[2] = {INFINITY, INFINITY};
  const int ops[2] = {R_MIN, R_MIN};
  for (int64_t j = gtid(); j < n; j += gstride()) {
    if (dv[j] < 0.0) r[0] = fmin(r[0], (-v[j]) / dv[j]);
    if (dw[j] < 0.0) r[1] = fmin(r[1], (-w[j]) / dw[j]);
  }
  grid_reduce<2>(r, ops, part, ticket, out);
}

// For K step lengths a_k: prod = (x + a dx)(s + a ds); out[3k..3k+2] =
// {min prod, sum prod, count(prod <= 0)} (theta = min/mean in the reference).
constexpr int kGridK = 8;
__global__ void __launch_bounds__(kRedThreads)
    centering_grid_kernel(const double* __restrict__ x, const double* __restrict__ s,
                          const double* __restrict__ dx, const double* __restrict__ ds,
                          const double* __restrict__ alphas, int64_t n, double* part,
                          unsigned* ticket, double* out) {
  double v[3 * kGridK];
  int ops[3 * kGridK];
  double a[kGridK];
#pragma unroll
  for (int k = 0; k < kGridK; ++k) {
    v[3 * k] = INFINITY;
    v[3 * k + 1] = 0.0;
    v[3 * k + 2] = 0.0;
    ops[3 * k] = R_MIN;
    ops[3 * k + 1] = R_SUM;
    ops[3 * k + 2] = R_SUM;
    a[k] = alphas[k];
  }
  for (int64_t j = gtid(); j < n; j += gstride()) {
    const double xj = x[j], sj = s[j], dxj = dx[j], dsj = ds[j];
#pragma unroll
    for (int k = 0; k < kGridK; ++k) {
      const double p = (xj + a[k] * dxj) * (sj + a[k] * dsj);
      v[3 * k] = fmin(v[3 * k], p);
      v[3 * k + 1] += p;
      v[3 * k + 2] += p <= 0.0 ? 1.0 : 0.0;
    }
  }
  grid_reduce<3 * kGridK>(v, ops, part, ticket, out);
}

// x[j] = 1 for every all-zero column j of A (phase1_point pins them, ipm_core.py:834-835).
__global__ void zero_col_fill_kernel(const double* __restrict__ A, int64_t lda, int m, int64_t n,
                                     double* __restrict__ x) {
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= n) return;
  const double* col = A + j * lda;
  int nz = 0;
  for (int i = lane; i < m; i += 32) nz |= col[i] != 0.0;
  nz = __any_sync(0xffffffffu, nz);
  if (!nz && lane == 0) x[j] = 1.0;
}

// v = sqrt(x s) * t   (correction.py:58 for a dense / identity W)
__global__ void sqrt_xs_scale_kernel(const double* __restrict__ t, const double* __restrict__ x,
                                     const double* __restrict__ s, double* __restrict__ v,
                                     int64_t n) {
  for (int64_t j = gtid(); j < n; j += gstride()) v[j] = sqrt(x[j] * s[j]) * t[j];
}

// y = x + alpha * d   (numpy: it.y + a * dirn.dy)
__global__ void axpy_kernel(const double* __restrict__ x, double alpha,
                            const double* __restrict__ d, double* __restrict__ y, int64_t n) {
  for (int64_t j = gtid(); j < n; j += gstride()) y[j] = x[j] + alpha * d[j];
}

// x_new = x + alpha dx, s_new = s + alpha ds with make_iterate's rounding
// (round-to-nearest multiply then add, no FMA: skb_stream.cu OpIter).
__global__ void step_xs_kernel(const double* __restrict__ x, const double* __restrict__ dx,
                               const double* __restrict__ s, const double* __restrict__ ds,
                               double alpha, double* __restrict__ xn, double* __restrict__ sn,
                               int64_t n) {
  for (int64_t j = gtid(); j < n; j += gstride()) {
    xn[j] = __dadd_rn(x[j], __dmul_rn(alpha, dx[j]));
    sn[j] = __dadd_rn(s[j], __dmul_rn(alpha, ds[j]));
  }
}

// out[0] = sigma * (sum / n): the next step's sigma * mu, exactly the host's
// `sigma * (float(sum) / n)`
__global__ void sigma_mu_kernel(const double* __restrict__ sum, double n, double sigma,
                                double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = __dmul_rn(sigma, __ddiv_rn(sum[0], n));
}

// out = a - b (m-vectors, e.g. infeas = A D^2 A' dy - p)
__global__ void sub_kernel(const double* __restrict__ a, const double* __restrict__ b,
                           double* __restrict__ out, int64_t n) {
  for (int64_t j = gtid(); j < n; j += gstride()) out[j] = a[j] - b[j];
}

}  // namespace skb

using namespace skb;

constexpr int kRedBlocksPerSm = 8;  // full occupancy: enough loads in flight for HBM

static int red_grid(int64_t n) {
  int64_t g = (n + kRedThreads - 1) / kRedThreads;
  const int64_t cap = kRedBlocksPerSm * (int64_t)skb_num_sms();
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

// Reduction scratch: partials (grid * 16 doubles) + ticket.
extern "C" size_t skb_reduce_workspace_bytes(void) {
  return (size_t)kRedBlocksPerSm * skb_num_sms() * 32 * 8 + 512;
}

#define RED_WS                                                                   \
  skb_ws ws = skb_ws_make(workspace, ws_bytes);                                  \
  unsigned* ticket = (unsigned*)skb_ws_take(&ws, 256);                           \
  double* part = (double*)skb_ws_take(&ws, (size_t)kRedBlocksPerSm * skb_num_sms() * 32 * 8); \
  if (!ticket || !part) return SKB_ERR_WORKSPACE;                                \
  cudaStream_t st = (cudaStream_t)stream

#define LAUNCH_OK return skb_launch_status(__func__)

// The ticket word (first 4 bytes of the workspace) must be zero before the
// first use; every kernel leaves it zero. skb_reduce_workspace_init zeroes it.
extern "C" int skb_reduce_workspace_init(void* workspace, void* stream) {
  cudaMemsetAsync(workspace, 0, 256, (cudaStream_t)stream);
  LAUNCH_OK;
}

extern "C" int skb_step_prep(const double* x, const double* s, int64_t n, double* d, double* d2,
                             double* out, void* workspace, size_t ws_bytes, void* stream) {
  RED_WS;
  step_prep_kernel<<<red_grid(n), kRedThreads, 0, st>>>(x, s, n, d, d2, part, ticket, out);
  LAUNCH_OK;
}

extern "C" int skb_iter_stats(const double* x, const double* s, const double* r_d, int64_t n,
                              double* out, void* workspace, size_t ws_bytes, void* stream) {
  RED_WS;
  iter_stats_kernel<<<red_grid(n), kRedThreads, 0, st>>>(x, s, r_d, n, part, ticket, out);
  LAUNCH_OK;
}

extern "C" int skb_dir_stats(const double* x, const double* s, const double* dx,
                             const double* ds, const double* v, double sigma_mu, int64_t n,
                             double* out, void* workspace, size_t ws_bytes, void* stream) {
  RED_WS;
  dir_stats_kernel<<<red_grid(n), kRedThreads, 0, st>>>(x, s, dx, ds, v, sigma_mu, n, part,
                                                        ticket, out);
  LAUNCH_OK;
}

extern "C" int skb_crossing(const double* x, const double* s, const double* dx, const double* ds,
                            double g1a, double g1b, double g1mu, int64_t n, double* out,
                            void* workspace, size_t ws_bytes, void* stream) {
  RED_WS;
  crossing_kernel<<<red_grid(n), kRedThreads, 0, st>>>(x, s, dx, ds, g1a, g1b, g1mu, n, part,
                                                       ticket, out);
  LAUNCH_OK;
}

extern "C" int skb_vec_stats(const double* a, const double* sub, int64_t n, double* out,
                             void* workspace, size_t ws_bytes, void* stream) {
  RED_WS;
  vec_stats_kernel<<<red_grid(n), kRedThreads, 0, st>>>(a, sub, n, part, ticket, out);
  LAUNCH_OK;
}

extern "C" int skb_ratio_min(const double* v, const double* dv, const double* w, const double* dw,
                             int64_t n, double* out, void* workspace, size_t ws_bytes,
                             void* stream) {
  RED_WS;
  ratio_min_kernel<<<red_grid(n), kRedThreads, 0, st>>>(v, dv, w, dw, n, part, ticket, out);
  LAUNCH_OK;
}

extern "C" int skb_centering_grid(const double* x, const double* s, const double* dx,
                                  const double* ds, const double* alphas, int64_t n, double* out,
                                  void* workspace, size_t ws_bytes, void* stream) {
  skb_ws ws = skb_ws_make(workspace, ws_bytes);
  unsigned* ticket = (unsigned*)skb_ws_take(&ws, 256);
  double* part = (double*)skb_ws_take(&ws, (size_t)2 * skb_num_sms() * 3 * kGridK * 8);
  if (!ticket || !part) return SKB_ERR_WORKSPACE;
  centering_grid_kernel<<<red_grid(n), kRedThreads, 0, (cudaStream_t)stream>>>(
      x, s, dx, ds, alphas, n, part, ticket, out);
  LAUNCH_OK;
}

extern "C" int skb_zero_col_fill(const double* A, int64_t m, int64_t n, int64_t lda, double* x,
                                 void* stream) {
  if (n <= 0) return 0;
  zero_col_fill_kernel<<<(unsigned)((n * 32 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      A, lda, (int)m, n, x);
  LAUNCH_OK;
}

extern "C" int skb_sqrt_xs_scale(const double* t, const double* x, const double* s, double* v,
                                 int64_t n, void* stream) {
  sqrt_xs_scale_kernel<<<red_grid(n), kRedThreads, 0, (cudaStream_t)stream>>>(t, x, s, v, n);
  LAUNCH_OK;
}

extern "C" int skb_step_xs(const double* x, const double* dx, const double* s, const double* ds,
                           double alpha, double* xn, double* sn, int64_t n, void* stream) {
  if (n <= 0) return 0;
  step_xs_kernel<<<red_grid(n), kRedThreads, 0, (cudaStream_t)stream>>>(x, dx, s, ds, alpha, xn,
                                                                       sn, n);
  return skb_launch_status(__func__);
}

extern "C" int skb_sigma_mu(const double* sum, double n, double sigma, double* out, void* stream) {
  sigma_mu_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(sum, n, sigma, out);
  return skb_launch_status(__func__);
}

extern "C" int skb_axpy(const double* x, double alpha, const double* d, double* y, int64_t n,
                        void* stream) {
  axpy_kernel<<<red_grid(n), kRedThreads, 0, (cudaStream_t)stream>>>(x, alpha, d, y, n);
  LAUNCH_OK;
}

extern "C" int skb_sub(const double* a, const double* b, double* out, int64_t n, void* stream) {
  sub_kernel<<<red_grid(n), kRedThreads, 0, (cudaStream_t)stream>>>(a, b, out, n);
  LAUNCH_OK;
}
