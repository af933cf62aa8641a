// Phase timing (clock64) of the 64x64 diagonal Cholesky + inverse leaf on one CTA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o diag_micro diag_micro.cu
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
constexpr int NB = 64, LDP = NB + 1, kLeafThreads = 256;

__device__ void leaf_inverse(const double (*Lsm)[LDP], const double* rinv, double* out, long ld) {
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
      out[(long)q * ld + j] = xq;
#pragma unroll
      for (int k = u + 1; k < NB + u; ++k) x[k] = fma(-Lsm[(q0 + k) & (NB - 1)][q], xq, x[k]);
    }
#pragma unroll
    for (int k = 0; k < NB; ++k) x[k] = x[k + R];
#pragma unroll
    for (int k = NB; k < NB + R; ++k) x[k] = 0.0;
  }
}

__global__ void __launch_bounds__(256) diag_old(const double* src, double* dst, double* Dinv, long long* clk, int mode) {
  __shared__ double Lsm[NB][LDP];
  __shared__ double colc[2][NB];
  __shared__ double rinv[NB];
  const int t = threadIdx.x, i = t >> 2, q4 = t & 3;
  long long c0c = clock64();
  double r[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int k = q4 + 4 * j;
    r[j] = k <= i ? src[i * 64 + k] : 0.0;
    Lsm[i][k] = 0.0;
  }
  __syncthreads();
  long long c1 = clock64();
  for (int c0 = 0; c0 < NB; c0 += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c0 + u, buf = u & 1;
      if (q4 == u && i >= c) colc[buf][i] = r[0];
      __syncthreads();
      const double piv = colc[buf][c];
      const double rs = mode & 1 ? 1.0 / sqrt(piv) : rsqrt(piv);
      if (t == 0) rinv[c] = rs;
      const double ai = colc[buf][i];
      if (q4 == u && i >= c) Lsm[i][c] = i == c ? piv * rs : ai * rs;
      if (i > c) {
        const double air = ai * (rs * rs);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int k = q4 + 4 * j + c0;
          if (k > c && k <= i) r[j] = fma(-air, colc[buf][k], r[j]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 15; ++j) r[j] = r[j + 1];
    r[15] = 0.0;
  }
  __syncthreads();
  long long c2 = clock64();
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int k = q4 + 4 * j;
    dst[i * 64 + k] = Lsm[i][k];
  }
  leaf_inverse(Lsm, rinv, Dinv, NB);
  __syncthreads();
  long long c3 = clock64();
  if (t == 0) { clk[0] = c1 - c0c; clk[1] = c2 - c1; clk[2] = c3 - c2; }
}

constexpr int kFLD = NB + 1;
constexpr size_t kDiagSmem = (size_t)(2 * NB + 32) * kFLD * sizeof(double) + (NB + 2) * 8;

__device__ __forceinline__ bool warp_factor16(double* S, int c0, double* rinv, double* colb) {
  // lane l < 16 owns row c0 + l in registers; column c's values go through a
  // warp-private shared vector (one store, LDS.128 broadcast reads) -- 8 loads
  // per column instead of 30 shuffles; the column loop is unrolled (static
  // register indices, no rotation).
  const int l = threadIdx.x & 31, lr = l & 15;
  const int row = c0 + lr;
  double a[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) a[j] = j <= lr ? S[row * kFLD + c0 + j] : 0.0;
  bool ok = true;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const double piv = __shfl_sync(0xffffffffu, a[c], c);
    const double rs = rsqrt(piv);
    ok = ok && piv > 0.0;
    const double lc = lr == c ? piv * rs : (lr > c ? a[c] * rs : 0.0);
    a[c] = lc;
    if (l < 16) colb[l] = lc;
    if (l == c) rinv[c0 + c] = rs;
    __syncwarp();
#pragma unroll
    for (int j = c + 1; j < 16; ++j)
      if (j <= lr) a[j] = fma(-lc, colb[j], a[j]);
    __syncwarp();
  }
  if (l < 16) {
#pragma unroll
    for (int c = 0; c < 16; ++c) S[row * kFLD + c0 + c] = a[c];
  }
  return ok;
}

// D (b, b) = inverse of the 16 x 16 lower block of S at (16 b, 16 b): lane j < 16
// computes column j by right-looking substitution.
__device__ __forceinline__ void leaf16_inverse(const double* S, double* D, int b, const double* rinv) {
  const int j = threadIdx.x & 31;
  if (j >= 16) return;
  const int o = 16 * b;
  double x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = k == j ? 1.0 : 0.0;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const double xq = x[q] * rinv[o + q];
    D[(o + q) * kFLD + o + j] = xq;
#pragma unroll
    for (int k = q + 1; k < 16; ++k) x[k] = fma(-S[(o + k) * kFLD + o + q], xq, x[k]);
  }
}

// Merge level h (16 or 32): for each aligned pair of h-blocks at o:
// T = L[o+h.., o..] Li[o.., o..] (h x h), then D[o+h.., o..] = -Li[o+h.., o+h..] T.
__device__ __forceinline__ void inverse_merge(const double* S, double* D, double* T, int h) {
  const int t = threadIdx.x, pairs = NB / (2 * h), per = h * h;
  for (int e = t; e < pairs * per; e += kLeafThreads) {
    const int o = (e / per) * 2 * h, r = (e % per) / h, c = e % h;
    const double* Lr = S + (o + h + r) * kFLD + o;
    double acc = 0.0;
    for (int p = c; p < h; ++p) acc = fma(Lr[p], D[(o + p) * kFLD + o + c], acc);  // Li lower
    T[(e / per) * h * kFLD / 2 + r * kFLD / 2 + c] = acc;
  }
  __syncthreads();
  for (int e = t; e < pairs * per; e += kLeafThreads) {
    const int o = (e / per) * 2 * h, r = (e % per) / h, c = e % h;
    const double* Lr = D + (o + h + r) * kFLD + o + h;
    double acc = 0.0;
    for (int p = 0; p <= r; ++p) acc = fma(Lr[p], T[(e / per) * h * kFLD / 2 + p * kFLD / 2 + c], acc);
    D[(o + h + r) * kFLD + o + c] = -acc;
  }
  __syncthreads();
}

__device__ __forceinline__ void diag_factor(const double* src, long ld, double* dst, long ld_dst, int* status,
                         double* Dinv, double* smem, long long* clkp) {
  long long cA = clock64();
  double* S = smem;
  double* D = S + NB * kFLD;
  double* T = D + NB * kFLD;  // 32 rows of kFLD: room for two 16 x 16 or one 32 x 32 (stride kFLD / 2)
  double* rinv = T + 32 * kFLD;
  int* bad = reinterpret_cast<int*>(rinv + NB);
  const int t = threadIdx.x, warp = t >> 5;
  for (int e = t; e < NB * NB; e += kLeafThreads) {
    const int r = e >> 6, c = e & 63;
    S[r * kFLD + c] = c <= r ? src[(long)r * ld + c] : 0.0;
    D[r * kFLD + c] = 0.0;
  }
  if (t == 0) *bad = 0;
  __syncthreads();
  long long cB = clock64(), cF = 0, cS = 0, cU = 0;
  for (int c0 = 0; c0 < NB; c0 += 16) {
    long long x0 = clock64();
    if (warp == 0 && !warp_factor16(S, c0, rinv, T) && t == 0) *bad = 1;
    __syncthreads();
    long long x1 = clock64(); cF += x1 - x0;
    const int rows = NB - c0 - 16;
    if (rows == 0) break;
    if (t < rows) {  // L[r][c0..c0+15] = A[r][..] L_bb^-T, r = c0 + 16 + t
      double* Sr = S + (c0 + 16 + t) * kFLD + c0;
      double x[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) x[c] = Sr[c];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        x[c] *= rinv[c0 + c];
#pragma unroll
        for (int k = c + 1; k < 16; ++k) x[k] = fma(-x[c], S[(c0 + k) * kFLD + c0 + c], x[k]);
      }
#pragma unroll
      for (int c = 0; c < 16; ++c) Sr[c] = x[c];
    }
    __syncthreads();
    long long x2 = clock64(); cS += x2 - x1;
    for (int e = t; e < rows * rows; e += kLeafThreads) {  // trailing lower update
      const int r = e / rows, q = e - r * rows;
      if (q > r) continue;
      const double* Lr = S + (c0 + 16 + r) * kFLD + c0;
      const double* Lq = S + (c0 + 16 + q) * kFLD + c0;
      double acc = S[(c0 + 16 + r) * kFLD + c0 + 16 + q];
#pragma unroll
      for (int p = 0; p < 16; ++p) acc = fma(-Lr[p], Lq[p], acc);
      S[(c0 + 16 + r) * kFLD + c0 + 16 + q] = acc;
    }
    __syncthreads();
    cU += clock64() - x2;
  }
  long long cC = clock64();
  for (int e = t; e < NB * NB; e += kLeafThreads) {
    const int r = e >> 6, c = e & 63;
    dst[(long)r * ld_dst + c] = S[r * kFLD + c];
  }
  if (*bad) {
    if (t == 0) atomicOr(status, 4);
    return;
  }
  if (!Dinv) return;
  if (warp < 4) leaf16_inverse(S, D, warp, rinv);
  __syncthreads();
  inverse_merge(S, D, T, 16);
  inverse_merge(S, D, T, 32);
  for (int e = t; e < NB * NB; e += kLeafThreads) {
    const int r = e >> 6, c = e & 63;
    Dinv[r * NB + c] = D[r * kFLD + c];
  }
  __syncthreads();
  if (t == 0) { clkp[0] = cB - cA; clkp[1] = cF; clkp[2] = cS; clkp[3] = cU; clkp[4] = clock64() - cC; }
}

__global__ void __launch_bounds__(256) diag_new(const double* src, double* dst, double* Dinv, int* st, long long* clk) {
  extern __shared__ double dsm[];
  long long a = clock64();
  diag_factor(src, 64, dst, 64, st, Dinv, dsm, clk + 4);
  __syncthreads();
  if (threadIdx.x == 0) clk[10] = clock64() - a;
  a = clock64();
  diag_factor(src, 64, dst, 64, st, Dinv, dsm, clk + 4);
  __syncthreads();
  if (threadIdx.x == 0) clk[3] = clock64() - a;
}
__global__ void rsqrt_lat(double* out, int iters, int mode) {
  double a = threadIdx.x + 2.0;
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) a = (mode ? 1.0 / sqrt(a) : rsqrt(a)) + 2.0;
  long long c1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) out[256] = (double)(c1 - c0) / iters;
}
__global__ void bar_lat(double* out, int iters) {
  __shared__ double s[256];
  double a = threadIdx.x;
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) { s[(threadIdx.x + i) & 255] = a; __syncthreads(); a += s[(threadIdx.x * 7 + i) & 255]; }
  long long c1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) out[256] = (double)(c1 - c0) / iters;
}


__global__ void shfl_tput(double* out, int iters) {
  double v[8];
  for (int k = 0; k < 8; ++k) v[k] = threadIdx.x + k;
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __shfl_sync(0xffffffffu, v[k], (i + k) & 31) + 1.0;
  }
  long long c1 = clock64();
  double s = 0; for (int k = 0; k < 8; ++k) s += v[k];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) out[256] = (double)(c1 - c0) / iters / 8;
}
__global__ void lds_tput(double* out, int iters) {
  __shared__ double sm[64];
  if (threadIdx.x < 64) sm[threadIdx.x] = threadIdx.x;
  __syncwarp();
  double v[8];
  for (int k = 0; k < 8; ++k) v[k] = k;
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] += sm[(i + k) & 63];
  }
  long long c1 = clock64();
  double s = 0; for (int k = 0; k < 8; ++k) s += v[k];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) out[256] = (double)(c1 - c0) / iters / 8;
}
int main() {
  double *src, *dst, *Dinv, *o; long long* clk;
  cudaMalloc(&src, 64 * 64 * 8); cudaMalloc(&dst, 64 * 64 * 8); cudaMalloc(&Dinv, 64 * 64 * 8);
  cudaMalloc(&o, 512 * 8); cudaMallocManaged(&clk, 128);
  double h[64 * 64];
  for (int i = 0; i < 64; ++i) for (int j = 0; j < 64; ++j) h[i * 64 + j] = (i == j ? 64.0 : 0.0) + 1.0 / (1 + i + j);
  cudaMemcpy(src, h, sizeof h, cudaMemcpyHostToDevice);
  for (int mode = 0; mode < 2; ++mode) {
    for (int r = 0; r < 3; ++r) diag_old<<<1, 256>>>(src, dst, Dinv, clk, mode);
    cudaDeviceSynchronize();
    printf("diag_old mode %d: load %lld  factor %lld  store+inverse %lld cycles\n", mode, clk[0], clk[1], clk[2]);
  }
  int* st; cudaMalloc(&st, 4);
  cudaFuncSetAttribute(diag_new, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDiagSmem);
  for (int r = 0; r < 3; ++r) diag_new<<<1, 256, kDiagSmem>>>(src, dst, Dinv, st, clk);
  cudaDeviceSynchronize();
  printf("cold first call %lld\n", clk[10]);
  printf("diag_new (warm 2nd call): total %lld  load %lld factor16s %lld trsm %lld update %lld store+inverse %lld cycles (%s)\n", clk[3], clk[4], clk[5], clk[6], clk[7], clk[8], cudaGetErrorString(cudaGetLastError()));
  double ho;
  for (int mode = 0; mode < 2; ++mode) {
    rsqrt_lat<<<1, 32>>>(o, 1000, mode); cudaDeviceSynchronize();
    cudaMemcpy(&ho, o + 256, 8, cudaMemcpyDeviceToHost); printf("rsqrt mode %d latency %.1f cycles\n", mode, ho);
  }
  shfl_tput<<<1, 32>>>(o, 1000); cudaDeviceSynchronize();
  cudaMemcpy(&ho, o + 256, 8, cudaMemcpyDeviceToHost); printf("shfl.f64 (runtime lane) + dadd per op, 1 warp: %.1f cycles\n", ho);
  lds_tput<<<1, 32>>>(o, 1000); cudaDeviceSynchronize();
  cudaMemcpy(&ho, o + 256, 8, cudaMemcpyDeviceToHost); printf("lds.f64 broadcast + dadd per op, 1 warp: %.1f cycles\n", ho);
  bar_lat<<<1, 256>>>(o, 1000); cudaDeviceSynchronize();
  cudaMemcpy(&ho, o + 256, 8, cudaMemcpyDeviceToHost); printf("syncthreads+lds round %.1f cycles\n", ho);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 100; ++r) diag_old<<<1, 256>>>(src, dst, Dinv, clk, 0);
  cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
  printf("diag_old back-to-back: %.2f us per launch\n", ms * 10);
  return 0;
}
