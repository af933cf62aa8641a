// clock64 timing of the 64 x 64 leaf inverse: one thread per column (round 2
// before) vs four lanes per column (csrc/skb_dense.cu leaf_inverse). Dev aid.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NB = 64, LDP = NB + 1;
__device__ void inv_1t(const double (*Lsm)[LDP], const double* rinv, double* out, long ld) {
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
__device__ void inv_4l(const double (*Lsm)[LDP], const double* rinv, double* out, long ld) {
  const int t = threadIdx.x, j = t >> 2, sub = t & 3, lane = t & 31;
  const int src0 = lane & ~3;
  double x[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) x[r] = (sub + 4 * r == j) ? 1.0 : 0.0;
  for (int g = 0; g < 16; ++g) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = 4 * g + u;
      double xq = sub == u ? x[0] * rinv[q] : 0.0;
      xq = __shfl_sync(0xffffffffu, xq, src0 | u);
      if (sub == u) out[(long)q * ld + j] = xq;
      if (sub > u) x[0] = fma(-Lsm[sub + 4 * g][q], xq, x[0]);
#pragma unroll
      for (int r = 1; r < 16; ++r) x[r] = fma(-Lsm[(sub + 4 * (g + r)) & (NB - 1)][q], xq, x[r]);
    }
#pragma unroll
    for (int r = 0; r < 15; ++r) x[r] = x[r + 1];
    x[15] = 0.0;
  }
}
__global__ void k(const double* L, double* out, long long* clk, int mode) {
  __shared__ double Lsm[NB][LDP];
  __shared__ double rinv[NB];
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) Lsm[e / NB][e % NB] = L[e];
  __syncthreads();
  if (threadIdx.x < NB) rinv[threadIdx.x] = 1.0 / Lsm[threadIdx.x][threadIdx.x];
  __syncthreads();
  long long c0 = clock64();
  if (mode == 0) inv_1t(Lsm, rinv, out, NB); else inv_4l(Lsm, rinv, out, NB);
  __syncthreads();
  long long c1 = clock64();
  if (threadIdx.x == 0) clk[mode] = c1 - c0;
}
int main() {
  double h[NB * NB];
  for (int i = 0; i < NB; ++i) for (int j = 0; j < NB; ++j) h[i * NB + j] = j > i ? 0.0 : (i == j ? 2.0 : 1.0 / (1 + i + j));
  double *L, *o0, *o1; long long* clk;
  cudaMalloc(&L, sizeof h); cudaMalloc(&o0, sizeof h); cudaMalloc(&o1, sizeof h); cudaMallocManaged(&clk, 64);
  cudaMemcpy(L, h, sizeof h, cudaMemcpyHostToDevice);
  for (int r = 0; r < 3; ++r) { k<<<1, 256>>>(L, o0, clk, 0); k<<<1, 256>>>(L, o1, clk, 1); }
  cudaDeviceSynchronize();
  double a[NB * NB], b[NB * NB];
  cudaMemcpy(a, o0, sizeof a, cudaMemcpyDeviceToHost); cudaMemcpy(b, o1, sizeof b, cudaMemcpyDeviceToHost);
  int diff = 0;
  for (int i = 0; i < NB; ++i) for (int j = 0; j <= i; ++j) diff += a[i * NB + j] != b[i * NB + j];
  printf("inverse: one thread per column %lld cycles, four lanes per column %lld cycles, lower entries differing %d\n", clk[0], clk[1], diff);
  return 0;
}
