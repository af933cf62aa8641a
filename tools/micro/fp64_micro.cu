// FP64 microbenchmarks on B200: DFMA latency/throughput, DDIV/DSQRT latency, DMMA throughput.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_lat(double* out, int iters) {
  double a = threadIdx.x * 1e-3 + 1.0, b = 0.999999, c = 1e-9;
  for (int i = 0; i < iters; ++i) a = fma(a, b, c);
  out[threadIdx.x] = a;
}
__global__ void dfma_tput(double* out, int iters) {
  double a[8];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], 0.999999, 1e-9);
  double s = 0; for (int k = 0; k < 8; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void ddiv_lat(double* out, int iters) {
  double a = threadIdx.x + 2.0;
  for (int i = 0; i < iters; ++i) a = 1.0000001 / a + 0.5;
  out[threadIdx.x] = a;
}
__global__ void dsqrt_lat(double* out, int iters) {
  double a = threadIdx.x + 2.0;
  for (int i = 0; i < iters; ++i) a = sqrt(a) + 1.0;
  out[threadIdx.x] = a;
}
__global__ void dmma_tput(double* out, int iters) {
  double c[8][2] = {};
  double a = threadIdx.x * 1e-3, b = 1e-3;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  double s = 0; for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dmma_lat(double* out, int iters) {
  double c[2] = {};
  double a = threadIdx.x * 1e-3, b = 1e-3;
  for (int i = 0; i < iters; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
  out[threadIdx.x] = c[0] + c[1];
}
__global__ void sync_lat(double* out, int iters) {
  double a = threadIdx.x;
  for (int i = 0; i < iters; ++i) { __syncthreads(); a += 1.0; }
  out[threadIdx.x] = a;
}
template <class F> float tm(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}
int main() {
  double* out; cudaMalloc(&out, 1 << 26);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); double ghz = clk / 1e6;
  int it = 1 << 16;
  float ms = tm([&] { dfma_lat<<<1, 32>>>(out, it); });
  printf("DFMA dependent latency: %.1f cycles\n", ms * 1e-3 * ghz * 1e9 / it);
  ms = tm([&] { ddiv_lat<<<1, 32>>>(out, it); });
  printf("DDIV+DADD dependent latency: %.1f cycles\n", ms * 1e-3 * ghz * 1e9 / it);
  ms = tm([&] { dsqrt_lat<<<1, 32>>>(out, it); });
  printf("DSQRT+DADD dependent latency: %.1f cycles\n", ms * 1e-3 * ghz * 1e9 / it);
  ms = tm([&] { dmma_lat<<<1, 32>>>(out, it); });
  printf("DMMA m8n8k4 dependent latency: %.1f cycles\n", ms * 1e-3 * ghz * 1e9 / it);
  ms = tm([&] { sync_lat<<<1, 64>>>(out, it); });
  printf("__syncthreads (2 warps): %.1f cycles\n", ms * 1e-3 * ghz * 1e9 / it);
  int it2 = 1 << 14;
  ms = tm([&] { dfma_tput<<<148 * 8, 256>>>(out, it2); });
  printf("DFMA throughput: %.2f TFLOP/s\n", 2.0 * 148 * 8 * 256 * 8.0 * it2 / (ms * 1e-3) / 1e12);
  ms = tm([&] { dmma_tput<<<148 * 8, 256>>>(out, it2); });
  printf("DMMA throughput: %.2f TFLOP/s\n", 512.0 * 148 * 8 * 8 * 8.0 * it2 / (ms * 1e-3) / 1e12);
  printf("sm clock %.3f GHz\n", ghz);
  return 0;
}
