// L2 -> SM ingress through the TMA bulk engine (development aid): one producer
// lane per CTA streams 8 KB chunks (one c2 column) of a buffer into a 16-stage
// shared-memory ring; consumer warps only wait and release. Buffer sizes below
// (L2-resident) and above (HBM) the 126 MB L2, evict_normal vs evict_first.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2209_08722_b200/csrc/skb_common.cuh"
using namespace skb;

SKB_DEV void mbar_arrive1(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
constexpr int kStages = 16, kChunk = 8000, kCons = 4;  // consumer warps

__global__ void __launch_bounds__(32 * (kCons + 1), 2)
    ingress(const char* buf, size_t nchunks, int reps, int evict_first, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + kStages;
  unsigned char* ring = sm + 256;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], kCons); }
    fence_mbar_init();
  }
  __syncthreads();
  const size_t total = nchunks * (size_t)reps;
  // CTA c takes chunks c, c + G, ... (wrapping over the buffer reps times)
  if (warp == 0) {
    if (lane == 0) {
      uint64_t pol;
      if (evict_first) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
      int st = 0; uint32_t ph = 0;
      for (size_t t = blockIdx.x; t < total; t += gridDim.x) {
        mbar_wait(&empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&full[st], kChunk);
        bulk_g2s(ring + (size_t)st * kChunk, buf + (t % nchunks) * kChunk, kChunk, &full[st], pol);
        if (++st == kStages) { st = 0; ph ^= 1; }
      }
    }
  } else {
    int st = 0; uint32_t ph = 0; unsigned long long acc = 0;
    for (size_t t = blockIdx.x; t < total; t += gridDim.x) {
      mbar_wait(&full[st], ph);
      if (lane == 0) acc += ring[(size_t)st * kChunk + warp];
      __syncwarp();
      if (lane == 0) mbar_arrive1(&empty[st]);
      if (++st == kStages) { st = 0; ph ^= 1; }
    }
    if (lane == 0 && acc == 12345) *sink = acc;
  }
}

// plain 16-byte loads by every thread, 4 in flight per thread
__global__ void __launch_bounds__(512) ldg_stream(const int4* buf, size_t n16, int reps,
                                                  unsigned long long* sink) {
  unsigned long long acc = 0;
  const size_t total = n16 * (size_t)reps, stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < total; i += 4 * stride) {
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcg(buf + (i + u * stride) % n16);
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += (unsigned)(v[u].x ^ v[u].w);
  }
  if (acc == 12345) *sink = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = 256 + (size_t)kStages * kChunk;
  cudaFuncSetAttribute(ingress, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const size_t big = 8000ull << 20;
  char* buf; cudaMalloc(&buf, big); cudaMemset(buf, 1, big);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  struct { size_t bytes; int reps; } cases[] = {{32ull << 20, 200}, {48ull << 20, 150}, {96ull << 20, 80}, {big, 1}};
  for (int ef = 0; ef < 2; ++ef)
    for (auto c : cases)
      for (int cps = 1; cps <= 2; ++cps) {
        const size_t nch = c.bytes / kChunk;
        ingress<<<sms * cps, 32 * (kCons + 1), smem>>>(buf, nch, 1, ef, sink);
        cudaEventRecord(a);
        ingress<<<sms * cps, 32 * (kCons + 1), smem>>>(buf, nch, c.reps, ef, sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const double gb = (double)nch * kChunk * c.reps / 1e9;
        printf("evict_first=%d buffer %6zu MB x%3d  CTAs/SM %d: %8.3f ms  %7.0f GB/s  (%s)\n", ef,
               c.bytes >> 20, c.reps, cps, ms, gb / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
      }
  for (auto c : cases)
    for (int cps = 2; cps <= 4; cps += 2) {
      const size_t n16 = c.bytes / 16;
      ldg_stream<<<sms * cps, 512>>>((const int4*)buf, n16, 1, sink);
      cudaEventRecord(a);
      ldg_stream<<<sms * cps, 512>>>((const int4*)buf, n16, c.reps, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double gb = (double)c.bytes * c.reps / 1e9;
      printf("LDG.128 buffer %6zu MB x%3d  CTAs/SM %d: %8.3f ms  %7.0f GB/s\n", c.bytes >> 20,
             c.reps, cps, ms, gb / (ms * 1e-3));
    }
  return 0;
}
