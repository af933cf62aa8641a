// Shared device helpers for the skb (sketched IPM, B200) kernels.
// sm_100a only: cp.async.bulk + mbarrier staging, Philox4x64-10, warp reductions.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define SKB_DEV __device__ __forceinline__

namespace skb {

constexpr int kWarp = 32;

// ------------------------------------------------------------------ status
// Bit flags written by kernels into a device status word; the host maps
// them onto the reference exception classes (include/skb.h).
enum : int {
  ST_OK = 0,
  ST_BREAKDOWN_CURV = 1,   // krylov_solvers.py:89-90 (chebyshev :191-192)
  ST_BREAKDOWN_RZ = 2,     // krylov_solvers.py:77-78,96-97
  ST_CHOL_FAIL = 4,        // nonpositive pivot in a Cholesky (rank loss)
  ST_NONPOSITIVE = 8,      // nonpositive scaling / point
  ST_BAD_ARG = 16,
};

// --------------------------------------------------------------- mbarrier
SKB_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

SKB_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

SKB_DEV void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

SKB_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

SKB_DEV bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}

SKB_DEV void mbar_wait(uint64_t* bar, uint32_t phase) {
  while (!mbar_try_wait(bar, phase)) {
  }
}

// L2 policy for streaming operands that are read once per pass (A columns):
// evict-first keeps the small reused vectors / factor resident in L2.
SKB_DEV uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// Read-only gathers that should not displace L2-resident working data:
// no L1 allocation, L2 evict-first.
SKB_DEV double ldg_ef(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
SKB_DEV int ldg_ef(const int* p, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
               : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
SKB_DEV long long ldg_ef(const long long* p, uint64_t pol) {
  long long v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s64 %0, [%1], %2;"
               : "=l"(v) : "l"(p), "l"(pol));
  return v;
}

// 1-D bulk async copy global -> shared (TMA engine, no tensor map), completes
// as tx bytes on the mbarrier. dst/src 16-byte aligned, bytes % 16 == 0.
SKB_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// ------------------------------------------------------------- reductions
SKB_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
SKB_DEV double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
SKB_DEV double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum in a fixed order (deterministic). buf: >= 32 doubles smem.
SKB_DEV double block_sum(double v, double* buf) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) buf[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < nw ? buf[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) buf[0] = t;
  }
  __syncthreads();
  t = buf[0];
  __syncthreads();
  return t;
}

// ------------------------------------------------------------------ Philox
// Philox4x64-10 (Random123 round function, as used by numpy's Philox).
struct u64x4 {
  uint64_t v[4];
};

SKB_DEV u64x4 philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3, uint64_t k0,
                            uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ULL;
      k1 += 0xBB67AE8584CAA73BULL;
    }
    const uint64_t h0 = __umul64hi(0xD2E7470EE14C6C93ULL, c0), l0 = 0xD2E7470EE14C6C93ULL * c0;
    const uint64_t h1 = __umul64hi(0xCA5A826395121157ULL, c2), l1 = 0xCA5A826395121157ULL * c2;
    const uint64_t n0 = h1 ^ c1 ^ k0, n2 = h0 ^ c3 ^ k1;
    c0 = n0;
    c1 = l1;
    c2 = n2;
    c3 = l0;
  }
  u64x4 o;
  o.v[0] = c0;
  o.v[1] = c1;
  o.v[2] = c2;
  o.v[3] = c3;
  return o;
}

}  // namespace skb
