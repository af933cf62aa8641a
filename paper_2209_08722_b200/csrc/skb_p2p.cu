// One-shot all-reduce of an m-vector over NVLink peer memory (one process per
// GPU, one node), replacing NCCL for the per-pass exchange of SURVEY.md §8(e):
// every A-pass that produces an m-vector (the PCG normal matvec above all)
// ends with an all-reduce of m doubles (8 KB at c2, 80 KB at c4), a
// latency-bound message.
//
// Each rank owns a symmetric buffer (two m-slots, by epoch parity) and one flag
// word per block, opened by every peer through CUDA IPC. Block b of every rank
// handles the same row slice: it copies its slice of the local sum into its
// slot, publishes flag[b] = epoch (system-scope release), waits for flag[b] of
// every peer (acquire, P2P loads), then sums the peers' slices in rank order
// (bypassing L1). The result is identical on every rank and independent of
// arrival order. Two slots suffice: a rank cannot publish epoch e + 2 into a
// slot a peer still reads for epoch e, because finishing e + 1 needs that
// peer's epoch e + 1 flag, which it sets only after its epoch e kernel ended.
// A spin that exceeds ~2 s writes NaN (and sets *err) instead of hanging.
#include <cuda_runtime.h>

#include <string.h>

#include "skb_common.cuh"
#include "skb_internal.h"

namespace skb {

constexpr int kP2PMaxRanks = 8;
constexpr int kP2PThreads = 256;

struct P2PPeers {
  double* data[kP2PMaxRanks];      // [2][ld] per rank
  uint64_t* flags[kP2PMaxRanks];   // [max_blocks] per rank
};

SKB_DEV void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
SKB_DEV uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// mode 0: publish + gather (production); 1: publish only; 2: gather only
// (the single-process tests run the ranks' halves in an order that never waits).
__global__ void __launch_bounds__(kP2PThreads)
    p2p_allreduce_kernel(const double* __restrict__ local, double* __restrict__ out, int m,
                         int64_t ld, int rank, int world, P2PPeers peers, uint64_t epoch,
                         int mode, long long timeout_cycles, int* err) {
  const int b = blockIdx.x;
  const int r0 = b * kP2PThreads, r = r0 + threadIdx.x;
  const int slot = (int)(epoch & 1);
  if (mode != 2) {
    if (r < m) peers.data[rank][slot * ld + r] = local[r];
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      st_release_sys(&peers.flags[rank][b], epoch);
    }
  }
  if (mode == 1) return;
  __shared__ int ok;
  if (threadIdx.x == 0) {
    ok = 1;
    const long long t0 = clock64();
    for (int g = 0; g < world; ++g) {
      while (ld_acquire_sys(&peers.flags[g][b]) < epoch) {
        if (clock64() - t0 > timeout_cycles) {  // default ~2 s at 1.9 GHz
          ok = 0;
          atomicExch(err, 1);
          break;
        }
      }
      if (!ok) break;
    }
  }
  __syncthreads();
  if (r >= m) return;
  if (!ok) {
    out[r] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  double s = __ldcv(&peers.data[0][slot * ld + r]);
  for (int g = 1; g < world; ++g) s += __ldcv(&peers.data[g][slot * ld + r]);
  out[r] = s;
}

}  // namespace skb

using namespace skb;

// Symmetric buffers come from cudaMalloc (an IPC handle names a whole
// allocation; a caching allocator's sub-block would open at the wrong offset).
extern "C" int skb_p2p_alloc(int64_t bytes, uint64_t* dev_ptr_out) {
  void* p = nullptr;
  if (bytes <= 0 || cudaMalloc(&p, (size_t)bytes) != cudaSuccess) return skb_launch_status(__func__);
  if (cudaMemset(p, 0, (size_t)bytes) != cudaSuccess) return skb_launch_status(__func__);
  *dev_ptr_out = (uint64_t)(uintptr_t)p;
  return 0;
}

extern "C" int skb_p2p_free(uint64_t dev_ptr) {
  if (cudaFree((void*)(uintptr_t)dev_ptr) != cudaSuccess) return skb_launch_status(__func__);
  return 0;
}

extern "C" int skb_ipc_handle(void* dev_ptr, void* handle_out) {
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, dev_ptr) != cudaSuccess) return skb_launch_status(__func__);
  memcpy(handle_out, &h, sizeof(h));
  return 0;
}

extern "C" int skb_ipc_open(const void* handle, uint64_t* dev_ptr_out) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
    return skb_launch_status(__func__);
  *dev_ptr_out = (uint64_t)(uintptr_t)p;
  return 0;
}

extern "C" int skb_ipc_close(uint64_t dev_ptr) {
  if (cudaIpcCloseMemHandle((void*)(uintptr_t)dev_ptr) != cudaSuccess)
    return skb_launch_status(__func__);
  return 0;
}

extern "C" int32_t skb_p2p_can_access(int32_t device, int32_t peer) {
  int ok = 0;
  if (device == peer) return 1;
  if (cudaDeviceCanAccessPeer(&ok, device, peer) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return ok;
}

extern "C" int32_t skb_p2p_max_blocks(int64_t m) {
  return (int32_t)((m + kP2PThreads - 1) / kP2PThreads);
}

// out = sum over ranks of local (m doubles) through the peers' symmetric
// buffers: data_ptrs[g] -> [2][ld] doubles, flag_ptrs[g] -> >= ceil(m/256) u64
// (host arrays of world device pointers, this rank's own at index rank).
extern "C" int skb_p2p_allreduce(const double* local, double* out, int64_t m, int64_t ld,
                                 int32_t rank, int32_t world, const uint64_t* data_ptrs,
                                 const uint64_t* flag_ptrs, uint64_t epoch, int32_t mode,
                                 int64_t timeout_cycles, int* err, void* stream) {
  if (world < 1 || world > kP2PMaxRanks || rank < 0 || rank >= world || m < 0 || ld < m ||
      epoch == 0 || timeout_cycles <= 0)
    return SKB_ERR_ARG;
  if (m == 0) return 0;
  P2PPeers p{};
  for (int g = 0; g < world; ++g) {
    p.data[g] = (double*)(uintptr_t)data_ptrs[g];
    p.flags[g] = (uint64_t*)(uintptr_t)flag_ptrs[g];
  }
  const int grid = (int)((m + kP2PThreads - 1) / kP2PThreads);
  p2p_allreduce_kernel<<<grid, kP2PThreads, 0, (cudaStream_t)stream>>>(
      local, out, (int)m, ld, rank, world, p, epoch, mode, (long long)timeout_cycles, err);
  return skb_launch_status(__func__);
}
