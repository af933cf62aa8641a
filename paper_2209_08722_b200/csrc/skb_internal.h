// Internal host-side helpers shared by the skb translation units.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/skb.h"

// Bump allocator over a caller-provided device workspace. Kernels never
// allocate: the Python side owns the buffer (a torch tensor) and passes it in.
struct skb_ws {
  char* base;
  size_t cap;
  size_t off;
};

static inline skb_ws skb_ws_make(void* p, size_t bytes) {
  skb_ws w;
  w.base = (char*)p;
  w.cap = bytes;
  w.off = 0;
  return w;
}

static inline void* skb_ws_take(skb_ws* w, size_t bytes) {
  size_t o = (w->off + 255) & ~(size_t)255;
  if (!w->base || o + bytes > w->cap) return nullptr;
  w->off = o + bytes;
  return w->base + o;
}

static inline int skb_num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

#include <stdio.h>

// Collect the last launch error; on failure report it on stderr (the C ABI
// only returns a code) and return SKB_ERR_CUDA.
static inline int skb_launch_status(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return 0;
  fprintf(stderr, "[skb] %s: CUDA error %s (%s)\n", where, cudaGetErrorName(e),
          cudaGetErrorString(e));
  return SKB_ERR_CUDA;
}

// FP64 GEMM on the INT8 tensor cores (skb_ozaki.cu). Operand x has R rows over
// K with element (r, k) at p[r * sr + k * sk]; C[i][j] (row-major, ldc) =
// alpha sum_k a(i,k) kscale[k] b(j,k) + beta C. Returns 0 done, 1 not
// applicable (workspace / cuBLASLt unavailable: the caller runs DMMA), < 0 error.
struct skb_oz_operand {
  const double* p;
  int64_t sr, sk;
};
struct skb_oz_args {
  skb_oz_operand a, b;
  const double* kscale;
  double* C;
  int64_t ldc;
  int M, N, K;
  double alpha, beta;
  int lower_only;
  int tri_a, tri_b;  // as GemmArgs: opA lower (1) / upper (2), opB lower (1) / upper (2)
};
int skb_oz_gemm(const skb_oz_args& g, skb_ws* ws, cudaStream_t st);
size_t skb_oz_bytes(int M, int N, int K, bool share);

#include <string.h>

// Small device -> host readbacks (status words, counts, a few statistics)
// through the calling thread's pinned buffer: a pageable destination makes the
// driver stage the copy, which costs tens of microseconds more per readback
// on a path that does several per IPM step. Usage: add() the copies, then
// sync() once; the values land in the caller's (pageable) variables.
struct skb_readback {
  struct Item {
    void* dst;
    size_t at, n;
  };
  Item items[8];
  int k = 0;
  size_t off = 0;
  char* pin = nullptr;
  cudaStream_t st;
  explicit skb_readback(cudaStream_t s) : st(s) {
    thread_local char* buf = nullptr;
    if (!buf && cudaHostAlloc((void**)&buf, 4096, cudaHostAllocDefault) != cudaSuccess) {
      buf = nullptr;
      cudaGetLastError();
    }
    pin = buf;
  }
  void add(void* dst, const void* src, size_t n) {
    if (!pin || k == 8 || off + n > 4096) {  // no pinned room: direct (staged) copy
      cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, st);
      return;
    }
    cudaMemcpyAsync(pin + off, src, n, cudaMemcpyDeviceToHost, st);
    items[k++] = Item{dst, off, n};
    off += (n + 15) & ~(size_t)15;
  }
  cudaError_t sync() {
    const cudaError_t e = cudaStreamSynchronize(st);
    for (int i = 0; i < k; ++i) memcpy(items[i].dst, pin + items[i].at, items[i].n);
    return e;
  }
};

// Batched INT8 GEMM on tcgen05 (skb_i8gemm.cu); declared in include/skb.h.
