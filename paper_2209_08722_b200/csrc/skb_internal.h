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
