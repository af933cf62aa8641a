/* A non-Python host driving the drop-in boundary (include/skb.h) directly:
 * sparse-sign hashes (K1) and one fused normal-operator pass (K4) on device
 * memory from cudaMalloc, results printed for tests/test_gpu_c_abi.py to check
 * against the oracle. Build: gcc abi_smoke.c -I include -L<pkg> -lskb -lcudart */
#include <stdio.h>
#include <stdlib.h>
#include <cuda_runtime_api.h>

#include "skb.h"

#define CK(x)                                                        \
  do {                                                               \
    int rc_ = (int)(x);                                              \
    if (rc_ != 0) {                                                  \
      fprintf(stderr, "%s failed: %d (line %d)\n", #x, rc_, __LINE__); \
      return 1;                                                      \
    }                                                                \
  } while (0)

int main(int argc, char** argv) {
  if (argc < 3) {
    fprintf(stderr, "usage: abi_smoke KEY0 KEY1\n");
    return 2;
  }
  const uint64_t k0 = strtoull(argv[1], NULL, 10), k1 = strtoull(argv[2], NULL, 10);
  const int64_t n = 1000;
  const int32_t w = 64, s = 2;
  void* ws = NULL;
  const size_t wsb = 64u << 20;
  CK(cudaMalloc(&ws, wsb));
  int32_t* cols;
  double* vals;
  CK(cudaMalloc((void**)&cols, n * s * sizeof(int32_t)));
  CK(cudaMalloc((void**)&vals, n * s * sizeof(double)));
  uint64_t used = 0;
  CK(skb_sparse_embedding(k0, k1, n, w, s, cols, vals, &used, ws, wsb, NULL));
  int32_t hc[8];
  double hv[8];
  CK(cudaMemcpy(hc, cols, sizeof(hc), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hv, vals, sizeof(hv), cudaMemcpyDeviceToHost));
  printf("words_used %llu\n", (unsigned long long)used);
  printf("cols");
  for (int i = 0; i < 8; ++i) printf(" %d", hc[i]);
  printf("\nvals");
  for (int i = 0; i < 8; ++i) printf(" %.17g", hv[i]);
  printf("\n");

  /* u = A diag(d2) A' z for A(i, j) = ((i + 2 j) % 7) - 3, column-major, lda = m (even) */
  const int64_t m = 6, lda = 6, nn = 50;
  double hA[6 * 50], hd2[50], hz[6], hu[6];
  for (int64_t j = 0; j < nn; ++j) {
    hd2[j] = 0.5 + 0.01 * (double)j;
    for (int64_t i = 0; i < m; ++i) hA[j * lda + i] = (double)((i + 2 * j) % 7) - 3.0;
  }
  for (int64_t i = 0; i < m; ++i) hz[i] = 1.0 + (double)i;
  double *A, *d2, *z, *u;
  CK(cudaMalloc((void**)&A, sizeof(hA)));
  CK(cudaMalloc((void**)&d2, sizeof(hd2)));
  CK(cudaMalloc((void**)&z, sizeof(hz)));
  CK(cudaMalloc((void**)&u, sizeof(hu)));
  CK(cudaMemcpy(A, hA, sizeof(hA), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d2, hd2, sizeof(hd2), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(z, hz, sizeof(hz), cudaMemcpyHostToDevice));
  CK(skb_normal_apply(A, m, nn, lda, d2, z, u, NULL, NULL, ws, wsb, NULL));
  CK(cudaMemcpy(hu, u, sizeof(hu), cudaMemcpyDeviceToHost));
  printf("u");
  for (int i = 0; i < 6; ++i) printf(" %.17g", hu[i]);
  printf("\n");
  return 0;
}
