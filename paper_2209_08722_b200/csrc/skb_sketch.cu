// K2: ADW = A diag(d) W for the sparse-sign / CountSketch W, bit-exact.
//
// Replaces apply_sketch (reference sketching.py:142-161): AD = A.multiply(d)
// then (AD @ W_csr).toarray() via scipy csr_matmat, which for every row i and
// bucket b sums fl(fl(A_ij d_j) v_jk) over the entries (j,k) with cols[j,k] = b
// in ascending j, one multiply and one add per term, starting from 0.
//
// B200 mapping (output stored bucket-major: X[b][i] = ADW[i][b], i.e. ADW'):
//  1. stable counting sort of the n*s entries by bucket (chunk histograms,
//     per-chunk exclusive offsets, warp-synchronous match_any ranking) ->
//     member lists in ascending j;
//  2. persistent CTAs, one bucket at a time (dynamic fetch): a producer warp
//     streams the member columns (contiguous, column-major A) through a ring
//     of shared-memory stages with the TMA bulk engine; 256 consumer threads
//     each own a pair of rows and accumulate in registers in member order with
//     __dmul_rn/__dadd_rn (no FMA). Splitting rows (not members) across
//     threads keeps the per-(i, b) summation order of the reference exactly.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include <cub/block/block_radix_sort.cuh>
#include <cub/device/device_histogram.cuh>
#include <cub/device/device_radix_sort.cuh>

#include "skb_common.cuh"
#include "skb_internal.h"

namespace skb {

__global__ void bucket_hist_kernel(const int32_t* __restrict__ cols, int64_t N, int64_t C, int w,
                                   int32_t* __restrict__ hist) {
  const int64_t e0 = (int64_t)blockIdx.x * C, e1 = min(N, e0 + C);
  int32_t* h = hist + (int64_t)blockIdx.x * w;
  for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) atomicAdd(&h[cols[e]], 1);
}

// In place: hist[c][b] <- sum_{c' < c} hist[c'][b]; total[b] <- sum_c hist[c][b].
__global__ void bucket_chunk_prefix_kernel(int32_t* __restrict__ hist, int nchunks, int w,
                                           uint32_t* __restrict__ total) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= w) return;
  int32_t run = 0;
  for (int c0 = 0; c0 < nchunks; c0 += 16) {  // batch the loads: they are independent
    int32_t t[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) t[q] = c0 + q < nchunks ? hist[(int64_t)(c0 + q) * w + b] : 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      if (c0 + q < nchunks) hist[(int64_t)(c0 + q) * w + b] = run;
      run += t[q];
    }
  }
  total[b] = (uint32_t)run;
}

// One CTA per chunk: the chunk's bucket ids are staged in shared memory by all
// threads, then warp 0 ranks them in entry order (match_any) against a
// shared-memory cursor per bucket and writes the entry index to its slot.
constexpr int kScatterSub = 4096;

// Member codes: the entry index (< 2^31) with the sign of its hash value in bit
// 31, so a bucket's consumers learn v = +-1/sqrt(s) without gathering vals.
SKB_DEV uint32_t sign_bit(const double* __restrict__ vals, int64_t e) {
  return vals[e] < 0.0 ? 0x80000000u : 0u;
}
constexpr uint32_t kMemIdx = 0x7FFFFFFFu;

__global__ void __launch_bounds__(256) bucket_scatter_kernel(
    const int32_t* __restrict__ cols, int64_t N, int64_t C, int w,
    const int32_t* __restrict__ hist, const uint64_t* __restrict__ start,
    const double* __restrict__ vals, int32_t* __restrict__ mem_e) {
  extern __shared__ uint32_t sm_scatter[];
  uint32_t* cursor = sm_scatter;
  int32_t* sb = reinterpret_cast<int32_t*>(sm_scatter + w);
  const int64_t c = blockIdx.x, e0 = c * C, e1 = min(N, e0 + C);
  for (int b = threadIdx.x; b < w; b += blockDim.x)
    cursor[b] = (uint32_t)(start[b] + hist[c * w + b]);
  const int lane = threadIdx.x & 31;
  for (int64_t s0 = e0; s0 < e1; s0 += kScatterSub) {
    const int cnt = (int)min((int64_t)kScatterSub, e1 - s0);
    __syncthreads();
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) sb[t] = cols[s0 + t];
    __syncthreads();
    if (threadIdx.x < 32) {
      for (int base = 0; base < cnt; base += 32) {
        const int t = base + lane;
        const bool act = t < cnt;
        const unsigned amask = __ballot_sync(0xffffffffu, act);
        if (!act) break;
        const int b = sb[t];
        const unsigned peers = __match_any_sync(amask, b);
        const int rank = __popc(peers & ((1u << lane) - 1u));
        mem_e[cursor[b] + rank] = (int32_t)((uint32_t)(s0 + t) | sign_bit(vals, s0 + t));
        __syncwarp(amask);
        if (rank == 0) cursor[b] += __popc(peers);
        __syncwarp(amask);
      }
    }
  }
}

// start[b] = first position of bucket b in the sorted keys (start[w] = N): each
// boundary i (keys[i-1] != keys[i], or the ends) fills the buckets in between.
__global__ void bucket_starts_kernel(const uint32_t* __restrict__ keys, int64_t N, int w,
                                     uint64_t* __restrict__ start) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > N) return;
  const int64_t kp = i == 0 ? -1 : (int64_t)keys[i - 1];
  const int64_t kc = i == N ? (int64_t)w : (int64_t)keys[i];
  for (int64_t b = kp + 1; b <= kc; ++b) start[b] = (uint64_t)i;
}

__global__ void scan_buckets_kernel(const uint32_t* __restrict__ in, uint64_t* __restrict__ out,
                                    int n) {
  __shared__ uint64_t part[1024];
  __shared__ uint64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < n; base += 1024) {
    const int i = base + threadIdx.x;
    const uint64_t v = i < n ? in[i] : 0;
    part[threadIdx.x] = v;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
      const uint64_t t = threadIdx.x >= off ? part[threadIdx.x - off] : 0;
      __syncthreads();
      part[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < n) out[i] = carry + part[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += part[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[n] = carry;
}

struct StageMeta {
  double d, v;
  int32_t bucket;  // -1: terminate
  int32_t flags;   // 1 first, 2 last, 4 empty bucket
};

constexpr int kConsumers = 256;

template <int KP>  // row pairs per consumer thread: m <= 512 * KP
__global__ void __launch_bounds__(kConsumers + 32, KP <= 4 ? 2 : 1)
    sketch_accumulate_kernel(const double* __restrict__ A, int64_t lda, int m,
                             const double* __restrict__ d, const uint64_t* __restrict__ start,
                             const int32_t* __restrict__ mem_e, const double* __restrict__ vals,
                             int s,
                             int w, int stages, unsigned int* __restrict__ counter,
                             double* __restrict__ X, int64_t ldx) {
  extern __shared__ __align__(128) unsigned char smem[];
  const size_t col_bytes = (size_t)((m + 1) & ~1) * 8;  // this row slice of a column
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + stages;
  StageMeta* meta = reinterpret_cast<StageMeta*>(empty + stages);
  size_t off = ((size_t)stages * (16 + sizeof(StageMeta)) + 127) & ~(size_t)127;
  unsigned char* bufs = smem + off;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kConsumers / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 0) {  // ---------------- producer warp (lane 0 issues, all lanes fetch metadata)
    const uint64_t pol = l2_evict_first_policy();
    int st = 0;
    uint32_t ph = 0;
    auto next = [&]() {
      if (++st == stages) {
        st = 0;
        ph ^= 1;
      }
    };
    for (;;) {
      int b = 0;
      if (lane == 0) b = (int)atomicAdd(counter, 1u);
      b = __shfl_sync(0xffffffffu, b, 0);
      if (b >= w) break;
      const uint64_t e0 = start[b], e1 = start[b + 1];
      if (e0 == e1) {
        if (lane == 0) {
          mbar_wait(&empty[st], ph ^ 1);
          meta[st] = StageMeta{0.0, 0.0, b, 1 | 2 | 4};
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[st]))
                       : "memory");
        }
        next();
        continue;
      }
      for (uint64_t eb = e0; eb < e1; eb += 32) {
        const uint64_t e = eb + lane;
        int64_t j = 0;
        double v = 0.0, dj = 0.0;
        if (e < e1) {
          const int64_t ei = (uint32_t)mem_e[e] & kMemIdx;
          j = ei / s;
          v = vals[ei];
          dj = d[j];
        }
        const int cnt = (int)min((uint64_t)32, e1 - eb);
        for (int q = 0; q < cnt; ++q) {
          const int64_t jq = __shfl_sync(0xffffffffu, j, q);
          const double vq = __shfl_sync(0xffffffffu, v, q);
          const double dq = __shfl_sync(0xffffffffu, dj, q);
          if (lane == 0) {
            const uint64_t eq = eb + q;
            mbar_wait(&empty[st], ph ^ 1);
            meta[st] = StageMeta{dq, vq, b, (eq == e0 ? 1 : 0) | (eq + 1 == e1 ? 2 : 0)};
            mbar_arrive_expect_tx(&full[st], (uint32_t)col_bytes);
            bulk_g2s(bufs + (size_t)st * col_bytes, A + jq * lda, (uint32_t)col_bytes, &full[st],
                     pol);
          }
          next();
        }
      }
    }
    if (lane == 0) {
      mbar_wait(&empty[st], ph ^ 1);
      meta[st] = StageMeta{0.0, 0.0, -1, 0};
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[st]))
                   : "memory");
    }
    return;
  }

  // ------------------------------------ consumers: thread p owns row pairs 2p + 512k
  const int p = threadIdx.x - 32;
  double2 acc[KP];
  int st = 0;
  uint32_t ph = 0;
  for (;;) {
    mbar_wait(&full[st], ph);
    const StageMeta mt = meta[st];
    if (mt.bucket < 0) break;
    if (mt.flags & 1) {
#pragma unroll
      for (int k = 0; k < KP; ++k) acc[k] = make_double2(0.0, 0.0);
    }
    if (!(mt.flags & 4)) {
      const double* col = reinterpret_cast<const double*>(bufs + (size_t)st * col_bytes);
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const int r = 512 * k + 2 * p;
        if (r < m) {
          const double2 a = *reinterpret_cast<const double2*>(col + r);
          acc[k].x = __dadd_rn(acc[k].x, __dmul_rn(__dmul_rn(a.x, mt.d), mt.v));
          acc[k].y = __dadd_rn(acc[k].y, __dmul_rn(__dmul_rn(a.y, mt.d), mt.v));
        }
      }
    }
    if (mt.flags & 2) {
      double* out = X + (int64_t)mt.bucket * ldx;
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const int r = 512 * k + 2 * p;
        if (r + 1 < m)
          *reinterpret_cast<double2*>(out + r) = acc[k];
        else if (r < m)
          out[r] = acc[k].x;
      }
    }
    __syncwarp();
    if (lane == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[st]))
                   : "memory");
    if (++st == stages) {
      st = 0;
      ph ^= 1;
    }
  }
}

// Identity sketch (w >= n): ADW = AD, X[j][i] = A_ij * d_j  (sketching.py:155-156).
__global__ void scale_columns_kernel(const double* __restrict__ A, int64_t lda, int m, int64_t n,
                                     const double* __restrict__ d, double* __restrict__ X,
                                     int64_t ldx) {
  const int64_t j = blockIdx.x;
  if (j >= n) return;
  const double dj = d[j];
  for (int i = threadIdx.x; i < m; i += blockDim.x) X[j * ldx + i] = __dmul_rn(A[j * lda + i], dj);
}

// v_j = sqrt(x_j s_j) * sum_k vals[j,k] u[cols[j,k]]   (correction.py:58; sketching.py:80)
__global__ void sketch_gather_kernel(const int32_t* __restrict__ cols,
                                     const double* __restrict__ vals, int s, int64_t n,
                                     const double* __restrict__ u, const double* __restrict__ x,
                                     const double* __restrict__ sv, double* __restrict__ v) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double t = __dmul_rn(vals[j * s], u[cols[j * s]]);
  for (int k = 1; k < s; ++k) t = __dadd_rn(t, __dmul_rn(vals[j * s + k], u[cols[j * s + k]]));
  if (x) t = __dmul_rn(__dsqrt_rn(__dmul_rn(x[j], sv[j])), t);
  v[j] = t;
}

}  // namespace skb

using namespace skb;

namespace skb {
__global__ void iota_kernel(int32_t* __restrict__ v, const double* __restrict__ vals, int64_t N) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) v[i] = (int32_t)((uint32_t)i | sign_bit(vals, i));
}
}  // namespace skb

// N >= 2^20: stable LSD radix sort (CUB) of the entries by bucket, ceil(log2 w)
// key bits; stability keeps ascending entry order inside each bucket, so the
// result equals the counting sort's.
constexpr int64_t kRadixMinN = 1ll << 20;

static size_t radix_temp_bytes(int64_t N, int32_t w) {
  size_t sort_b = 0, hist_b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_b, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)N, 0, 32);
  cub::DeviceHistogram::HistogramEven(nullptr, hist_b, (const int32_t*)nullptr,
                                      (uint32_t*)nullptr, (int)w + 1, 0, (int)w, (int)N);
  return std::max(sort_b, hist_b) + 256;
}

extern "C" size_t skb_sketch_workspace_bytes(int64_t n, int32_t w, int32_t s) {
  const int64_t N = n * (int64_t)s;
  int64_t C = std::max<int64_t>(4096, (N * (int64_t)w) / (16ll << 20) + 1);
  const int64_t nch = (N + C - 1) / C;
  const size_t counting =
      (size_t)nch * w * 4 + (size_t)w * 4 + (size_t)(w + 1) * 8 + (size_t)N * 4 + 16 + 8 * 256;
  if (N < kRadixMinN && !getenv("SKB_BUCKET_RADIX")) return counting;
  const size_t radix = (size_t)w * 4 + (size_t)(w + 1) * 8 + (size_t)N * 4 * 3 + 16 +
                       radix_temp_bytes(N, w) + 8 * 256;
  return std::max(counting, radix);
}

static int bucket_sort_radix(const int32_t* cols, const double* vals, int64_t N, int32_t w,
                             skb_ws* ws,
                             cudaStream_t st, uint64_t** start_out, int32_t** mem_out,
                             unsigned int** counter_out) {
  uint32_t* total = (uint32_t*)skb_ws_take(ws, (size_t)w * 4);
  uint64_t* start = (uint64_t*)skb_ws_take(ws, (size_t)(w + 1) * 8);
  int32_t* mem_e = (int32_t*)skb_ws_take(ws, (size_t)N * 4);
  uint32_t* keys = (uint32_t*)skb_ws_take(ws, (size_t)N * 4);
  int32_t* iota = (int32_t*)skb_ws_take(ws, (size_t)N * 4);
  unsigned int* counter = (unsigned int*)skb_ws_take(ws, 16);
  const size_t tb = radix_temp_bytes(N, w);
  void* tmp = skb_ws_take(ws, tb);
  if (!total || !start || !mem_e || !keys || !iota || !counter || !tmp) return SKB_ERR_WORKSPACE;
  cudaMemsetAsync(counter, 0, 16, st);
  int bits = 1;
  while ((1ll << bits) < (int64_t)w) ++bits;
  (void)total;
  iota_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(iota, vals, N);
  size_t b2 = tb;
  cub::DeviceRadixSort::SortPairs(tmp, b2, reinterpret_cast<const uint32_t*>(cols), keys, iota,
                                  mem_e, (int)N, 0, bits, st);
  // bucket starts from the sorted keys' boundaries (no separate histogram pass)
  bucket_starts_kernel<<<(unsigned)((N + 1 + 255) / 256), 256, 0, st>>>(keys, N, w, start);
  *start_out = start;
  *mem_out = mem_e;
  *counter_out = counter;
  return skb_launch_status("bucket_sort_radix");
}

// Stable counting sort of the n*s hash entries by bucket -> start[w+1], mem_e[N]
// (entry indices, ascending within each bucket), plus a zeroed work counter.
static int bucket_sort(const int32_t* cols, const double* vals, int64_t n, int32_t s, int32_t w,
                       skb_ws* ws,
                       cudaStream_t st, uint64_t** start_out, int32_t** mem_out,
                       unsigned int** counter_out) {
  const int64_t N = n * (int64_t)s;
  if ((N >= kRadixMinN || getenv("SKB_BUCKET_RADIX")) && N < (1ll << 31) &&
      !getenv("SKB_BUCKET_COUNTING"))
    return bucket_sort_radix(cols, vals, N, w, ws, st, start_out, mem_out, counter_out);
  const int64_t C = std::max<int64_t>(4096, (N * (int64_t)w) / (16ll << 20) + 1);
  const int64_t nch = (N + C - 1) / C;
  int32_t* hist = (int32_t*)skb_ws_take(ws, (size_t)nch * w * 4);
  uint32_t* total = (uint32_t*)skb_ws_take(ws, (size_t)w * 4);
  uint64_t* start = (uint64_t*)skb_ws_take(ws, (size_t)(w + 1) * 8);
  int32_t* mem_e = (int32_t*)skb_ws_take(ws, (size_t)std::max<int64_t>(N, 1) * 4);
  unsigned int* counter = (unsigned int*)skb_ws_take(ws, 16);
  if (!hist || !total || !start || !mem_e || !counter) return SKB_ERR_WORKSPACE;
  if (N >= (1ll << 31)) return SKB_ERR_UNSUPPORTED;
  cudaMemsetAsync(hist, 0, (size_t)nch * w * 4, st);
  cudaMemsetAsync(counter, 0, 16, st);
  if (N > 0) {
    bucket_hist_kernel<<<(unsigned)nch, 256, 0, st>>>(cols, N, C, w, hist);
  }
  bucket_chunk_prefix_kernel<<<(w + 255) / 256, 256, 0, st>>>(hist, (int)nch, w, total);
  scan_buckets_kernel<<<1, 1024, 0, st>>>(total, start, w);
  if (N > 0) {
    const size_t csm = (size_t)w * 4 + (size_t)kScatterSub * 4;
    static size_t conf_sc = 0;
    if (csm > 48 * 1024 && csm > conf_sc) {
      if (csm > 220 * 1024) return SKB_ERR_UNSUPPORTED;
      cudaFuncSetAttribute(bucket_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)csm);
      conf_sc = csm;
    }
    bucket_scatter_kernel<<<(unsigned)nch, 256, csm, st>>>(cols, N, C, w, hist, start, vals,
                                                           mem_e);
  }
  *start_out = start;
  *mem_out = mem_e;
  *counter_out = counter;
  return 0;
}

// ---- CSC A (c4): one warp per bucket, the bucket's m-vector in shared memory.
// Members are processed in ascending column order; a member's entries hit
// distinct rows, so its (<= 32 at a time) lanes update without conflicts and
// every (row, bucket) sum keeps scipy's ascending-j order, no FMA: bit-exact.
constexpr int kCscStage = 8;  // entries staged per member (longer columns loop)

__global__ void __launch_bounds__(32)
    csc_sketch_kernel(const int64_t* __restrict__ colptr, const int32_t* __restrict__ rowidx,
                      const double* __restrict__ av, int m, const double* __restrict__ d,
                      const uint64_t* __restrict__ start, const int32_t* __restrict__ mem_e,
                      const double* __restrict__ wvals, int s, int w,
                      unsigned int* __restrict__ counter, double* __restrict__ X, int64_t ldx) {
  extern __shared__ __align__(16) double sacc[];
  int32_t* srow = reinterpret_cast<int32_t*>(sacc + m);
  double* sval = reinterpret_cast<double*>(srow + 32 * kCscStage + 32);  // 8-aligned
  sval = reinterpret_cast<double*>(((uintptr_t)sval + 15) & ~(uintptr_t)15);
  const int lane = threadIdx.x;
  for (;;) {
    int b = 0;
    if (lane == 0) b = (int)atomicAdd(counter, 1u);
    b = __shfl_sync(0xffffffffu, b, 0);
    if (b >= w) break;
    for (int i = lane; i < m; i += 32) sacc[i] = 0.0;
    __syncwarp();
    const uint64_t e0 = start[b], e1 = start[b + 1];
    for (uint64_t eb = e0; eb < e1; eb += 32) {
      const uint64_t e = eb + lane;
      int64_t c0 = 0, cnt = 0;
      double scl = 0.0, wv = 0.0;
      if (e < e1) {
        const int64_t ei = (uint32_t)mem_e[e] & kMemIdx;
        const int64_t j = ei / s;
        wv = wvals[ei];
        scl = d[j];
        c0 = colptr[j];
        cnt = colptr[j + 1] - c0;
        for (int t = 0; t < kCscStage && t < cnt; ++t) {  // stage this member's entries
          srow[lane * kCscStage + t] = rowidx[c0 + t];
          sval[lane * kCscStage + t] = av[c0 + t];
        }
      }
      __syncwarp();
      const int nm = (int)min((uint64_t)32, e1 - eb);
      for (int q = 0; q < nm; ++q) {
        const int64_t cq = __shfl_sync(0xffffffffu, cnt, q);
        const int64_t c0q = __shfl_sync(0xffffffffu, c0, q);
        const double dq = __shfl_sync(0xffffffffu, scl, q);
        const double wq = __shfl_sync(0xffffffffu, wv, q);
        for (int64_t t = lane; t < cq; t += 32) {
          const int r = t < kCscStage ? srow[q * kCscStage + t] : rowidx[c0q + t];
          const double a = t < kCscStage ? sval[q * kCscStage + t] : av[c0q + t];
          sacc[r] = __dadd_rn(sacc[r], __dmul_rn(__dmul_rn(a, dq), wq));
        }
        __syncwarp();
      }
    }
    double* out = X + (int64_t)b * ldx;
    for (int i = lane; i < m; i += 32) out[i] = sacc[i];
    __syncwarp();
  }
}

// ---- CSC A, large m: one THREAD per bucket, its row of X (bucket-major, zeroed
// beforehand) updated in place in global memory. The thread walks the
// bucket's members in ascending j and applies each member's entries in
// order, so every (row, bucket) sum is the same left-to-right fl-sum as
// scipy's (bit-exact); buckets are independent, so all w threads run at once
// (a shared-memory m-vector per bucket would allow only ~2 buckets per SM at
// m = 1e4). Index loads of the next member are issued ahead of the RMWs.
constexpr int kRmwThreads = 256;
constexpr int kRmwStage = 8;

// (Development fallback, SKB_CSC_SKETCH_RMW=1: thread per bucket, or S threads
// per bucket owning row slices; random HBM read-modify-writes of X, 27 ms at
// c4 with s = 4 whatever S.)
template <int S>
__global__ void __launch_bounds__(kRmwThreads)
    csc_sketch_rmw_kernel(const int64_t* __restrict__ colptr, const int32_t* __restrict__ rowidx,
                          const double* __restrict__ av, const double* __restrict__ d,
                          const uint64_t* __restrict__ start, const int32_t* __restrict__ mem_e,
                          const double* __restrict__ wvals, int s, int w, int m,
                          double* __restrict__ X, int64_t ldx) {
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int b = (int)(gt / S), sl = (int)(gt % S);
  if (b >= w) return;
  const int rlo = (int)((int64_t)m * sl / S), rhi = (int)((int64_t)m * (sl + 1) / S);
  double* __restrict__ Xb = X + (int64_t)b * ldx;
  const uint64_t e0 = start[b], e1 = start[b + 1];
  int64_t ei_next = e0 < e1 ? ((uint32_t)mem_e[e0] & kMemIdx) : 0;
  for (uint64_t e = e0; e < e1; ++e) {
    const int64_t ei = ei_next;
    if (e + 1 < e1) ei_next = (uint32_t)mem_e[e + 1] & kMemIdx;
    const int64_t j = ei / s;
    const double wv = wvals[ei], dj = d[j];
    const int64_t c0 = colptr[j], c1 = colptr[j + 1];
    for (int64_t t0 = c0; t0 < c1; t0 += kRmwStage) {
      int r[kRmwStage];
      double a[kRmwStage];
#pragma unroll
      for (int q = 0; q < kRmwStage; ++q) {
        const bool ok = t0 + q < c1;
        r[q] = ok ? rowidx[t0 + q] : -1;
        a[q] = ok ? av[t0 + q] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < kRmwStage; ++q)
        if (r[q] >= rlo && r[q] < rhi)
          Xb[r[q]] = __dadd_rn(Xb[r[q]], __dmul_rn(__dmul_rn(a[q], dj), wv));
    }
  }
}

// Large m (c4: m = 1e4, w = 4e4, s = 4): a warp per bucket, the buckets in
// flight limited to the resident warps (~1,200 x 80 KB bucket rows of X stay
// in L2 while they are updated). The warp takes its members 32 at a time
// (lane = member, ascending = the reference's order) through a 3-stage load
// pipeline (member ids -> column meta -> the column's first kL2U row indices
// and values), so every HBM gather is in flight one chunk ahead. A chunk's
// entries are applied in parallel where their row is unique in the chunk (a
// hashed per-warp count table); entries whose row may repeat are applied
// lane by lane in ascending lane order. Each (bucket, row) sum thus runs in
// ascending member order exactly as scipy's, and X is touched only in L2.
constexpr int kL2Threads = 128, kL2U = 8, kL2Hash = 2048;

struct L2Meta {  // one member's column: first entry, count, d_j and the sketch value
  int64_t c0;
  int nn;
  double dj, wv;
};

__global__ void __launch_bounds__(kL2Threads)
    csc_sketch_l2_kernel(const int64_t* __restrict__ colptr, const int32_t* __restrict__ rowidx,
                         const double* __restrict__ av, const double* __restrict__ d,
                         const uint64_t* __restrict__ start, const int32_t* __restrict__ mem_e,
                         const double* __restrict__ wvals, int s, int w,
                         double* __restrict__ X, int64_t ldx) {
  __shared__ int cnt_all[(kL2Threads / 32) * kL2Hash];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int* cnt = cnt_all + wid * kL2Hash;
  for (int i = lane; i < kL2Hash; i += 32) cnt[i] = 0;
  __syncwarp();
  const int gw = blockIdx.x * (kL2Threads / 32) + wid, nw = gridDim.x * (kL2Threads / 32);
  const uint64_t pol = l2_evict_first_policy();  // gathers must not evict the X rows
  for (int b = gw; b < w; b += nw) {
    double* __restrict__ Xb = X + (int64_t)b * ldx;
    const int64_t e0 = (int64_t)start[b], e1 = (int64_t)start[b + 1];
    const int nchunk = (int)((e1 - e0 + 31) / 32);
    // pipeline registers: ei (chunk k+2), meta (chunk k+1), entries (chunk k)
    auto load_ei = [&](int k) -> int64_t {
      const int64_t e = e0 + 32 * (int64_t)k + lane;
      return (k < nchunk && e < e1) ? (int64_t)((uint32_t)ldg_ef(&mem_e[e], pol) & kMemIdx) : -1;
    };
    auto load_meta = [&](int64_t ei) -> L2Meta {
      L2Meta mt{0, 0, 0.0, 0.0};
      if (ei >= 0) {
        const int64_t j = ei / s;
        mt.c0 = ldg_ef(reinterpret_cast<const long long*>(colptr) + j, pol);
        mt.nn = (int)(ldg_ef(reinterpret_cast<const long long*>(colptr) + j + 1, pol) - mt.c0);
        mt.dj = ldg_ef(&d[j], pol);
        mt.wv = ldg_ef(&wvals[ei], pol);
      }
      return mt;
    };
    int rr[kL2U];
    double aa[kL2U];
    auto load_entries = [&](const L2Meta& mt) {
#pragma unroll
      for (int q = 0; q < kL2U; ++q) {
        const bool ok = q < mt.nn;
        rr[q] = ok ? ldg_ef(&rowidx[mt.c0 + q], pol) : -1;
        aa[q] = ok ? ldg_ef(&av[mt.c0 + q], pol) : 0.0;
      }
    };
    int64_t ei_next = load_ei(1);
    L2Meta mt_cur = load_meta(load_ei(0));
    L2Meta mt_next = load_meta(ei_next);
    ei_next = load_ei(2);
    load_entries(mt_cur);
    for (int k = 0; k < nchunk; ++k) {
      // values of chunk k (entries loaded one iteration ago)
      int r[kL2U];
      double v[kL2U];
#pragma unroll
      for (int q = 0; q < kL2U; ++q) {
        r[q] = rr[q];
        v[q] = __dmul_rn(__dmul_rn(aa[q], mt_cur.dj), mt_cur.wv);
      }
      const int nn = mt_cur.nn;
      const int64_t c0 = mt_cur.c0;
      const double dj = mt_cur.dj, wv = mt_cur.wv;
      // keep the pipeline going: entries of chunk k+1, meta of chunk k+2, ids of k+3
      mt_cur = mt_next;
      load_entries(mt_cur);
      mt_next = load_meta(ei_next);
      ei_next = load_ei(k + 3);
      const bool long_col = __any_sync(0xffffffffu, nn > kL2U);
      if (!long_col) {
#pragma unroll
        for (int q = 0; q < kL2U; ++q)
          if (q < nn) atomicAdd(&cnt[r[q] & (kL2Hash - 1)], 1);
        __syncwarp();
        bool uq[kL2U];
        bool any_rep = false;
#pragma unroll
        for (int q = 0; q < kL2U; ++q) {
          uq[q] = q < nn && cnt[r[q] & (kL2Hash - 1)] == 1;
          any_rep |= q < nn && !uq[q];
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < kL2U; ++q)
          if (q < nn) cnt[r[q] & (kL2Hash - 1)] = 0;
        // unique rows: all RMWs of the lane in flight together
        double x[kL2U];
#pragma unroll
        for (int q = 0; q < kL2U; ++q) x[q] = uq[q] ? Xb[r[q]] : 0.0;
#pragma unroll
        for (int q = 0; q < kL2U; ++q)
          if (uq[q]) Xb[r[q]] = __dadd_rn(x[q], v[q]);
        // possibly repeated rows: lane by lane, ascending (= member order)
        for (unsigned g = __ballot_sync(0xffffffffu, any_rep); g; g &= g - 1) {
          if (__ffs(g) - 1 == lane) {
#pragma unroll
            for (int q = 0; q < kL2U; ++q)
              if (q < nn && !uq[q]) Xb[r[q]] = __dadd_rn(Xb[r[q]], v[q]);
          }
          __syncwarp();
        }
        __syncwarp();
      } else {
        // a column longer than kL2U in this chunk: the whole chunk lane by lane
        for (int l = 0; l < 32; ++l) {
          if (l == lane) {
            for (int q = 0; q < nn; ++q) {
              const int rq = q < kL2U ? r[q] : __ldg(&rowidx[c0 + q]);
              const double vq =
                  q < kL2U ? v[q] : __dmul_rn(__dmul_rn(__ldg(&av[c0 + q]), dj), wv);
              Xb[rq] = __dadd_rn(Xb[rq], vq);
            }
          }
          __syncwarp();
        }
      }
    }
  }
}

namespace skb {
// ---- CSC A through ELL head records (m <= 65535): one CTA per bucket (dynamic
// fetch), the bucket's row of X as an m-vector in shared memory. Members are
// taken 256 at a time (one per thread, ascending j); each member's 64-byte
// record (rows, values, and d_j written into it for this call) arrives in one
// load, prefetched a batch ahead. The batch's terms fl(fl(A_ij d_j) v) are
// added to the accumulator in rounds of bids (below), so each row takes its
// terms in member order: every (row, bucket) sum is the reference's
// ascending-j left-to-right fl-sum (bit-exact) with no
// atomics on values. Columns longer than a record run member by member from
// the CSC arrays (the batch is split there, order kept).
constexpr int kEllSkT = 512;
struct __align__(16) SkEll {  // = EllRec of skb_stream.cu, spare = d_j for this call
  uint16_t row[5];
  uint8_t cnt, pad[5];
  double val[5];
  double d;
};
static_assert(sizeof(SkEll) == 64, "ELL record");

__global__ void ell_set_d_kernel(SkEll* __restrict__ ell, const double* __restrict__ d,
                                 int64_t n) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) ell[j].d = d[j];
}

// Ordered application of one batch's terms without sorting: in round k every
// pending term bids its member index for its row (shared atomicMin), the
// lowest bidder of each row adds its term and resets the row's bid, the others
// wait for the next round -- so each row receives its terms in ascending member
// (= ascending j) order. Rounds = the largest multiplicity of a row in the
// batch (~3 for 2,560 terms over 1e4 rows).
__global__ void __launch_bounds__(kEllSkT, 1)
    csc_sketch_ell_kernel(const SkEll* __restrict__ ell, const int64_t* __restrict__ colptr,
                          const int32_t* __restrict__ rowidx, const double* __restrict__ av,
                          const double* __restrict__ d, const uint64_t* __restrict__ start,
                          const int32_t* __restrict__ mem_e, double vmag, int s, int w, int m,
                          unsigned int* __restrict__ counter, double* __restrict__ X,
                          int64_t ldx) {
  __shared__ int sb;
  extern __shared__ __align__(16) double acc[];  // m doubles, then m int32 bids
  int* bid = reinterpret_cast<int*>(acc + m);
  const int tid = threadIdx.x;
  for (int i = tid; i < m; i += kEllSkT) {
    acc[i] = 0.0;
    bid[i] = 0x7fffffff;
  }
  for (;;) {
    __syncthreads();
    if (tid == 0) sb = (int)atomicAdd(counter, 1u);
    __syncthreads();
    const int b = sb;
    if (b >= w) break;
    const uint64_t e0 = start[b], e1 = start[b + 1];
    SkEll rec{};
    uint32_t code = 0;
    bool have = false;
    auto fetch = [&](uint64_t eb) {
      have = eb + tid < e1;
      if (have) {
        code = (uint32_t)mem_e[eb + tid];
        const int64_t j = (int64_t)(code & 0x7FFFFFFFu) / s;
        rec = ell[j];
      }
    };
    fetch(e0);
    for (uint64_t eb = e0; eb < e1; eb += kEllSkT) {
      const SkEll r = rec;
      const uint32_t c = code;
      const bool h = have;
      if (eb + kEllSkT < e1) fetch(eb + kEllSkT);  // next batch in flight during this one
      const double v = (c & 0x80000000u) ? -vmag : vmag;
      if (!__syncthreads_or(h && r.cnt > 5)) {
        double t[5];
        unsigned pend = 0;  // bit q: term q not applied yet
#pragma unroll
        for (int q = 0; q < 5; ++q) {
          t[q] = __dmul_rn(__dmul_rn(r.val[q], r.d), v);
          if (h && q < r.cnt) pend |= 1u << q;
        }
        while (__syncthreads_or(pend != 0)) {
#pragma unroll
          for (int q = 0; q < 5; ++q)
            if (pend & (1u << q)) atomicMin(&bid[r.row[q]], tid);
          __syncthreads();
#pragma unroll
          for (int q = 0; q < 5; ++q)
            if ((pend & (1u << q)) && bid[r.row[q]] == tid) {
              acc[r.row[q]] = __dadd_rn(acc[r.row[q]], t[q]);
              pend &= ~(1u << q);
              bid[r.row[q]] = 0x7fffffff;  // a member's rows are distinct: one reset each
            }
          __syncthreads();
        }
      } else {  // a long column in this batch: members one by one, in order
        const int cnt = (int)min((uint64_t)kEllSkT, e1 - eb);
        for (int q = 0; q < cnt; ++q) {
          __syncthreads();
          if (tid == q) sb = (int)c;  // broadcast the member code
          __syncthreads();
          const uint32_t cq = (uint32_t)sb;
          const int64_t j = (int64_t)(cq & 0x7FFFFFFFu) / s;
          const double vq = (cq & 0x80000000u) ? -vmag : vmag;
          const double dj = d[j];
          const int64_t a0 = colptr[j], a1 = colptr[j + 1];
          for (int64_t e = a0 + tid; e < a1; e += kEllSkT) {  // a column's rows are distinct
            const int row = rowidx[e];
            acc[row] = __dadd_rn(acc[row], __dmul_rn(__dmul_rn(av[e], dj), vq));
          }
        }
      }
    }
    __syncthreads();
    double* xr = X + (int64_t)b * ldx;
    for (int i = tid; i < m; i += kEllSkT) {
      xr[i] = acc[i];
      acc[i] = 0.0;
    }
  }
}

// ---- CSC A through ELL records, one counting sort by row per bucket (the
// default for 2048 < m <= ~40,000; the bid-round kernel above stays behind
// SKB_CSC_SKETCH_BIDS=1). Up to kRowsT * kRowsM members of a bucket at a time:
//   1. each thread loads its members' 64-byte records (all loads in flight
//      together), forms the terms t = fl(fl(A_ij d_j) v) in registers and
//      takes a ticket in its row with a packed-u16 shared atomic (count);
//   2. one block scan turns the counts into row offsets;
//   3. each term goes to slot offset(row) + ticket with its member index (the
//      order inside a row is arbitrary);
//   4. rows are summed straight into X (no accumulator in shared memory):
//      0 + t1 + t2 does not depend on the order of t1 and t2 (fl(0 + t) = t up
//      to the sign of zero, fl(a + b) = fl(b + a)), so rows with at most two
//      terms are summed at once, two rows per thread; rows with three or more
//      are queued and summed by one thread each in ascending member order.
// Every (row, bucket) sum is the ascending-j left-to-right fl-sum, bit-exact,
// with records read once and no rounds. Later chunks of a large bucket
// continue each row from X; a chunk holding a column longer than a record
// runs member by member on X in place.
constexpr int kRowsT = 768, kRowsM = 3;  // threads, members per thread
constexpr size_t kRowsSmemMax = 227 * 1024 - 1024;  // + the static shared words

static size_t rows_hard_entries(int m) {  // per-warp lists: every row a warp covers
  const size_t W = (size_t)(m + 1) / 2;
  return (size_t)(kRowsT / 32) * ((W + kRowsT - 1) / kRowsT) * 64;
}
static size_t rows_fixed_bytes(int m) {
  const size_t words = (size_t)(m + 1) / 2 + 1;
  return ((words * 4 + 15) & ~(size_t)15) + ((rows_hard_entries(m) * 2 + 15) & ~(size_t)15);
}
constexpr int kRowsCap = kRowsT * kRowsM * 5;  // terms per chunk (< 2^16)
static size_t rows_smem_bytes(int m) { return rows_fixed_bytes(m) + (size_t)kRowsCap * 10; }
SKB_DEV int half16(uint32_t wv, int r) { return (int)((wv >> ((r & 1) * 16)) & 0xFFFFu); }
SKB_DEV uint32_t row_inc(int r) { return 1u << ((r & 1) * 16); }

__global__ void __launch_bounds__(kRowsT, 1)
    csc_sketch_rows_kernel(const SkEll* __restrict__ ell, const int64_t* __restrict__ colptr,
                           const int32_t* __restrict__ rowidx, const double* __restrict__ av,
                           const uint64_t* __restrict__ start, const int32_t* __restrict__ mem_e,
                           double vmag, int s, int w, int m, unsigned int* __restrict__ counter,
                           double* __restrict__ X, int64_t ldx) {
  extern __shared__ __align__(16) unsigned char rs_sm[];
  const int W = (m + 1) / 2;
  uint32_t* offw = reinterpret_cast<uint32_t*>(rs_sm);  // row r: half (r & 1) of word r >> 1
  uint16_t* hard = reinterpret_cast<uint16_t*>(rs_sm + (((size_t)(W + 1) * 4 + 15) & ~(size_t)15));
  const int hcap = ((W + kRowsT - 1) / kRowsT) * 64;  // this warp's list capacity
  double* Sv = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(hard) +
                                         (((size_t)(kRowsT / 32) * hcap * 2 + 15) & ~(size_t)15));
  uint16_t* Sm = reinterpret_cast<uint16_t*>(Sv + kRowsCap);
  __shared__ int s_b;
  __shared__ int s_wtot[32];
  const unsigned FULL = 0xffffffffu;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kNW = kRowsT / 32;
  constexpr int cm = kRowsT * kRowsM;  // members per chunk
  for (;;) {
    __syncthreads();  // the previous bucket is done with offw / hard / S
    if (tid == 0) s_b = (int)atomicAdd(counter, 1u);
    __syncthreads();
    const int b = s_b;
    if (b >= w) break;
    const uint64_t e0 = start[b], e1 = start[b + 1];
    double* xb = X + (int64_t)b * ldx;
    const int64_t nmem = (int64_t)(e1 - e0);
    if (nmem == 0) {
      for (int r = tid; r < m; r += kRowsT) xb[r] = 0.0;
      continue;
    }
    for (int64_t c0 = 0; c0 < nmem; c0 += cm) {
      const int nc = (int)min((int64_t)cm, nmem - c0);
      const bool first = c0 == 0;
      const int32_t* mc = mem_e + e0 + c0;
      for (int i = tid; i <= W; i += kRowsT) offw[i] = 0u;
      // ---- 1. records (member i = tid + k * kRowsT), terms and tickets in registers
      SkEll rec[kRowsM];
      uint32_t code[kRowsM];
      bool has[kRowsM];
      bool lng = false;
#pragma unroll
      for (int k = 0; k < kRowsM; ++k) {
        const int i = tid + k * kRowsT;
        has[k] = i < nc;
        code[k] = has[k] ? (uint32_t)mc[i] : 0u;
      }
#pragma unroll
      for (int k = 0; k < kRowsM; ++k)
        if (has[k]) rec[k] = ell[(int64_t)(code[k] & 0x7FFFFFFFu) / s];
#pragma unroll
      for (int k = 0; k < kRowsM; ++k) lng |= has[k] && rec[k].cnt > 5;
      __syncthreads();  // offw zeroed
      if (!__syncthreads_or(lng)) {
        uint32_t tk[kRowsM][5];  // row | ticket << 16 (0xFFFF: no term)
        double tv[kRowsM][5];
#pragma unroll
        for (int k = 0; k < kRowsM; ++k) {
          const double v = (code[k] & 0x80000000u) ? -vmag : vmag;
#pragma unroll
          for (int q = 0; q < 5; ++q) {
            tk[k][q] = 0xFFFFu;
            if (has[k] && q < rec[k].cnt) {
              const int row = rec[k].row[q];
              tk[k][q] = (uint32_t)row |
                         ((uint32_t)half16(atomicAdd(&offw[row >> 1], row_inc(row)), row) << 16);
              tv[k][q] = __dmul_rn(__dmul_rn(rec[k].val[q], rec[k].d), v);
            }
          }
        }
        __syncthreads();
        // ---- 2. exclusive scan of the counts (thread t owns a run of words)
        const int per = (W + kRowsT - 1) / kRowsT;
        const int w0 = min(W, tid * per), w1 = min(W, w0 + per);
        int sum = 0;
        for (int i = w0; i < w1; ++i) {
          const uint32_t v = offw[i];
          sum += (int)(v & 0xFFFFu) + (int)(v >> 16);
        }
        int inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(FULL, inc, o);
          if (lane >= o) inc += y;
        }
        if (lane == 31) s_wtot[warp] = inc;
        __syncthreads();
        const int wt = lane < kNW ? s_wtot[lane] : 0;
        int winc = wt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(FULL, winc, o);
          if (lane >= o) winc += y;
        }
        int run = __shfl_sync(FULL, winc - wt, warp) + inc - sum;
        for (int i = w0; i < w1; ++i) {
          const uint32_t v = offw[i];
          const uint32_t lo = (uint32_t)run;
          run += (int)(v & 0xFFFFu);
          offw[i] = lo | ((uint32_t)run << 16);
          run += (int)(v >> 16);
        }
        if (tid == kRowsT - 1) offw[W] = (uint32_t)run;  // end of the last row (m odd: half 0)
        __syncthreads();
        // ---- 3. terms to their slots
#pragma unroll
        for (int k = 0; k < kRowsM; ++k)
#pragma unroll
          for (int q = 0; q < 5; ++q)
            if (tk[k][q] != 0xFFFFu) {
              const int row = (int)(tk[k][q] & 0xFFFFu);
              const int slot = half16(offw[row >> 1], row) + (int)(tk[k][q] >> 16);
              Sv[slot] = tv[k][q];
              Sm[slot] = (uint16_t)(tid + k * kRowsT);
            }
        __syncthreads();
        // ---- 4. two rows per thread (word k = rows 2k, 2k+1; offw[W] = total);
        // order-free rows now, rows with more terms queued
        const int lim = first ? 2 : 1;
        uint16_t* hl = hard + warp * hcap;  // this warp's queued rows
        int nh = 0;
#pragma unroll 1
        for (int k0 = 0; k0 < W; k0 += kRowsT) {
          const int k = k0 + tid;
          bool q0 = false, q1 = false;
          if (k < W) {
            const uint32_t v = offw[k], vn = offw[k + 1];
            const int s0 = (int)(v & 0xFFFFu), s1 = (int)(v >> 16), en = (int)(vn & 0xFFFFu);
            const int n0 = s1 - s0, n1 = en - s1;  // row 2k + 1 = m (m odd): n1 = 0
            q0 = n0 > lim;
            q1 = n1 > lim;
            double* xp = xb + 2 * k;
            if (first) {  // hard rows get a placeholder here, their sum below
              double x0 = 0.0, x1 = 0.0;
              if (n0 >= 1 && !q0) x0 = __dadd_rn(x0, Sv[s0]);
              if (n0 == 2) x0 = __dadd_rn(x0, Sv[s0 + 1]);
              if (n1 >= 1 && !q1) x1 = __dadd_rn(x1, Sv[s1]);
              if (n1 == 2) x1 = __dadd_rn(x1, Sv[s1 + 1]);
              if (2 * k + 1 < m)
                *reinterpret_cast<double2*>(xp) = make_double2(x0, x1);
              else
                xp[0] = x0;
            } else {
              if (n0 == 1) xp[0] = __dadd_rn(xp[0], Sv[s0]);
              if (n1 == 1) xp[1] = __dadd_rn(xp[1], Sv[s1]);
            }
          }
          const unsigned m0 = __ballot_sync(FULL, q0), m1 = __ballot_sync(FULL, q1);
          const unsigned lt = (1u << lane) - 1u;
          if (q0) hl[nh + __popc(m0 & lt)] = (uint16_t)(2 * k);
          if (q1) hl[nh + __popc(m0) + __popc(m1 & lt)] = (uint16_t)(2 * k + 1);
          nh += __popc(m0) + __popc(m1);
        }
        __syncwarp();  // the placeholders above are overwritten by other lanes below
        // this warp's queued rows, one per lane, terms in ascending member order: a
        // sorting network over eight (member, term) pairs, selection beyond eight
        for (int k0 = 0; k0 < nh; k0 += 32) {
          const int k = k0 + lane;
          int r = 0, lo = 0, c = 0;
          if (k < nh) {
            r = hl[k];
            const uint32_t v = offw[r >> 1];
            lo = half16(v, r);
            const int hi = (r & 1) ? (int)(offw[(r >> 1) + 1] & 0xFFFFu) : (int)(v >> 16);
            c = hi - lo;
          }
          double x = 0.0;
          if (k < nh && !first) x = xb[r];
          if (__any_sync(FULL, c > 8)) {
            int prev = -1;
            for (int u = 0; u < c; ++u) {  // the next member in ascending order
              int best = 0x7FFFFFFF, bi = lo;
              for (int q = lo; q < lo + c; ++q) {
                const int mm = Sm[q];
                if (mm > prev && mm < best) {
                  best = mm;
                  bi = q;
                }
              }
              x = __dadd_rn(x, Sv[bi]);
              prev = best;
            }
          } else {
            int key[8];
            double val[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              key[q] = q < c ? (int)Sm[lo + q] : 0x10000 + q;
              val[q] = q < c ? Sv[lo + q] : 0.0;
            }
            // Batcher odd-even merge sort, 8 inputs (19 compare-exchanges)
            auto cx = [&](int a, int b) {
              const bool sw = key[a] > key[b];
              const int ka = key[a];
              const double va = val[a];
              key[a] = sw ? key[b] : key[a];
              val[a] = sw ? val[b] : val[a];
              key[b] = sw ? ka : key[b];
              val[b] = sw ? va : val[b];
            };
            cx(0, 1); cx(2, 3); cx(4, 5); cx(6, 7);
            cx(0, 2); cx(1, 3); cx(4, 6); cx(5, 7);
            cx(1, 2); cx(5, 6);
            cx(0, 4); cx(1, 5); cx(2, 6); cx(3, 7);
            cx(2, 4); cx(3, 5);
            cx(1, 2); cx(3, 4); cx(5, 6);
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (q < c) x = __dadd_rn(x, val[q]);
          }
          if (k < nh) xb[r] = x;
        }
      } else {
        // a column longer than a record: member by member, rows split, X in place
        if (first) {
          for (int r = tid; r < m; r += kRowsT) xb[r] = 0.0;
          __syncthreads();
        }
        for (int i = 0; i < nc; ++i) {
          const uint32_t cd = (uint32_t)mc[i];
          const int64_t j = (int64_t)(cd & 0x7FFFFFFFu) / s;
          const double v = (cd & 0x80000000u) ? -vmag : vmag;
          const double dj = ell[j].d;
          const int64_t a0 = colptr[j], a1 = colptr[j + 1];
          for (int64_t e = a0 + tid; e < a1; e += kRowsT) {  // a column's rows are distinct
            const int row = rowidx[e];
            xb[row] = __dadd_rn(xb[row], __dmul_rn(__dmul_rn(av[e], dj), v));
          }
          __syncthreads();
        }
      }
      __syncthreads();  // the next chunk reuses offw / S / hard and reads X
    }
  }
}
}  // namespace skb

extern "C" int skb_csc_sketch_apply(const int64_t* colptr, const int32_t* rowidx,
                                    const double* av, void* ell, int64_t m, int64_t n,
                                    const double* d, const int32_t* cols, const double* vals,
                                    int32_t s, int32_t w, double* X, int64_t ldx,
                                    void* workspace, size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (m < 1 || ldx < m || s < 1 || w < 1) return SKB_ERR_ARG;
  skb_ws ws = skb_ws_make(workspace, ws_bytes);
  uint64_t* start;
  int32_t* mem_e;
  unsigned int* counter;
  int rc = bucket_sort(cols, vals, n, s, w, &ws, st, &start, &mem_e, &counter);
  if (rc) return rc;
  const bool use_ell = ell && m > 2048 && m <= 65535 && n > 0 && !getenv("SKB_CSC_SKETCH_L2");
  // s = 1 (500 members a bucket at c4): the bid-round kernel is faster
  // (2.93 vs 3.60 ms per c4 apply); s >= 2: the row-sorting kernel (s = 4:
  // 7.26 vs 7.71 ms), profiles/r02_csc_sketch_c4.txt
  // Each ELL kernel has a shared-memory ceiling in m (rows: ~27,000, bids: ~18,700);
  // beyond both the L2 kernel takes the sketch.
  const bool want_bids = getenv("SKB_CSC_SKETCH_BIDS") != nullptr || s == 1;
  const bool rows_ok = use_ell && !(ldx & 1) && rows_smem_bytes((int)m) <= kRowsSmemMax;
  const bool bids_ok = use_ell && (size_t)m * 12 <= 220 * 1024;
  if (rows_ok && !(want_bids && bids_ok)) {
    const size_t smem = rows_smem_bytes((int)m);
    static size_t conf_r = 0;
    if (smem > conf_r) {
      if (cudaFuncSetAttribute(csc_sketch_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem) != cudaSuccess)
        return SKB_ERR_UNSUPPORTED;
      conf_r = smem;
    }
    const double vmag = 1.0 / std::sqrt((double)s);  // as below
    ell_set_d_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>((SkEll*)ell, d, n);
    const int grid = std::min(skb_num_sms(), (int)w);
    csc_sketch_rows_kernel<<<grid, kRowsT, smem, st>>>((const SkEll*)ell, colptr, rowidx, av,
                                                       start, mem_e, vmag, s, w, (int)m, counter,
                                                       X, ldx);
    return skb_launch_status(__func__);
  }
  if (bids_ok) {
    const size_t smem = (size_t)m * 12;  // accumulator + bids
    static size_t conf_e = 0;
    if (smem > conf_e) {
      if (cudaFuncSetAttribute(csc_sketch_ell_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem) != cudaSuccess)
        return SKB_ERR_UNSUPPORTED;
      conf_e = smem;
    }
    // every hash value is +-1/sqrt(s) (skb_hash.cu: sign / sqrt(s), both correctly
    // rounded, so the host's IEEE quotient is the same double)
    const double vmag = 1.0 / std::sqrt((double)s);
    ell_set_d_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>((SkEll*)ell, d, n);
    const int grid = std::min(skb_num_sms(), (int)w);
    csc_sketch_ell_kernel<<<grid, kEllSkT, smem, st>>>((const SkEll*)ell, colptr, rowidx, av, d,
                                                       start, mem_e, vmag, s, w, (int)m, counter,
                                                       X, ldx);
    return skb_launch_status(__func__);
  }
  if (m > 2048 && !getenv("SKB_CSC_SKETCH_RMW")) {
    cudaMemsetAsync(X, 0, (size_t)w * ldx * 8, st);
    static const int l2cps = getenv("SKB_L2_CPS") ? atoi(getenv("SKB_L2_CPS")) : 2;
    const int grid = std::min(skb_num_sms() * l2cps, (int)((w + 3) / 4));
    csc_sketch_l2_kernel<<<grid, kL2Threads, 0, st>>>(colptr, rowidx, av, d, start, mem_e, vals,
                                                      s, w, X, ldx);
    return skb_launch_status(__func__);
  }
  if (m > 2048) {
    cudaMemsetAsync(X, 0, (size_t)w * ldx * 8, st);
    csc_sketch_rmw_kernel<1><<<(unsigned)((w + kRmwThreads - 1) / kRmwThreads), kRmwThreads, 0,
                               st>>>(colptr, rowidx, av, d, start, mem_e, vals, s, w, (int)m, X,
                                     ldx);
    return skb_launch_status(__func__);
  }
  const size_t smem = (size_t)m * 8 + 32 * kCscStage * 4 + 32 * 4 + 16 + 32 * kCscStage * 8;
  if (smem > 220 * 1024) return SKB_ERR_UNSUPPORTED;
  static size_t conf = 0;
  if (smem > 48 * 1024 && smem > conf) {
    if (cudaFuncSetAttribute(csc_sketch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return SKB_ERR_CUDA;
    conf = smem;
  }
  const int per_sm = std::max(1, (int)((220 * 1024) / smem));
  const int grid = std::min(skb_num_sms() * std::min(per_sm, 16), std::max(1, (int)w));
  csc_sketch_kernel<<<grid, 32, smem, st>>>(colptr, rowidx, av, (int)m, d, start, mem_e, vals, s,
                                            w, counter, X, ldx);
  return skb_launch_status(__func__);
}

// One launch of the bucket-streaming kernel over rows [0, m) of A / X (a slice).
static int sketch_slice(const double* A, int64_t lda, int64_t m, const double* d,
                        const uint64_t* start, const int32_t* mem_e, const double* vals, int s,
                        int w, unsigned int* counter, double* X, int64_t ldx, cudaStream_t st) {
  const size_t col_bytes = (size_t)(m + (m & 1)) * 8;
  // tuning knobs (development): CTAs per SM and ring depth
  // Two CTAs per SM (two producers per SM): 1.73 -> 1.32 ms at c2 (round-1 sweep).
  // CTAs (bulk-copy producers) per SM: 4 for m <= 1024 (c2 s = 4: 4.91 -> 4.72 ms with 6
  // stages each, s = 1: 1.289 -> 1.279 ms; sweep in profiles/r02_sketch_s4_analysis.txt),
  // 2 up to m = 2048, one CTA above (register budget)
  static const int cps_env = getenv("SKB_SKETCH_CPS") ? atoi(getenv("SKB_SKETCH_CPS")) : 0;
  const int ctas_per_sm = m > 2048 ? 1 : cps_env > 0 ? cps_env : (m <= 1024 ? 4 : 2);
  static const int max_stages = getenv("SKB_SKETCH_STAGES") ? atoi(getenv("SKB_SKETCH_STAGES")) : 16;
  const size_t budget = (size_t)(200 * 1024) / std::max(1, ctas_per_sm);
  int stages = (int)std::min<size_t>((size_t)max_stages, budget / col_bytes);
  stages = std::max(stages, 2);
  const size_t smem =
      (((size_t)stages * (16 + sizeof(StageMeta)) + 127) & ~(size_t)127) + stages * col_bytes;
  const int grid = std::min(skb_num_sms() * std::max(1, ctas_per_sm), (int)std::max(1, w));
  int rc = 0;
  // one configured-smem watermark per kernel instantiation
  static size_t conf[6] = {0, 0, 0, 0, 0, 0};
  auto launch = [&](auto kern, int which) {
    if (smem > conf[which]) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
          cudaSuccess)
        rc = SKB_ERR_CUDA;
      conf[which] = smem;
    }
    kern<<<grid, kConsumers + 32, smem, st>>>(A, lda, (int)m, d, start, mem_e, vals, s, w,
                                              stages, counter, X, ldx);
  };
  if (m <= 512)
    launch(sketch_accumulate_kernel<1>, 0);
  else if (m <= 1024)
    launch(sketch_accumulate_kernel<2>, 1);
  else if (m <= 2048)
    launch(sketch_accumulate_kernel<4>, 2);
  else if (m <= 4096)
    launch(sketch_accumulate_kernel<8>, 3);
  else if (m <= 8192)
    launch(sketch_accumulate_kernel<16>, 4);
  else
    launch(sketch_accumulate_kernel<32>, 5);
  return rc;
}

extern "C" int skb_sketch_apply(const double* A, int64_t m, int64_t n, int64_t lda,
                                const double* d, const int32_t* cols, const double* vals,
                                int32_t s, int32_t w, double* X, int64_t ldx, void* workspace,
                                size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (m < 1 || lda < m || (lda & 1) || ldx < m || (ldx & 1) || s < 1 || w < 1)
    return SKB_ERR_ARG;
  skb_ws ws = skb_ws_make(workspace, ws_bytes);
  uint64_t* start;
  int32_t* mem_e;
  unsigned int* counter;
  {
    int rc0 = bucket_sort(cols, vals, n, s, w, &ws, st, &start, &mem_e, &counter);
    if (rc0) return rc0;
  }
  // Rows are independent sums: past two staged columns per ring (m > ~12,800) the
  // sketch runs over 8192-row slices of A and X (the same chains, bit-exact).
  const int64_t m_full = m;
  const bool sliced = (size_t)2 * (m + (m & 1)) * 8 + 256 > (size_t)200 * 1024;
  const int64_t ms_max = sliced ? 8192 : m;
  int rc = 0;
  for (int64_t r0 = 0; r0 < m_full && !rc; r0 += ms_max) {
    const int64_t ms = std::min<int64_t>(ms_max, m_full - r0);
    if (r0 > 0) cudaMemsetAsync(counter, 0, 16, st);  // the bucket counter, per launch
    rc = sketch_slice(A + r0, lda, ms, d, start, mem_e, vals, s, w, counter, X + r0, ldx, st);
  }
  if (rc) return rc;
  return skb_launch_status(__func__);
}

extern "C" int skb_scale_columns(const double* A, int64_t m, int64_t n, int64_t lda,
                                 const double* d, double* X, int64_t ldx, void* stream) {
  if (n <= 0) return 0;
  scale_columns_kernel<<<(unsigned)n, 128, 0, (cudaStream_t)stream>>>(A, lda, (int)m, n, d, X,
                                                                      ldx);
  return skb_launch_status(__func__);
}

extern "C" int skb_sketch_gather(const int32_t* cols, const double* vals, int32_t s, int64_t n,
                                 const double* u, const double* x, const double* sv, double* v,
                                 void* stream) {
  if (n <= 0) return 0;
  sketch_gather_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      cols, vals, s, n, u, x, sv, v);
  return skb_launch_status(__func__);
}
