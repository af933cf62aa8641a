// K1: sparse-sign sketch hashes, bit-exact with numpy's Philox stream.
//
// Replaces build_sparse_embedding (reference sketching.py:93-119):
//   cols = rng.integers(0, w, (n, s)); duplicate rows redrawn; signs drawn after.
// The 32-bit word stream is W_q = half (q&1) of Philox4x64-10 output q>>1,
// block counter (q>>3)+1 (numpy counter pre-increment). A bounded draw in
// [0, w) takes the next word with lo32(W*w) >= (2^32 - w) mod w (Lemire) and
// returns hi32(W*w). Acceptance depends only on the word, so the draw is a
// stream compaction: flag, count per tile, scan tile counts, emit.
#include "skb_common.cuh"
#include "skb_internal.h"

namespace skb {

constexpr int kHashThreads = 256;           // one Philox block (8 words) per thread
constexpr int kWordsPerTile = kHashThreads * 8;

SKB_DEV void words8(uint64_t blk, uint64_t k0, uint64_t k1, uint32_t w[8]) {
  u64x4 o = philox4x64_10(blk + 1, 0, 0, 0, k0, k1);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    w[2 * i] = (uint32_t)o.v[i];
    w[2 * i + 1] = (uint32_t)(o.v[i] >> 32);
  }
}

// Count accepted words of each tile. Words [q0, q1) are eligible.
__global__ void lemire_count_kernel(uint64_t k0, uint64_t k1, uint64_t q0, uint64_t q1,
                                    uint32_t bound, uint32_t thr, uint32_t* tile_cnt) {
  __shared__ double buf[32];
  const uint64_t blk = (q0 >> 3) + (uint64_t)blockIdx.x * kHashThreads + threadIdx.x;
  uint32_t w[8];
  words8(blk, k0, k1, w);
  int c = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint64_t q = blk * 8 + i;
    const uint64_t prod = (uint64_t)w[i] * bound;
    c += (q >= q0 && q < q1 && (uint32_t)prod >= thr) ? 1 : 0;
  }
  const double tot = block_sum((double)c, buf);
  if (threadIdx.x == 0) tile_cnt[blockIdx.x] = (uint32_t)tot;
}

// Exclusive scan of tile counts (single CTA, fixed order). Also writes the total.
__global__ void scan_u32_kernel(const uint32_t* in, uint64_t* out, int n, uint64_t* total) {
  __shared__ uint64_t part[1024];
  __shared__ uint64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < n; base += 1024) {
    const int i = base + threadIdx.x;
    uint64_t v = i < n ? in[i] : 0;
    part[threadIdx.x] = v;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
      uint64_t t = threadIdx.x >= off ? part[threadIdx.x - off] : 0;
      __syncthreads();
      part[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < n) out[i] = carry + part[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += part[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

// Emit the first `need` accepted draws; record words consumed (relative to q0).
__global__ void lemire_emit_kernel(uint64_t k0, uint64_t k1, uint64_t q0, uint64_t q1,
                                   uint32_t bound, uint32_t thr, const uint64_t* tile_off,
                                   uint64_t need, uint32_t* out, uint64_t* consumed) {
  __shared__ uint32_t sc[kHashThreads];
  const uint64_t blk = (q0 >> 3) + (uint64_t)blockIdx.x * kHashThreads + threadIdx.x;
  uint32_t w[8];
  words8(blk, k0, k1, w);
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint64_t q = blk * 8 + i;
    const uint64_t prod = (uint64_t)w[i] * bound;
    acc |= (q >= q0 && q < q1 && (uint32_t)prod >= thr) ? (1u << i) : 0u;
  }
  const uint32_t c = __popc(acc);
  sc[threadIdx.x] = c;
  __syncthreads();
  for (int off = 1; off < kHashThreads; off <<= 1) {  // inclusive scan
    uint32_t t = threadIdx.x >= off ? sc[threadIdx.x - off] : 0;
    __syncthreads();
    sc[threadIdx.x] += t;
    __syncthreads();
  }
  uint64_t idx = tile_off[blockIdx.x] + sc[threadIdx.x] - c;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (acc & (1u << i)) {
      if (idx < need) {
        out[idx] = (uint32_t)(((uint64_t)w[i] * bound) >> 32);
        if (idx == need - 1) *consumed = blk * 8 + i + 1 - q0;
      }
      ++idx;
    }
  }
}

// Duplicate detection per row (s small): flag rows that repeat a bucket.
__global__ void dup_flag_kernel(const uint32_t* cols, int64_t nrows, int s, const int64_t* rows,
                                uint32_t* flag) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const int64_t row = rows ? rows[r] : r;
  const uint32_t* c = cols + row * s;
  uint32_t f = 0;
  for (int a = 0; a < s && !f; ++a)
    for (int b = a + 1; b < s; ++b)
      if (c[a] == c[b]) {
        f = 1;
        break;
      }
  flag[r] = f;
}

// Stable compaction of indices with flag != 0: tile counts -> scan -> emit.
__global__ void flag_count_kernel(const uint32_t* flag, int64_t n, uint32_t* tile_cnt) {
  __shared__ double buf[32];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const double c = (i < n && flag[i]) ? 1.0 : 0.0;
  const double t = block_sum(c, buf);
  if (threadIdx.x == 0) tile_cnt[blockIdx.x] = (uint32_t)t;
}

__global__ void flag_emit_kernel(const uint32_t* flag, int64_t n, const uint64_t* tile_off,
                                 const int64_t* rows, int64_t* out) {
  __shared__ uint32_t sc[1024];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t c = (i < n && flag[i]) ? 1u : 0u;
  sc[threadIdx.x] = c;
  __syncthreads();
  for (int off = 1; off < (int)blockDim.x; off <<= 1) {
    uint32_t t = threadIdx.x >= off ? sc[threadIdx.x - off] : 0;
    __syncthreads();
    sc[threadIdx.x] += t;
    __syncthreads();
  }
  if (c) out[tile_off[blockIdx.x] + sc[threadIdx.x] - 1] = rows ? rows[i] : i;
}

__global__ void scatter_rows_kernel(const uint32_t* vals, const int64_t* rows, int64_t nrows,
                                    int s, uint32_t* cols) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nrows * s) return;
  const int64_t r = e / s;
  cols[rows[r] * s + (e - r * s)] = vals[e];
}

// Signs: Lemire with bound 2 never rejects; sign = 2*(W>>31) - 1, val = sign/sqrt(s).
// One thread per Philox block (8 consecutive 32-bit words): one Philox call for
// its 8 signs (one call per sign computed the same block 8 times over), and
// sign / sqrt(s) = +-(1 / sqrt(s)) exactly, so the quotient is formed once.
__global__ void sign_kernel(uint64_t k0, uint64_t k1, uint64_t q0, int64_t cnt, int s,
                            double* vals) {
  const uint64_t blk = (q0 >> 3) + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t qa = blk * 8 > q0 ? blk * 8 : q0;
  const uint64_t qe = q0 + (uint64_t)cnt, qb = blk * 8 + 8 < qe ? blk * 8 + 8 : qe;
  if (qa >= qb) return;
  const u64x4 o = philox4x64_10(blk + 1, 0, 0, 0, k0, k1);
  const double vmag = __ddiv_rn(1.0, __dsqrt_rn((double)s));
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const uint64_t q = blk * 8 + u;
    if (q >= qa && q < qb) {
      const uint64_t v = o.v[u >> 1];
      const uint32_t wd = (u & 1) ? (uint32_t)(v >> 32) : (uint32_t)v;
      vals[q - q0] = (wd >> 31) ? vmag : -vmag;
    }
  }
}

// 2s >= w branch: cols[j] = argsort(random((n, w))[j])[:s]. next_double =
// (out64 >> 11) * 2^-53 from 64-bit outputs j*w + c. Selection by repeated
// minimum (values distinct with probability 1 - O(w^2 2^-53)). Small w only.
SKB_DEV double philox_double(uint64_t k0, uint64_t k1, uint64_t k) {
  u64x4 o = philox4x64_10((k >> 2) + 1, 0, 0, 0, k0, k1);
  return (double)(o.v[k & 3] >> 11) * (1.0 / 9007199254740992.0);
}

__global__ void argsort_select_kernel(uint64_t k0, uint64_t k1, int64_t n, int w, int s,
                                      uint32_t* cols) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double prev = -1.0;
  for (int r = 0; r < s; ++r) {
    double best = 2.0;
    int bi = 0;
    for (int c = 0; c < w; ++c) {
      const double v = philox_double(k0, k1, (uint64_t)j * w + c);
      if (v > prev && v < best) {
        best = v;
        bi = c;
      }
    }
    cols[j * s + r] = (uint32_t)bi;
    prev = best;
  }
}

}  // namespace skb

using namespace skb;

// ---------------------------------------------------------------- host side

static inline uint32_t lemire_threshold(uint32_t bound) {
  return (uint32_t)((0x100000000ULL - bound) % bound);
}

// Draw `cnt` bounded integers in [0, bound) from word position *pos.
// Workspace: tiles*(4+8) + 16 bytes. Synchronises the stream.
static int lemire_draw(uint64_t k0, uint64_t k1, uint64_t* pos, uint32_t bound, uint64_t cnt,
                       uint32_t* out, skb_ws* ws, cudaStream_t st) {
  if (cnt == 0) return 0;
  const uint32_t thr = lemire_threshold(bound);
  const double prej = (double)thr / 4294967296.0;
  uint64_t margin = 64 + (uint64_t)(cnt * prej * 4.0) + (uint64_t)(8.0 * sqrt(cnt * prej + 1.0));
  for (int attempt = 0; attempt < 8; ++attempt) {
    const uint64_t q0 = *pos, q1 = q0 + cnt + margin;
    const uint64_t blk0 = q0 >> 3, blk1 = (q1 + 7) >> 3;
    const uint64_t tiles = (blk1 - blk0 + kHashThreads - 1) / kHashThreads;
    const size_t mark = ws->off;
    uint32_t* tile_cnt = (uint32_t*)skb_ws_take(ws, tiles * 4);
    uint64_t* tile_off = (uint64_t*)skb_ws_take(ws, tiles * 8);
    uint64_t* scal = (uint64_t*)skb_ws_take(ws, 16);
    if (!tile_cnt || !tile_off || !scal) return SKB_ERR_WORKSPACE;
    lemire_count_kernel<<<(unsigned)tiles, kHashThreads, 0, st>>>(k0, k1, q0, q1, bound, thr,
                                                                  tile_cnt);
    scan_u32_kernel<<<1, 1024, 0, st>>>(tile_cnt, tile_off, (int)tiles, scal);
    cudaMemsetAsync(scal + 1, 0xff, 8, st);
    lemire_emit_kernel<<<(unsigned)tiles, kHashThreads, 0, st>>>(k0, k1, q0, q1, bound, thr,
                                                                 tile_off, cnt, out, scal + 1);
    uint64_t h[2];
    skb_readback rb(st);
    rb.add(h, scal, 16);
    cudaError_t e = rb.sync();
    ws->off = mark;
    if (e != cudaSuccess) return SKB_ERR_CUDA;
    if (h[0] >= cnt) {
      *pos = q0 + h[1];
      return 0;
    }
    margin *= 4;
  }
  return SKB_ERR_INTERNAL;
}

static int compact_flags(const uint32_t* flag, int64_t n, const int64_t* rows, int64_t* out,
                         int64_t* count, skb_ws* ws, cudaStream_t st) {
  const int64_t tiles = (n + 1023) / 1024;
  const size_t mark = ws->off;
  uint32_t* tc = (uint32_t*)skb_ws_take(ws, tiles * 4);
  uint64_t* to = (uint64_t*)skb_ws_take(ws, tiles * 8);
  uint64_t* tot = (uint64_t*)skb_ws_take(ws, 8);
  if (!tc || !to || !tot) return SKB_ERR_WORKSPACE;
  flag_count_kernel<<<(unsigned)tiles, 1024, 0, st>>>(flag, n, tc);
  scan_u32_kernel<<<1, 1024, 0, st>>>(tc, to, (int)tiles, tot);
  flag_emit_kernel<<<(unsigned)tiles, 1024, 0, st>>>(flag, n, to, rows, out);
  uint64_t h = 0;
  skb_readback rb(st);
  rb.add(&h, tot, 8);
  cudaError_t e = rb.sync();
  ws->off = mark;
  if (e != cudaSuccess) return SKB_ERR_CUDA;
  *count = (int64_t)h;
  return 0;
}

extern "C" int skb_lemire_draw(uint64_t key0, uint64_t key1, uint64_t word_offset,
                               uint32_t bound, uint64_t count, uint32_t* out,
                               uint64_t* words_used, void* workspace, size_t ws_bytes,
                               void* stream) {
  if (bound == 0) return SKB_ERR_ARG;
  skb_ws ws = skb_ws_make(workspace, ws_bytes);
  uint64_t pos = word_offset;
  int rc = lemire_draw(key0, key1, &pos, bound, count, out, &ws, (cudaStream_t)stream);
  if (words_used) *words_used = pos - word_offset;
  return rc;
}

extern "C" int skb_sparse_embedding(uint64_t key0, uint64_t key1, int64_t n, int32_t w,
                                    int32_t s, int32_t* cols, double* vals,
                                    uint64_t* words_used, void* workspace, size_t ws_bytes,
                                    void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (s < 1 || s > w || (int64_t)w > n * (int64_t)s) return SKB_ERR_DIMS;
  skb_ws ws = skb_ws_make(workspace, ws_bytes);
  uint32_t* ucols = (uint32_t*)cols;
  uint64_t pos = 0;
  if (2 * (int64_t)s >= w) {
    argsort_select_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(key0, key1, n, w, s,
                                                                       ucols);
    pos = 2ull * (uint64_t)n * (uint64_t)w;  // n*w 64-bit outputs consumed by random()
  } else {
    int rc = lemire_draw(key0, key1, &pos, (uint32_t)w, (uint64_t)n * s, ucols, &ws, st);
    if (rc) return rc;
    if (s > 1) {
      // duplicate-row redraw rounds (sketching.py:110-115)
      uint32_t* flag = (uint32_t*)skb_ws_take(&ws, (size_t)n * 4);
      int64_t* rows = (int64_t*)skb_ws_take(&ws, (size_t)n * 8);
      int64_t* rows2 = (int64_t*)skb_ws_take(&ws, (size_t)n * 8);
      uint32_t* tmp = (uint32_t*)skb_ws_take(&ws, (size_t)n * s * 4);
      if (!flag || !rows || !rows2 || !tmp) return SKB_ERR_WORKSPACE;
      const int64_t* cand = nullptr;  // first round: all rows
      int64_t ncand = n;
      for (;;) {
        dup_flag_kernel<<<(unsigned)((ncand + 255) / 256), 256, 0, st>>>(ucols, ncand, s, cand,
                                                                         flag);
        int64_t nd = 0;
        rc = compact_flags(flag, ncand, cand, rows, &nd, &ws, st);
        if (rc) return rc;
        if (nd == 0) break;
        rc = lemire_draw(key0, key1, &pos, (uint32_t)w, (uint64_t)nd * s, tmp, &ws, st);
        if (rc) return rc;
        scatter_rows_kernel<<<(unsigned)((nd * s + 255) / 256), 256, 0, st>>>(tmp, rows, nd, s,
                                                                             ucols);
        // only redrawn rows can still hold duplicates
        cudaMemcpyAsync(rows2, rows, (size_t)nd * 8, cudaMemcpyDeviceToDevice, st);
        cand = rows2;
        ncand = nd;
      }
    }
  }
  const int64_t cnt = n * (int64_t)s;
  if (cnt > 0) {
    const int64_t nblk = (int64_t)(((pos + (uint64_t)cnt - 1) >> 3) - (pos >> 3)) + 1;
    sign_kernel<<<(unsigned)((nblk + 255) / 256), 256, 0, st>>>(key0, key1, pos, cnt, s, vals);
  }
  pos += (uint64_t)cnt;
  if (words_used) *words_used = pos;
  return skb_launch_status(__func__);
}
