// K9: the dense Gaussian sketch W, bit-exact with numpy's standard_normal.
//
// Replaces build_gaussian_sketch (reference sketching.py:131-139):
//   W = Generator(Philox(seed)).standard_normal((n, w)) / sqrt(w)
// numpy draws N(0,1) with a 256-layer ziggurat over 64-bit Philox outputs.
// An attempt at stream position q reads word q: idx = low 8 bits, then a sign
// bit and a 52-bit magnitude rabs; if rabs < ki[idx] (99.3%) it returns
// rabs * wi[idx] (signed). Otherwise it reads further words: the wedge test
// (one uniform, accept or restart at q + 2) or, for idx == 0, the tail loop
// (two uniforms per round). Attempt lengths vary, so draw k's position
// depends on every earlier slow attempt: a sequential recurrence.
//
// B200 mapping: positions are tiled (4096 per CTA). Each thread classifies 16
// positions (fast/slow) from its Philox blocks; one walker thread per tile
// resolves the rare slow attempts in order, starting from a provably visited
// anchor (a position preceded by 64 fast positions is always an attempt start
// when every attempt is <= 64 words, which is checked), and marks the words
// they consume. Accepted draws are then compacted with a tile-count scan, as
// for the Lemire hashes. The tables come from numpy's own build
// (ziggurat_tables.py -> generated header).
#include "skb_common.cuh"
#include "skb_internal.h"
#include "skb_ziggurat_tables.h"

namespace skb {

constexpr int kZThreads = 256;
constexpr int kZPer = 16;
constexpr int kZTile = kZThreads * kZPer;  // 4096 positions
constexpr int kZMaxLen = 64;
constexpr double kZigR = 3.6541528853610088;      // numpy ziggurat_nor_r
constexpr double kZigInvR = 0.27366123732975828;  // numpy ziggurat_nor_inv_r

SKB_DEV uint64_t zig_ki(int i) { return zig_ki_double_bits[i]; }
SKB_DEV double zig_wi(int i) { return __longlong_as_double((long long)zig_wi_double_bits[i]); }
SKB_DEV double zig_fi(int i) { return __longlong_as_double((long long)zig_fi_double_bits[i]); }

SKB_DEV uint64_t out64(uint64_t k0, uint64_t k1, uint64_t q) {
  const u64x4 o = philox4x64_10((q >> 2) + 1, 0, 0, 0, k0, k1);
  return o.v[q & 3];
}

SKB_DEV double to_unit(uint64_t r) {  // numpy next_double
  return (double)(r >> 11) * (1.0 / 9007199254740992.0);
}

SKB_DEV bool zig_fast(uint64_t r) {
  const int idx = (int)(r & 0xff);
  const uint64_t rabs = (r >> 9) & 0x000fffffffffffffULL;
  return rabs < zig_ki(idx);
}

SKB_DEV double zig_fast_value(uint64_t r) {
  const int idx = (int)(r & 0xff);
  const uint64_t rabs = (r >> 9) & 0x000fffffffffffffULL;
  const double x = __dmul_rn((double)rabs, zig_wi(idx));
  return ((r >> 8) & 1) ? -x : x;
}

// A slow attempt starting at q (word r): -> accepted?, value, length in words.
SKB_DEV bool zig_slow(uint64_t k0, uint64_t k1, uint64_t q, uint64_t r, double* val, int* len) {
  const int idx = (int)(r & 0xff);
  const uint64_t rabs = (r >> 9) & 0x000fffffffffffffULL;
  double x = __dmul_rn((double)rabs, zig_wi(idx));
  if ((r >> 8) & 1) x = -x;
  if (idx == 0) {
    uint64_t p = q + 1;
    for (;;) {
      const double u1 = to_unit(out64(k0, k1, p)), u2 = to_unit(out64(k0, k1, p + 1));
      p += 2;
      const double xx = __dmul_rn(-kZigInvR, log1p(-u1));
      const double yy = -log1p(-u2);
      if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
        *val = ((rabs >> 8) & 1) ? -__dadd_rn(kZigR, xx) : __dadd_rn(kZigR, xx);
        *len = (int)(p - q);
        return true;
      }
      if (p - q > (uint64_t)kZMaxLen) {  // flagged by the caller (len > max)
        *len = kZMaxLen + 1;
        return false;
      }
    }
  }
  const double u = to_unit(out64(k0, k1, q + 1));
  const double lhs =
      __dadd_rn(__dmul_rn(__dsub_rn(zig_fi(idx - 1), zig_fi(idx)), u), zig_fi(idx));
  *len = 2;
  if (lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x))) {
    *val = x;
    return true;
  }
  return false;
}

// One tile of positions [t0, t0 + 4096). emit == 0: write the tile's draw
// count; emit == 1: write draws (value / sqrtw) at tile_off[tile] + rank.
__global__ void __launch_bounds__(kZThreads)
    gauss_tile_kernel(uint64_t k0, uint64_t k1, int emit, const uint64_t* __restrict__ tile_off,
                      uint64_t lo, uint64_t need, double sqrtw, double* __restrict__ out,
                      uint32_t* __restrict__ tile_cnt, int* __restrict__ err) {
  __shared__ uint32_t slow_bits[kZTile / 32];
  __shared__ uint32_t skip_bits[kZTile / 32];
  __shared__ uint32_t acc_bits[kZTile / 32];  // accepted slow attempts
  __shared__ double slow_val[kZTile];
  __shared__ uint32_t scan[kZThreads];
  const int tid = threadIdx.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * kZTile;
  const uint64_t my0 = t0 + (uint64_t)tid * kZPer;
  uint64_t r[kZPer];
#pragma unroll
  for (int b = 0; b < kZPer / 4; ++b) {
    const u64x4 o = philox4x64_10(((my0 >> 2) + b) + 1, 0, 0, 0, k0, k1);
#pragma unroll
    for (int i = 0; i < 4; ++i) r[4 * b + i] = o.v[i];
  }
  uint32_t mask = 0;
#pragma unroll
  for (int i = 0; i < kZPer; ++i) mask |= zig_fast(r[i]) ? 0u : (1u << i);
  const uint32_t other = __shfl_xor_sync(0xffffffffu, mask, 1);
  if ((tid & 1) == 0) slow_bits[tid >> 1] = mask | (other << 16);
  if (tid < kZTile / 32) {
    skip_bits[tid] = 0;
    acc_bits[tid] = 0;
  }
  __syncthreads();

  if (tid == 0) {  // ---- walker
    // anchor: the latest a <= t0 whose 64 predecessors are all fast (a = 0 at the start)
    uint64_t pre[kZMaxLen];
    int npre = 0, run = 0;
    uint64_t a = 0;
    bool anchored = (t0 == 0);
    for (uint64_t p = t0; p > 0 && !anchored;) {
      --p;
      if (zig_fast(out64(k0, k1, p))) {
        if (++run == kZMaxLen) {
          a = p + kZMaxLen;
          anchored = true;
        }
      } else {
        run = 0;
        if (npre < kZMaxLen) pre[npre++] = p;  // slow positions in (a, t0), newest first
        else {
          atomicOr(err, 2);
          break;
        }
      }
      if (p == 0 && !anchored) {
        a = 0;
        anchored = true;
      }
    }
    // walk the slow positions of [a, t0) in ascending order
    uint64_t next_free = a;
    for (int k = npre - 1; k >= 0; --k) {
      const uint64_t s = pre[k];
      if (s < a || s < next_free) continue;
      double v;
      int len;
      zig_slow(k0, k1, s, out64(k0, k1, s), &v, &len);
      if (len > kZMaxLen) atomicOr(err, 1);
      next_free = s + len;
    }
    for (uint64_t p = t0; p < next_free && p < t0 + kZTile; ++p)
      skip_bits[(p - t0) >> 5] |= 1u << ((p - t0) & 31);
    // the tile's slow positions in order
    for (int wd = 0; wd < kZTile / 32; ++wd) {
      uint32_t bits = slow_bits[wd];
      while (bits) {
        const int bpos = __ffs(bits) - 1;
        bits &= bits - 1;
        const uint64_t s = t0 + (uint64_t)(wd * 32 + bpos);
        if (s < next_free) continue;  // consumed by an earlier slow attempt
        double v = 0.0;
        int len;
        const bool ok = zig_slow(k0, k1, s, out64(k0, k1, s), &v, &len);
        if (len > kZMaxLen) atomicOr(err, 1);
        if (ok) {
          acc_bits[wd] |= 1u << bpos;
          slow_val[wd * 32 + bpos] = v;
        }
        for (uint64_t p = s + 1; p < s + len && p < t0 + kZTile; ++p)
          skip_bits[(p - t0) >> 5] |= 1u << ((p - t0) & 31);
        next_free = s + len;
      }
    }
  }
  __syncthreads();

  const uint32_t sk = (skip_bits[tid >> 1] >> ((tid & 1) * 16)) & 0xffffu;
  const uint32_t ac = (acc_bits[tid >> 1] >> ((tid & 1) * 16)) & 0xffffu;
  const uint32_t outm = ((~mask & 0xffffu) & ~sk) | ac;  // visited fast | accepted slow
  const uint32_t c = __popc(outm);
  scan[tid] = c;
  __syncthreads();
  for (int off = 1; off < kZThreads; off <<= 1) {
    const uint32_t t = tid >= off ? scan[tid - off] : 0;
    __syncthreads();
    scan[tid] += t;
    __syncthreads();
  }
  if (!emit) {
    if (tid == kZThreads - 1) tile_cnt[blockIdx.x] = scan[tid];
    return;
  }
  uint64_t idx = tile_off[blockIdx.x] + scan[tid] - c;
#pragma unroll
  for (int i = 0; i < kZPer; ++i) {
    if (outm & (1u << i)) {
      if (idx >= lo && idx < need) {
        const double v = (ac & (1u << i)) ? slow_val[tid * kZPer + i] : zig_fast_value(r[i]);
        out[idx - lo] = __ddiv_rn(v, sqrtw);
      }
      ++idx;
    }
  }
}

__global__ void scan_tiles_kernel(const uint32_t* in, uint64_t* out, int n, uint64_t* total) {
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
  if (threadIdx.x == 0) *total = carry;
}

}  // namespace skb

using namespace skb;

// W = draws [lo, count) of standard_normal / sqrt(w) (row-major n x w when
// lo = 0, count = n*w; a rank's row block with lo = j0*w, count = j1*w).
// Synchronises the stream (tile count check).
extern "C" int skb_gaussian_sketch(uint64_t key0, uint64_t key1, int64_t lo, int64_t count,
                                   int32_t w, double* W, void* workspace, size_t ws_bytes,
                                   void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (count < 0 || lo < 0 || lo > count || w < 1) return SKB_ERR_ARG;
  if (count == lo) return 0;
  skb_ws ws = skb_ws_make(workspace, ws_bytes);
  const double sqrtw = __builtin_sqrt((double)w);
  uint64_t positions = (uint64_t)count + (uint64_t)count / 64 + 4 * kZTile;
  for (int attempt = 0; attempt < 4; ++attempt) {
    const uint64_t tiles = (positions + kZTile - 1) / kZTile;
    if (tiles > 0x7fffffffULL) return SKB_ERR_UNSUPPORTED;
    const size_t mark = ws.off;
    uint32_t* cnt = (uint32_t*)skb_ws_take(&ws, tiles * 4);
    uint64_t* off = (uint64_t*)skb_ws_take(&ws, tiles * 8);
    uint64_t* tot = (uint64_t*)skb_ws_take(&ws, 16);
    int* err = (int*)skb_ws_take(&ws, 16);
    if (!cnt || !off || !tot || !err) return SKB_ERR_WORKSPACE;
    cudaMemsetAsync(err, 0, 16, st);
    gauss_tile_kernel<<<(unsigned)tiles, kZThreads, 0, st>>>(key0, key1, 0, nullptr, 0, 0,
                                                             sqrtw, nullptr, cnt, err);
    scan_tiles_kernel<<<1, 1024, 0, st>>>(cnt, off, (int)tiles, tot);
    gauss_tile_kernel<<<(unsigned)tiles, kZThreads, 0, st>>>(key0, key1, 1, off, (uint64_t)lo,
                                                             (uint64_t)count, sqrtw, W, cnt, err);
    uint64_t total = 0;
    int herr = 0;
    cudaMemcpyAsync(&total, tot, 8, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return SKB_ERR_CUDA;
    ws.off = mark;
    if (herr) return SKB_ERR_INTERNAL;  // an attempt longer than 64 words (never observed)
    if (total >= (uint64_t)count) return skb_launch_status(__func__);
    positions *= 2;
  }
  return SKB_ERR_INTERNAL;
}

extern "C" size_t skb_gaussian_workspace_bytes(int64_t count) {
  const uint64_t tiles = ((uint64_t)count * 2 + 8 * kZTile) / kZTile + 1;
  return (size_t)tiles * 12 + 4096;
}
