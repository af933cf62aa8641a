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
// B200 mapping (one pass, persistent CTAs, tiles of 4096 positions taken in
// ticket order): each thread draws and classifies 16 words; the rare slow
// attempts (~1.2%) are listed in position order and evaluated by the whole
// CTA in parallel; their chaining (which listed words start attempts) needs
// only integer work from an anchor — the latest position preceded by 64 fast
// words, found in a backward halo — and is resolved per run between "sync
// points". The tile's draw count feeds a decoupled look-back that gives its
// global offset; values are staged in shared memory and stored coalesced.
// The tables come from numpy's own build (ziggurat_tables.py -> generated
// header) and are copied to shared memory (random per-lane index).
#include <algorithm>
#include <climits>

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

// The tables live in shared memory inside the kernel: idx is random per lane,
// and a divergent __constant__ index serialises the constant cache (LDC).
struct ZigTables {
  uint64_t ki[256];
  double wi[256];
  double fi[256];
};

SKB_DEV void zig_load_tables(ZigTables* t) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    t->ki[i] = zig_ki_double_bits[i];
    t->wi[i] = __longlong_as_double((long long)zig_wi_double_bits[i]);
    t->fi[i] = __longlong_as_double((long long)zig_fi_double_bits[i]);
  }
}

SKB_DEV uint64_t out64(uint64_t k0, uint64_t k1, uint64_t q) {
  const u64x4 o = philox4x64_10((q >> 2) + 1, 0, 0, 0, k0, k1);
  return o.v[q & 3];
}

SKB_DEV double to_unit(uint64_t r) {  // numpy next_double
  return (double)(r >> 11) * (1.0 / 9007199254740992.0);
}

SKB_DEV bool zig_fast(const ZigTables& T, uint64_t r) {
  const int idx = (int)(r & 0xff);
  const uint64_t rabs = (r >> 9) & 0x000fffffffffffffULL;
  return rabs < T.ki[idx];
}

SKB_DEV double zig_fast_value(const ZigTables& T, uint64_t r) {
  const int idx = (int)(r & 0xff);
  const uint64_t rabs = (r >> 9) & 0x000fffffffffffffULL;
  const double x = __dmul_rn((double)rabs, T.wi[idx]);
  return ((r >> 8) & 1) ? -x : x;
}

// A slow attempt starting at q (word r): -> accepted?, value, length in words.
SKB_DEV bool zig_slow(const ZigTables& T, uint64_t k0, uint64_t k1, uint64_t q, uint64_t r,
                      double* val, int* len) {
  const int idx = (int)(r & 0xff);
  const uint64_t rabs = (r >> 9) & 0x000fffffffffffffULL;
  double x = __dmul_rn((double)rabs, T.wi[idx]);
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
      __dadd_rn(__dmul_rn(__dsub_rn(T.fi[idx - 1], T.fi[idx]), u), T.fi[idx]);
  *len = 2;
  if (lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x))) {
    *val = x;
    return true;
  }
  return false;
}

// x / c correctly rounded (numpy's true division) without DDIV: with
// rc = RN(1/c), q = RN(x rc) is within an ulp and the FMA residual correction
// RN(q + (x - q c) rc) is the correctly rounded quotient (Markstein; the
// operands here are far from the subnormal range). Zero keeps its sign.
SKB_DEV double div_by(double x, double c, double rc) {
  const double q = __dmul_rn(x, rc);
  if (x == 0.0) return q;
  const double r = __fma_rn(-q, c, x);
  return __fma_rn(r, rc, q);
}

// Tile state words for the decoupled look-back: flag in bits 62-63.
constexpr uint64_t kZFlagAgg = 1ULL << 62;   // tile's own draw count published
constexpr uint64_t kZFlagIncl = 2ULL << 62;  // inclusive prefix published
constexpr uint64_t kZValMask = (1ULL << 62) - 1;
constexpr int kZHalo = 256;       // positions per backward halo chunk (64 Philox blocks)
constexpr int kZHaloChunks = 16;  // anchor search depth (4096 positions)
constexpr int kZListMax = 192;    // slow positions per tile + halo (mean ~30)

struct GaussSmem {
  ZigTables T;
  uint32_t slow_bits[kZTile / 32];  // tile positions whose word fails the fast test
  uint32_t skip_bits[kZTile / 32];  // consumed by a slow attempt
  uint32_t acc_bits[kZTile / 32];   // accepted slow attempt starts
  uint32_t halo_w[kZHalo * kZHaloChunks / 32];  // halo_w[k]: [t0-32(k+1), t0-32k)
  int32_t l_off[kZListMax];         // slow positions from the anchor on, ascending (rel. t0)
  int32_t l_pm[kZListMax];          // prefix max of earlier attempt ends (chain bound)
  double l_val[kZListMax];
  uint8_t l_len[kZListMax];
  uint8_t l_ok[kZListMax];
  uint32_t warp_sum[kZThreads / 32];
  uint64_t prefix;
  uint32_t tile;
  int32_t anchor;  // relative to t0 (<= 0)
  int list_n;
  int anchored;
};

// Slow-bit word at relative word index r (r >= 0: tile, r < 0: halo).
SKB_DEV uint32_t gs_word(const GaussSmem& S, int r) {
  return r >= 0 ? S.slow_bits[r] : S.halo_w[-r - 1];
}

// Persistent kernel; each CTA takes tiles of positions [t0, t0 + 4096) in
// ticket order, so the look-back only ever waits on running/finished tiles:
//  1. every thread draws its 16 words (4 Philox blocks), keeps their fast
//     values in registers and flags the slow ones (~0.7%) in a bitmap;
//  2. backward halo chunks of 256 positions until the anchor is found: the
//     latest a <= t0 preceded by 64 fast words (an attempt start whenever
//     every attempt is <= 64 words, which the chain checks);
//  3. warp 0 compacts the slow positions in [a, t0 + 4096) into an ascending
//     list; the whole CTA evaluates those attempts in parallel (value,
//     accept, length); one lane chains them with the stored lengths and
//     marks the consumed words;
//  4. block scan of the emitted draws, decoupled look-back for the tile's
//     global offset, values staged in shared memory and written coalesced.
__global__ void __launch_bounds__(kZThreads, 3)
    gauss_onepass_kernel(uint64_t k0, uint64_t k1, uint64_t p0, uint64_t lo, uint64_t need,
                         double sqrtw,
                         double* __restrict__ out, uint64_t* __restrict__ state,
                         uint32_t* __restrict__ ticket, uint32_t tiles, int* __restrict__ err) {
  __shared__ GaussSmem S;
  extern __shared__ double stage[];  // kZTile outputs by rank (dynamic: 32 KB)
  const double rsqrtw = __drcp_rn(sqrtw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  zig_load_tables(&S.T);
  for (;;) {
    if (tid == 0) S.tile = atomicAdd(ticket, 1u);
    if (tid < kZTile / 32) {
      S.skip_bits[tid] = 0;
      S.acc_bits[tid] = 0;
    }
    __syncthreads();
    const uint32_t tile = S.tile;
    if (tile >= tiles) break;
    const uint64_t t0 = p0 + (uint64_t)tile * kZTile;  // p0: first position (a tile multiple)
    const uint64_t my0 = t0 + (uint64_t)tid * kZPer;

    // ---- 1. classify this thread's words
    double vv[kZPer];
    uint32_t mask = 0;
#pragma unroll
    for (int b = 0; b < kZPer / 4; ++b) {
      const u64x4 o = philox4x64_10(((my0 >> 2) + b) + 1, 0, 0, 0, k0, k1);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        vv[4 * b + i] = zig_fast_value(S.T, o.v[i]);
        if (!zig_fast(S.T, o.v[i])) mask |= 1u << (4 * b + i);
      }
    }
    {
      const uint32_t other = __shfl_xor_sync(0xffffffffu, mask, 1);
      if ((tid & 1) == 0) S.slow_bits[tid >> 1] = mask | (other << 16);
    }
    if (tid == 0) {
      S.anchored = (t0 == 0);
      S.anchor = 0;
    }
    __syncthreads();

    // ---- 2. anchor from backward halo chunks
    int32_t a_rel = 0;  // thread 0: current candidate (relative to t0)
    int chunks = 0;
    while (!S.anchored) {
      const int c = chunks;
      if (c == kZHaloChunks) {
        if (tid == 0) atomicOr(err, 2);  // (never observed: 4096 words without a 64-run)
        break;
      }
      if (tid < 8) S.halo_w[8 * c + tid] = 0;
      __syncthreads();
      if (tid < kZHalo / 4) {
        const int64_t p0 = (int64_t)t0 - (int64_t)kZHalo * (c + 1) + 4 * tid;
        if (p0 >= 0) {
          const u64x4 o = philox4x64_10(((uint64_t)p0 >> 2) + 1, 0, 0, 0, k0, k1);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (!zig_fast(S.T, o.v[i])) {
              const int dd = kZHalo * (c + 1) - 4 * tid - i;  // t0 - p, in [1, 256 (c+1)]
              const int k = (dd - 1) >> 5;
              atomicOr(&S.halo_w[k], 1u << (32 * (k + 1) - dd));
            }
          }
        }
      }
      __syncthreads();
      ++chunks;
      if (tid == 0) {
        // lowest relative position covered (clipped at the stream start)
        const int32_t low = (int64_t)t0 - (int64_t)kZHalo * chunks < 0 ? -(int32_t)t0
                                                                       : -kZHalo * chunks;
        for (;;) {
          // highest slow position s in [low, a_rel)
          int32_t s = INT32_MIN;
          for (int32_t q = a_rel - 1; q >= low;) {
            const int r = q >> 5;  // floor division (arithmetic shift)
            uint32_t wbits = gs_word(S, r) & (0xffffffffu >> (31 - (q & 31)));
            if (wbits) {
              s = r * 32 + (31 - __clz(wbits));
              break;
            }
            q = r * 32 - 1;
          }
          if (s == INT32_MIN) {
            if (a_rel - low >= kZMaxLen || low == -(int32_t)t0) {
              S.anchor = a_rel;
              S.anchored = 1;
            }
            break;  // else: need another chunk
          }
          if (a_rel - s > kZMaxLen) {
            S.anchor = a_rel;
            S.anchored = 1;
            break;
          }
          a_rel = s;
        }
      }
      __syncthreads();
    }

    // ---- 3a. ascending list of slow positions in [anchor, t0 + 4096)
    if (warp == 0) {
      const int32_t anc = S.anchor;
      const int r_lo = anc >> 5;  // floor
      const int nw = kZTile / 32 - r_lo;
      const int per = (nw + 31) / 32;
      const int rb = r_lo + lane * per;
      int cnt = 0;
      for (int t = 0; t < per; ++t) {
        const int r = rb + t;
        if (r >= kZTile / 32) break;
        uint32_t wbits = gs_word(S, r);
        if (r * 32 < anc) wbits &= 0xffffffffu << (anc - r * 32);
        cnt += __popc(wbits);
      }
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      int pos = incl - cnt;
      for (int t = 0; t < per; ++t) {
        const int r = rb + t;
        if (r >= kZTile / 32) break;
        uint32_t wbits = gs_word(S, r);
        if (r * 32 < anc) wbits &= 0xffffffffu << (anc - r * 32);
        while (wbits) {
          const int b = __ffs(wbits) - 1;
          wbits &= wbits - 1;
          if (pos < kZListMax) S.l_off[pos] = r * 32 + b;
          ++pos;
        }
      }
      if (lane == 31) {
        S.list_n = min(incl, kZListMax);
        if (incl > kZListMax) atomicOr(err, 4);
      }
    }
    __syncthreads();
    // ---- 3b. evaluate every listed attempt in parallel
    const int nlist = S.list_n;
    for (int i = tid; i < nlist; i += kZThreads) {
      const uint64_t q = (uint64_t)((int64_t)t0 + S.l_off[i]);
      double v = 0.0;
      int len;
      const bool ok = zig_slow(S.T, k0, k1, q, out64(k0, k1, q), &v, &len);
      S.l_val[i] = v;
      S.l_len[i] = (uint8_t)min(len, 255);
      S.l_ok[i] = ok;
    }
    __syncthreads();
    // ---- 3c. chain. PM_i = max(anchor, ends of all earlier entries as if
    // every entry were an attempt) bounds the true next free word, so an
    // entry with off_i >= PM_i is certainly an attempt (a sync point). Each
    // lane owning a sync point resolves, in order, the entries up to the
    // next sync point (short runs: only adjacent slow words conflict).
    if (warp == 0) {
      int32_t carry = S.anchor;
      for (int b = 0; b < nlist; b += 32) {
        const int i = b + lane;
        const bool valid = i < nlist;
        const int32_t e = valid ? S.l_off[i] + (int32_t)S.l_len[i] : INT32_MIN;
        int32_t pm = e;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int32_t t = __shfl_up_sync(0xffffffffu, pm, o);
          if (lane >= o) pm = max(pm, t);
        }
        int32_t before = __shfl_up_sync(0xffffffffu, pm, 1);
        before = lane == 0 ? carry : max(before, carry);
        if (valid) S.l_pm[i] = before;
        carry = max(carry, __shfl_sync(0xffffffffu, pm, 31));
      }
      __syncwarp();
      for (int i = lane; i < nlist; i += 32) {
        if (S.l_off[i] < S.l_pm[i]) continue;  // not a sync point
        int32_t next_free = INT32_MIN;
        for (int k = i; k < nlist && (k == i || S.l_off[k] < S.l_pm[k]); ++k) {
          const int32_t so = S.l_off[k];
          if (so < next_free) continue;  // consumed by the previous attempt
          const int len = S.l_len[k];
          if (len > kZMaxLen) atomicOr(err, 1);
          if (so >= 0 && S.l_ok[k]) atomicOr(&S.acc_bits[so >> 5], 1u << (so & 31));
          const int32_t e = min(so + len, kZTile);
          for (int32_t p = max(so + 1, 0); p < e;) {  // consumed words in the tile
            const int r = p >> 5, b0 = p & 31;
            const int nb = min(32 - b0, e - p);
            atomicOr(&S.skip_bits[r], (nb == 32 ? 0xffffffffu : ((1u << nb) - 1u)) << b0);
            p += nb;
          }
          next_free = so + len;
        }
      }
    }
    __syncthreads();

    // ---- 4. scan, look-back, staged coalesced store
    const uint32_t sk = (S.skip_bits[tid >> 1] >> ((tid & 1) * 16)) & 0xffffu;
    const uint32_t ac = (S.acc_bits[tid >> 1] >> ((tid & 1) * 16)) & 0xffffu;
    const uint32_t outm = ((~mask & 0xffffu) & ~sk) | ac;  // visited fast | accepted slow
    const uint32_t cnt = __popc(outm);
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) S.warp_sum[warp] = incl;
    if (ac) {  // accepted slow values from the list (binary search; rare)
#pragma unroll
      for (int i = 0; i < kZPer; ++i) {
        if (ac & (1u << i)) {
          const int32_t off = tid * kZPer + i;
          int lo_i = 0, hi_i = nlist - 1;
          while (lo_i < hi_i) {
            const int mid = (lo_i + hi_i) >> 1;
            if (S.l_off[mid] < off) lo_i = mid + 1;
            else hi_i = mid;
          }
          vv[i] = S.l_val[lo_i];
        }
      }
    }
    __syncthreads();
    uint32_t wbase = 0, total = 0;
#pragma unroll
    for (int w2 = 0; w2 < kZThreads / 32; ++w2) {
      const uint32_t t = S.warp_sum[w2];
      if (w2 < warp) wbase += t;
      total += t;
    }
    const uint32_t excl = wbase + incl - cnt;
#pragma unroll
    for (int i = 0, k = 0; i < kZPer; ++i) {
      if (outm & (1u << i)) {
        stage[excl + k] = div_by(vv[i], sqrtw, rsqrtw);
        ++k;
      }
    }
    if (warp == 0) {
      volatile uint64_t* vs = state;
      if (lane == 0)
        vs[tile] = (tile == 0 ? uint64_t(kZFlagIncl) : uint64_t(kZFlagAgg)) | (uint64_t)total;
      uint64_t prefix = 0;
      int64_t j = (int64_t)tile - 1;
      while (j >= 0) {
        const int64_t idx = j - lane;
        uint64_t sv = idx >= 0 ? uint64_t(vs[idx]) : uint64_t(kZFlagIncl);
        int first;
        for (;;) {
          const uint32_t ready = __ballot_sync(0xffffffffu, (sv >> 62) != 0);
          const uint32_t incl_m = __ballot_sync(0xffffffffu, (sv >> 62) == 2);
          first = incl_m ? __ffs(incl_m) - 1 : 32;
          const uint32_t need_m = first == 32 ? 0xffffffffu : ((2u << first) - 1u);
          if ((ready & need_m) == need_m) break;
          if ((sv >> 62) == 0) sv = vs[idx];
        }
        uint64_t part = (lane <= first && idx >= 0) ? (sv & kZValMask) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        prefix += part;
        if (first < 32) break;
        j -= 32;
      }
      if (lane == 0) {
        if (tile > 0) vs[tile] = kZFlagIncl | (prefix + total);
        S.prefix = prefix;
      }
    }
    __syncthreads();
    const uint64_t base = S.prefix;
    for (uint32_t k = tid; k < total; k += kZThreads) {
      const uint64_t idx = base + k;
      if (idx >= lo && idx < need) out[idx - lo] = stage[k];
    }
    __syncthreads();
  }
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
    if (tiles > 0xffffff00ULL) return SKB_ERR_UNSUPPORTED;
    const size_t mark = ws.off;
    uint64_t* state = (uint64_t*)skb_ws_take(&ws, tiles * 8);
    uint32_t* ticket = (uint32_t*)skb_ws_take(&ws, 16);
    int* err = (int*)skb_ws_take(&ws, 16);
    if (!state || !ticket || !err) return SKB_ERR_WORKSPACE;
    cudaMemsetAsync(state, 0, tiles * 8, st);
    cudaMemsetAsync(ticket, 0, 16, st);
    cudaMemsetAsync(err, 0, 16, st);
    static int grid = 0;
    if (!grid) {
      cudaFuncSetAttribute(gauss_onepass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kZTile * 8);
      int per = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, gauss_onepass_kernel, kZThreads,
                                                    kZTile * 8);
      grid = std::max(1, per) * skb_num_sms();
    }
    gauss_onepass_kernel<<<(unsigned)std::min<uint64_t>(tiles, (uint64_t)grid), kZThreads,
                           kZTile * 8, st>>>(key0, key1, 0, (uint64_t)lo, (uint64_t)count, sqrtw,
                                             W, state, ticket, (uint32_t)tiles, err);
    uint64_t last = 0;
    int herr = 0;
    cudaMemcpyAsync(&last, state + (tiles - 1), 8, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return SKB_ERR_CUDA;
    ws.off = mark;
    if (herr) return SKB_ERR_INTERNAL;  // an attempt longer than 64 words (never observed)
    if ((last & kZValMask) >= (uint64_t)count) return skb_launch_status(__func__);
    positions *= 2;
  }
  return SKB_ERR_INTERNAL;
}

// The draws whose attempts START in stream positions [p0, p1) (multiples of
// 4096), in stream order, into out[0, count) (count <= cap; *count_host gets
// the number of draws of the range even when it exceeds cap). Consecutive
// ranges partition the draw sequence, so ranks can each generate one range
// and exchange by global draw index (sketching.build_gaussian_sketch).
// Synchronises the stream.
extern "C" int skb_gaussian_range(uint64_t key0, uint64_t key1, uint64_t p0, uint64_t p1,
                                  int32_t w, double* out, int64_t cap, uint64_t* count_host,
                                  void* workspace, size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (w < 1 || cap < 0 || p1 < p0 || (p0 % kZTile) || (p1 % kZTile)) return SKB_ERR_ARG;
  *count_host = 0;
  if (p1 == p0) return 0;
  skb_ws ws = skb_ws_make(workspace, ws_bytes);
  const double sqrtw = __builtin_sqrt((double)w);
  const uint64_t tiles = (p1 - p0) / kZTile;
  if (tiles > 0xffffff00ULL) return SKB_ERR_UNSUPPORTED;
  uint64_t* state = (uint64_t*)skb_ws_take(&ws, tiles * 8);
  uint32_t* ticket = (uint32_t*)skb_ws_take(&ws, 16);
  int* err = (int*)skb_ws_take(&ws, 16);
  if (!state || !ticket || !err) return SKB_ERR_WORKSPACE;
  cudaMemsetAsync(state, 0, tiles * 8, st);
  cudaMemsetAsync(ticket, 0, 16, st);
  cudaMemsetAsync(err, 0, 16, st);
  static int grid = 0;
  if (!grid) {
    cudaFuncSetAttribute(gauss_onepass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kZTile * 8);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, gauss_onepass_kernel, kZThreads,
                                                  kZTile * 8);
    grid = std::max(1, per) * skb_num_sms();
  }
  gauss_onepass_kernel<<<(unsigned)std::min<uint64_t>(tiles, (uint64_t)grid), kZThreads,
                         kZTile * 8, st>>>(key0, key1, p0, 0, (uint64_t)cap, sqrtw, out, state,
                                           ticket, (uint32_t)tiles, err);
  uint64_t last = 0;
  int herr = 0;
  cudaMemcpyAsync(&last, state + (tiles - 1), 8, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return SKB_ERR_CUDA;
  if (herr) return SKB_ERR_INTERNAL;
  *count_host = last & kZValMask;
  return skb_launch_status(__func__);
}

extern "C" size_t skb_gaussian_workspace_bytes(int64_t count) {
  const uint64_t tiles = ((uint64_t)count * 2 + 8 * kZTile) / kZTile + 1;
  return (size_t)tiles * 8 + 4096;
}
