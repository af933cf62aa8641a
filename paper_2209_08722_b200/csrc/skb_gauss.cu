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
// B200 mapping: four kernels over tiles of 4096 stream positions, every one
// of them parallel across tiles (no tile waits on another):
//  K9a classify: Philox + the fast test for every word -> a 1-bit-per-word
//      "slow" bitmap (1/8 byte per draw), no barriers;
//  K9b chain (one warp per tile): anchor = the latest position before the
//      tile preceded by 64 fast words (read from the bitmap), the tile's slow
//      positions listed in order, their attempts evaluated by the lanes, and
//      chained between "sync points" into consumed / accepted bitmaps and the
//      tile's draw count;
//  K9c exclusive scan of the counts (CUB) -> each tile's first draw index;
//  K9d emit: Philox again, fast values, accepted slow values recomputed,
//      block ranks, staged in shared memory and stored coalesced.
// The tables come from numpy's own build (ziggurat_tables.py -> generated
// header) and live in shared memory (random per-lane index).
#include <algorithm>
#include <climits>

#include <cub/device/device_scan.cuh>

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

// log1p(x) for x in (-1, 0], bit-identical to the host libm numpy calls in the
// ziggurat tail (npy_log1p -> glibc 2.39 log1p). glibc's log1p is the fdlibm
// algorithm (argument reduction to 1 + f, s = f / (2 + f), a degree-7 odd
// polynomial in s evaluated in Estrin form), and on FMA-capable x86 hosts
// glibc runs its FMA build of it: the contractions below are that build's
// (checked bit for bit against glibc on 4e8 arguments, tests/golden/log1p_check.c).
// CUDA's own log1p differs from it in the last place on ~0.4% of arguments.
SKB_DEV double glibc_log1p(double x) {
  constexpr double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  constexpr double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
                   Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
                   Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
                   Lp7 = 1.479819860511658591e-01;
  const int hx = __double2hiint(x), ax = hx & 0x7fffffff;
  if (ax >= 0x3ff00000) return x == -1.0 ? -INFINITY : __longlong_as_double(0x7ff8000000000000ll);
  if (ax < 0x3e200000) return ax < 0x3c900000 ? x : __fma_rn(-__dmul_rn(x, x), 0.5, x);
  int k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx <= (int)0xbfd2bec3) {  // -0.2929 < x <= 0 (x is never positive here)
    k = 0;
    f = x;
    hu = 1;
  } else {
    double u = __dadd_rn(1.0, x);
    hu = __double2hiint(u);
    k = (hu >> 20) - 1023;
    c = k > 0 ? __dsub_rn(1.0, __dsub_rn(u, x)) : __dsub_rn(x, __dsub_rn(u, 1.0));
    c = __ddiv_rn(c, u);
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = __hiloint2double(hu | 0x3ff00000, __double2loint(u));
    } else {
      k += 1;
      u = __hiloint2double(hu | 0x3fe00000, __double2loint(u));
      hu = (0x00100000 - hu) >> 2;
    }
    f = __dsub_rn(u, 1.0);
  }
  const double hfsq = __dmul_rn(__dmul_rn(0.5, f), f);
  const double kd = (double)k;
  if (hu == 0) {
    if (f == 0.0) return k == 0 ? 0.0 : __fma_rn(kd, ln2_hi, __fma_rn(kd, ln2_lo, c));
    const double R = __dmul_rn(hfsq, __fma_rn(-0.66666666666666666, f, 1.0));
    if (k == 0) return __dsub_rn(f, R);
    return __fma_rn(kd, ln2_hi, -__dsub_rn(__dsub_rn(R, __fma_rn(kd, ln2_lo, c)), f));
  }
  const double s = __ddiv_rn(f, __dadd_rn(2.0, f));
  const double z = __dmul_rn(s, s);
  const double R2 = __fma_rn(Lp3, z, Lp2), R3 = __fma_rn(Lp5, z, Lp4), R4 = __fma_rn(Lp7, z, Lp6);
  const double z2 = __dmul_rn(z, z), z4 = __dmul_rn(z2, z2), z6 = __dmul_rn(z4, z2);
  double R = __fma_rn(z, Lp1, __dmul_rn(z2, R2));
  R = __fma_rn(z4, R3, R);
  R = __fma_rn(z6, R4, R);
  const double t = __dmul_rn(s, __dadd_rn(hfsq, R));
  if (k == 0) return __dsub_rn(f, __dsub_rn(hfsq, t));
  return __fma_rn(kd, ln2_hi,
                  -__dsub_rn(__dsub_rn(hfsq, __dadd_rn(__fma_rn(kd, ln2_lo, c), t)), f));
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
      const double xx = __dmul_rn(-kZigInvR, glibc_log1p(-u1));
      const double yy = -glibc_log1p(-u2);
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

constexpr int kZHaloTiles = 4;           // anchor search depth before a range start
constexpr int kZWords = kZTile / 32;     // bitmap words per tile
constexpr int kZListMax = 512;           // listed slow positions per tile (mean ~50)
constexpr int kZChainWarps = 4;

// ---- K9a: slow bitmap of positions [base, base + 32 * nwords). With `vals`
// (the stored-values mode, when the workspace has room for 8 bytes per
// position) the fast positions' final values W = x / sqrt(w) are written too,
// at their POSITION index, and K9d only compacts them instead of running
// Philox a second time (the slow ones are recomputed there as before).
__global__ void __launch_bounds__(256)
    zig_classify_kernel(uint64_t k0, uint64_t k1, uint64_t base, int64_t nwords,
                        uint32_t* __restrict__ bits, double* __restrict__ vals, double sqrtw) {
  __shared__ ZigTables T;
  zig_load_tables(&T);
  const double rsqrtw = __drcp_rn(sqrtw);
  __syncthreads();
  for (int64_t wd = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; wd < nwords;
       wd += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t p = base + 32 * (uint64_t)wd;
    uint32_t mask = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const u64x4 o = philox4x64_10(((p >> 2) + b) + 1, 0, 0, 0, k0, k1);
      double v4[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint64_t r = o.v[i];
        if (!zig_fast(T, r)) mask |= 1u << (4 * b + i);
        v4[i] = vals ? div_by(zig_fast_value(T, r), sqrtw, rsqrtw) : 0.0;
      }
      if (vals) {
        double2* dst = reinterpret_cast<double2*>(vals + 32 * wd + 4 * b);
        dst[0] = make_double2(v4[0], v4[1]);
        dst[1] = make_double2(v4[2], v4[3]);
      }
    }
    bits[wd] = mask;
  }
}

struct ZigChainWarp {
  int32_t off[kZListMax];   // slow positions from the anchor on, ascending (relative t0)
  int32_t pm[kZListMax];    // prefix max of earlier attempt ends
  uint8_t len[kZListMax];
  uint8_t ok[kZListMax];
  uint32_t skip[kZWords];
  uint32_t acc[kZWords];
};

// ---- K9b: one warp per tile; bits cover positions [base, ...) with base <= P0 - halo
__global__ void __launch_bounds__(32 * kZChainWarps)
    zig_chain_kernel(uint64_t k0, uint64_t k1, uint64_t P0, uint64_t base,
                     const uint32_t* __restrict__ bits, int64_t tiles,
                     uint32_t* __restrict__ gskip, uint32_t* __restrict__ gacc,
                     uint64_t* __restrict__ cnt, int* __restrict__ err,
                     double* __restrict__ vals, double sqrtw) {
  __shared__ ZigTables T;
  __shared__ ZigChainWarp W[kZChainWarps];
  zig_load_tables(&T);
  __syncthreads();
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  ZigChainWarp& S = W[wl];
  for (int64_t tile = (int64_t)blockIdx.x * kZChainWarps + wl; tile < tiles;
       tile += (int64_t)gridDim.x * kZChainWarps) {
    const uint64_t t0 = P0 + (uint64_t)tile * kZTile;
    const int64_t r_t0 = (int64_t)((t0 - base) / 32);  // bitmap word of t0
    auto word = [&](int64_t r_rel) -> uint32_t {       // word at relative index (t0 = 0)
      const int64_t g = r_t0 + r_rel;
      return g >= 0 ? bits[g] : 0u;
    };
    for (int q = lane; q < kZWords; q += 32) {
      S.skip[q] = 0;
      S.acc[q] = 0;
    }
    // anchor (lane 0): latest a <= 0 with 64 fast predecessors, or the stream start
    int32_t anc = 0;
    if (lane == 0 && t0 > 0) {
      const int32_t low = -(int32_t)(t0 - base);  // lowest position with known bits
      int32_t a = 0;
      bool found = false;
      for (;;) {
        int32_t sl = INT32_MIN;
        for (int32_t q = a - 1; q >= low;) {
          const int32_t r = q >> 5;
          const uint32_t wbits = word(r) & (0xffffffffu >> (31 - (q & 31)));
          if (wbits) {
            sl = r * 32 + (31 - __clz(wbits));
            break;
          }
          q = r * 32 - 1;
        }
        if (sl == INT32_MIN) {
          found = (a - low >= kZMaxLen) || base == 0;  // ... or fast back to the stream start
          break;
        }
        if (a - sl > kZMaxLen) {
          found = true;
          break;
        }
        a = sl;
      }
      if (!found) atomicOr(err, 2);  // (never observed: 16K words without a 64-run)
      anc = a;
    }
    anc = __shfl_sync(0xffffffffu, anc, 0);
    // ascending list of slow positions in [anc, 4096)
    {
      const int r_lo = anc >> 5;
      const int nw = kZWords - r_lo;
      const int per = (nw + 31) / 32;
      const int rb = r_lo + lane * per;
      int c = 0;
      for (int t = 0; t < per; ++t) {
        const int r = rb + t;
        if (r >= kZWords) break;
        uint32_t wbits = word(r);
        if (r * 32 < anc) wbits &= 0xffffffffu << (anc - r * 32);
        c += __popc(wbits);
      }
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      int pos = incl - c;
      for (int t = 0; t < per; ++t) {
        const int r = rb + t;
        if (r >= kZWords) break;
        uint32_t wbits = word(r);
        if (r * 32 < anc) wbits &= 0xffffffffu << (anc - r * 32);
        while (wbits) {
          const int b = __ffs(wbits) - 1;
          wbits &= wbits - 1;
          if (pos < kZListMax) S.off[pos] = r * 32 + b;
          ++pos;
        }
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      if (lane == 0 && total > kZListMax) atomicOr(err, 4);
      __syncwarp();
      const int nlist = min(total, kZListMax);
      // evaluate every listed attempt (lanes in parallel)
      for (int i = lane; i < nlist; i += 32) {
        const uint64_t q = (uint64_t)((int64_t)t0 + S.off[i]);
        double v;
        int len;
        const bool ok = zig_slow(T, k0, k1, q, out64(k0, k1, q), &v, &len);
        S.len[i] = (uint8_t)min(len, 255);
        S.ok[i] = ok;
        // stored-values mode: an accepted attempt's value goes into its start
        // position's slot (a slow position: K9a's fast value there is unused),
        // so the emit pass never recomputes a slow attempt (tiles evaluating
        // the same attempt write the same value)
        if (vals && ok) vals[q - base] = div_by(v, sqrtw, __drcp_rn(sqrtw));
      }
      __syncwarp();
      // prefix max of attempt ends (as if every entry were an attempt)
      int32_t carry = anc;
      for (int b = 0; b < nlist; b += 32) {
        const int i = b + lane;
        const bool valid = i < nlist;
        const int32_t e = valid ? S.off[i] + (int32_t)S.len[i] : INT32_MIN;
        int32_t pmv = e;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int32_t t = __shfl_up_sync(0xffffffffu, pmv, o);
          if (lane >= o) pmv = max(pmv, t);
        }
        int32_t before = __shfl_up_sync(0xffffffffu, pmv, 1);
        before = lane == 0 ? carry : max(before, carry);
        if (valid) S.pm[i] = before;
        carry = max(carry, __shfl_sync(0xffffffffu, pmv, 31));
      }
      __syncwarp();
      // chain between sync points
      for (int i = lane; i < nlist; i += 32) {
        if (S.off[i] < S.pm[i]) continue;
        int32_t next_free = INT32_MIN;
        for (int k = i; k < nlist && (k == i || S.off[k] < S.pm[k]); ++k) {
          const int32_t so = S.off[k];
          if (so < next_free) continue;
          const int len = S.len[k];
          if (len > kZMaxLen) atomicOr(err, 1);
          if (so >= 0 && S.ok[k]) atomicOr(&S.acc[so >> 5], 1u << (so & 31));
          const int32_t e = min(so + len, kZTile);
          for (int32_t p = max(so + 1, 0); p < e;) {
            const int r = p >> 5, b0 = p & 31;
            const int nb = min(32 - b0, e - p);
            atomicOr(&S.skip[r], (nb == 32 ? 0xffffffffu : ((1u << nb) - 1u)) << b0);
            p += nb;
          }
          next_free = so + len;
        }
      }
      __syncwarp();
    }
    // the tile's draws: visited fast words + accepted slow attempts
    uint64_t c = 0;
    for (int q = lane; q < kZWords; q += 32) {
      const uint32_t sk = S.skip[q], ac = S.acc[q];
      c += __popc((~word(q) & ~sk) | ac);
      gskip[tile * kZWords + q] = sk;
      gacc[tile * kZWords + q] = ac;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[tile] = c;
    __syncwarp();
  }
}

// ---- K9d: emit the tile's draws at their global indices (offs: exclusive scan).
// Each thread's draws are consecutive in the output (its rank range), so
// they are stored directly (no staging barrier); the warp's ranges abut.
__global__ void __launch_bounds__(kZThreads, 3)
    zig_emit_kernel(uint64_t k0, uint64_t k1, uint64_t P0, int64_t tiles,
                    const uint32_t* __restrict__ gskip, const uint32_t* __restrict__ gacc,
                    const uint64_t* __restrict__ offs, uint64_t lo, uint64_t need,
                    double sqrtw, double* __restrict__ out, const uint32_t* __restrict__ bits,
                    const double* __restrict__ vals, uint64_t vbase) {
  __shared__ ZigTables T;
  __shared__ uint32_t warp_sum[2][kZThreads / 32];
  __shared__ double wbuf[kZThreads / 32][32 * kZPer];
  zig_load_tables(&T);
  const double rsqrtw = __drcp_rn(sqrtw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __syncthreads();
  int par = 0;  // warp_sum buffer: flips per processed tile (skipped tiles have no barrier)
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const uint64_t t0 = P0 + (uint64_t)tile * kZTile;
    const uint64_t my0 = t0 + (uint64_t)tid * kZPer;
    const uint64_t base = offs[tile];
    const uint64_t tcount = offs[tile + 1] - base;
    if (base >= need || base + tcount <= lo) continue;  // uniform across the CTA
    const uint32_t sk = (gskip[tile * kZWords + (tid >> 1)] >> ((tid & 1) * 16)) & 0xffffu;
    const uint32_t ac = (gacc[tile * kZWords + (tid >> 1)] >> ((tid & 1) * 16)) & 0xffffu;
    double vv[kZPer];
    uint32_t slow = 0;
    if (vals) {  // stored-values mode: K9a's values (already / sqrt(w)) and slow bits
      const uint64_t rel = my0 - vbase;  // a multiple of 16
      slow = (bits[rel >> 5] >> (rel & 31)) & 0xffffu;
      const double2* src = reinterpret_cast<const double2*>(vals + rel);
#pragma unroll
      for (int i = 0; i < kZPer / 2; ++i) {
        const double2 t2 = src[i];
        vv[2 * i] = t2.x;
        vv[2 * i + 1] = t2.y;
      }
    } else {
#pragma unroll
      for (int b = 0; b < kZPer / 4; ++b) {
        const u64x4 o = philox4x64_10(((my0 >> 2) + b) + 1, 0, 0, 0, k0, k1);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          vv[4 * b + i] = zig_fast_value(T, o.v[i]);
          if (!zig_fast(T, o.v[i])) slow |= 1u << (4 * b + i);
        }
      }
    }
    const uint32_t outm = ((~slow & 0xffffu) & ~sk) | ac;
    const uint32_t c = __popc(outm);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_sum[par][warp] = incl;  // double-buffered: one barrier per tile
    __syncthreads();
    uint32_t wbase = 0;
#pragma unroll
    for (int w2 = 0; w2 < kZThreads / 32; ++w2)
      if (w2 < warp) wbase += warp_sum[par][w2];
    const uint64_t first = base + wbase + incl - c;  // global index of this thread's first draw
    // the warp's draws are one contiguous range: stage them in shared memory
    // and store coalesced (direct per-thread stores touch 32 lines per instruction)
    const uint64_t wfirst = __shfl_sync(0xffffffffu, first, 0);
    const uint32_t wcount = __shfl_sync(0xffffffffu, incl, 31);
    double* buf = wbuf[warp];
    const uint32_t off = (uint32_t)(first - wfirst);
#pragma unroll
    for (int i = 0, k = 0; i < kZPer; ++i) {
      if (outm & (1u << i)) {
        if (vals || !((ac >> i) & 1u)) buf[off + k] = vals ? vv[i] : div_by(vv[i], sqrtw, rsqrtw);
        ++k;
      }
    }
    // accepted slow attempts (rare): recompute their values in a rolled loop
    // (stored-values mode: K9b already put them into vals)
    for (uint32_t rest = vals ? 0u : ac; rest; rest &= rest - 1) {
      const int i = __ffs(rest) - 1;
      const uint64_t q = my0 + i;
      double v;
      int len;
      zig_slow(T, k0, k1, q, out64(k0, k1, q), &v, &len);
      buf[off + __popc(outm & ((1u << i) - 1u))] = div_by(v, sqrtw, rsqrtw);
    }
    __syncwarp();
    // the warp's slice of [lo, need): 32-bit offsets from one 64-bit base
    const uint32_t p_lo =
        wfirst >= lo ? 0u : (lo - wfirst < wcount ? (uint32_t)(lo - wfirst) : wcount);
    const uint32_t p_hi =
        wfirst >= need ? 0u : (need - wfirst < wcount ? (uint32_t)(need - wfirst) : wcount);
    double* ow = out + (int64_t)(wfirst - lo);  // only dereferenced at p in [p_lo, p_hi)
    for (uint32_t p = p_lo + lane; p < p_hi; p += 32) ow[p] = buf[p];
    __syncwarp();
    par ^= 1;
  }
}

// ---- K9d in the stored-values mode: every value it emits (fast ones from K9a,
// accepted slow ones from K9b) is already in vals, so the pass is a stream
// compaction; the next tile's values are loaded while this tile's draws are
// stored (the two-phase loop above left the loads idle during the stores).
struct ZigPre {
  double v[kZPer];
  uint32_t slow, sk, ac;
  uint64_t base, tcount;
};

__global__ void __launch_bounds__(kZThreads, 3)
    zig_emit_vals_kernel(uint64_t P0, int64_t tiles, const uint32_t* __restrict__ gskip,
                         const uint32_t* __restrict__ gacc, const uint64_t* __restrict__ offs,
                         uint64_t lo, uint64_t need, double* __restrict__ out,
                         const uint32_t* __restrict__ bits, const double* __restrict__ vals,
                         uint64_t vbase) {
  __shared__ uint32_t warp_sum[2][kZThreads / 32];
  __shared__ __align__(16) double wbuf[kZThreads / 32][32 * kZPer + 2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto fetch = [&](int64_t tile, ZigPre& f) {
    f.base = offs[tile];
    f.tcount = offs[tile + 1] - f.base;
    const uint64_t rel = P0 + (uint64_t)tile * kZTile + (uint64_t)tid * kZPer - vbase;
    f.slow = (bits[rel >> 5] >> (rel & 31)) & 0xffffu;
    f.sk = (gskip[tile * kZWords + (tid >> 1)] >> ((tid & 1) * 16)) & 0xffffu;
    f.ac = (gacc[tile * kZWords + (tid >> 1)] >> ((tid & 1) * 16)) & 0xffffu;
    const double2* src = reinterpret_cast<const double2*>(vals + rel);
#pragma unroll
    for (int i = 0; i < kZPer / 2; ++i) {
      const double2 t2 = src[i];
      f.v[2 * i] = t2.x;
      f.v[2 * i + 1] = t2.y;
    }
  };
  ZigPre cur;
  int64_t tile = blockIdx.x;
  if (tile < tiles) fetch(tile, cur);
  int par = 0;
  for (; tile < tiles; tile += gridDim.x) {
    const int64_t nt = tile + gridDim.x;
    const uint64_t base = cur.base, tcount = cur.tcount;
    if (base >= need || base + tcount <= lo) {  // uniform across the CTA
      if (nt < tiles) fetch(nt, cur);
      continue;
    }
    const uint32_t outm = ((~cur.slow & 0xffffu) & ~cur.sk) | cur.ac;
    const uint32_t c = __popc(outm);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_sum[par][warp] = incl;
    __syncthreads();
    uint32_t wbase = 0;
#pragma unroll
    for (int w2 = 0; w2 < kZThreads / 32; ++w2)
      if (w2 < warp) wbase += warp_sum[par][w2];
    const uint64_t first = base + wbase + incl - c;
    const uint64_t wfirst = __shfl_sync(0xffffffffu, first, 0);
    const uint32_t wcount = __shfl_sync(0xffffffffu, incl, 31);
    double* ow = out + (int64_t)(wfirst - lo);  // only dereferenced in [p_lo, p_hi)
    // stage with the global alignment (buf + sa + p and ow + p agree mod 16 bytes)
    const uint32_t sa = (uint32_t)((reinterpret_cast<uintptr_t>(ow) >> 3) & 1);
    double* buf = wbuf[warp] + sa;
    if (lane == 0)  // the previous tile's bulk store has read the buffer
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncwarp();
    const uint32_t off = (uint32_t)(first - wfirst);
#pragma unroll
    for (int i = 0, k = 0; i < kZPer; ++i) {
      if (outm & (1u << i)) {
        buf[off + k] = cur.v[i];
        ++k;
      }
    }
    if (nt < tiles) fetch(nt, cur);  // in flight during the stores below
    __syncwarp();
    const uint32_t p_lo =
        wfirst >= lo ? 0u : (lo - wfirst < wcount ? (uint32_t)(lo - wfirst) : wcount);
    const uint32_t p_hi =
        wfirst >= need ? 0u : (need - wfirst < wcount ? (uint32_t)(need - wfirst) : wcount);
    // the warp's range as one TMA bulk store (16-byte aligned middle) plus <= 2 edges
    const uint32_t pa = p_lo + ((reinterpret_cast<uintptr_t>(ow + p_lo) >> 3) & 1);
    const uint32_t pb = pa < p_hi ? pa + ((p_hi - pa) & ~1u) : pa;
    if (lane == 0 && p_lo < pa && p_lo < p_hi) ow[p_lo] = buf[p_lo];
    if (lane == 1 && pb < p_hi) ow[pb] = buf[pb];
    if (lane == 0 && pb > pa) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   ::"l"(ow + pa), "r"(smem_u32(buf + pa)), "r"((pb - pa) * 8u)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    par ^= 1;
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Draws of the stream positions [P0, P1) (tile multiples), written as
// out[idx - lo] for global draw indices lo <= idx < need (idx counted from the
// first attempt starting at or after P0). *total = draws of the range.
static int zig_generate(uint64_t k0, uint64_t k1, uint64_t P0, uint64_t P1, uint64_t lo,
                        uint64_t need, int32_t w, double* out, uint64_t* total, skb_ws* ws,
                        cudaStream_t st) {
  const int64_t tiles = (int64_t)((P1 - P0) / kZTile);
  *total = 0;
  if (tiles <= 0) return 0;
  const uint64_t base = P0 >= (uint64_t)kZHaloTiles * kZTile ? P0 - kZHaloTiles * kZTile : 0;
  const int64_t nwords = (int64_t)((P1 - base) / 32);
  uint32_t* bits = (uint32_t*)skb_ws_take(ws, (size_t)nwords * 4);
  uint32_t* gskip = (uint32_t*)skb_ws_take(ws, (size_t)tiles * kZWords * 4);
  uint32_t* gacc = (uint32_t*)skb_ws_take(ws, (size_t)tiles * kZWords * 4);
  uint64_t* cnt = (uint64_t*)skb_ws_take(ws, (size_t)(tiles + 1) * 8);
  uint64_t* offs = (uint64_t*)skb_ws_take(ws, (size_t)(tiles + 1) * 8);
  int* err = (int*)skb_ws_take(ws, 16);
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, cnt, offs, (int)(tiles + 1), st);
  void* scan_tmp = skb_ws_take(ws, scan_bytes + 16);
  if (!bits || !gskip || !gacc || !cnt || !offs || !err || !scan_tmp) return SKB_ERR_WORKSPACE;
  // stored-values mode when the workspace has room for 8 bytes per position
  const char* sv = getenv("SKB_ZIG_STORE");
  double* vals = (sv && sv[0] == '0') || need <= lo
                     ? nullptr
                     : (double*)skb_ws_take(ws, (size_t)nwords * 32 * 8);
  if (tiles + 1 > 0x7fffffffLL) return SKB_ERR_UNSUPPORTED;
  cudaMemsetAsync(err, 0, 16, st);
  cudaMemsetAsync(cnt + tiles, 0, 8, st);
  const int sms = skb_num_sms();
  zig_classify_kernel<<<(unsigned)std::min<int64_t>((nwords + 255) / 256, 64LL * sms), 256, 0,
                        st>>>(k0, k1, base, nwords, bits, vals, __builtin_sqrt((double)w));
  zig_chain_kernel<<<(unsigned)std::min<int64_t>((tiles + kZChainWarps - 1) / kZChainWarps,
                                                 16LL * sms),
                     32 * kZChainWarps, 0, st>>>(k0, k1, P0, base, bits, tiles, gskip, gacc, cnt,
                                                 err, vals, __builtin_sqrt((double)w));
  cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, cnt, offs, (int)(tiles + 1), st);
  if (need > lo && vals)
    zig_emit_vals_kernel<<<(unsigned)std::min<int64_t>(tiles, 8LL * sms), kZThreads, 0, st>>>(
        P0, tiles, gskip, gacc, offs, lo, need, out, bits, vals, base);
  else if (need > lo)
    zig_emit_kernel<<<(unsigned)std::min<int64_t>(tiles, 8LL * sms), kZThreads, 0, st>>>(
        k0, k1, P0, tiles, gskip, gacc, offs, lo, need, __builtin_sqrt((double)w), out, bits,
        vals, base);
  int herr = 0;
  skb_readback rb(st);
  rb.add(total, offs + tiles, 8);
  rb.add(&herr, err, 4);
  if (rb.sync() != cudaSuccess) return SKB_ERR_CUDA;
  if (herr) return SKB_ERR_INTERNAL;  // an attempt longer than 64 words (never observed)
  return skb_launch_status("zig_generate");
}

// numpy's ziggurat consumes 1.0220 words per draw on average (fast-path
// acceptance 98.9%; slow attempts take extra words and may restart), with a
// relative spread ~1e-5 at 1e9 draws: 1 + 1/32 covers it with one pass.
static uint64_t zig_positions_for(uint64_t count) {
  const uint64_t p = count + count / 32 + 8 * (uint64_t)kZTile;
  return (p + kZTile - 1) / kZTile * kZTile;
}

}  // namespace skb

using namespace skb;

// W = draws [lo, count) of standard_normal / sqrt(w) (row-major n x w when
// lo = 0, count = n*w; a rank's row block with lo = j0*w, count = j1*w).
// Synchronises the stream.
extern "C" int skb_gaussian_sketch(uint64_t key0, uint64_t key1, int64_t lo, int64_t count,
                                   int32_t w, double* W, void* workspace, size_t ws_bytes,
                                   void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (count < 0 || lo < 0 || lo > count || w < 1) return SKB_ERR_ARG;
  if (count == lo) return 0;
  uint64_t positions = zig_positions_for((uint64_t)count);
  for (int attempt = 0; attempt < 4; ++attempt) {
    skb_ws ws = skb_ws_make(workspace, ws_bytes);
    uint64_t total = 0;
    const int rc = zig_generate(key0, key1, 0, positions, (uint64_t)lo, (uint64_t)count, w, W,
                                &total, &ws, st);
    if (rc) return rc;
    if (total >= (uint64_t)count) return 0;
    positions = (positions + positions / 16 + kZTile - 1) / kZTile * kZTile;  // (never observed)
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
  return zig_generate(key0, key1, p0, p1, 0, (uint64_t)cap, w, out, count_host, &ws, st);
}

// Workspace for `count` draws (or a range of ~count positions): the slow
// bitmap, consumed / accepted bitmaps, counts, offsets and the scan scratch.
// The stored-values mode's extra workspace (8 bytes per stream position): add it
// to skb_gaussian_workspace_bytes when device memory allows; without it the
// generator runs Philox twice instead.
extern "C" size_t skb_gaussian_value_bytes(int64_t count) {
  const uint64_t p = zig_positions_for((uint64_t)std::max<int64_t>(count, 1));
  const uint64_t pos = p + p / 16 + (uint64_t)(kZHaloTiles + 1) * kZTile;  // one retry's growth
  return (size_t)pos * 8 + (1u << 20);
}

extern "C" size_t skb_gaussian_workspace_bytes(int64_t count) {
  const uint64_t pos = zig_positions_for((uint64_t)std::max<int64_t>(count, 1)) * 2 +
                       (uint64_t)kZHaloTiles * kZTile;
  const uint64_t tiles = pos / kZTile + 2;
  return (size_t)(pos / 32 * 4 + tiles * kZWords * 8 + tiles * 16) + (1u << 20);
}
