// K3e core: batched INT8 x INT8 -> INT32 GEMM on the 5th-generation tensor
// cores (tcgen05.mma kind::i8, accumulators in TMEM, operands staged by TMA).
//
// The FP64-on-INT8 emulation (skb_ozaki.cu, CRT / Ozaki scheme II) reduces one
// FP64 product to n (12..20) exact INT8 products, one per modulus:
//   C_l (rows x cols, int32, row-major) = A_l (rows x K) * B_l (cols x K)^T
// with both operands K-major int8 residue slabs. This kernel is that batch.
// Replaces the cuBLASLt call of round 1 (the reference operations behind it:
// preconditioning.py:46 gesdd's products, sketching.py:158-159 AD @ W).
//
// Structure (one 128 x 256 output tile per CTA, grid.z = modulus):
//   * a 3-D TMA tensor map per operand ({K, rows, modulus}, 128-byte boxes,
//     SWIZZLE_128B) fills a 4-stage shared-memory ring (16 KB A + 32 KB B per
//     stage) behind full/empty mbarriers; one elected thread issues the loads;
//   * one elected thread issues tcgen05.mma.cta_group::1.kind::i8
//     (M = 128, N = 256, K = 32; four per 128-byte stage) into a 256-column
//     TMEM accumulator and returns each stage with tcgen05.commit;
//   * after the last commit the four warps read their 32 TMEM lanes
//     (tcgen05.ld 32x32b.x32) and store the int32 tile.
// One CTA per SM (the ring takes 193 KB); at the emulation's sizes the grid
// covers the 148 SMs many times over.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "skb_common.cuh"
#include "skb_internal.h"

namespace skb {
namespace i8 {

constexpr int BM = 128, BN = 256, BK = 128, NST = 4;
constexpr int A_BYTES = BM * BK, B_BYTES = BN * BK, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM_BYTES = NST * STAGE_BYTES + 1024;  // + 1 KB for 1024-byte alignment
constexpr int TMEM_COLS = BN;                         // int32 accumulator columns

// Instruction descriptor (kind::i8): D s32, A s8, B s8, both K-major, M=128, N=256.
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

// Shared-memory matrix descriptor: K-major, SWIZZLE_128B (rows of 128 bytes,
// 8-row swizzle atoms 1024 bytes apart), sm_100 version bit.
SKB_DEV uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

SKB_DEV void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                         int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

SKB_DEV void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(
          tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate), "r"(0u), "r"(0u), "r"(0u), "r"(0u));
}

SKB_DEV void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__global__ void __launch_bounds__(128, 1)
    i8gemm_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                  int32_t* __restrict__ C, int64_t ldc, int64_t mstride, int rows, int cols,
                  int arow0, int brow0, int kb0, int nkb) {
  extern __shared__ uint8_t smraw[];
  __shared__ __align__(8) uint64_t full[NST], empty[NST], done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = (smem_u32(smraw) + 1023u) & ~1023u;
  const int tm = blockIdx.y, tn = blockIdx.x, z = blockIdx.z;

  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
  }
  if (warp == 0) {  // the whole warp allocates TMEM (and later frees it)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;

  if (tid == 0) {  // ------------------------------------------------ TMA producer
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % NST;
      if (kb >= NST) mbar_wait(&empty[s], (uint32_t)(((kb / NST) - 1) & 1));
      mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
      const uint32_t sa = sbase + s * STAGE_BYTES;
      const int k = kb0 + kb * BK;
      tma_load_3d(sa, &ta, &full[s], k, arow0 + tm * BM, z);
      tma_load_3d(sa + A_BYTES, &tb, &full[s], k, brow0 + tn * BN, z);
    }
  } else if (tid == 32) {  // ------------------------------------------ MMA issuer
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % NST;
      mbar_wait(&full[s], (uint32_t)((kb / NST) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t sa = sbase + s * STAGE_BYTES, sb = sa + A_BYTES;
#pragma unroll
      for (int k = 0; k < BK / 32; ++k)  // K = 32 bytes per MMA, inside the 128-byte row
        mma_i8(tmem, sdesc(sa + 32 * k), sdesc(sb + 32 * k), (kb | k) != 0 ? 1u : 0u);
      mma_commit(&empty[s]);  // the stage returns to the producer once these MMAs are done
    }
    mma_commit(&done);
  }
  __syncwarp();

  // ------------------------------------------------------------- epilogue
  mbar_wait(&done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = tm * BM + warp * 32 + lane;
  int32_t* crow = C + (int64_t)z * mstride + (int64_t)row * ldc + (int64_t)tn * BN;
  const int cmax = cols - tn * BN;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 32) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
        "%28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
          "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (row < rows) {
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (c0 + 4 * q < cmax)  // cols is a multiple of 16: 4-column groups are whole
          *reinterpret_cast<int4*>(crow + c0 + 4 * q) =
              make_int4((int)v[4 * q], (int)v[4 * q + 1], (int)v[4 * q + 2], (int)v[4 * q + 3]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(TMEM_COLS)
                 : "memory");
}

}  // namespace i8
}  // namespace skb

// ---------------------------------------------------------------- 2-SM
// The same batch with CTA pairs (cluster 2x1x1, tcgen05 cta_group::2): one
// 256 x 256 output tile per pair, M = 256 per MMA. Each CTA stages half of the
// A rows and half of the B rows (16 + 16 KB per 128-byte K block, 6 stages),
// both CTAs' TMA loads complete on the leader's full barrier, the leader
// alone issues the MMAs, and its commits arrive on both CTAs' empty / done
// barriers (multicast). Each CTA's TMEM holds its 128 rows x 256 columns.
namespace skb {
namespace i8 {

constexpr int P_BM = 256, P_BN = 256, P_NST = 6;
constexpr int P_A_BYTES = 128 * BK, P_B_BYTES = 128 * BK, P_STAGE = P_A_BYTES + P_B_BYTES;
constexpr int P_SMEM_BYTES = P_NST * P_STAGE + 1024;
constexpr uint32_t kIdesc2 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(P_BN >> 3) << 17) |
                             ((uint32_t)(P_BM >> 4) << 24);

SKB_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
SKB_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    i8gemm2_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                   int32_t* __restrict__ C, int64_t ldc, int64_t mstride, int rows, int cols,
                   int arow0, int brow0, int kb0, int nkb) {
  extern __shared__ uint8_t smraw[];
  __shared__ __align__(8) uint64_t full[P_NST], empty[P_NST], done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();
  const uint32_t sbase = (smem_u32(smraw) + 1023u) & ~1023u;
  const int tn = blockIdx.x >> 1, tm = blockIdx.y, z = blockIdx.z;

  if (tid == 0) {
    for (int s = 0; s < P_NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;

  if (tid == 0) {  // ------------------------------------------ TMA producer (both CTAs)
    const int arow = arow0 + tm * P_BM + (int)rank * 128, brow = brow0 + tn * P_BN + (int)rank * 128;
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % P_NST;
      if (kb >= P_NST) mbar_wait(&empty[s], (uint32_t)(((kb / P_NST) - 1) & 1));
      const uint32_t lead_full = smem_u32(&full[s]) & 0xFEFFFFFFu;  // the leader's barrier
      if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * P_STAGE);
      const uint32_t sa = sbase + s * P_STAGE;
      const int k = kb0 + kb * BK;
      asm volatile(
          "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(sa),
          "l"(reinterpret_cast<uint64_t>(&ta)), "r"(lead_full), "r"(k), "r"(arow), "r"(z)
          : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(sa + P_A_BYTES),
          "l"(reinterpret_cast<uint64_t>(&tb)), "r"(lead_full), "r"(k), "r"(brow), "r"(z)
          : "memory");
    }
  } else if (tid == 32 && rank == 0) {  // ----------------------- MMA issuer (leader)
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % P_NST;
      mbar_wait(&full[s], (uint32_t)((kb / P_NST) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t sa = sbase + s * P_STAGE, sb = sa + P_A_BYTES;
#pragma unroll
      for (int k = 0; k < BK / 32; ++k) {
        const uint32_t acc = (kb | k) != 0 ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, "
            "%5}, p;\n\t}" ::"r"(tmem),
            "l"(sdesc(sa + 32 * k)), "l"(sdesc(sb + 32 * k)), "r"(kIdesc2), "r"(acc), "r"(0u));
      }
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
          " [%0], %1;" ::"r"(smem_u32(&empty[s])),
          "h"((uint16_t)3)
          : "memory");
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(smem_u32(&done)),
        "h"((uint16_t)3)
        : "memory");
  }
  __syncwarp();

  // ------------------------------------------------------------- epilogue
  mbar_wait(&done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = tm * P_BM + (int)rank * 128 + warp * 32 + lane;
  int32_t* crow = C + (int64_t)z * mstride + (int64_t)row * ldc + (int64_t)tn * P_BN;
  const int cmax = cols - tn * P_BN;
#pragma unroll 1
  for (int c0 = 0; c0 < P_BN; c0 += 32) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
        "%28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
          "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (row < rows) {
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (c0 + 4 * q < cmax)
          *reinterpret_cast<int4*>(crow + c0 + 4 * q) =
              make_int4((int)v[4 * q], (int)v[4 * q + 1], (int)v[4 * q + 2], (int)v[4 * q + 3]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // both CTAs done with TMEM and barriers
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(TMEM_COLS)
                 : "memory");
}

// -------------------------------------------------- 2-SM, persistent
// Persistent CTA pairs over a static tile schedule (tile t = cluster +
// i * clusters, grouped order below). NB = 1: 256 x 256 pair tiles and two
// 256-column TMEM accumulators, so the epilogue of tile i overlaps the main
// loop of tile i+1. NB = 2: 256 x 512 pair tiles (two N = 256 MMAs per K step
// sharing the staged A), one 512-column accumulator: a third less operand
// traffic per MAC through L2 (the INT8 pipe outruns L2 -> SM at 256 x 256),
// for long K where the exposed epilogue is a few percent.
//   warps 0-3  epilogue (TMEM lanes 0-127 -> int32 tile), release the
//              accumulator to the leader (remote mbarrier arrive from CTA 1)
//   warp 4     TMA producer (both CTAs: their A half and B halves)
//   warp 5     MMA issuer (leader CTA only)
constexpr int Q_THREADS = 192;
constexpr int Q_TMEM_COLS = 512;

SKB_DEV void arrive_cluster(uint64_t* local_bar, uint32_t target_rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(local_bar)),
               "r"(target_rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(r) : "memory");
}

// Tile order: per modulus, groups of kGM tile rows; inside a group tm runs
// fastest, then tn. The ~74 co-resident pairs then cover a ~8 x 9 block of
// (tm, tn), so every A and B K-slice they stream is shared by ~8 pairs while
// in L2 (row-major order would re-read each B panel from HBM per tile row).
// With tri = 1 only tiles meeting the lower triangle col <= row + tri_off
// exist, and the enumeration is compact over them (no idle pairs).
constexpr int kGM = 8;
SKB_DEV int tri_tmin(int tn, int bn, int tri, int tri_off) {  // first tile row reaching tn
  if (!tri) return 0;
  const int v = tn * bn - (P_BM - 1) - tri_off;
  return v <= 0 ? 0 : (v + P_BM - 1) / P_BM;
}
SKB_DEV int group_col_count(int g0, int gm, int tn, int bn, int tri, int tri_off) {
  const int lo = max(g0, tri_tmin(tn, bn, tri, tri_off));
  return max(0, g0 + gm - lo);
}
SKB_DEV int tiles_per_z(int TM, int TN, int bn, int tri, int tri_off) {
  int tot = 0;
  for (int g0 = 0; g0 < TM; g0 += kGM)
    for (int tn = 0; tn < TN; ++tn)
      tot += group_col_count(g0, min(kGM, TM - g0), tn, bn, tri, tri_off);
  return tot;
}
SKB_DEV void decode_tile(int t, int TM, int TN, int bn, int per_z, int tri, int tri_off, int& z,
                         int& tm, int& tn) {
  z = t / per_z;
  int r = t - z * per_z;
  for (int g0 = 0; g0 < TM; g0 += kGM) {
    const int gm = min(kGM, TM - g0);
    for (tn = 0; tn < TN; ++tn) {
      const int c = group_col_count(g0, gm, tn, bn, tri, tri_off);
      if (r < c) {
        tm = max(g0, tri_tmin(tn, bn, tri, tri_off)) + r;
        return;
      }
      r -= c;
    }
  }
  tm = tn = 0;  // not reached
}

template <int NB>
struct PCfg {
  static constexpr int BN = 256 * NB;                  // pair tile columns
  static constexpr int NST = NB == 1 ? 6 : 4;           // stages
  static constexpr int A = 128 * BK, B = 128 * NB * BK;  // per-CTA bytes per K block
  static constexpr int STAGE = A + B;
  static constexpr int SMEM = NST * STAGE + 1024;
  static constexpr int NACC = NB == 1 ? 2 : 1;          // TMEM accumulators
};

// Residue epilogue (res.on): instead of the int32 products, store their symmetric
// residues mod p_z as int8 (r = c - rint(c / p) p, exact: |c| < 2^31, and a
// non-tie quotient is >= 0.5/p from a half-integer; p = 256 ties store -128),
// so the CRT reads 1 byte per product instead of 4 (skb_ozaki.cu).
struct ResMod {
  int on;
  double p[24], pinv[24];
};

template <int NB>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Q_THREADS, 1)
    i8gemm2p_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                    int32_t* __restrict__ C, int64_t ldc, int64_t mstride, int rows, int cols,
                    int arow0, int brow0, int kb0, int nkb, int TM, int TN, int nz, int tri,
                    int tri_off, const __grid_constant__ ResMod res) {
  using Cfg = PCfg<NB>;
  extern __shared__ uint8_t smraw[];
  __shared__ __align__(8) uint64_t full[Cfg::NST], empty[Cfg::NST], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();
  const uint32_t sbase = (smem_u32(smraw) + 1023u) & ~1023u;
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int per_z = tiles_per_z(TM, TN, Cfg::BN, tri, tri_off);
  const int ntiles = per_z * nz;

  if (tid == 0) {
    for (int s = 0; s < Cfg::NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);  // 4 epilogue warps x 2 CTAs
    }
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "n"(Q_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;

  if (warp == 4) {  // ------------------------------------------------ TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int64_t it = 0;
      for (int t = cl; t < ntiles; t += ncl) {
        int z, tm, tn;
        decode_tile(t, TM, TN, Cfg::BN, per_z, tri, tri_off, z, tm, tn);
        const int arow = arow0 + tm * P_BM + (int)rank * 128;
        const int brow = brow0 + tn * Cfg::BN + (int)rank * 128;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          if (it >= Cfg::NST) mbar_wait(&empty[s], ph ^ 1);
          const uint32_t lead_full = smem_u32(&full[s]) & 0xFEFFFFFFu;
          if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * Cfg::STAGE);
          const uint32_t sa = sbase + s * Cfg::STAGE;
          const int k = kb0 + kb * BK;
          asm volatile(
              "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx"
              "::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(sa),
              "l"(reinterpret_cast<uint64_t>(&ta)), "r"(lead_full), "r"(k), "r"(arow), "r"(z)
              : "memory");
#pragma unroll
          for (int h = 0; h < NB; ++h)  // B rows of MMA h: [h*256 + rank*128, +128)
            asm volatile(
                "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::"
                "complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(sa + Cfg::A +
                                                                           h * 128 * BK),
                "l"(reinterpret_cast<uint64_t>(&tb)), "r"(lead_full), "r"(k),
                "r"(brow + h * 256), "r"(z)
                : "memory");
          if (++s == Cfg::NST) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 5) {  // ------------------------------------- MMA issuer (leader)
    if (lane == 0 && rank == 0) {
      int s = 0;
      uint32_t ph = 0;
      int i = 0;
      for (int t = cl; t < ntiles; t += ncl, ++i) {
        const int b = Cfg::NACC == 2 ? (i & 1) : 0;
        const int use = Cfg::NACC == 2 ? (i >> 1) : i;  // prior uses of this accumulator
        if (use >= 1) mbar_wait(&tempty[b], (uint32_t)((use - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc_t = tmem + (uint32_t)(b * 256);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = sbase + s * Cfg::STAGE, sb = sa + Cfg::A;
#pragma unroll
          for (int k = 0; k < BK / 32; ++k) {
            const uint32_t acc = (kb | k) != 0 ? 1u : 0u;
#pragma unroll
            for (int h = 0; h < NB; ++h)
              asm volatile(
                  "{\n\t.reg .pred p;\n\t"
                  "setp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, "
                  "%5, %5}, p;\n\t}" ::"r"(acc_t + (uint32_t)(h * 256)),
                  "l"(sdesc(sa + 32 * k)), "l"(sdesc(sb + h * 128 * BK + 32 * k)),
                  "r"(kIdesc2), "r"(acc), "r"(0u));
          }
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::"
              "cluster.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])),
              "h"((uint16_t)3)
              : "memory");
          if (++s == Cfg::NST) {
            s = 0;
            ph ^= 1;
          }
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster"
            ".b64 [%0], %1;" ::"r"(smem_u32(&tfull[b])),
            "h"((uint16_t)3)
            : "memory");
      }
    }
  } else {  // ------------------------------------------------ epilogue (warps 0-3)
    int i = 0;
    for (int t = cl; t < ntiles; t += ncl, ++i) {
      int z, tm, tn;
      decode_tile(t, TM, TN, Cfg::BN, per_z, tri, tri_off, z, tm, tn);
      const int b = Cfg::NACC == 2 ? (i & 1) : 0;
      const int use = Cfg::NACC == 2 ? (i >> 1) : i;
      mbar_wait(&tfull[b], (uint32_t)(use & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row = tm * P_BM + (int)rank * 128 + warp * 32 + lane;
      int32_t* crow = res.on ? C
                             : C + (int64_t)z * mstride + (int64_t)row * ldc + (int64_t)tn * Cfg::BN;
      const int cmax = cols - tn * Cfg::BN;
#pragma unroll 1
      for (int c0 = 0; c0 < Cfg::BN; c0 += 32) {
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(b * 256 + c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, "
            "%10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, "
            "%26, %27, %28, %29, %30, %31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
              "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
              "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
              "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row < rows) {
          if (res.on) {  // int8 residues: C is a byte slab (ldc, mstride in bytes)
            const double pz = res.p[z], piz = res.pinv[z];
            constexpr double kMg = 6755399441055744.0;  // 1.5 * 2^52
            uint32_t w[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              uint32_t bytes[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const double dd = (double)(int)v[4 * q + u];
                const double qq = fma(dd, piz, kMg) - kMg;
                bytes[u] = (uint32_t)__double2loint(fma(-qq, pz, dd) + kMg);
              }
              w[q] = __byte_perm(__byte_perm(bytes[0], bytes[1], 0x0040),
                                 __byte_perm(bytes[2], bytes[3], 0x0040), 0x5410);
            }
            int8_t* c8 = reinterpret_cast<int8_t*>(C) + (int64_t)z * mstride +
                         (int64_t)row * ldc + (int64_t)tn * Cfg::BN + c0;
            if (c0 < cmax) *reinterpret_cast<uint4*>(c8) = make_uint4(w[0], w[1], w[2], w[3]);
            if (c0 + 16 < cmax)
              *reinterpret_cast<uint4*>(c8 + 16) = make_uint4(w[4], w[5], w[6], w[7]);
          } else {
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (c0 + 4 * q < cmax)
                *reinterpret_cast<int4*>(crow + c0 + 4 * q) =
                    make_int4((int)v[4 * q], (int)v[4 * q + 1], (int)v[4 * q + 2],
                              (int)v[4 * q + 3]);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) arrive_cluster(&tempty[b], 0);  // the accumulator is free again
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(Q_TMEM_COLS)
                 : "memory");
}

}  // namespace i8
}  // namespace skb

namespace skb {
namespace i8 {
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encoder() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeFn)p;
  });
  return fn;
}

// {K, rows, batch} int8 slab: row stride ld bytes, batch stride bs bytes.
static bool make_map(CUtensorMap* m, const int8_t* base, int64_t K, int64_t R, int64_t nb,
                     int64_t ld, int64_t bs, int box_rows) {
  EncodeFn enc = encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)R, (cuuint64_t)nb};
  const cuuint64_t strides[2] = {(cuuint64_t)ld, (cuuint64_t)bs};
  const cuuint32_t box[3] = {(cuuint32_t)BK, (cuuint32_t)box_rows, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)base, dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

}  // namespace i8
}  // namespace skb

using namespace skb;

// C_l[r][c] (int32, row stride ldc, batch stride sc) = sum_k A_l[ar0 + r][k] B_l[br0 + c][k]
// over k in [k0, k1) for l < n, r < rows, c < cols. A / B: K-major int8 slabs with
// Kp bytes per row, Ra / Rb rows and batch strides sa / sb; k0 % 128 == 0, k1 <= Kp,
// and the slab entries in [k0, k1) outside the caller's range must be zero
// (the K tail is rounded up to whole 128-byte boxes; past Kp TMA fills zeros).
// cols % 16 == 0. tri = 1: only the tiles meeting the lower triangle col <= row
// + tri_off are computed (the others are left untouched; persistent 2-SM path).
// Returns 0, or SKB_ERR_* (no CPU or library fallback).
static int i8gemm_run(const int8_t* A, int64_t Ra, int64_t sa, const int8_t* B, int64_t Rb,
                      int64_t sb, int64_t Kp, int32_t* C, int64_t ldc, int64_t sc, int32_t rows,
                      int32_t cols, int32_t ar0, int32_t br0, int32_t k0, int32_t k1, int32_t n,
                      int32_t tri, int32_t tri_off, const skb::i8::ResMod& res, void* stream) {
  using namespace skb::i8;
  if (rows <= 0 || cols <= 0 || n <= 0) return 0;
  if (k1 <= k0 || (k0 % BK) || (cols % 16) || (Kp % 16) || ((uintptr_t)A & 15) ||
      ((uintptr_t)B & 15) || (ldc % (res.on ? 16 : 4)) || (sc % (res.on ? 16 : 4)) ||
      ((uintptr_t)C & 15) || (res.on && n > 24))
    return SKB_ERR_ARG;
  CUtensorMap ma, mb;
  static const bool one_sm0 = getenv("SKB_I8_1SM") && getenv("SKB_I8_1SM")[0] == '1';
  if (!make_map(&ma, A, Kp, Ra, n, Kp, sa, one_sm0 ? BM : 128) ||
      !make_map(&mb, B, Kp, Rb, n, Kp, sb, one_sm0 ? BN : 128))
    return SKB_ERR_CUDA;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(i8gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(i8gemm2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             P_SMEM_BYTES) != cudaSuccess)
      return SKB_ERR_CUDA;
    configured = true;
  }
  const int nkb = (k1 - k0 + BK - 1) / BK;
  static const bool one_sm = getenv("SKB_I8_1SM") && getenv("SKB_I8_1SM")[0] == '1';
  if (!res.on && one_sm) {
    dim3 grid((unsigned)((cols + BN - 1) / BN), (unsigned)((rows + BM - 1) / BM), (unsigned)n);
    i8gemm_kernel<<<grid, 128, SMEM_BYTES, (cudaStream_t)stream>>>(ma, mb, C, ldc, sc, rows,
                                                                   cols, ar0, br0, k0, nkb);
  } else if (!res.on && getenv("SKB_I8_NP") && getenv("SKB_I8_NP")[0] == '1') {  // non-persistent
    dim3 grid((unsigned)(2 * ((cols + P_BN - 1) / P_BN)), (unsigned)((rows + P_BM - 1) / P_BM),
              (unsigned)n);
    i8gemm2_kernel<<<grid, 128, P_SMEM_BYTES, (cudaStream_t)stream>>>(ma, mb, C, ldc, sc, rows,
                                                                      cols, ar0, br0, k0, nkb);
  } else {
    static bool cfg2 = false;
    if (!cfg2) {
      if (cudaFuncSetAttribute(i8gemm2p_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               PCfg<1>::SMEM) != cudaSuccess ||
          cudaFuncSetAttribute(i8gemm2p_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               PCfg<2>::SMEM) != cudaSuccess)
        return SKB_ERR_CUDA;
      cfg2 = true;
    }
    // 512-wide pair tiles when K is long enough to hide their exposed epilogue
    static const int wide_env = getenv("SKB_I8_WIDE") ? atoi(getenv("SKB_I8_WIDE")) : -1;
    const bool wide = wide_env >= 0 ? wide_env == 1 : (nkb >= 48 && cols > 256);
    const int bn = wide ? 512 : 256;
    const int TN = (cols + bn - 1) / bn, TM = (rows + P_BM - 1) / P_BM;
    int per_z = 0;  // tiles that exist (the kernel enumerates them compactly)
    for (int tm = 0; tm < TM; ++tm) {
      const int last = tm * P_BM + P_BM - 1 + tri_off;
      per_z += !tri ? TN : (last < 0 ? 0 : std::min(TN, last / bn + 1));
    }
    if (per_z == 0) return 0;
    const int pairs = std::max(1, std::min(skb_num_sms() / 2, per_z * n));
    if (wide)
      i8gemm2p_kernel<2><<<2 * pairs, Q_THREADS, PCfg<2>::SMEM, (cudaStream_t)stream>>>(
          ma, mb, C, ldc, sc, rows, cols, ar0, br0, k0, nkb, TM, TN, n, tri ? 1 : 0, tri_off,
          res);
    else
      i8gemm2p_kernel<1><<<2 * pairs, Q_THREADS, PCfg<1>::SMEM, (cudaStream_t)stream>>>(
          ma, mb, C, ldc, sc, rows, cols, ar0, br0, k0, nkb, TM, TN, n, tri ? 1 : 0, tri_off,
          res);
  }
  return skb_launch_status("skb_i8gemm");
}

extern "C" int skb_i8gemm_batched(const int8_t* A, int64_t Ra, int64_t sa, const int8_t* B,
                                  int64_t Rb, int64_t sb, int64_t Kp, int32_t* C, int64_t ldc,
                                  int64_t sc, int32_t rows, int32_t cols, int32_t ar0,
                                  int32_t br0, int32_t k0, int32_t k1, int32_t n, int32_t tri,
                                  int32_t tri_off, void* stream) {
  skb::i8::ResMod res{};
  return i8gemm_run(A, Ra, sa, B, Rb, sb, Kp, C, ldc, sc, rows, cols, ar0, br0, k0, k1, n, tri,
                    tri_off, res, stream);
}

// As skb_i8gemm_batched, but each product is stored as its symmetric residue mod
// mod[l] (int8 slab C8: row stride ldc8 and batch stride sc8 in bytes, multiples
// of 16): the FP64 emulation's CRT then reads one byte per product. Persistent
// 2-SM kernel only; n <= 24.
extern "C" int skb_i8gemm_residues(const int8_t* A, int64_t Ra, int64_t sa, const int8_t* B,
                                   int64_t Rb, int64_t sb, int64_t Kp, int8_t* C8, int64_t ldc8,
                                   int64_t sc8, int32_t rows, int32_t cols, int32_t ar0,
                                   int32_t br0, int32_t k0, int32_t k1, int32_t n, int32_t tri,
                                   int32_t tri_off, const double* mod, void* stream) {
  if (n > 24) return SKB_ERR_ARG;
  skb::i8::ResMod res{};
  res.on = 1;
  for (int l = 0; l < n; ++l) {
    res.p[l] = mod[l];
    res.pinv[l] = 1.0 / mod[l];
  }
  return i8gemm_run(A, Ra, sa, B, Rb, sb, Kp, reinterpret_cast<int32_t*>(C8), ldc8, sc8, rows,
                    cols, ar0, br0, k0, k1, n, tri, tri_off, res, stream);
}
