// Planned CSC passes (K4c): every A-pass of a sparse LP that produces an
// m-vector (normal operator, gemv, rhs, directions, iterate), without atomics.
// Included by skb_stream.cu (shares its Op family and reduce_partials_kernel).
//
// A is fixed for the whole solve, so a one-time plan per matrix reorganises
// it into chunks of whole columns sized to a shared-memory stage (column j
// weighs 12 B per entry + 10 B). Per chunk the plan stream holds, 16-byte
// aligned and contiguous:
//   vals  (8 B/entry, CSC order; each region padded to 16 bytes)
//   rp32  (4 B/entry: row (u16) | position of the entry in the chunk's
//          row-sorted order (u16) << 16)
//   coff  (2 B/column: first entry of each column, chunk-local)
// plus a header with 33 cut points of the row-sorted order at the row
// boundaries w * m / 32. A pass then streams 12 B/entry + 10 B/column --
// the CSC roofline's algorithmic bytes -- through a TMA bulk-copy ring
// (cp.async.bulk + mbarrier; the op's first n-vector (d2, x, ...) rides in
// the same stage) and, per chunk,
//   pass 1  (4 lanes per column)  dot = sum vals * z[row] (strided fma per
//           lane, fixed xor tree across the 4), the op's coefficient and
//           elementwise outputs; each product cf * val lands at its
//           row-sorted slot;
//   pass 2  (warp per row range)  the products in row order: each run of a
//           row is summed into its last lane, which adds one value per row
//           into the CTA's m-vector partial. Warp ranges (the plan's cut
//           points) start at row boundaries: rows are disjoint across warps,
//           no atomics.
// Pass 1 of chunk k+1 and pass 2 of chunk k run in the same phase (one
// barrier per chunk). Summation order is fixed by the plan: deterministic.
#pragma once

namespace skb {

constexpr int kCpNS = 3;                   // stages in the bulk-copy ring
constexpr int kCpHdr = 128;                // chunk header bytes (first in a stage)
constexpr int kCpSmemMax = 232448;         // opt-in dynamic shared memory per CTA
constexpr int kCpMaxSB = 256 + 12 * 2047;  // sorted positions fit 11 bits

struct CscChunk {   // 128 bytes
  int64_t j0;       // first column
  int32_t nc;       // columns
  int32_t sbytes;   // stream bytes of this chunk (multiple of 16)
  int64_t soff;     // byte offset of the chunk's stream data in the plan
  int32_t ne;       // entries
  int32_t pad0;
  uint16_t cut[33];
  uint16_t pad1[15];
};
static_assert(sizeof(CscChunk) == kCpHdr, "chunk header layout");

struct CscPlanHdr {  // first 256 bytes of the plan buffer
  int64_t magic, m, n, nnz, nchunks, wb, sb, stream_off;
};
constexpr int64_t kCscPlanMagic = 0x534b42435343504cll;  // "SKBCSCPL"

__host__ __device__ inline int64_t cscp_pad16(int64_t b) { return (b + 15) & ~(int64_t)15; }

// stage bytes for a shared-memory budget: 3 stages + 2 product buffers of
// (8 + 2) B per entry, entries <= (sb - 256) / 12
inline int64_t cscp_stage_bytes(int64_t m, bool dot) {
  const int64_t mp = (m + 1) & ~(int64_t)1;
  const int64_t fixed = (dot ? 16 : 8) * mp + 1024;
  const int64_t budget = kCpSmemMax - fixed;
  // kCpNS * sb + 2 * 10 * (sb - 256) / 12 <= budget
  int64_t sb = (budget + 2 * 10 * 256 / 12) * 12 / (12 * kCpNS + 20);
  sb &= ~(int64_t)15;
  return sb > kCpMaxSB ? (int64_t)kCpMaxSB & ~(int64_t)15 : sb;
}

inline size_t cscp_smem(int m, bool dot, int64_t sb) {
  const int64_t mp = (m + 1) & ~1;
  const int64_t emax = (sb - 256) / 12;
  return (size_t)((dot ? mp : 0) + mp) * 8 + (size_t)kCpNS * sb + (size_t)2 * emax * 10 +
         2 * 33 * 4 + 8 * (2 * kCpNS + 4) + 64;
}

__global__ void cscp_bounds_kernel(const int64_t* __restrict__ colptr, int64_t n, int64_t wb,
                                   int64_t nchunks, CscChunk* __restrict__ ch) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  // first j in [0, n] with 12 (colptr[j] - colptr[0]) + 10 j >= c wb (monotone in j)
  const int64_t key = c * wb, base = colptr[0];
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (12 * (colptr[mid] - base) + 10 * mid >= key) hi = mid; else lo = mid + 1;
  }
  ch[c].j0 = lo;
}

constexpr int kCpSortT = 512, kCpSortIPT = 4;  // 2048 keys per chunk at most

__global__ void __launch_bounds__(kCpSortT)
    cscp_build_kernel(const int64_t* __restrict__ colptr, const int32_t* __restrict__ rowidx,
                      const double* __restrict__ vals, int64_t m, int64_t n, int64_t nchunks,
                      int64_t sb,
                      CscChunk* __restrict__ ch, uint8_t* __restrict__ stream) {
  using Sort = cub::BlockRadixSort<uint32_t, kCpSortT, kCpSortIPT>;
  __shared__ typename Sort::TempStorage tmp;
  __shared__ uint32_t keys_s[kCpSortT * kCpSortIPT];
  __shared__ uint16_t inv_s[kCpSortT * kCpSortIPT];
  const int64_t c = blockIdx.x;
  const int64_t j0 = ch[c].j0, j1 = (c + 1 < nchunks) ? ch[c + 1].j0 : n;
  const int64_t e0 = colptr[j0];
  const int ne = (int)(colptr[j1] - e0), nc = (int)(j1 - j0);
  uint8_t* sp = stream + c * sb;
  double* sv = reinterpret_cast<double*>(sp);
  uint32_t* rp = reinterpret_cast<uint32_t*>(sp + cscp_pad16(8 * (int64_t)ne));
  uint16_t* co = reinterpret_cast<uint16_t*>(sp + cscp_pad16(8 * (int64_t)ne) +
                                             cscp_pad16(4 * (int64_t)ne));
  uint32_t k[kCpSortIPT];
#pragma unroll
  for (int q = 0; q < kCpSortIPT; ++q) {
    const int i = threadIdx.x * kCpSortIPT + q;  // blocked arrangement
    if (i < ne) {
      const uint32_t r = (uint32_t)rowidx[e0 + i];
      keys_s[i] = r;
      k[q] = (r << 11) | (uint32_t)i;
      sv[i] = vals[e0 + i];
    } else {
      k[q] = 0xFFFFFFFFu;
    }
  }
  for (int jl = threadIdx.x; jl < nc; jl += kCpSortT) co[jl] = (uint16_t)(colptr[j0 + jl] - e0);
  __syncthreads();
  Sort(tmp).Sort(k);
#pragma unroll
  for (int q = 0; q < kCpSortIPT; ++q) {
    const int pos = threadIdx.x * kCpSortIPT + q;
    if (pos < ne) inv_s[k[q] & 2047u] = (uint16_t)pos;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ne; i += kCpSortT) rp[i] = keys_s[i] | ((uint32_t)inv_s[i] << 16);
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kCpSortIPT; ++q) keys_s[threadIdx.x * kCpSortIPT + q] = k[q];
  __syncthreads();
  if (threadIdx.x <= 32) {  // cut w: first sorted position with row >= ceil(w m / 32)
    const uint32_t rb = (uint32_t)(((int64_t)threadIdx.x * m + 31) / 32);
    int lo = 0, hi = ne;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((keys_s[mid] >> 11) >= rb) hi = mid; else lo = mid + 1;
    }
    ch[c].cut[threadIdx.x] = (uint16_t)lo;
  }
  if (threadIdx.x == 0) {
    ch[c].nc = nc;
    ch[c].ne = ne;
    ch[c].sbytes = (int32_t)(cscp_pad16(8 * (int64_t)ne) + cscp_pad16(4 * (int64_t)ne) +
                             cscp_pad16(2 * (int64_t)nc));
    ch[c].soff = c * sb;
  }
}

// ------------------------------------------------------------ the pass
// Warp-specialised pipeline, one CTA per SM, persistent over its chunks:
//   warp 0            producer: TMA bulk copies of chunk k into stage k % NS
//                     (waits on empty[s]; headers prefetched two ahead)
//   kCpGW gather warps  pass 1 of chunk k (waits full[s] and pempty[b]),
//                     products into buffer b = k % 2, then arrives on
//                     empty[s] and pfull[b]
//   kCpSW scatter warps pass 2 of chunk k (waits pfull[b]), then pempty[b]
// Only scatter warps touch the m-vector partial, and scatter warp w owns the
// FIXED row block [w m / kCpSW, (w+1) m / kCpSW) in every chunk (the plan's
// cut points sit at multiples of m / 32), so warps working on different
// chunks never share a row: no atomics, fixed order.
constexpr int kCpGW = 8, kCpSW = 16;
constexpr int kCpThreads = 32 * (1 + kCpGW + kCpSW);

SKB_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <class Op>
__global__ void __launch_bounds__(kCpThreads, 1)
    cscp_kernel(const CscChunk* __restrict__ hdrs, const uint8_t* __restrict__ stream,
                int sb, int nchunks, int m, const double* __restrict__ z,
                double* __restrict__ part, Op op, const int* __restrict__ gate, int dbg) {
  if (gate && *gate) return;
  extern __shared__ __align__(128) uint8_t cpsm[];
  const int mp = (m + 1) & ~1;
  const int emax = (sb - 256) / 12;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint8_t* stages = cpsm;                                          // kCpNS * sb
  double* zs = reinterpret_cast<double*>(stages + kCpNS * sb);    // mp (kDot)
  double* us = zs + (Op::kDot ? mp : 0);                           // mp
  double* svb = us + mp;                                           // 2 * emax products
  uint16_t* srb = reinterpret_cast<uint16_t*>(svb + 2 * emax);     // 2 * emax rows
  int* cutb = reinterpret_cast<int*>(srb + 2 * emax + 2);          // 2 x 33 cut points
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(cutb + 66) + 7) & ~(uintptr_t)7);
  uint64_t* full = bars;                 // kCpNS
  uint64_t* empty = bars + kCpNS;        // kCpNS
  uint64_t* pfull = bars + 2 * kCpNS;    // 2
  uint64_t* pempty = bars + 2 * kCpNS + 2;  // 2

  if (Op::kDot)
    for (int i = tid; i < m; i += kCpThreads) zs[i] = z[i];
  for (int i = tid; i < m; i += kCpThreads) us[i] = 0.0;
  if (tid == 0) {
    for (int s = 0; s < kCpNS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 32 * kCpGW);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&pfull[b], 32 * kCpGW);
      mbar_init(&pempty[b], 32 * kCpSW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int grid = gridDim.x;
  const int nloc = nchunks > (int)blockIdx.x ? (nchunks - 1 - (int)blockIdx.x) / grid + 1 : 0;

  if (warp == 0) {  // ------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      int64_t hj[2] = {0, 0};
      int hn[2] = {0, 0}, hs[2] = {0, 0};
      auto hdr_load = [&](int kl, int q) {
        if (kl < nloc) {
          const int4 v = __ldg(reinterpret_cast<const int4*>(hdrs + blockIdx.x + (int64_t)kl * grid));
          hj[q] = ((int64_t)(uint32_t)v.y << 32) | (uint32_t)v.x;
          hn[q] = v.z;
          hs[q] = v.w;
        }
      };
      hdr_load(0, 0);
      hdr_load(1, 1);
      int s = 0;
      uint32_t ph = 0;
      for (int kl = 0; kl < nloc; ++kl) {
        if (kl >= kCpNS) mbar_wait(&empty[s], ph ^ 1);
        const int q = kl & 1;
        const int64_t c = blockIdx.x + (int64_t)kl * grid;
        uint8_t* stage = stages + s * sb;
        const uintptr_t a0 = reinterpret_cast<uintptr_t>(op.src(0) + hj[q]) & ~(uintptr_t)15;
        const uintptr_t a1 =
            reinterpret_cast<uintptr_t>(op.src(0) + hj[q] + hn[q]) & ~(uintptr_t)15;
        const uint32_t pbytes = a1 > a0 ? (uint32_t)(a1 - a0) : 0u;
        mbar_arrive_expect_tx(&full[s], (uint32_t)(kCpHdr + hs[q]) + pbytes);
        bulk_g2s(stage, hdrs + c, kCpHdr, &full[s], pol);
        if (hs[q]) bulk_g2s(stage + kCpHdr, stream + c * sb, (uint32_t)hs[q], &full[s], pol);
        if (pbytes)
          bulk_g2s(stage + kCpHdr + hs[q], reinterpret_cast<const void*>(a0), pbytes, &full[s],
                   pol);
        hdr_load(kl + 2, q);
        if (++s == kCpNS) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp <= kCpGW) {  // ---------------------------- gather (pass 1)
    const int gt = tid - 32;  // 0 .. 32*kCpGW-1
    int s = 0;
    uint32_t ph = 0;
    for (int kl = 0; kl < nloc; ++kl) {
      const int b = kl & 1;
      mbar_wait(&full[s], ph);
      if (kl >= 2) mbar_wait(&pempty[b], ((kl >> 1) - 1) & 1);
      const uint8_t* stage = stages + s * sb;
      const CscChunk* h = reinterpret_cast<const CscChunk*>(stage);
      const int64_t j0 = h->j0;
      const int nc = h->nc, ne = h->ne, sbytes = h->sbytes;
      const double* vs = reinterpret_cast<const double*>(stage + kCpHdr);
      const uint32_t* rp = reinterpret_cast<const uint32_t*>(stage + kCpHdr + cscp_pad16(8 * ne));
      const uint16_t* co = reinterpret_cast<const uint16_t*>(
          stage + kCpHdr + cscp_pad16(8 * ne) + cscp_pad16(4 * ne));
      const uintptr_t a0 = reinterpret_cast<uintptr_t>(op.src(0) + j0) & ~(uintptr_t)15;
      const uintptr_t a1 = reinterpret_cast<uintptr_t>(op.src(0) + j0 + nc) & ~(uintptr_t)15;
      const uint8_t* ps = stage + kCpHdr + sbytes;
      double* sv = svb + b * emax;
      uint16_t* sr = srb + b * emax;
      if (gt <= 32) cutb[b * 33 + gt] = h->cut[gt];
      if (dbg != 1)
        for (int jl = gt; jl < nc; jl += 32 * kCpGW) {
          const int64_t j = j0 + jl;
          const int a = co[jl], e1 = jl + 1 < nc ? co[jl + 1] : ne;
          Pre p;
          if (Op::kPre > 1) op.load(j, p);
          const uintptr_t aj = reinterpret_cast<uintptr_t>(op.src(0) + j);
          p.v[0] = aj < a1 ? *reinterpret_cast<const double*>(ps + (aj - a0)) : op.src(0)[j];
          double dot = 0.0;
          if (Op::kDot)
            for (int e = a; e < e1; ++e) dot = fma(vs[e], zs[rp[e] & 0xFFFFu], dot);
          const double cf = op.coef(j, p, dot);
          op.emit(j, p, dot, cf);
          if (Op::kAxpy)
            for (int e = a; e < e1; ++e) {
              const uint32_t w = rp[e];
              sv[w >> 16] = cf * vs[e];
              sr[w >> 16] = (uint16_t)(w & 0xFFFFu);
            }
        }
      mbar_arrive(&empty[s]);  // every lane: its reads of the stage and writes
      mbar_arrive(&pfull[b]);  // of products are released to the waiting roles
      if (++s == kCpNS) {
        s = 0;
        ph ^= 1;
      }
    }
  } else {  // ------------------------------------------------ scatter (pass 2)
    const int sw = warp - 1 - kCpGW;  // 0 .. kCpSW-1
    for (int kl = 0; kl < nloc; ++kl) {
      const int b = kl & 1;
      mbar_wait(&pfull[b], (kl >> 1) & 1);
      if (Op::kAxpy && dbg == 0) {
        const double* sv = svb + b * emax;
        const uint16_t* sr = srb + b * emax;
        const int* cut = cutb + b * 33;
        const int lo = cut[(sw * 32) / kCpSW], hi = cut[((sw + 1) * 32) / kCpSW];
        // lane l takes a contiguous piece of [lo, hi) starting at a row boundary:
        // each row's run is summed by one lane, sequentially
        int st = lo + (int)(((int64_t)lane * (hi - lo)) >> 5);
        while (st > lo && st < hi && sr[st] == sr[st - 1]) ++st;
        int en = __shfl_down_sync(0xffffffffu, st, 1);
        if (lane == 31) en = hi;
        int e = st;
        while (e < en) {
          const int r = sr[e];
          double acc = sv[e];
          for (++e; e < en && sr[e] == r; ++e) acc += sv[e];
          us[r] += acc;
        }
      }
      mbar_arrive(&pempty[b]);
    }
  }
  if (!Op::kAxpy) return;
  __syncthreads();
  for (int i = tid; i < m; i += kCpThreads) part[(size_t)blockIdx.x * m + i] = us[i];
}

struct CscPlanView {
  const CscChunk* ch;
  const uint8_t* stream;
  int64_t nchunks, sb;
};

// The host passes the plan's chunk count (from skb_csc_plan_build; the stage
// size follows from m) so no launch reads the plan header back.
static bool cscp_view(const void* plan, int64_t nchunks, int64_t m, CscPlanView* v) {
  const int64_t sb = m >= 1 && m <= 65535 ? cscp_stage_bytes(m, true) : 0;
  if (!plan || nchunks <= 0 || sb < 2048) return false;
  const uint8_t* base = (const uint8_t*)plan;
  v->ch = (const CscChunk*)(base + 256);
  v->stream = base + ((256 + nchunks * kCpHdr + 255) & ~(int64_t)255);
  v->nchunks = nchunks;
  v->sb = sb;
  return true;
}

template <class Op>
static int run_cscp(const CscPlanView& pv, int m, const double* z, double* out, const double* sub,
                    const Op& op, skb_ws* ws, cudaStream_t st, const int* gate) {
  const size_t smem = cscp_smem(m, Op::kDot, pv.sb);
  if (smem > (size_t)kCpSmemMax) return SKB_ERR_UNSUPPORTED;
  auto kern = cscp_kernel<Op>;
  static size_t configured = 0;
  if (smem > configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return SKB_ERR_CUDA;
    configured = smem;
  }
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(skb_num_sms(), pv.nchunks));
  double* part = nullptr;
  if (Op::kAxpy) {
    part = (double*)skb_ws_take(ws, (size_t)grid * m * 8);
    if (!part) return SKB_ERR_WORKSPACE;
  }
  static const int dbg = getenv("SKB_CSCP_DBG") ? atoi(getenv("SKB_CSCP_DBG")) : 0;
  kern<<<grid, kCpThreads, smem, st>>>(pv.ch, pv.stream, (int)pv.sb, (int)pv.nchunks, m, z, part,
                                       op, gate, dbg);
  if (Op::kAxpy)
    reduce_partials_kernel<<<(m + 31) / 32, 256, 0, st>>>(part, grid, m, sub, out, gate);
  return skb_launch_status(__func__);
}

}  // namespace skb

// Plan bytes for a CSC matrix (m rows, n columns, nnz entries, longest column
// maxlen); 0 when the planned passes do not apply (m > 65535, a column too long
// for a stage, or the m-vectors leave no shared memory for the ring).
extern "C" size_t skb_csc_plan_bytes(int64_t m, int64_t n, int64_t nnz, int64_t maxlen) {
  using namespace skb;
  if (m < 1 || m > 65535 || n < 1 || nnz < 0 || maxlen < 0) return 0;
  const int64_t sb = cscp_stage_bytes(m, true);
  const int64_t wmax = 12 * maxlen + 10;
  if (sb < 2048 || 2 * wmax >= sb - 256) return 0;
  const int64_t wb = sb - 256 - wmax;
  const int64_t nchunks = (12 * nnz + 10 * n + wb - 1) / wb;
  return (size_t)(((256 + nchunks * kCpHdr + 255) & ~(int64_t)255) + nchunks * sb);
}

// Build the plan (one pass over A + a per-chunk radix sort); *nchunks_out is
// passed back to every planned call.
extern "C" int skb_csc_plan_build(const int64_t* colptr, const int32_t* rowidx, const double* vals,
                                  int64_t m, int64_t n, int64_t nnz, int64_t maxlen, void* plan,
                                  size_t plan_bytes, int64_t* nchunks_out, void* stream) {
  using namespace skb;
  const size_t need = skb_csc_plan_bytes(m, n, nnz, maxlen);
  if (!need) return SKB_ERR_UNSUPPORTED;
  if (!plan || plan_bytes < need) return SKB_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  CscPlanHdr h;
  h.magic = kCscPlanMagic;
  h.m = m;
  h.n = n;
  h.nnz = nnz;
  h.sb = cscp_stage_bytes(m, true);
  h.wb = h.sb - 256 - (12 * maxlen + 10);
  h.nchunks = (12 * nnz + 10 * n + h.wb - 1) / h.wb;
  h.stream_off = (256 + h.nchunks * kCpHdr + 255) & ~(int64_t)255;
  uint8_t* base = (uint8_t*)plan;
  CscChunk* ch = (CscChunk*)(base + 256);
  if (cudaMemsetAsync(ch, 0, (size_t)h.nchunks * kCpHdr, st) != cudaSuccess) return SKB_ERR_CUDA;
  cscp_bounds_kernel<<<(unsigned)((h.nchunks + 255) / 256), 256, 0, st>>>(colptr, n, h.wb,
                                                                         h.nchunks, ch);
  cscp_build_kernel<<<(unsigned)h.nchunks, kCpSortT, 0, st>>>(
      colptr, rowidx, vals, m, n, h.nchunks, h.sb, ch, base + h.stream_off);
  if (cudaMemcpyAsync(plan, &h, sizeof(h), cudaMemcpyHostToDevice, st) != cudaSuccess)
    return SKB_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return skb_launch_status(__func__);
  if (nchunks_out) *nchunks_out = h.nchunks;
  return skb_launch_status(__func__);
}
