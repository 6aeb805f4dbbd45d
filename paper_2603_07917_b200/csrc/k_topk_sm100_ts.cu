// Stage 1, large-batch path (nq > 128): the query block (A operand) lives in TMEM.
//
// Same math and parity contract as k_topk_sm100.cu (tcgen05.mma kind::i8,
// exact int32 dots, fused per-query top-k), restructured so the epilogue is
// three warps per SM sub-partition and overlaps the MMA:
//   * A (128 queries x dim int8) is written once into TMEM columns
//     [A_COL, A_COL + dim/4) by the epilogue warps (tcgen05.st); the MMA
//     reads it there ("TS" form), so no shared memory holds A;
//   * two accumulators of BN = 192 columns (2 x 192 + 96 = 480 TMEM columns
//     at dim 384; 2 x 192 + 128 = 512 at dim 512): each epilogue warp pulls
//     its 64 columns into registers, releases the accumulator at once, and
//     filters from registers while the MMA of the next tile runs;
//   * 12 epilogue warps, three per TMEM lane quarter, split every tile's 192
//     columns in thirds; the three warps serving a query share its heap under
//     a per-query shared-memory lock (inserts are rare).  Three warps per
//     sub-partition (instead of two with 104 columns each) hide the filter's
//     latency chains; 64 data registers per thread keep the kernel at
//     <= 128 registers for 448 threads;
//   * bank tiles come through a two-tile ring (RING, below) so the MMA issuer
//     waits once per tile.
// Warps: 0 TMA producer (bank tiles + inverse norms), 1 TMEM allocator + MMA
// issuer, 2..13 epilogue (group g = (warp-2)/4 owns columns [64g, 64g + 64)).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>

#include <algorithm>
#include <type_traits>

#include "ss_common.cuh"
#include "ss_internal.h"
#include "topk_heap.cuh"

namespace ss {
namespace ts {

constexpr int BM = 128;          // queries (TMEM lanes)
constexpr int BN = 192;          // bank rows per tile (UMMA N): 2 x 192 accumulator columns + A's dim / 4 <= 512
constexpr int BK = 128;          // bytes per K-block (128B swizzle atom)
constexpr int UK = 32;           // int8 K per MMA
#ifndef SS_TS_EPW
#define SS_TS_EPW 3
#endif
constexpr int EPW = SS_TS_EPW;        // epilogue warps per TMEM lane quarter (3: 64 columns each, 4: 48)
constexpr int EPI_WARPS = 4 * EPW;    // 12
constexpr int THREADS = 64 + EPI_WARPS * 32;
constexpr int KMAX = 64;
constexpr int ISLOTS = 4;  // inverse-norm ring (tiles)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
#ifndef SS_TS_SLEEP
#define SS_TS_SLEEP 1
#endif
// waits with a suspend-time hint (the thread sleeps in the barrier instead of
// spinning) -- the epilogue warps' form -- and without (the single-thread
// producer / MMA issuer, whose wake-up latency would delay the pipeline)
__device__ __forceinline__ void bar_wait_sleep(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra W_%=;\n}\n" ::"r"(su32(b)),
      "r"(parity), "r"(0x989680)
      : "memory");
}
__device__ __forceinline__ void bar_wait_spin(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
#if SS_TS_SLEEP == 1
  bar_wait_sleep(b, parity);
#else
  bar_wait_spin(b, parity);
#endif
}
__device__ __forceinline__ void bar_wait_epi(uint64_t* b, uint32_t parity) {
#if SS_TS_SLEEP >= 1
  bar_wait_sleep(b, parity);
#else
  bar_wait_spin(b, parity);
#endif
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* b, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];\n" ::"r"(su32(dst)),
      "l"(m), "r"(su32(b)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(b))
      : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(b))
               : "memory");
}
// D[tmem] (+)= A[tmem] x B[smem]^T
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
// K-major, 128B swizzle: rows of 128 B, 8-row atoms 1024 B apart (SBO)
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// kind::i8 instruction descriptor: s32 accumulator, s8 x s8, K-major A and B
constexpr uint32_t idesc(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void ld32_async(uint32_t taddr, int (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void wait_ld(int (&v)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                 "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]),
                 "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]), "+r"(v[16]), "+r"(v[17]),
                 "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]),
                 "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]),
                 "+r"(v[30]), "+r"(v[31])
               :
               : "memory");
}
__device__ __forceinline__ void ld8_async(uint32_t taddr, int (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                 "=r"(v[7])
               : "r"(taddr));
}
__device__ __forceinline__ void wait_ld8(int (&v)[8]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]),
                 "+r"(v[7])
               :
               : "memory");
}
__device__ __forceinline__ void ld16_async(uint32_t taddr, int (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void wait_ld16(int (&v)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                 "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]),
                 "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15])
               :
               : "memory");
}
__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
      "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
      "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]),
      "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]),
      "r"(v[30]), "r"(v[31])
      : "memory");
}

__device__ __noinline__ uint64_t heapify(uint64_t* heap, int k) {
  for (int i = k / 2 - 1; i >= 0; --i) heap_sift_down<BM>(heap, k, i, heap[i * BM]);
  return heap[0];
}
__device__ __noinline__ uint64_t heap_replace(uint64_t* heap, int k, uint64_t x) {
  heap_sift_down<BM>(heap, k, 0, x);
  return heap[0];
}

// The slow path of the pure-top-k (SHARE) filter, out of line: many chunks
// pass there, and one copy of this code (instead of one per inlined chunk)
// measured faster (1.29 vs 1.45 ms at c2, theta = -1); with a similarity
// floor the path is rare and the call's register traffic makes it slower, so
// the default instantiation keeps it inline.  Under the query's heap lock (the heap is shared with
// the other column-half warp), insert the columns in `mask` whose exact key
// passes theta; returns the tightened s-domain threshold.
template <bool SHARE>
__device__ __noinline__ float insert_locked(uint32_t mask, const float* sl, float iq, float theta,
                                            int64_t gbase, int64_t gcap, uint64_t* heap, int k,
                                            int* s_hlock, int* s_hcnt, uint64_t* s_hroot, int qrow,
                                            uint32_t* s_rtop, int rshare, uint32_t* gslots,
                                            int64_t slot_idx, float thr) {
  while (atomicCAS(&s_hlock[qrow], 0, 1) != 0) {
  }
  __threadfence_block();
  int hcnt = s_hcnt[qrow];
  uint64_t hroot = s_hroot[qrow];
  uint32_t rth0 = 0u;
  if constexpr (SHARE) rth0 = s_rtop[qrow * 4 + rshare - 1];
  while (mask) {
    const int j = __ffs(mask) - 1;
    mask &= mask - 1;
    const float key = __fmul_rn(sl[j], iq);
    if (key >= theta) {
      int64_t rel = gbase + j;
      if (rel < 0) rel += gcap;
      const uint64_t comp = make_comp(key, (uint32_t)rel);
      bool kept = true;
      if (hcnt < k) {
        heap[hcnt * BM] = comp;
        if (++hcnt == k) hroot = heapify(heap, k);
      } else if (comp > hroot) {
        hroot = heap_replace(heap, k, comp);
      } else {
        kept = false;
      }
      if constexpr (SHARE) {
        if (kept) {  // this slice's top-R keys, descending
          uint32_t x = f32_order(key);
          for (int i = 0; i < rshare; ++i) {
            const uint32_t cur = s_rtop[qrow * 4 + i];
            if (x > cur) { s_rtop[qrow * 4 + i] = x; x = cur; }
          }
        }
      }
    }
  }
  uint32_t rth1 = 0u;
  if constexpr (SHARE) rth1 = s_rtop[qrow * 4 + rshare - 1];
  s_hcnt[qrow] = hcnt;
  s_hroot[qrow] = hroot;
  __threadfence_block();
  atomicExch(&s_hlock[qrow], 0);
  if (hcnt >= k) thr = fmaxf(thr, s_threshold(comp_key(hroot), iq));
  if constexpr (SHARE) {
    if (rth1 != rth0) __stcg(gslots + slot_idx, rth1);  // publish
  }
  return thr;
}

// SHARE (pure top-k): every slice publishes the R-th best key it keeps per
// query (gslots[slice][q], R = ceil(k / slices)); each tile, every slice
// filters with the minimum over all slices' published keys -- once every
// slice has published, the union of their top-R holds >= k rows at or above
// that minimum, so it bounds the global k-th key from below.  Slots that are
// still 0 make the minimum 0 (no bound).
constexpr int SHARE_EVERY = 2;
// Per-tile timeline of CTA (0, 0) for scripts/trace_ts.py, compiled only with
// -DSS_TRACE (scripts/exp_build.sh): clock64 stamps per [event][tile].
// Epilogue warp 2 (lane 0): 1 before the accumulator wait, 2 after it; the
// last of the 12 epilogue warps: 3 after the release, 4 after the filter;
// MMA issuer: 5 before the tile wait, 6 after it, 7 after the tile's
// commits; producer: 8 first part issued.  g_wtrace[e][warp][tile]: events
// 1..4 of every epilogue warp, and (e = 4) after its inverse-norm wait.
// (Stamps closer than a few hundred cycles are dominated by the stores.)
#ifdef SS_TRACE
__device__ long long g_trace[9][512];
__device__ long long g_wtrace[5][EPI_WARPS][512];
#define TRACE(ev, t)                                                                               \
  do {                                                                                             \
    if (blockIdx.x == 0 && blockIdx.y == 0 && (t) < 512) {                                         \
      if ((ev) <= 4) {                                                                             \
        if ((threadIdx.x & 31) == 0) {                                                             \
          const long long c_ = clock64();                                                          \
          g_wtrace[(ev) == 0 ? 4 : (ev) - 1][(threadIdx.x >> 5) - 2][t] = c_;                      \
          if ((ev) >= 3)                                                                           \
            atomicMax(reinterpret_cast<unsigned long long*>(&g_trace[ev][t]), (unsigned long long)c_); \
          else if (threadIdx.x == 64)                                                              \
            g_trace[ev][t] = c_;                                                                   \
        }                                                                                          \
      } else {                                                                                     \
        g_trace[ev][t] = clock64();                                                                \
      }                                                                                            \
    }                                                                                              \
  } while (0)
#else
#define TRACE(ev, t) \
  do {               \
  } while (0)
#endif
constexpr int NACC = 2;  // accumulators: the MMA of tile t+1 runs while tile t drains

// RING selects the bank-tile pipeline:
//   RING = true (tile ring, the default where it fits in shared memory): two
//     whole-tile stages; the MMA issuer waits ONCE per tile, on a barrier
//     that completes when the tile's K-blocks have landed AND the epilogue has
//     released the accumulator the tile will overwrite (the epilogue warps
//     arrive on it).  Issuing one tcgen05.mma takes the issuing thread about
//     as long as the MMA runs, so every barrier wait between MMAs is a bubble
//     in the tensor pipe (profiles/r2c_ts_ablation.md): per-K-block waits cost
//     ~30% of the kernel.  The producer still refills each K-block part as
//     soon as the MMAs that read it retire (per-part empty barriers).
//   RING = false: a ring of `stages` K-block stages, waited per K-block (for
//     shapes whose two tiles do not fit, e.g. dim 512).
template <int BN, bool SHARE, bool RING>
__global__ void __launch_bounds__(THREADS, 1)
k_topk_ts(const __grid_constant__ CUtensorMap tmB, const int8_t* __restrict__ Q,
          const float* __restrict__ q_inv, int64_t nq, const float* __restrict__ inv,
          const float2* __restrict__ ibnd, int64_t n_rows,
          int dim, int stages, int k, float theta, int64_t hmod, int64_t gcap, int64_t slot_offset,
          int64_t tiles_per_slice, uint64_t* __restrict__ partials,
          uint32_t* __restrict__ gslots, int rshare, int* __restrict__ counts,
          const int* __restrict__ resolved) {
  constexpr int A_COL = NACC * BN;
  constexpr int B_STAGE = BN * BK;
  constexpr int IS = ISLOTS;       // inverse-norm ring slots
  constexpr int CW = BN / EPW;     // columns per epilogue warp per tile
  static_assert(CW == 64 || CW == 48, "tile shape: 32 + 32 or 32 + 16 columns per epilogue warp");
  constexpr int CW2 = CW - 32;     // the second chunk's columns
  constexpr uint32_t IDESC = idesc(BN);
  const int nkb = dim / BK;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sB = smem;                                                    // stages x BN x 128 B
  uint64_t* s_heap = reinterpret_cast<uint64_t*>(sB + (RING ? NACC * nkb : stages) * B_STAGE);  // [k][128]
  uint64_t* s_hroot = s_heap + (size_t)k * BM;                           // [128]
  int* s_hcnt = reinterpret_cast<int*>(s_hroot + BM);                    // [128]
  int* s_hlock = s_hcnt + BM;                                            // [128]
  float* s_inv = reinterpret_cast<float*>(s_hlock + BM);                 // [ISLOTS][256]
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_inv + IS * 256);
  // barriers: RING -- full[2] (a tile's parts landed + its accumulator
  // released), empty[2 * nkb] (one per K-block part); else full/empty[stages]
  const int nfull = RING ? NACC : stages, nempty = RING ? NACC * nkb : stages;
  uint64_t* a_full = bars;
  uint64_t* full = bars + 1;
  uint64_t* empty = full + nfull;
  uint64_t* tfull = empty + nempty;
  uint64_t* tempty = tfull + NACC;   // (RING: unused -- the release goes to full)
  uint64_t* ifull = tempty + NACC;   // [IS] tile's inverse norms landed
  uint64_t* iempty = ifull + IS;     // [IS] consumed by every epilogue warp
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(iempty + IS);
  // SHARE: this slice's top-R keys per query, after everything else
  uint32_t* s_rtop = s_tmem + 4;  // [128][4]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = blockIdx.x, slice = blockIdx.y;
  const int64_t tile0 = (int64_t)slice * tiles_per_slice;
  const int64_t total_tiles = (n_rows + BN - 1) / BN;
  const int ntiles = (int)max((int64_t)0, min(total_tiles, tile0 + tiles_per_slice) - tile0);

  // Pure top-k cascade, second pass: this query tile is done if every query
  // already has >= k keys at or above the threshold pass's theta (their
  // top-k lie above it, and the threshold pass's lists hold them); the CTA
  // leaves before it allocates anything.
  if (resolved) {
    int need = 0;
    for (int i = threadIdx.x; i < BM; i += blockDim.x) {
      const int64_t qq = (int64_t)qt * BM + i;
      if (qq < nq) {
        int sum = 0;
        for (int s2 = 0; s2 < (int)gridDim.y; ++s2) sum += resolved[(int64_t)s2 * nq + qq];
        need |= sum < k;
      }
    }
    if (!__syncthreads_or(need)) return;
  }
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmB) : "memory");
    bar_init(a_full, 4);  // the 4 warps writing A into TMEM
    // RING: the producer's expect_tx arrival + every epilogue warp's release
    for (int s = 0; s < nfull; ++s) bar_init(&full[s], RING ? 1 + EPI_WARPS : 1);
    for (int s = 0; s < nempty; ++s) bar_init(&empty[s], 1);
    for (int b = 0; b < NACC; ++b) { bar_init(&tfull[b], 1); bar_init(&tempty[b], EPI_WARPS); }
    for (int b = 0; b < IS; ++b) { bar_init(&ifull[b], 1); bar_init(&iempty[b], EPI_WARPS); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int i = threadIdx.x; i < BM; i += blockDim.x) { s_hcnt[i] = 0; s_hroot[i] = 0; s_hlock[i] = 0; }
  if constexpr (SHARE)
    for (int i = threadIdx.x; i < BM * 4; i += blockDim.x) s_rtop[i] = 0u;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *s_tmem;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer ---
    if (lane == 0 && ntiles > 0) {
      int it = 0;
      for (int t = 0; t < ntiles; ++t) {
        const int row0 = (int)((tile0 + t) * BN);
        // the tile's BN inverse norms into the ring (the bank pads inv with
        // one NaN tile, so the copy never leaves the allocation); the
        // epilogue then issues no global loads in its tile loop
        const int sl = t % IS;
        if constexpr (!RING) {
          bar_wait(&iempty[sl], ((t / IS) & 1) ^ 1);
          bar_expect(&ifull[sl], BN * 4 + BN / 2);
          bulk_g2s(s_inv + sl * 256, inv + row0, BN * 4, &ifull[sl]);
          bulk_g2s(s_inv + sl * 256 + BN, ibnd + row0 / 16, BN / 2, &ifull[sl]);
        }
        if constexpr (RING) {
          // part kb of stage t & 1 is free once tile t - 2's K-block kb MMAs
          // retired; the tile's one expect_tx arrival follows the first such
          // wait (so it cannot land in the previous phase of full)
          const int st = t & 1;
          const uint32_t par = ((t >> 1) & 1) ^ 1;
          for (int kb = 0; kb < nkb; ++kb) {
            bar_wait(&empty[st * nkb + kb], par);
            if (kb == 0) bar_expect(&full[st], (uint32_t)(nkb * B_STAGE));
            tma2d(sB + (st * nkb + kb) * B_STAGE, &tmB, &full[st], kb * BK, row0);
            if (kb == 0) TRACE(8, t);
          }
          // the norms after the tile's bank parts: with two slots, the slot
          // frees only when the epilogue is done with tile t - 2, which must
          // not hold back the bank loads
          bar_wait(&iempty[sl], ((t / IS) & 1) ^ 1);
          bar_expect(&ifull[sl], BN * 4 + BN / 2);
          bulk_g2s(s_inv + sl * 256, inv + row0, BN * 4, &ifull[sl]);
          bulk_g2s(s_inv + sl * 256 + BN, ibnd + row0 / 16, BN / 2, &ifull[sl]);
        } else {
          for (int kb = 0; kb < nkb; ++kb, ++it) {
            const int s = it % stages;
            bar_wait(&empty[s], ((it / stages) & 1) ^ 1);
            bar_expect(&full[s], B_STAGE);
            tma2d(sB + s * B_STAGE, &tmB, &full[s], kb * BK, row0);
          }
        }
      }
      if constexpr (!RING)
        for (int i = max(0, it - stages); i < it; ++i) bar_wait(&empty[i % stages], (i / stages) & 1);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer ----
    if (lane == 0 && ntiles > 0) {
      bar_wait(a_full, 0);
      fence_after();
      const uint32_t b_base = su32(sB);
      int it = 0;
      for (int t = 0; t < ntiles; ++t) {
        const int acc = t % NACC;
        const uint32_t dacc = tmem + acc * BN;
        if constexpr (RING) {
          // one wait per tile: its parts landed and accumulator acc released
          TRACE(5, t);
          bar_wait_spin(&full[acc], (t >> 1) & 1);
          TRACE(6, t);
          fence_after();
          for (int kb = 0; kb < nkb; ++kb) {
            const uint32_t bst = b_base + (acc * nkb + kb) * B_STAGE;
#pragma unroll
            for (int kk = 0; kk < BK / UK; ++kk)
              mma_ts(dacc, tmem + A_COL + (kb * (BK / UK) + kk) * (UK / 4), desc_sw128(bst + kk * UK),
                     IDESC, (kb | kk) != 0);
            commit(&empty[acc * nkb + kb]);
          }
        } else {
          // every epilogue warp has pulled tile t - NACC out of this accumulator
          bar_wait(&tempty[acc], ((t / NACC) & 1) ^ 1);
          fence_after();
          for (int kb = 0; kb < nkb; ++kb, ++it) {
            const int s = it % stages;
            bar_wait(&full[s], (it / stages) & 1);
            fence_after();
#pragma unroll
            for (int kk = 0; kk < BK / UK; ++kk)
              mma_ts(dacc, tmem + A_COL + (kb * (BK / UK) + kk) * (UK / 4),
                     desc_sw128(b_base + s * B_STAGE + kk * UK), IDESC, (kb | kk) != 0);
            commit(&empty[s]);
          }
        }
        commit(&tfull[acc]);
        TRACE(7, t);
      }
    }
  } else {
    // --------------------------------------------------------- epilogue ----
    const int ew = warp - 2;                // 0..7
    const int grp = ew >> 2;                // column third of each tile
    const int quarter = warp & 3;           // TMEM lane quarter
    const int qrow = quarter * 32 + lane;
    const int64_t q = (int64_t)qt * BM + qrow;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    // group 0 writes this query's int8 vector into TMEM (A operand)
    if (grp == 0) {
      const int ncol = dim / 4;
      for (int c0 = 0; c0 < ncol; c0 += 32) {
        uint32_t v[32];
        const uint4* src = reinterpret_cast<const uint4*>(Q + q * dim) + c0 / 4;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          uint4 x = (q < nq) ? __ldg(src + u) : make_uint4(0, 0, 0, 0);
          v[4 * u + 0] = x.x; v[4 * u + 1] = x.y; v[4 * u + 2] = x.z; v[4 * u + 3] = x.w;
        }
        st32(tmem + lane_base + A_COL + c0, v);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      fence_before();
      __syncwarp();
      if (lane == 0) bar_arrive(a_full);
    }
    if constexpr (RING) {
      // both accumulators start free: release them for tiles 0 and 1
      if (lane == 0) { bar_arrive(&full[0]); bar_arrive(&full[1]); }
    }
    const float iq = (q < nq) ? q_inv[q] : __int_as_float(0x7fc00000);
    uint64_t* heap = s_heap + qrow;  // shared by the two column-half warps of this quarter
    float thr = (iq == iq) ? s_threshold(theta, iq) : INFINITY;
    for (int t = 0; t < ntiles; ++t) {
      const int64_t row0 = (tile0 + t) * BN + grp * CW;  // first bank row of my columns
      const int acc = t % NACC, sl = t % IS;
      const float* ciw = s_inv + sl * 256 + grp * CW;
      if constexpr (SHARE) {
        // minimum over the slices' published R-th best keys (independent
        // loads; their latency overlaps the wait for this tile's MMA), every
        // SHARE_EVERY tiles: a staler bound only prunes less, and the
        // gridDim.y L2 loads per query were a visible share of the tile loop
        if (q < nq && (t % SHARE_EVERY) == 0) {
          uint32_t m = ~0u;
          for (int s2 = 0; s2 < (int)gridDim.y; ++s2) m = min(m, __ldcg(gslots + (int64_t)s2 * nq + q));
          if (m != 0u && m != ~0u) thr = fmaxf(thr, s_threshold(f32_unorder(m), iq));
        }
      }
      bar_wait_epi(&ifull[sl], (t / IS) & 1);
      TRACE(0, t);
      // this warp's four 16-column filter bounds (hi0, lo0, hi1, lo1 per
      // 32-column chunk), precomputed per 16-row group by every bank write
      const float2* cb = reinterpret_cast<const float2*>(s_inv + sl * 256 + BN) + grp * (CW / 16);
      TRACE(1, t);
      bar_wait_epi(&tfull[acc], (t / NACC) & 1);
      TRACE(2, t);
      fence_after();
      const uint32_t tbase = tmem + lane_base + acc * BN + grp * CW;
      // pull my chunks into registers, then hand the accumulator back
      int v0[32], v1[CW2];
      ld32_async(tbase, v0);
      if constexpr (CW2 == 32) ld32_async(tbase + 32, v1);
      else ld16_async(tbase + 32, v1);
      wait_ld(v0);
      if constexpr (CW2 == 32) wait_ld(v1);
      else wait_ld16(v1);
      fence_before();
      __syncwarp();
      if (lane == 0) bar_arrive(RING ? &full[acc] : &tempty[acc]);  // accumulator free for tile t + 2
      TRACE(3, t);
#ifdef SS_ABLATE_FILTER  // scripts/exp_build.sh ablation: pull + release only, no filter
      if (v0[0] == 0x7fffffff && v1[5] == 0x7fffffff) thr = -thr;
      __syncwarp();
      if (lane == 0) bar_arrive(&iempty[sl]);
      continue;
#endif
      // Filter per 16-column half: a half can only hold a score >= thr if
      // fl(fl(max dot) * (max inv_w)) >= thr (or the min inv_w when every dot
      // is negative) -- monotone rounding makes this a superset test, so the
      // exact scores (one quarter-rate int->float conversion each) are only
      // formed for the rare halves that pass it.
      auto exact = [&](const auto& v, const int c, auto off_c, auto w_c) {
        constexpr int OFF = decltype(off_c)::value;
        constexpr int WW = decltype(w_c)::value;
        float s[WW];
        const float4* iw4 = reinterpret_cast<const float4*>(ciw + c * 32 + OFF);
#pragma unroll
        for (int j4 = 0; j4 < WW / 4; ++j4) {
          const float4 w = iw4[j4];
          s[4 * j4 + 0] = __fmul_rn(__int2float_rn(v[OFF + 4 * j4 + 0]), w.x);
          s[4 * j4 + 1] = __fmul_rn(__int2float_rn(v[OFF + 4 * j4 + 1]), w.y);
          s[4 * j4 + 2] = __fmul_rn(__int2float_rn(v[OFF + 4 * j4 + 2]), w.z);
          s[4 * j4 + 3] = __fmul_rn(__int2float_rn(v[OFF + 4 * j4 + 3]), w.w);
        }
        const int64_t gbase = slot_offset + row0 + c * 32 + OFF - hmod;
        uint32_t mask = 0;
#pragma unroll
        for (int j = 0; j < WW; ++j) mask |= (s[j] >= thr ? 1u : 0u) << j;
        if (!mask) return;
        float sl[WW];
#pragma unroll
        for (int j = 0; j < WW; ++j) sl[j] = s[j];
        if constexpr (SHARE) {
          thr = insert_locked<true>(mask, sl, iq, theta, gbase, gcap, heap, k, s_hlock, s_hcnt,
                                    s_hroot, qrow, s_rtop, rshare, gslots,
                                    (int64_t)slice * nq + q, thr);
        } else {
          // this query's heap is shared with the other column-half warp: take
          // its lock (one lock per thread at a time, never nested)
          while (atomicCAS(&s_hlock[qrow], 0, 1) != 0) {
          }
          __threadfence_block();
          int hcnt = s_hcnt[qrow];
          uint64_t hroot = s_hroot[qrow];
          while (mask) {
            const int j = __ffs(mask) - 1;
            mask &= mask - 1;
            const float key = __fmul_rn(sl[j], iq);
            if (key >= theta) {
              int64_t rel = gbase + j;
              if (rel < 0) rel += gcap;
              const uint64_t comp = make_comp(key, (uint32_t)rel);
              if (hcnt < k) {
                heap[hcnt * BM] = comp;
                if (++hcnt == k) hroot = heapify(heap, k);
              } else if (comp > hroot) {
                hroot = heap_replace(heap, k, comp);
              }
            }
          }
          s_hcnt[qrow] = hcnt;
          s_hroot[qrow] = hroot;
          __threadfence_block();
          atomicExch(&s_hlock[qrow], 0);
          if (hcnt >= k) thr = fmaxf(thr, s_threshold(comp_key(hroot), iq));
        }
      };
      auto chunk = [&](const auto& v, const int c) {
        constexpr int W = sizeof(v) / sizeof(v[0]);  // 32, or 16 (the second chunk at CW = 48)
        const int a0 = __vimax3_s32(v[0], v[1], v[2]), a1 = __vimax3_s32(v[3], v[4], v[5]);
        const int a2 = __vimax3_s32(v[6], v[7], v[8]), a3 = __vimax3_s32(v[9], v[10], v[11]);
        const int a4 = __vimax3_s32(v[12], v[13], v[14]);
        const int mdl = __vimax3_s32(__vimax3_s32(a0, a1, a2), __vimax3_s32(a3, a4, v[15]), a0);
        const float2 b0 = cb[2 * c];
        const float bl = __fmul_rn(__int2float_rn(mdl), mdl >= 0 ? b0.x : b0.y);
        if constexpr (W == 32) {
          const int b0_ = __vimax3_s32(v[16], v[17], v[18]), b1 = __vimax3_s32(v[19], v[20], v[21]);
          const int b2 = __vimax3_s32(v[22], v[23], v[24]), b3 = __vimax3_s32(v[25], v[26], v[27]);
          const int b4 = __vimax3_s32(v[28], v[29], v[30]);
          const int mdh = __vimax3_s32(__vimax3_s32(b0_, b1, b2), __vimax3_s32(b3, b4, v[31]), b0_);
          const float2 b1h = cb[2 * c + 1];
          const float bh = __fmul_rn(__int2float_rn(mdh), mdh >= 0 ? b1h.x : b1h.y);
          if constexpr (SHARE) {
            // pure top-k: many chunks pass while the bounds rise -- one exact
            // pass (and one heap lock) per 32 columns is cheaper there
            if (fmaxf(bl, bh) >= thr)
              exact(v, c, std::integral_constant<int, 0>(), std::integral_constant<int, 32>());
          } else {
            if (bl >= thr) exact(v, c, std::integral_constant<int, 0>(), std::integral_constant<int, 16>());
            if (bh >= thr) exact(v, c, std::integral_constant<int, 16>(), std::integral_constant<int, 16>());
          }
        } else {
          if (bl >= thr) exact(v, c, std::integral_constant<int, 0>(), std::integral_constant<int, 16>());
        }
      };
      chunk(v0, 0);
      chunk(v1, 1);
      __syncwarp();
      if (lane == 0) bar_arrive(&iempty[sl]);  // this tile's inverse norms consumed
      TRACE(4, t);
    }
    asm volatile("bar.sync 1, %0;\n" ::"n"(EPI_WARPS * 32) : "memory");  // every column third done
    if (grp == 0 && q < nq) {
      uint64_t* out = partials + ((int64_t)slice * nq + q) * k;
      const int hc = s_hcnt[qrow];
      for (int i = 0; i < k; ++i) out[i] = (i < hc) ? heap[i * BM] : 0ull;
      if (counts) counts[(int64_t)slice * nq + q] = hc;  // (pure top-k cascade, first pass)
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}

}  // namespace ts
#ifdef SS_TRACE
extern "C" int ss_exp_trace_reset(void) {
  static long long zeros[9][512];
  return cudaMemcpyToSymbol(ts::g_trace, zeros, sizeof(zeros)) == cudaSuccess ? 0 : 1;
}
extern "C" int ss_exp_trace(long long* host, long long* whost) {
  if (cudaMemcpyFromSymbol(host, ts::g_trace, sizeof(ts::g_trace)) != cudaSuccess) return 1;
  return cudaMemcpyFromSymbol(whost, ts::g_wtrace, sizeof(ts::g_wtrace)) == cudaSuccess ? 0 : 1;
}
#endif

static PFN_cuTensorMapEncodeTiled_v12000 ts_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

static size_t ts_fixed_smem(int k, int islots) {
  // heaps, per-query root / count / lock, the norms + bounds ring, barriers,
  // 1 KB alignment slack
  return (size_t)k * ts::BM * 8 + ts::BM * 16 + (size_t)islots * 256 * 4 + 512 + 1024;
}

// Shape of one launch: tile rows BN (the widest double buffer of accumulators
// that fits beside A's dim / 4 TMEM columns: 2 x 208 + 96 = 512 at dim 384
// and below, 2 x 192 + 128 at dim 512), and the pipeline: the tile ring (two
// whole tiles, see k_topk_ts) when it fits in shared memory, else a ring of
// K-block stages.  Pure top-k (SHARE) needs 2 KB more for the shared bounds.
struct TsShape {
  int bn = 0;
  bool ring = false;
  int stages = 0;
  size_t smem = 0;
};
static TsShape ts_shape(int dim, int k, bool share) {
  const int nkb = dim / ts::BK;
  const size_t extra = share ? ts::BM * 16 : 0;
  TsShape sh;
  if (dim / 4 + 2 * ts::BN > 512) return sh;
  sh.bn = ts::BN;
  const size_t fixed = ts_fixed_smem(k, ts::ISLOTS) + extra;
  const size_t ring = fixed + (size_t)2 * nkb * ts::BN * ts::BK;
  if (ring <= 227 * 1024) {
    sh.ring = true; sh.stages = 2 * nkb; sh.smem = ring;
    return sh;
  }
  for (int s = 8; s >= 3; --s) {
    const size_t smem = fixed + (size_t)s * ts::BN * ts::BK;
    if (smem <= 227 * 1024) {
      sh.stages = s; sh.smem = smem;
      return sh;
    }
  }
  sh.bn = 0;
  return sh;
}

bool topk_ts_supported(const TopkArgs& a) {
  if (a.dim % ts::BK || a.dim < ts::BK || a.k < 1 || a.k > ts::KMAX) return false;
  if (a.n_rows >= (1LL << 31) || a.nq >= (1LL << 31)) return false;
  if (!a.inv_padded || !a.ibnd) return false;  // tiles of norms and bounds are bulk-copied whole
  return ts_shape(a.dim, a.k, true).bn > 0 && ts_shape(a.dim, a.k, false).bn > 0;
}

// one partial list per CTA slice
int topk_ts_lists(const TopkArgs& a, int device) {
  const int64_t qtiles = (a.nq + ts::BM - 1) / ts::BM;
  const int bn = ts_shape(a.dim, a.k, false).bn;
  const int64_t tiles = (a.n_rows + bn - 1) / bn;
#ifdef SS_EXP_SLICES  // scripts/exp_build.sh ablation: a fixed slice count
  return (int)std::min<int64_t>(SS_EXP_SLICES, tiles);
#endif
  return pick_slices(qtiles, tiles, sm_count(device));
}

template <int BN>
static int launch_ts_t(const TopkArgs& a, const TsShape& sh, int rshare, uint64_t* partials, int n_slices,
                       cudaStream_t st, int* counts = nullptr, const int* resolved = nullptr) {
  auto enc = ts_encode();
  if (!enc) return set_error(SS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap mb;
  cuuint64_t gdim[2] = {(cuuint64_t)a.dim, (cuuint64_t)a.n_rows};
  cuuint64_t gstride[1] = {(cuuint64_t)a.dim};
  cuuint32_t box[2] = {(cuuint32_t)ts::BK, (cuuint32_t)BN};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&mb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(a.emb), gdim, gstride,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(SS_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  auto kern = rshare ? (sh.ring ? ts::k_topk_ts<BN, true, true> : ts::k_topk_ts<BN, true, false>)
                     : (sh.ring ? ts::k_topk_ts<BN, false, true> : ts::k_topk_ts<BN, false, false>);
  SS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh.smem));
  if (rshare)
    SS_CUDA_TRY(cudaMemsetAsync(a.gslots, 0, (size_t)n_slices * a.nq * sizeof(uint32_t), st));
  const int64_t tiles = (a.n_rows + BN - 1) / BN;
  const int64_t tps = (tiles + n_slices - 1) / n_slices;
  dim3 grid((unsigned)((a.nq + ts::BM - 1) / ts::BM), (unsigned)n_slices);
  count_launch();
  kern<<<grid, ts::THREADS, sh.smem, st>>>(mb, a.q, a.q_inv, a.nq, a.inv, a.ibnd, a.n_rows, a.dim,
                                           sh.stages, a.k, a.theta, a.head % a.gcap, a.gcap, a.slot_offset, tps,
                                           partials, a.gslots, rshare, counts, resolved);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

// Pure top-k (theta <= 0) runs as a cascade when the bank's scratch is there:
// (1) the threshold kernel at kCascadeTheta (the paper's similarity
// threshold) writes every slice's list of keys >= it and their
// counts; (2) the pure top-k kernel (bound sharing, SHARE) runs only for the
// query tiles holding a query with fewer than k such keys in total -- the
// other tiles exit at once.  Exact: a query with >= k keys at or above the
// threshold has its whole top-k there, and each of those rows is in its
// slice's top-k of keys >= the threshold, so the first pass's lists merge to
// the same top-k.  When every query resolves (clustered prompts), pure top-k
// costs the threshold pass plus an empty launch; when none does, the
// threshold pass is overhead (~1/3 of the pure top-k kernel).

int launch_topk_ts(const TopkArgs& a, uint64_t* partials, int n_lists, cudaStream_t st) {
  if (n_lists < 1) return set_error(SS_ERR_ARG, "ts: no slices");
  // pure top-k: share per-slice bounds (see k_topk_ts SHARE)
  int rshare = 0;
  if (a.gslots && a.theta <= 0.f && n_lists >= 2 && n_lists <= kMaxShareSlices) {
    const int R = (a.k + n_lists - 1) / n_lists;
    if (R <= 4) rshare = R;
  }
  const TsShape sh = ts_shape(a.dim, a.k, rshare > 0);
  if (sh.bn != ts::BN) return set_error(SS_ERR_UNSUPPORTED, "ts: no shape fits shared memory");
  if (a.gslots && a.theta <= 0.f && n_lists <= kMaxShareSlices) {
    // the bank's pure-top-k scratch: [kMaxShareSlices][nq] bounds, then
    // [kMaxShareSlices][nq] per-slice counts
    int* counts = reinterpret_cast<int*>(a.gslots + (size_t)kMaxShareSlices * a.nq);
    TopkArgs a1 = a;
    a1.theta = kCascadeTheta;
    const TsShape sh1 = ts_shape(a.dim, a.k, false);
    if (int rc = launch_ts_t<ts::BN>(a1, sh1, 0, partials, n_lists, st, counts, nullptr)) return rc;
    return launch_ts_t<ts::BN>(a, sh, rshare, partials, n_lists, st, nullptr, counts);
  }
  return launch_ts_t<ts::BN>(a, sh, rshare, partials, n_lists, st);
}

}  // namespace ss
