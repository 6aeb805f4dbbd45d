// Stage 1, large-batch path, v4: CTA-pair tcgen05 GEMM with a decoupled
// 8-warp epilogue.  Same math and parity contract as k_topk_sm100.cu
// (tcgen05.mma kind::i8, exact int32 dots, fused per-query top-k).
//
// Why this shape (profiles/ROUND1.md, round-1b ablation): tcgen05.mma with
// M=128 and K=32 takes the same time at N=192 as at N=256, so the full MMA
// rate needs N=256, and hiding the TMEM drain behind the next MMA needs two
// N=256 accumulators = all 512 TMEM columns -- A must then live in shared
// memory.  A (48 KB) + the per-query heaps (64 KB) leave room for only 3
// whole 32 KB bank stages in one CTA, which starves the MMA; a CTA pair
// (cluster of 2, cta_group::2, M=256) loads half of every bank tile per CTA
// (16 KB stages, 6 of them) and halves the L2->SM traffic.
//
// Per CTA (352 threads):
//   warp 0      producer: A once (TMA), then per tile the tile's inverse
//               norms (1 KB bulk copy into a 4-slot ring, this CTA's own
//               barrier) and this CTA's half of every B K-block (TMA,
//               completion on the leader's barrier)
//   warp 1      TMEM allocator; in the leader, the single-thread MMA issuer
//               (M=256 = both CTAs' queries, N=256, K=384 in 12 MMAs) into
//               accumulator t % 2
//   warps 2..9  epilogue: two warps per TMEM lane quarter split the 256
//               columns; each pulls its 4 x 32 columns into registers,
//               releases the accumulator (arrive on the leader's barrier),
//               and filters from registers while the next MMA runs -- integer
//               max-tree per 32 columns, one I2F + FMUL bound vs the per-query
//               threshold, exact keys + heap inserts only for passing chunks;
//               the two warps of a query share its smem heap under a lock.
// The inverse norms come from shared memory, so the epilogue issues no
// global loads inside the tile loop.
#include <stdlib.h>

#include "ss_common.cuh"
#include "ss_internal.h"
#include "tc_util.cuh"
#include "topk_heap.cuh"

namespace ss {
namespace pr {

constexpr int BM = 128;                 // queries per CTA (TMEM lanes)
constexpr int BN = 256;                 // bank rows per tile (UMMA N)
constexpr int HN = BN / 2;              // B rows loaded per CTA per tile
constexpr int BK = 128;                 // bytes per K-block (128B swizzle atom)
constexpr int UK = 32;                  // int8 K per MMA
constexpr int EPW = 2;                  // epilogue warps per TMEM lane quarter
constexpr int EPI_WARPS = 4 * EPW;      // 8: each owns BN / EPW columns of a tile
constexpr int CW = BN / EPW;            // 128 columns per epilogue warp per tile
constexpr int CPW = CW / 32;            // 4 chunks of 32 columns
constexpr int THREADS = 64 + EPI_WARPS * 32;
constexpr int A_BLK = BM * BK;          // 16 KB per K-block of A
constexpr int B_STAGE = HN * BK;        // 16 KB per stage per CTA
constexpr int ISLOTS = 4;               // inverse-norm ring (tiles)
constexpr int KMAX = 64;
// M = 256 (pair), N = 256, s32 accumulate, s8 x s8, K-major
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)((2 * BM) >> 4) << 24);

__device__ __noinline__ uint64_t heapify(uint64_t* heap, int k) {
  for (int i = k / 2 - 1; i >= 0; --i) heap_sift_down<BM>(heap, k, i, heap[i * BM]);
  return heap[0];
}
__device__ __noinline__ uint64_t heap_replace(uint64_t* heap, int k, uint64_t x) {
  heap_sift_down<BM>(heap, k, 0, x);
  return heap[0];
}

// v[j] for a run-time j without indexing a register array (which would put
// it in local memory): a 5-level select tree
__device__ __forceinline__ int pick32(const int (&v)[32], int j) {
  int a[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) a[u] = (j & 1) ? v[2 * u + 1] : v[2 * u];
  int b[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) b[u] = (j & 2) ? a[2 * u + 1] : a[2 * u];
  int c[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) c[u] = (j & 4) ? b[2 * u + 1] : b[2 * u];
  const int d0 = (j & 8) ? c[1] : c[0];
  const int d1 = (j & 8) ? c[3] : c[2];
  return (j & 16) ? d1 : d0;
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__global__ void __launch_bounds__(THREADS, 1)
k_topk_pair(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmB,
            const float* __restrict__ q_inv, int64_t nq, const float* __restrict__ inv,
            int64_t n_rows, int nkb, int stages, int k, float theta, int64_t hmod, int64_t gcap,
            int64_t slot_offset, int64_t tiles_per_slice, uint64_t* __restrict__ partials, int dbg) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                                                       // nkb x 16 KB
  uint8_t* sB = sA + nkb * A_BLK;                                           // stages x 16 KB
  float* s_inv = reinterpret_cast<float*>(sB + stages * B_STAGE);           // [ISLOTS][256]
  uint64_t* s_heap = reinterpret_cast<uint64_t*>(s_inv + ISLOTS * BN);      // [k][128]
  uint64_t* s_hroot = s_heap + (size_t)k * BM;                              // [128]
  int* s_hcnt = reinterpret_cast<int*>(s_hroot + BM);                       // [128]
  int* s_hlock = s_hcnt + BM;                                               // [128]
  float* s_ib = reinterpret_cast<float*>(s_hlock + BM);                     // [8 warps][8]
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_ib + EPI_WARPS * 8);
  uint64_t* a_full = bars;
  uint64_t* full = bars + 1;
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;    // [2]
  uint64_t* tempty = tfull + 2;        // [2]
  uint64_t* ifull = tempty + 2;        // [ISLOTS]
  uint64_t* iempty = ifull + ISLOTS;   // [ISLOTS]
  uint64_t* mdone = iempty + ISLOTS;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(mdone + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int qt = blockIdx.x, slice = blockIdx.y;
  const int64_t tile0 = (int64_t)slice * tiles_per_slice;
  const int64_t total_tiles = (n_rows + BN - 1) / BN;
  const int ntiles = (int)max((int64_t)0, min(total_tiles, tile0 + tiles_per_slice) - tile0);

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmQ) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmB) : "memory");
    mbar_init(a_full, 1);
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 2 * EPI_WARPS); }
    for (int b = 0; b < ISLOTS; ++b) { mbar_init(&ifull[b], 1); mbar_init(&iempty[b], EPI_WARPS); }
    mbar_init(mdone, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int i = threadIdx.x; i < BM; i += blockDim.x) { s_hcnt[i] = 0; s_hroot[i] = 0; s_hlock[i] = 0; }
  if (warp == 1) tmem_alloc512<2>(s_tmem);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  if (warp == 0) {
    // ------------------------------------------------------ producer -------
    if (lane == 0 && ntiles > 0) {
      if (leader) mbar_expect_tx(a_full, 2 * nkb * A_BLK);
      for (int kb = 0; kb < nkb; ++kb) tma_load_2d<2>(sA + kb * A_BLK, &tmQ, a_full, kb * BK, qt * BM);
      int it = 0;
      for (int t = 0; t < ntiles; ++t) {
        const int64_t row0 = (tile0 + t) * BN;
        // this tile's 256 inverse norms (the bank pads inv by one tile of NaN)
        const int sl = t % ISLOTS;
        if (!(dbg & 64)) {  // (debug 64 runs no epilogue, so nothing frees the slots)
          mbar_wait(&iempty[sl], ((t / ISLOTS) & 1) ^ 1);
          mbar_expect_tx(&ifull[sl], BN * 4);
          bulk_g2s(s_inv + sl * BN, inv + row0, BN * 4, &ifull[sl]);
        }
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % stages;
          mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
          if (dbg & 8) {  // debug: no bank traffic
            if (leader) mbar_expect_tx(&full[s], 0);
            continue;
          }
          if (leader) mbar_expect_tx(&full[s], 2 * B_STAGE);
          tma_load_2d<2>(sB + s * B_STAGE, &tmB, &full[s], kb * BK, (int)(row0 + rank * HN));
        }
      }
      // every stage's last MMA commit has landed before this CTA may exit
      for (int i = max(0, it - stages); i < it; ++i) mbar_wait(&empty[i % stages], (i / stages) & 1);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer ----
    if (leader && lane == 0 && ntiles > 0) {
      mbar_wait(a_full, 0);
      tc_fence_after();
      const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
      int it = 0;
      for (int t = 0; t < ntiles; ++t) {
        const int acc = t & 1;
        if (!(dbg & 64)) mbar_wait_cluster(&tempty[acc], ((t >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % stages;
          mbar_wait(&full[s], (it / stages) & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < BK / UK; ++kk) {
            const uint64_t ad = umma_desc_sw128(a_base + kb * A_BLK + kk * UK);
            const uint64_t bd = umma_desc_sw128(b_base + s * B_STAGE + kk * UK);
            if (!(dbg & 2)) tc_mma_i8<2>(d, ad, bd, IDESC, (kb | kk) != 0);
          }
          tc_commit<2>(&empty[s]);  // frees the stage in both CTAs once these MMAs retire
        }
        tc_commit<2>(&tfull[acc]);  // accumulator ready in both CTAs
      }
      if (dbg & 64) {
        tc_commit<2>(mdone);
        mbar_wait(mdone, 0);
      }
    }
  } else {
    // --------------------------------------------------------- epilogue ----
    const int ew = warp - 2;         // 0..7
    const int grp = ew >> 2;         // column half of each tile
    const int quarter = warp & 3;    // TMEM lane quarter
    const int qrow = quarter * 32 + lane;
    const int64_t q = (int64_t)qt * BM + qrow;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const float iq = (q < nq) ? q_inv[q] : __int_as_float(0x7fc00000);
    uint64_t* heap = s_heap + qrow;
    float* cib = s_ib + ew * 8;  // [max inv_w of chunk 0..3][min inv_w of chunk 0..3]
    float thr = (iq == iq) ? s_threshold(theta, iq) : INFINITY;
    const int nt_epi = (dbg & 64) ? 0 : ntiles;
    for (int t = 0; t < nt_epi; ++t) {
      const int acc = t & 1, sl = t % ISLOTS;
      const int64_t row0 = (tile0 + t) * BN + grp * CW;  // first bank row of my columns
      const float* ciw = s_inv + sl * BN + grp * CW;
      mbar_wait(&ifull[sl], (t / ISLOTS) & 1);
      {
        // chunk bounds of the inverse norms; rows past the end are NaN (never
        // match) and stay out of the bounds
        const float4 w = (lane * 4 < CW) ? reinterpret_cast<const float4*>(ciw)[lane]
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
        float hi = fmaxf(fmaxf(fmaxf(w.x, w.y), fmaxf(w.z, w.w)), 0.f);
        float lo = fminf(fminf(fminf(w.x, w.y), fminf(w.z, w.w)), INFINITY);
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
          hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
          lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        }
        if ((lane & 7) == 0 && lane * 4 < CW) {
          cib[lane >> 3] = hi;
          cib[4 + (lane >> 3)] = lo;
        }
      }
      __syncwarp();
      mbar_wait(&tfull[acc], (t >> 1) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem + lane_base + acc * BN + grp * CW;
      if (dbg & 16) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) { mbar_arrive_leader(&tempty[acc]); mbar_arrive(&iempty[sl]); }
        continue;
      }
      static_assert(CPW == 4, "four chunks per warp");
      int v0[32], v1[32], v2[32], v3[32];
      tmem_ld32_async(tbase, v0);
      tmem_ld32_async(tbase + 32, v1);
      tmem_ld32_async(tbase + 64, v2);
      tmem_ld32_async(tbase + 96, v3);
      tmem_wait_regs(v0);
      tmem_wait_regs(v1);
      tmem_wait_regs(v2);
      tmem_wait_regs(v3);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&tempty[acc]);
      if (!(dbg & 4)) {
        auto chunk = [&](const int (&v)[32], const int c) {
          int m[11];
#pragma unroll
          for (int j = 0; j < 10; ++j) m[j] = __vimax3_s32(v[3 * j], v[3 * j + 1], v[3 * j + 2]);
          m[10] = max(v[30], v[31]);
          const int md = __vimax3_s32(__vimax3_s32(m[0], m[1], m[2]), __vimax3_s32(m[3], m[4], m[5]),
                                      __vimax3_s32(__vimax3_s32(m[6], m[7], m[8]), m[9], m[10]));
          // fl(fl(max dot) * max inv_w) bounds every score of the chunk from
          // above (min inv_w when all dots are negative): monotone rounding
          const float bnd = __fmul_rn(__int2float_rn(md), md >= 0 ? cib[c] : cib[4 + c]);
          if (!(dbg & 1) && bnd >= thr) {
            // Candidate columns.  thr > 0: fl(v * w) >= thr needs v > 0 and,
            // as w <= mx, v >= thr (1 - 2^-24) / mx >= d0 (round-toward-zero
            // reciprocal and product, then a 1e-5 margin) -- one integer
            // compare per column.  Survivors are evaluated one at a time with
            // a register pick (no local memory: the smem carve-out leaves
            // little L1 for it).
            uint32_t m0 = 0xffffffffu;
            if (thr > 0.f && !(dbg & 32)) {
              const float mx = cib[c];
              const int d0 = __float2int_rz(__fmul_rz(__fmul_rz(thr, __frcp_rz(mx)), 0.99999f));
              m0 = 0;
#pragma unroll
              for (int jj = 0; jj < 32; ++jj) m0 |= (v[jj] >= d0 ? 1u : 0u) << jj;
            }
            const int64_t gbase = slot_offset + row0 + c * 32 - hmod;
            bool locked = false;
            int hcnt = 0;
            uint64_t hroot = 0;
            while (m0) {
              const int jj = __ffs(m0) - 1;
              m0 &= m0 - 1;
              const float sj = __fmul_rn(__int2float_rn(pick32(v, jj)), ciw[c * 32 + jj]);
              if (!(sj >= thr)) continue;
              const float key = __fmul_rn(sj, iq);
              if (!(key >= theta)) continue;
              if (dbg & 128) {  // debug: evaluate candidates, skip the heap
                thr = fmaxf(thr, -INFINITY);
                continue;
              }
              if (!locked) {
                // this query's heap is shared with the other column-half warp
                while (atomicCAS(&s_hlock[qrow], 0, 1) != 0) {
                }
                __threadfence_block();
                hcnt = s_hcnt[qrow];
                hroot = s_hroot[qrow];
                locked = true;
              }
              int64_t rel = gbase + jj;
              if (rel < 0) rel += gcap;
              const uint64_t comp = make_comp(key, (uint32_t)rel);
              if (hcnt < k) {
                heap[hcnt * BM] = comp;
                if (++hcnt == k) hroot = heapify(heap, k);
              } else if (comp > hroot) {
                hroot = heap_replace(heap, k, comp);
              }
            }
            if (locked) {
              s_hcnt[qrow] = hcnt;
              s_hroot[qrow] = hroot;
              __threadfence_block();
              atomicExch(&s_hlock[qrow], 0);
              if (hcnt >= k) thr = fmaxf(thr, s_threshold(comp_key(hroot), iq));
            }
          }
        };
        chunk(v0, 0);
        chunk(v1, 1);
        chunk(v2, 2);
        chunk(v3, 3);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&iempty[sl]);  // inverse norms of tile t consumed
    }
    asm volatile("bar.sync 1, %0;\n" ::"n"(EPI_WARPS * 32) : "memory");  // both halves done
    if (grp == 0 && q < nq) {
      uint64_t* out = partials + ((int64_t)slice * nq + q) * k;
      const int hc = s_hcnt[qrow];
      for (int i = 0; i < k; ++i) out[i] = (i < hc) ? heap[i * BM] : 0ull;
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc512<2>(tmem);
  }
}

}  // namespace pr

static size_t pair_fixed_smem(int dim, int k) {
  return (size_t)(dim / pr::BK) * pr::A_BLK + (size_t)pr::ISLOTS * pr::BN * 4 +
         (size_t)k * pr::BM * 8 + pr::BM * 16 + pr::EPI_WARPS * 8 * 4 + 512 + 1024;
}
static int pair_stages(int dim, int k) {
  for (int s = 8; s >= 3; --s)
    if (pair_fixed_smem(dim, k) + (size_t)s * pr::B_STAGE <= 227 * 1024) return s;
  return 0;
}

bool topk_pair_supported(const TopkArgs& a) {
  if (a.dim % pr::BK || a.dim > 512 || a.k < 1 || a.k > pr::KMAX) return false;
  if (a.n_rows >= (1LL << 31) || a.nq >= (1LL << 31)) return false;
  if (!a.inv_padded) return false;  // the tile's inverse norms are bulk-copied whole
  return pair_stages(a.dim, a.k) >= 4;
}

int topk_pair_lists(const TopkArgs& a, int device) {
  int64_t qtiles = (a.nq + pr::BM - 1) / pr::BM;
  qtiles = (qtiles + 1) / 2 * 2;
  const int64_t tiles = (a.n_rows + pr::BN - 1) / pr::BN;
  return pick_slices(qtiles, tiles, sm_count(device));
}

int launch_topk_pair(const TopkArgs& a, uint64_t* partials, int n_slices, cudaStream_t st,
                     const CUtensorMap& mq, const CUtensorMap& mb) {
  if (n_slices < 1) return set_error(SS_ERR_ARG, "pair: no slices");
  const int stages = pair_stages(a.dim, a.k);
  const size_t smem = pair_fixed_smem(a.dim, a.k) + (size_t)stages * pr::B_STAGE;
  SS_CUDA_TRY(cudaFuncSetAttribute(pr::k_topk_pair, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
  const int64_t tiles = (a.n_rows + pr::BN - 1) / pr::BN;
  const int64_t tps = (tiles + n_slices - 1) / n_slices;
  int64_t qtiles = (a.nq + pr::BM - 1) / pr::BM;
  qtiles = (qtiles + 1) / 2 * 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)qtiles, (unsigned)n_slices);
  cfg.blockDim = dim3(pr::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const char* dv = getenv("SS_TC_DEBUG");
  count_launch();
  SS_CUDA_TRY(cudaLaunchKernelEx(&cfg, pr::k_topk_pair, mq, mb, a.q_inv, a.nq, a.inv, a.n_rows,
                                 a.dim / pr::BK, stages, a.k, a.theta, a.head % a.gcap, a.gcap,
                                 a.slot_offset, tps, partials, dv ? atoi(dv) : 0));
  return SS_OK;
}

}  // namespace ss
