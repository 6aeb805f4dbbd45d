// Stage 1, large-batch path: int8 query x bank similarity on the 5th-gen
// tensor cores (tcgen05.mma kind::i8, int32 accumulators in TMEM), operands
// staged by TMA, fused with a per-query top-k in the epilogue -- the score
// matrix is never written to memory.
//
// Reference semantics: query_similar + north-star top-k;
// scores exactly as DESIGN.md section 3 (int8 dot products are exact in
// int32, so the tensor-core result is bit-identical to the CPU oracle).
//
// A CTA owns 128 queries (M = TMEM lanes) and streams one slice of the bank
// in 256-row tiles (N); with nq <= 128 (one query tile, 148 bank slices) it
// is the HBM-streaming scan of the north star.  6 warps per CTA:
//   warp 0      TMA producer: A (queries, once) and B (bank K-blocks, ring)
//   warp 1      TMEM allocator + single-thread MMA issuer (leader CTA)
//   warps 2..5  epilogue: tcgen05.ld 32 columns at a time, s = dot*inv_w,
//               one max-tree compare per 32 columns against the per-query
//               heap threshold; rare exact inserts into the per-query
//               shared-memory min-heap
// Two TMEM accumulator buffers (2 x 256 columns) let the MMA of tile t+1
// overlap the epilogue of tile t.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>

#include "ss_common.cuh"
#include "ss_internal.h"
#include "topk_heap.cuh"
#include "tc_util.cuh"

namespace ss {

// out-of-line heap maintenance for the epilogue (rare): returns the new root
__device__ __noinline__ uint64_t tc_heapify(uint64_t* heap, int k) {
  for (int i = k / 2 - 1; i >= 0; --i) heap_sift_down<tc::BM>(heap, k, i, heap[i * tc::BM]);
  return heap[0];
}
__device__ __noinline__ uint64_t tc_heap_replace(uint64_t* heap, int k, uint64_t x) {
  heap_sift_down<tc::BM>(heap, k, 0, x);
  return heap[0];
}

__global__ void __launch_bounds__(tc::THREADS, 1)
k_topk_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmB,
          const float* __restrict__ q_inv, int64_t nq, const float* __restrict__ inv,
          int64_t n_rows, int nkb, int stages, int k, float theta, int64_t hmod, int64_t gcap,
          int64_t slot_offset, int64_t tiles_per_slice, uint64_t* __restrict__ partials,
          int spread, int* __restrict__ counts, const int* __restrict__ resolved) {
  constexpr int B_STAGE = tc::BN * tc::BK;     // bytes per K-block stage
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment for the 128B-swizzle atoms; index the __shared__ array
  // (not an integer round trip) so every access stays LDS/STS, not generic.
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                                        // nkb x 16 KB
  uint8_t* sB = sA + nkb * tc::A_BLK;                        // stages x B_STAGE
  uint64_t* s_heap = reinterpret_cast<uint64_t*>(sB + stages * B_STAGE);  // [k][128]
  float* s_iw = reinterpret_cast<float*>(s_heap + (size_t)k * tc::BM);  // [4 warps][2][256]
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_iw + 8 * tc::BN);
  uint64_t* a_full = bars;
  uint64_t* full = bars + 1;
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = blockIdx.x, slice = blockIdx.y;  // qt: 128-query tile of this CTA
  const int64_t tile0 = (int64_t)slice * tiles_per_slice;
  const int64_t total_tiles = (n_rows + tc::BN - 1) / tc::BN;
  const int64_t tile1 = min(total_tiles, tile0 + tiles_per_slice);
  const int ntiles = (int)max((int64_t)0, tile1 - tile0);
  // pure top-k cascade, second pass (see launch_topk_ts): leave at once when
  // every query of this tile already holds >= k keys above the threshold
  // pass's theta
  if (resolved) {
    int need = 0;
    for (int i = threadIdx.x; i < tc::BM; i += blockDim.x) {
      const int64_t qq = (int64_t)qt * tc::BM + i;
      if (qq < nq) {
        int sum = 0;
        for (int s2 = 0; s2 < (int)gridDim.y; ++s2) sum += resolved[(int64_t)s2 * nq + qq];
        need |= sum < k;
      }
    }
    if (!__syncthreads_or(need)) return;
  }

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmQ) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmB) : "memory");
    mbar_init(a_full, 1);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) tmem_alloc512(s_tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer ---
    if (lane == 0 && ntiles > 0) {
      mbar_expect_tx(a_full, nkb * tc::A_BLK);
      for (int kb = 0; kb < nkb; ++kb)
        tma_load_2d(sA + kb * tc::A_BLK, &tmQ, a_full, kb * tc::BK, qt * tc::BM);
      int it = 0;
      for (int t = 0; t < ntiles; ++t) {
        const int row0 = (int)((tile0 + t) * tc::BN);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % stages;
          mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
          mbar_expect_tx(&full[s], B_STAGE);
          tma_load_2d(sB + s * B_STAGE, &tmB, &full[s], kb * tc::BK, row0);
        }
      }
      // drain: wait for the final MMA commits on every stage, so no arrive
      // can target this CTA's shared memory after it exits
      for (int i = max(0, it - stages); i < it; ++i) mbar_wait(&empty[i % stages], (i / stages) & 1);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer ----
    if (lane == 0 && ntiles > 0) {
      mbar_wait(a_full, 0);
      tc_fence_after();
      const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
      int it = 0;
      for (int t = 0; t < ntiles; ++t) {
        const int acc = t & 1;
        mbar_wait(&tempty[acc], ((t >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * tc::BN;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % stages;
          mbar_wait(&full[s], (it / stages) & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < tc::BK / tc::UK; ++kk) {
            const uint64_t ad = umma_desc_sw128(a_base + kb * tc::A_BLK + kk * tc::UK);
            const uint64_t bd = umma_desc_sw128(b_base + s * B_STAGE + kk * tc::UK);
            tc_mma_i8(d, ad, bd, idesc_i8(), (kb | kk) != 0);
          }
          tc_commit(&empty[s]);  // frees the B stage once these MMAs retire
        }
        tc_commit(&tfull[acc]);  // accumulator ready for the epilogue
      }
    }
  } else {
    // --------------------------------------------------------- epilogue ----
    const int ew = warp - tc::EPI_WARP0;        // 0..3
    const int quarter = warp & 3;               // TMEM lane quarter this warp may access
    const int qrow = quarter * 32 + lane;       // query row within the tile
    // spread (one query tile, nq <= 128): query i sits in TMEM row
    // (i % 4) * 32 + i / 4, so a few queries occupy all four lane quarters and
    // all four epilogue warps share the slow path (pure top-k)
    const int64_t q = spread ? (int64_t)((qrow & 31) * 4 + (qrow >> 5)) : (int64_t)qt * tc::BM + qrow;
    const float iq = (q < nq) ? q_inv[q] : __int_as_float(0x7fc00000);
    // per-query heap state in registers (see topk_heap.cuh for the invariant)
    int hcnt = 0;
    uint64_t hroot = 0;
    uint64_t* heap = s_heap + qrow;
    float* wiw = s_iw + ew * 2 * tc::BN;  // double-buffered per warp
    const float NaNf = __int_as_float(0x7fc00000);
    // register prefetch of a tile's inverse norms (8 per lane)
    float pre[8];
    auto fetch_iw = [&](int t) {
      const int64_t r0 = (tile0 + t) * tc::BN + lane * 8;
      if (r0 + 8 <= n_rows) {
        const float4* p = reinterpret_cast<const float4*>(inv + r0);
        float4 a = __ldg(p), b = __ldg(p + 1);
        pre[0] = a.x; pre[1] = a.y; pre[2] = a.z; pre[3] = a.w;
        pre[4] = b.x; pre[5] = b.y; pre[6] = b.z; pre[7] = b.w;
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) pre[u] = (r0 + u < n_rows) ? inv[r0 + u] : NaNf;
      }
    };
    if (ntiles > 0) fetch_iw(0);
    // conservative s-domain filter: admits every row whose exact key can reach
    // the current k-th best (or theta while the heap fills)
    float thr = (iq == iq) ? s_threshold(theta, iq) : INFINITY;
    for (int t = 0; t < ntiles; ++t) {
      const int acc = t & 1;
      const int64_t row0 = (tile0 + t) * tc::BN;
      float* ciw = wiw + (t & 1) * tc::BN;
      {
        float4* d = reinterpret_cast<float4*>(ciw + lane * 8);
        d[0] = make_float4(pre[0], pre[1], pre[2], pre[3]);
        d[1] = make_float4(pre[4], pre[5], pre[6], pre[7]);
      }
      __syncwarp();
      if (t + 1 < ntiles) fetch_iw(t + 1);  // overlaps this tile's epilogue
      mbar_wait(&tfull[acc], (t >> 1) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem + ((uint32_t)(quarter * 32) << 16) + acc * tc::BN;
      auto chunk = [&](const int (&v)[32], const int c) {
        // hot path: 32 independent s = fl(dot * inv_w), one max tree, one branch
        float s[32];
        const float4* iw4 = reinterpret_cast<const float4*>(ciw + c * 32);
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          const float4 w = iw4[j4];  // broadcast LDS.128
          s[4 * j4 + 0] = __fmul_rn(__int2float_rn(v[4 * j4 + 0]), w.x);
          s[4 * j4 + 1] = __fmul_rn(__int2float_rn(v[4 * j4 + 1]), w.y);
          s[4 * j4 + 2] = __fmul_rn(__int2float_rn(v[4 * j4 + 2]), w.z);
          s[4 * j4 + 3] = __fmul_rn(__int2float_rn(v[4 * j4 + 3]), w.w);
        }
        float m[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) m[j] = fmaxf(s[j], s[j + 16]);
#pragma unroll
        for (int j = 0; j < 8; ++j) m[j] = fmaxf(m[j], m[j + 8]);
#pragma unroll
        for (int j = 0; j < 4; ++j) m[j] = fmaxf(m[j], m[j + 4]);
        const float mx = fmaxf(fmaxf(m[0], m[1]), fmaxf(m[2], m[3]));
        if (mx >= thr) {  // rare: exact keys and heap inserts for this chunk
          // key = fl(s * iq) is exactly the oracle's fl(fl(dot*iw)*iq); the
          // common case is an append while the heap fills, inlined here; only
          // heapify / root replacement leave the hot code (noinline helpers)
          const int64_t gbase = slot_offset + row0 + c * 32 - hmod;
          uint32_t mask = 0;
#pragma unroll
          for (int j = 0; j < 32; ++j) mask |= (s[j] >= thr ? 1u : 0u) << j;
          float sl[32];  // dynamic indexing below: the compiler stages these in local memory
#pragma unroll
          for (int j = 0; j < 32; ++j) sl[j] = s[j];
          while (mask) {
            const int j = __ffs(mask) - 1;
            mask &= mask - 1;
            const float key = __fmul_rn(sl[j], iq);
            if (key >= theta) {
              int64_t rel = gbase + j;
              if (rel < 0) rel += gcap;
              const uint64_t comp = make_comp(key, (uint32_t)rel);
              if (hcnt < k) {
                heap[hcnt * tc::BM] = comp;
                if (++hcnt == k) {
                  hroot = tc_heapify(heap, k);
                  thr = fmaxf(thr, s_threshold(comp_key(hroot), iq));
                }
              } else if (comp > hroot) {
                hroot = tc_heap_replace(heap, k, comp);
                thr = fmaxf(thr, s_threshold(comp_key(hroot), iq));
              }
            }
          }
        }
      };
      // software pipeline: the TMEM load of chunk c+1 is in flight while
      // chunk c is scanned
      int va[32], vb[32];
      tmem_ld32_async(tbase, va);
      tmem_wait_regs(va);
#pragma unroll 1
      for (int c = 0; c < tc::BN / 32; c += 2) {
        tmem_ld32_async(tbase + (c + 1) * 32, vb);
        chunk(va, c);
        tmem_wait_regs(vb);
        if (c + 2 < tc::BN / 32) {
          tmem_ld32_async(tbase + (c + 2) * 32, va);
        } else {  // accumulator drained: hand it back to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        chunk(vb, c + 1);
        if (c + 2 < tc::BN / 32) tmem_wait_regs(va);
      }
      __syncwarp();
    }
    if (q < nq) {
      uint64_t* out = partials + ((int64_t)slice * nq + q) * k;
      for (int i = 0; i < k; ++i) out[i] = (i < hcnt) ? heap[i * tc::BM] : 0ull;
      if (counts) counts[(int64_t)slice * nq + q] = hcnt;  // (pure top-k cascade, first pass)
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc512(tmem);
  }
}

// ---------------------------------------------------------------- host ----
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

static int make_map(CUtensorMap* m, const void* base, int64_t rows, int dim, int box_rows) {
  auto enc = get_encode();
  if (!enc) return set_error(SS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t gdim[2] = {(cuuint64_t)dim, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)dim};
  cuuint32_t box[2] = {(cuuint32_t)tc::BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), gdim, gstride, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(SS_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return SS_OK;
}

static size_t tc_fixed_smem(int dim, int k) {
  return (size_t)(dim / tc::BK) * tc::A_BLK + (size_t)k * tc::BM * 8 + 8 * tc::BN * 4 + 512 + 1024;
}

// as many B stages as fit beside A, the heaps and the inverse-norm buffers
static int tc_stages(int dim, int k) {
  const size_t stage = (size_t)tc::BN * tc::BK;
  const size_t fixed = tc_fixed_smem(dim, k);
  for (int c = 8; c >= 2; --c)
    if (fixed + c * stage <= 227 * 1024) return c;
  return 0;
}

bool topk_tc_supported(const TopkArgs& a) {
  if (a.dim % tc::BK || a.dim > 512 || a.k > tc::KMAX || a.k < 1) return false;
  if (a.n_rows >= (1LL << 31) || a.nq >= (1LL << 31)) return false;
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0) return false;  // built for sm_100a only
  return tc_stages(a.dim, a.k) >= 2;
}

// One kernel per regime: above one 128-query tile the A-in-TMEM kernel
// (k_topk_sm100_ts.cu, two epilogue warps per sub-partition); at or below it
// this kernel, as a bank-streaming scan over 148 slices.
static bool use_ts(const TopkArgs& a) { return a.nq > tc::BM && topk_ts_supported(a); }

int topk_tc_slices(const TopkArgs& a, int device) {
  if (use_ts(a)) return topk_ts_lists(a, device);
  const int sms = sm_count(device);
  const int64_t qtiles = (a.nq + tc::BM - 1) / tc::BM;
  const int64_t tiles = (a.n_rows + tc::BN - 1) / tc::BN;
  int64_t want = sms / qtiles;
  if (want < 1) want = 1;
  if (want > tiles) want = tiles;
  return (int)want;
}

// queries of a single tile copied to rows (i % 4) * 32 + i / 4 (see `spread`)
__global__ void k_spread_queries(const int8_t* __restrict__ q, int64_t nq, int dim,
                                 int8_t* __restrict__ out) {
  const int i = blockIdx.x;
  if (i >= nq) return;
  const int r = (i & 3) * 32 + (i >> 2);
  const int4* src = reinterpret_cast<const int4*>(q + (int64_t)i * dim);
  int4* dst = reinterpret_cast<int4*>(out + (int64_t)r * dim);
  for (int j = threadIdx.x; j < dim / 16; j += blockDim.x) dst[j] = src[j];
}

static int launch_tc(const TopkArgs& a, uint64_t* partials, int n_slices, cudaStream_t st,
                     int* counts = nullptr, const int* resolved = nullptr) {
  const int stages = tc_stages(a.dim, a.k);
  if (stages < 2) return set_error(SS_ERR_UNSUPPORTED, "tcgen05: not enough shared memory");
  const size_t smem = tc_fixed_smem(a.dim, a.k) + (size_t)stages * tc::BN * tc::BK;
  CUtensorMap mq, mb;
  // pure top-k on a single query tile: spread the queries over the four TMEM
  // lane quarters so every epilogue warp shares the (then frequent) exact
  // path (rows past nq in the scratch are never used: their query index maps
  // >= nq).  With a similarity floor the exact path is rare and the extra
  // copy launch would only cost time.
  const int spread = (a.nq <= tc::BM && a.qscratch && a.theta <= 0.f) ? 1 : 0;
  if (spread) {
    count_launch();
    k_spread_queries<<<(unsigned)a.nq, 32, 0, st>>>(a.q, a.nq, a.dim, a.qscratch);
    SS_LAUNCH_CHECK();
    if (int rc = make_map(&mq, a.qscratch, tc::BM, a.dim, tc::BM)) return rc;
  } else if (int rc = make_map(&mq, a.q, a.nq, a.dim, tc::BM)) {
    return rc;
  }
  if (int rc = make_map(&mb, a.emb, a.n_rows, a.dim, tc::BN)) return rc;
  SS_CUDA_TRY(cudaFuncSetAttribute(k_topk_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t tiles = (a.n_rows + tc::BN - 1) / tc::BN;
  const int64_t tps = (tiles + n_slices - 1) / n_slices;
  const int64_t qtiles = (a.nq + tc::BM - 1) / tc::BM;
  count_launch();
  k_topk_tc<<<dim3((unsigned)qtiles, (unsigned)n_slices), tc::THREADS, smem, st>>>(
      mq, mb, a.q_inv, a.nq, a.inv, a.n_rows, a.dim / tc::BK, stages, a.k, a.theta,
      a.head % a.gcap, a.gcap, a.slot_offset, tps, partials, spread, counts, resolved);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

int launch_topk_tc(const TopkArgs& a, uint64_t* partials, int n_slices, cudaStream_t st) {
  if (!topk_tc_supported(a)) return set_error(SS_ERR_UNSUPPORTED, "tcgen05 path unsupported");
  if (use_ts(a)) return launch_topk_ts(a, partials, n_slices, st);
  if (a.gslots && a.theta <= 0.f && n_slices <= kMaxShareSlices) {
    // pure top-k as the threshold cascade (see launch_topk_ts); the counts
    // live in the bank's pure-top-k scratch after the bound slots
    int* counts = reinterpret_cast<int*>(a.gslots + (size_t)kMaxShareSlices * a.nq);
    TopkArgs a1 = a;
    a1.theta = kCascadeTheta;
    if (int rc = launch_tc(a1, partials, n_slices, st, counts, nullptr)) return rc;
    return launch_tc(a, partials, n_slices, st, nullptr, counts);
  }
  return launch_tc(a, partials, n_slices, st);
}

}  // namespace ss
