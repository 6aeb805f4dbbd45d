// Stage 1, large-batch path: int8 query x bank similarity on the 5th-gen
// tensor cores (tcgen05.mma kind::i8, int32 accumulators in TMEM), operands
// staged by TMA, fused with a per-query top-k in the epilogue -- the score
// matrix is never written to memory.
//
// Reference semantics: query_similar + north-star top-k;
// scores exactly as DESIGN.md section 3 (int8 dot products are exact in
// int32, so the tensor-core result is bit-identical to the CPU oracle).
//
// CTA = 128 queries (M, = TMEM lanes) x one slice of the bank streamed in
// 256-row tiles (N).  6 warps:
//   warp 0      TMA producer: A (queries, once) and B (bank K-blocks, ring)
//   warp 1      TMEM allocator + single-thread MMA issuer
//   warps 2..5  epilogue: tcgen05.ld 32 columns at a time, s = dot*inv_w,
//               one compare against the per-query heap threshold, rare
//               exact insert into the per-query shared-memory min-heap
// Two TMEM accumulator buffers (2 x 256 columns) let the MMA of tile t+1
// overlap the epilogue of tile t.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "ss_common.cuh"
#include "ss_internal.h"
#include "topk_heap.cuh"

namespace ss {

namespace tc {
constexpr int BM = 128;          // queries per CTA (TMEM lanes)
constexpr int BN = 256;          // bank rows per tile (UMMA N)
constexpr int BK = 128;          // bytes per K-block (one 128B swizzle atom)
constexpr int UK = 32;           // int8 K per tcgen05.mma
constexpr int THREADS = 192;
constexpr int EPI_WARP0 = 2;
constexpr int KMAX = 64;         // heap capacity (k <= 64 on this path)
constexpr int A_BLK = BM * BK;   // 16 KB per K-block of A
constexpr int B_STAGE = BN * BK; // 32 KB per K-block of B
}  // namespace tc

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int (&v)[32]) {
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
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// UMMA shared-memory descriptor, K-major, 128B swizzle: rows of 128 B, 8-row
// atoms 1024 B apart (SBO), LBO unused for swizzled K-major, version 1.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;                 // LBO (ignored)
  d |= (uint64_t)(1024 >> 4) << 32;       // SBO
  d |= (uint64_t)1 << 46;                 // descriptor version (tcgen05)
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}

// instruction descriptor: D=S32, A=B=signed int8, K-major both, N=256, M=128
constexpr uint32_t IDESC_I8 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(tc::BN >> 3) << 17) |
                              ((uint32_t)(tc::BM >> 4) << 24);

__device__ __noinline__ void tc_consider(uint64_t* heap, int k, HeapState* st, int dot, float iw,
                                         float iq, float theta, int64_t gslot, int64_t head,
                                         int64_t gcap) {
  heap_consider<tc::BM>(heap, k, *st, dot, iw, iq, theta, gslot, head, gcap);
}

__global__ void __launch_bounds__(tc::THREADS, 1)
k_topk_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmB,
          const float* __restrict__ q_inv, int64_t nq, const float* __restrict__ inv,
          int64_t n_rows, int nkb, int stages, int k, float theta, int64_t head, int64_t gcap,
          int64_t slot_offset, int64_t tiles_per_slice, uint64_t* __restrict__ partials) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~(uintptr_t)1023);
  uint8_t* sA = smem;                                        // nkb x 16 KB
  uint8_t* sB = sA + nkb * tc::A_BLK;                        // stages x 32 KB
  uint64_t* s_heap = reinterpret_cast<uint64_t*>(sB + stages * tc::B_STAGE);  // [k][128]
  float* s_iw = reinterpret_cast<float*>(s_heap + (size_t)k * tc::BM);      // [4][256]
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_iw + 4 * tc::BN);
  uint64_t* a_full = bars;
  uint64_t* full = bars + 1;
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = blockIdx.x, slice = blockIdx.y;
  const int64_t tile0 = (int64_t)slice * tiles_per_slice;
  const int64_t total_tiles = (n_rows + tc::BN - 1) / tc::BN;
  const int64_t tile1 = min(total_tiles, tile0 + tiles_per_slice);
  const int ntiles = (int)max((int64_t)0, tile1 - tile0);

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
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
                     smem_u32(s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
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
          mbar_expect_tx(&full[s], tc::B_STAGE);
          tma_load_2d(sB + s * tc::B_STAGE, &tmB, &full[s], kb * tc::BK, row0);
        }
      }
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
            uint64_t ad = umma_desc_sw128(a_base + kb * tc::A_BLK + kk * tc::UK);
            uint64_t bd = umma_desc_sw128(b_base + s * tc::B_STAGE + kk * tc::UK);
            tc_mma_i8(d, ad, bd, IDESC_I8, (kb | kk) != 0);
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
    const int64_t q = (int64_t)qt * tc::BM + qrow;
    const float iq = (q < nq) ? q_inv[q] : __int_as_float(0x7fc00000);
    HeapState st;
    st.cnt = 0;
    st.root = 0;
    st.thr_s = (iq == iq) ? s_threshold(theta, iq) : INFINITY;
    uint64_t* heap = s_heap + qrow;
    float* wiw = s_iw + ew * tc::BN;
    for (int t = 0; t < ntiles; ++t) {
      const int acc = t & 1;
      const int64_t row0 = (tile0 + t) * tc::BN;
      // this tile's inverse norms -> warp-private smem (8 per lane)
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        int64_t r = row0 + lane * 8 + u;
        wiw[lane * 8 + u] = (r < n_rows) ? inv[r] : __int_as_float(0x7fc00000);
      }
      __syncwarp();
      mbar_wait(&tfull[acc], (t >> 1) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem + ((uint32_t)(quarter * 32) << 16) + acc * tc::BN;
#pragma unroll 1
      for (int c = 0; c < tc::BN / 32; ++c) {
        int v[32];
        tmem_ld32(tbase + c * 32, v);
        if (c == tc::BN / 32 - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        float thr = st.thr_s;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float iw = wiw[c * 32 + j];
          const float s = __fmul_rn(__int2float_rn(v[j]), iw);
          if (s >= thr) {
            tc_consider(heap, k, &st, v[j], iw, iq, theta, slot_offset + row0 + c * 32 + j, head,
                        gcap);
            thr = st.thr_s;
          }
        }
      }
      __syncwarp();
    }
    if (q < nq) {
      uint64_t* out = partials + ((int64_t)slice * nq + q) * k;
      for (int i = 0; i < k; ++i) out[i] = (i < st.cnt) ? heap[i * tc::BM] : 0ull;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
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

static int tc_stages(int dim, int k) {
  const int fixed = (dim / tc::BK) * tc::A_BLK + k * tc::BM * 8 + 4 * tc::BN * 4 + 256 + 1024;
  for (int s = 4; s >= 2; --s)
    if (fixed + s * tc::B_STAGE <= 227 * 1024) return s;
  return 0;
}

static size_t tc_smem(int dim, int k, int stages) {
  return (size_t)(dim / tc::BK) * tc::A_BLK + (size_t)stages * tc::B_STAGE +
         (size_t)k * tc::BM * 8 + 4 * tc::BN * 4 + 256 + 1024;
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

int topk_tc_slices(const TopkArgs& a, int device) {
  int sms = sm_count(device);
  int64_t qtiles = (a.nq + tc::BM - 1) / tc::BM;
  int64_t tiles = (a.n_rows + tc::BN - 1) / tc::BN;
  int64_t want = sms / qtiles;
  if (want < 1) want = 1;
  if (want > tiles) want = tiles;
  return (int)want;
}

int launch_topk_tc(const TopkArgs& a, uint64_t* partials, int n_slices, cudaStream_t st) {
  if (!topk_tc_supported(a)) return set_error(SS_ERR_UNSUPPORTED, "tcgen05 path unsupported");
  const int stages = tc_stages(a.dim, a.k);
  const size_t smem = tc_smem(a.dim, a.k, stages);
  CUtensorMap mq, mb;
  if (int rc = make_map(&mq, a.q, a.nq, a.dim, tc::BM)) return rc;
  if (int rc = make_map(&mb, a.emb, a.n_rows, a.dim, tc::BN)) return rc;
  SS_CUDA_TRY(cudaFuncSetAttribute(k_topk_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t tiles = (a.n_rows + tc::BN - 1) / tc::BN;
  const int64_t tps = (tiles + n_slices - 1) / n_slices;
  dim3 grid((unsigned)((a.nq + tc::BM - 1) / tc::BM), (unsigned)n_slices);
  count_launch();
  k_topk_tc<<<grid, tc::THREADS, smem, st>>>(mq, mb, a.q_inv, a.nq, a.inv, a.n_rows, a.dim / tc::BK,
                                             stages, a.k, a.theta, a.head, a.gcap, a.slot_offset,
                                             tps, partials);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

}  // namespace ss
