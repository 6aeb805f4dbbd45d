// Stage 4: rank requests by ascending (G, id) -- SPEC.md:393-395 (primary key
// = Gittins index, smaller served first; tie -> arrival order, ids are
// assigned in arrival order).  Equivalently descending north-star index 1/G.
//
//   n <= 4096 : one CTA, bitonic sort of (orderable64(G), id, index) in smem
//   n  > 4096 : LSD radix sort, 8-bit digits: 4 passes over the low 32 bits of
//               id, then 8 passes over orderable64(G); each pass is
//               histogram -> exclusive scan -> stable scatter (warp match_any
//               ranking), so ties keep id order.
#include "ss_common.cuh"
#include "ss_internal.h"

namespace ss {

constexpr int SMALL_SORT_MAX = 4096;

__global__ void __launch_bounds__(1024)
k_rank_small(const double* __restrict__ G, const int64_t* __restrict__ ids, int n, int npad,
             int64_t* __restrict__ perm) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* key = reinterpret_cast<uint64_t*>(smem);
  int64_t* id = reinterpret_cast<int64_t*>(key + npad);
  int32_t* idx = reinterpret_cast<int32_t*>(id + npad);
  for (int i = threadIdx.x; i < npad; i += blockDim.x) {
    if (i < n) {
      key[i] = f64_order(G[i]);
      id[i] = ids ? ids[i] : i;
    } else {
      key[i] = ~0ull;
      id[i] = INT64_MAX;
    }
    idx[i] = i;
  }
  __syncthreads();
  for (int size = 2; size <= npad; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < npad; i += blockDim.x) {
        int j = i ^ stride;
        if (j > i) {
          bool asc = ((i & size) == 0);
          uint64_t ka = key[i], kb = key[j];
          int64_t ia = id[i], ib = id[j];
          bool gt = (ka > kb) || (ka == kb && ia > ib);
          if (gt == asc) {
            key[i] = kb; key[j] = ka;
            id[i] = ib; id[j] = ia;
            int32_t t = idx[i]; idx[i] = idx[j]; idx[j] = t;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) perm[i] = idx[i];
}

// ------------------------------------------------------- rank by counting --
// n <= 8192: every thread owns one request and counts the requests that
// precede it in the total order (G, id, index) -- a strict total order, so
// the ranks form a permutation and perm[rank_i] = i is exact and stable.
// Keys are staged through shared memory in 1024-entry tiles.
constexpr int COUNT_MAX = 8192;

// 8 lanes per request: lane t of a group compares against j = t, t+8, ...
// (L1-resident loads), then the group sums its partial ranks with shuffles.
constexpr int RC_LANES = 8;

__global__ void __launch_bounds__(256)
k_rank_count(const double* __restrict__ G, const int64_t* __restrict__ ids, int n,
             int64_t* __restrict__ perm) {
  __shared__ uint64_t sk[2048];
  __shared__ int64_t sid[2048];
  const int t = threadIdx.x & (RC_LANES - 1);
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) / RC_LANES;
  const bool live = i < n;
  const uint64_t ki = live ? f64_order(G[i]) : 0ull;
  const int64_t ii = live ? (ids ? ids[i] : i) : 0;
  int rank = 0;
  for (int t0 = 0; t0 < n; t0 += 2048) {
    const int m = min(2048, n - t0);
    __syncthreads();
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
      sk[j] = f64_order(G[t0 + j]);
      sid[j] = ids ? ids[t0 + j] : t0 + j;
    }
    __syncthreads();
    if (live) {
#pragma unroll 8
      for (int j = t; j < m; j += RC_LANES) {
        const uint64_t kj = sk[j];
        const int64_t ij = sid[j];
        rank += (kj < ki) | ((kj == ki) & ((ij < ii) | ((ij == ii) & (t0 + j < i))));
      }
    }
  }
#pragma unroll
  for (int o = RC_LANES / 2; o > 0; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
  if (live && t == 0) perm[rank] = i;
}

// ---------------------------------------------------------------- radix ----
constexpr int RT_THREADS = 256;
constexpr int RT_ITEMS = 8;
constexpr int RT_TILE = RT_THREADS * RT_ITEMS;

__global__ void k_rank_init(const double* __restrict__ G, const int64_t* __restrict__ ids,
                            int64_t n, uint64_t* __restrict__ key, uint32_t* __restrict__ id32,
                            uint32_t* __restrict__ idx) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  key[i] = f64_order(G[i]);
  id32[i] = ids ? (uint32_t)ids[i] : (uint32_t)i;
  idx[i] = (uint32_t)i;
}

__device__ __forceinline__ int digit_of(uint64_t key, uint32_t id, int pass) {
  return pass < 4 ? (int)((id >> (8 * pass)) & 255u) : (int)((key >> (8 * (pass - 4))) & 255ull);
}

__global__ void __launch_bounds__(RT_THREADS)
k_radix_hist(const uint64_t* __restrict__ key, const uint32_t* __restrict__ id32, int64_t n,
             int pass, int nblocks, uint32_t* __restrict__ bhist) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t base = (int64_t)blockIdx.x * RT_TILE;
  for (int it = 0; it < RT_ITEMS; ++it) {
    int64_t i = base + (int64_t)it * RT_THREADS + threadIdx.x;
    bool live = i < n;
    int d = live ? digit_of(key[i], id32[i], pass) : 0;
    unsigned am = __ballot_sync(0xffffffffu, live);
    if (live) {
      unsigned peers = __match_any_sync(am, d);
      if ((peers & ((1u << lane) - 1u)) == 0u) atomicAdd(&h[d], __popc(peers));
    }
  }
  __syncthreads();
  bhist[threadIdx.x * nblocks + blockIdx.x] = h[threadIdx.x];  // digit-major
}

// exclusive scan of 256*nblocks counters (digit-major) in one CTA
__global__ void __launch_bounds__(1024)
k_radix_scan(uint32_t* __restrict__ bhist, int total) {
  __shared__ uint32_t s_warp[32];
  __shared__ uint32_t s_carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < total; b0 += 1024) {
    int i = b0 + threadIdx.x;
    uint32_t v = i < total ? bhist[i] : 0;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint32_t y = s_warp[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= o) y += t;
      }
      s_warp[lane] = y;
    }
    __syncthreads();
    uint32_t pre = (warp ? s_warp[warp - 1] : 0) + s_carry;
    if (i < total) bhist[i] = pre + x - v;
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = pre + x;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(RT_THREADS)
k_radix_scatter(const uint64_t* __restrict__ key, const uint32_t* __restrict__ id32,
                const uint32_t* __restrict__ idx, int64_t n, int pass, int nblocks,
                const uint32_t* __restrict__ offs, uint64_t* __restrict__ okey,
                uint32_t* __restrict__ oid, uint32_t* __restrict__ oidx) {
  __shared__ uint32_t cnt[RT_THREADS / 32][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = lane; d < 256; d += 32) cnt[warp][d] = 0;
  __syncwarp();
  const int64_t base = (int64_t)blockIdx.x * RT_TILE + (int64_t)warp * (RT_TILE / 8);
  uint64_t k_[RT_ITEMS];
  uint32_t id_[RT_ITEMS], ix_[RT_ITEMS], rk[RT_ITEMS];
  int dg[RT_ITEMS];
#pragma unroll
  for (int it = 0; it < RT_ITEMS; ++it) {
    int64_t i = base + it * 32 + lane;
    bool live = i < n;
    k_[it] = live ? key[i] : 0;
    id_[it] = live ? id32[i] : 0;
    ix_[it] = live ? idx[i] : 0;
    int d = live ? digit_of(k_[it], id_[it], pass) : 0;
    dg[it] = live ? d : -1;
    unsigned am = __ballot_sync(0xffffffffu, live);
    uint32_t r = 0;
    if (live) {
      unsigned peers = __match_any_sync(am, d);
      uint32_t before = cnt[warp][d];
      r = before + __popc(peers & ((1u << lane) - 1u));
      __syncwarp(am);
      if ((peers & ((1u << lane) - 1u)) == 0u) cnt[warp][d] = before + __popc(peers);
    }
    __syncwarp();
    rk[it] = r;
  }
  __syncthreads();
  // per-digit exclusive scan across warps -> cnt[w][d] becomes warp offset
  {
    const int d = threadIdx.x;  // 256 threads, 256 digits
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < RT_THREADS / 32; ++w) {
      uint32_t c = cnt[w][d];
      cnt[w][d] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < RT_ITEMS; ++it) {
    if (dg[it] < 0) continue;
    int d = dg[it];
    uint32_t pos = offs[d * nblocks + blockIdx.x] + cnt[warp][d] + rk[it];
    okey[pos] = k_[it];
    oid[pos] = id_[it];
    oidx[pos] = ix_[it];
  }
}

__global__ void k_rank_out(const uint32_t* __restrict__ idx, int64_t n, int64_t* __restrict__ perm) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) perm[i] = idx[i];
}

int64_t rank_workspace_bytes(int64_t n) {
  if (n <= SMALL_SORT_MAX) return 256;
  int64_t nblocks = (n + RT_TILE - 1) / RT_TILE;
  return 2 * n * (8 + 4 + 4) + 256 * nblocks * 4 + 1024;
}

int launch_rank(const double* G, const int64_t* ids, int64_t n, int64_t* perm, void* ws,
                int64_t ws_bytes, cudaStream_t st) {
  if (n <= 0) return SS_OK;
  if (n <= COUNT_MAX) {
    count_launch();
    k_rank_count<<<(unsigned)((n * RC_LANES + 255) / 256), 256, 0, st>>>(G, ids, (int)n, perm);
    SS_LAUNCH_CHECK();
    return SS_OK;
  }
  if (n <= SMALL_SORT_MAX) {
    int npad = 1;
    while (npad < n) npad <<= 1;
    size_t smem = (size_t)npad * (8 + 8 + 4);
    if (smem > 48 * 1024)
      SS_CUDA_TRY(cudaFuncSetAttribute(k_rank_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    count_launch();
    k_rank_small<<<1, 1024, smem, st>>>(G, ids, (int)n, npad, perm);
    SS_LAUNCH_CHECK();
    return SS_OK;
  }
  if (n > 0x7fffffffLL) return set_error(SS_ERR_UNSUPPORTED, "rank n too large");
  if (ws_bytes < rank_workspace_bytes(n))
    return set_error(SS_ERR_ARG, "rank workspace too small (%lld < %lld)", (long long)ws_bytes,
                     (long long)rank_workspace_bytes(n));
  const int nblocks = (int)((n + RT_TILE - 1) / RT_TILE);
  unsigned char* p = reinterpret_cast<unsigned char*>(ws);
  uint64_t* key[2];
  uint32_t* id[2];
  uint32_t* ix[2];
  key[0] = reinterpret_cast<uint64_t*>(p); p += n * 8;
  key[1] = reinterpret_cast<uint64_t*>(p); p += n * 8;
  id[0] = reinterpret_cast<uint32_t*>(p); p += n * 4;
  id[1] = reinterpret_cast<uint32_t*>(p); p += n * 4;
  ix[0] = reinterpret_cast<uint32_t*>(p); p += n * 4;
  ix[1] = reinterpret_cast<uint32_t*>(p); p += n * 4;
  uint32_t* bhist = reinterpret_cast<uint32_t*>(p);
  count_launch();
  k_rank_init<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(G, ids, n, key[0], id[0], ix[0]);
  SS_LAUNCH_CHECK();
  int cur = 0;
  for (int pass = 0; pass < 12; ++pass) {
    if (pass < 4 && ids == nullptr) continue;  // identity ids: input already in id order
    count_launch();
    k_radix_hist<<<nblocks, RT_THREADS, 0, st>>>(key[cur], id[cur], n, pass, nblocks, bhist);
    count_launch();
    k_radix_scan<<<1, 1024, 0, st>>>(bhist, 256 * nblocks);
    count_launch();
    k_radix_scatter<<<nblocks, RT_THREADS, 0, st>>>(key[cur], id[cur], ix[cur], n, pass, nblocks,
                                                     bhist, key[cur ^ 1], id[cur ^ 1], ix[cur ^ 1]);
    SS_LAUNCH_CHECK();
    cur ^= 1;
  }
  count_launch();
  k_rank_out<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ix[cur], n, perm);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

}  // namespace ss
