// Stage 4: rank requests by ascending (G, id) -- SPEC.md:393-395 (primary key
// = Gittins index, smaller served first; tie -> arrival order, ids are
// assigned in arrival order).  Equivalently descending north-star index 1/G.
//
//   n <= 5120 : rank by counting (32 lanes per request up to 2048, else 8)
//   n <= 8192 : 1024-request chunks bitonic-sorted per CTA, then ranks by
//               binary search across the sorted chunks
//   n  > 8192 : onesweep LSD radix sort (see below), stable, ties keep id
//               order.
#include "ss_common.cuh"
#include "ss_internal.h"

namespace ss {

// ------------------------------------------------------- rank by counting --
// n <= 5120: every thread owns one request and counts the requests that
// precede it in the total order (G, id, index) -- a strict total order, so
// the ranks form a permutation and perm[rank_i] = i is exact and stable.
// Keys are staged through shared memory in 1024-entry tiles.
constexpr int COUNT_MAX = 5120;  // measured crossover with the chunked rank (scripts/time_rank.py)

// L lanes per request (32 up to 2048 requests, else 8): lane t of a group
// compares against j = t, t+L, ... (shared-memory tiles), then the group sums
// its partial ranks with shuffles.
template <int L>
__global__ void __launch_bounds__(256)
k_rank_count(const double* __restrict__ G, const int64_t* __restrict__ ids, int n,
             int64_t* __restrict__ perm) {
  constexpr int RC_LANES = L;
  pdl_wait();  // G from the previous kernel
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

// ------------------------------------------------------ 5120 < n <= 8192 ---
// Chunked rank: each 1024-request chunk is bitonic-sorted by one CTA on the
// strict total order (orderable64(G), id, index) -- strides below 32 through
// warp shuffles, the rest through shared memory -- and a request's rank is
// its position in its own chunk plus, for every other chunk, the number of
// that chunk's entries before it (binary search over all sorted chunks staged
// in shared memory).  O(n log n) instead of the counting rank's O(n^2):
// 25-27 us against 39-52 us at n = 6000-8192.  Keys are unique (index breaks
// every tie), so the ranks form a permutation and perm[rank] = index is exact
// and stable.
constexpr int CH_N = 1024;
constexpr int CHUNK_MAX = 8192;  // chunks staged whole in shared memory by the merge

struct RkKey {
  uint64_t k;
  int64_t id;
  int32_t ix;
};
__device__ __forceinline__ bool rk_less(const RkKey& a, const RkKey& b) {
  return a.k < b.k || (a.k == b.k && (a.id < b.id || (a.id == b.id && a.ix < b.ix)));
}

__global__ void __launch_bounds__(CH_N)
k_rank_chunk(const double* __restrict__ G, const int64_t* __restrict__ ids, int n,
             uint64_t* __restrict__ sk, int64_t* __restrict__ sid, int32_t* __restrict__ six) {
  pdl_wait();  // G from the previous kernel
  __shared__ uint64_t xk[CH_N];
  __shared__ int64_t xid[CH_N];
  __shared__ int32_t xix[CH_N];
  const int t = threadIdx.x;
  const int i = blockIdx.x * CH_N + t;
  RkKey me;
  if (i < n) {
    me.k = f64_order(G[i]);
    me.id = ids ? ids[i] : i;
    me.ix = i;
  } else {  // sentinels sort last
    me.k = ~0ull;
    me.id = INT64_MAX;
    me.ix = INT32_MAX;
  }
  for (int size = 2; size <= CH_N; size <<= 1) {
    const bool asc = (t & size) == 0;
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      RkKey o;
      if (stride >= 32) {
        xk[t] = me.k; xid[t] = me.id; xix[t] = me.ix;
        __syncthreads();
        o.k = xk[t ^ stride]; o.id = xid[t ^ stride]; o.ix = xix[t ^ stride];
        __syncthreads();
      } else {
        o.k = __shfl_xor_sync(0xffffffffu, me.k, stride);
        o.id = __shfl_xor_sync(0xffffffffu, me.id, stride);
        o.ix = __shfl_xor_sync(0xffffffffu, me.ix, stride);
      }
      const bool lower = (t & stride) == 0;
      const bool take = (lower == asc) ? rk_less(o, me) : rk_less(me, o);  // keep min / max
      if (take) me = o;
    }
  }
  const int m = min(CH_N, n - blockIdx.x * CH_N);
  const int o = blockIdx.x * CH_N + t;
  if (t < m) { sk[o] = me.k; sid[o] = me.id; six[o] = me.ix; }
}

__global__ void __launch_bounds__(CH_N)
k_rank_merge(const uint64_t* __restrict__ sk, const int64_t* __restrict__ sid,
             const int32_t* __restrict__ six, int n, int64_t* __restrict__ perm) {
  pdl_wait();  // the sorted chunks
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* xk = reinterpret_cast<uint64_t*>(smem);
  int64_t* xid = reinterpret_cast<int64_t*>(xk + n);
  int32_t* xix = reinterpret_cast<int32_t*>(xid + n);
  for (int j = threadIdx.x; j < n; j += CH_N) { xk[j] = sk[j]; xid[j] = sid[j]; xix[j] = six[j]; }
  __syncthreads();
  const int c = blockIdx.x, t = threadIdx.x;
  const int i = c * CH_N + t;
  if (i >= n) return;
  const RkKey me{xk[i], xid[i], xix[i]};
  int rank = t;
  const int nch = (n + CH_N - 1) / CH_N;
  for (int c2 = 0; c2 < nch; ++c2) {
    if (c2 == c) continue;
    int lo = c2 * CH_N, hi = min(n, lo + CH_N);  // first entry not before me
    const int base = lo;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (rk_less(RkKey{xk[mid], xid[mid], xix[mid]}, me)) lo = mid + 1; else hi = mid;
    }
    rank += lo - base;
  }
  perm[rank] = me.ix;
}

// ---------------------------------------------------------------- radix ----
// n > 8192: onesweep LSD radix sort of (id, orderable64(G)) -- 16 passes of
// 8-bit digits over the 128-bit key (id digits first, then G digits), stable,
// so the result is ascending (G, id).
//   1. k_os_init   one read of G/ids: key/id/index arrays + all 16 digit
//                  histograms (block-private smem, then global atomics)
//   2. k_os_scan   per-pass exclusive digit offsets; a pass whose digit is
//                  constant over all keys is marked trivial and skipped (the
//                  high id bytes and the sign/exponent byte of G usually are),
//                  with the ping-pong parity of every pass resolved here
//   3. k_os_pass   x16: tiles of 2048 keys claimed in order, warp-striped
//                  match_any ranks, per-digit decoupled look-back across tiles
//                  (flag in the top 2 bits of a 32-bit status word), one
//                  stable scatter -- no separate histogram/scan launches
//   4. k_os_out    perm = final index array
constexpr int RT_THREADS = 256;
#ifndef SS_RT_ITEMS
#define SS_RT_ITEMS 8
#endif
constexpr int RT_ITEMS = SS_RT_ITEMS;
#ifndef SS_OS_LB
#define SS_OS_LB 8
#endif
constexpr int OS_LB = SS_OS_LB;  // look-back window (predecessor tiles per round trip)
constexpr int RT_TILE = RT_THREADS * RT_ITEMS;
constexpr int OS_PASSES = 16;
constexpr int OS_SMEM = RT_TILE * (8 + 8 + 4);
constexpr uint32_t OS_AGG = 1u << 30, OS_PRE = 2u << 30, OS_VAL = (1u << 30) - 1;

struct OsMeta {
  uint32_t trivial[OS_PASSES];
  uint32_t src[OS_PASSES + 1];  // source buffer of each pass; src[16] = final
};

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int os_digit(uint64_t key, uint64_t id, int pass) {
  return pass < 8 ? (int)((id >> (8 * pass)) & 255u) : (int)((key >> (8 * (pass - 8))) & 255u);
}

__global__ void __launch_bounds__(RT_THREADS)
k_os_init(const double* __restrict__ G, const int64_t* __restrict__ ids, int64_t n,
          uint64_t* __restrict__ key, uint64_t* __restrict__ idk, uint32_t* __restrict__ idx,
          uint32_t* __restrict__ ghist, uint32_t* __restrict__ unsorted) {
  __shared__ uint32_t h[OS_PASSES][256];
  __shared__ int s_uns;
  if (threadIdx.x == 0) s_uns = 0;
  for (int i = threadIdx.x; i < OS_PASSES * 256; i += RT_THREADS) (&h[0][0])[i] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * RT_TILE;
  for (int it = 0; it < RT_ITEMS; ++it) {
    const int64_t i = base + (int64_t)it * RT_THREADS + threadIdx.x;
    if (i >= n) break;
    const uint64_t k = f64_order(G[i]);
    // signed id -> order-preserving unsigned
    const uint64_t d = (uint64_t)(ids ? ids[i] : i) ^ 0x8000000000000000ull;
    key[i] = k;
    idk[i] = d;
    idx[i] = (uint32_t)i;
    // ids already ascending in input order -> the id passes are no-ops for a
    // stable sort (detected here, applied in k_os_scan)
    if (ids && i > 0 && ids[i - 1] > ids[i]) s_uns = 1;
#pragma unroll
    for (int p = 0; p < OS_PASSES; ++p) atomicAdd(&h[p][os_digit(k, d, p)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < OS_PASSES * 256; i += RT_THREADS) {
    const uint32_t c = (&h[0][0])[i];
    if (c) atomicAdd(&ghist[i], c);
  }
  if (threadIdx.x == 0 && s_uns) atomicOr(unsorted, 1u);
}

// one CTA: ghist[p][d] -> exclusive offsets in place; trivial passes; parities
__global__ void __launch_bounds__(256)
k_os_scan(uint32_t* __restrict__ ghist, int64_t n, const uint32_t* __restrict__ unsorted,
          OsMeta* __restrict__ meta) {
  pdl_wait();  // k_os_init's histograms
  __shared__ uint32_t s_warp[OS_PASSES][8];
  __shared__ int s_triv[OS_PASSES];
  const int d = threadIdx.x, lane = d & 31, warp = d >> 5;
  uint32_t hv[OS_PASSES];
#pragma unroll
  for (int p = 0; p < OS_PASSES; ++p) hv[p] = ghist[p * 256 + d];  // all loads in flight
  if (d < OS_PASSES) s_triv[d] = 0;
  __syncthreads();
#pragma unroll
  for (int p = 0; p < OS_PASSES; ++p) {
    const uint32_t v = hv[p];
    if ((int64_t)v == n) s_triv[p] = 1;  // one digit holds every key
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    if (lane == 31) s_warp[p][warp] = x;
    hv[p] = x - v;
  }
  __syncthreads();
#pragma unroll
  for (int p = 0; p < OS_PASSES; ++p) {
    uint32_t pre = 0;
    for (int w = 0; w < warp; ++w) pre += s_warp[p][w];
    ghist[p * 256 + d] = pre + hv[p];
  }
  if (d == 0) {
    // ids already ascending in input order: the stable key passes alone
    // produce (G, id) order, so the id passes are skipped
    const bool ids_sorted = *unsorted == 0u;
    uint32_t par = 0;
    for (int p = 0; p < OS_PASSES; ++p) {
      const int triv = s_triv[p] || (p < 8 && ids_sorted);
      meta->trivial[p] = (uint32_t)triv;
      meta->src[p] = par;
      if (!triv) par ^= 1u;
    }
    meta->src[OS_PASSES] = par;
  }
}

__global__ void __launch_bounds__(RT_THREADS)
k_os_pass(uint64_t* __restrict__ key0, uint64_t* __restrict__ key1, uint64_t* __restrict__ id0,
          uint64_t* __restrict__ id1, uint32_t* __restrict__ ix0, uint32_t* __restrict__ ix1,
          int64_t n, int pass, const uint32_t* __restrict__ gofs, uint32_t* __restrict__ status,
          uint32_t* __restrict__ tile_ctr, const OsMeta* __restrict__ meta) {
  // PDL: the previous pass (or k_os_scan) has completed and flushed; let the
  // next pass's CTAs launch now, so a trivial pass costs little more than
  // its predecessor's tail (they wait for this grid in their pdl_wait)
  pdl_wait();
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (meta->trivial[pass]) return;
  __shared__ uint32_t cnt[RT_THREADS / 32][256];
  __shared__ uint32_t s_excl[256];   // global offset of the tile's run of each digit
  __shared__ uint32_t s_tstart[256]; // start of each digit's run inside the tile
  __shared__ uint32_t s_wsum[RT_THREADS / 32];
  __shared__ int s_tile;
  extern __shared__ __align__(16) unsigned char os_smem[];
  uint64_t* skey = reinterpret_cast<uint64_t*>(os_smem);  // tile sorted by digit
  uint64_t* sidk = skey + RT_TILE;
  uint32_t* six = reinterpret_cast<uint32_t*>(sidk + RT_TILE);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool flip = meta->src[pass] != 0;
  const uint64_t* key = flip ? key1 : key0;
  const uint64_t* idk = flip ? id1 : id0;
  const uint32_t* idx = flip ? ix1 : ix0;
  uint64_t* okey = flip ? key0 : key1;
  uint64_t* oid = flip ? id0 : id1;
  uint32_t* oidx = flip ? ix0 : ix1;
  if (threadIdx.x == 0) s_tile = (int)atomicAdd(tile_ctr, 1u);
  for (int d = lane; d < 256; d += 32) cnt[warp][d] = 0;
  __syncthreads();
  const int tile = s_tile;
  const int64_t base = (int64_t)tile * RT_TILE + (int64_t)warp * (RT_TILE / 8);
  uint64_t k_[RT_ITEMS], d_[RT_ITEMS];
  uint32_t ix_[RT_ITEMS], rk[RT_ITEMS];
  int dg[RT_ITEMS];
#pragma unroll
  for (int it = 0; it < RT_ITEMS; ++it) {
    const int64_t i = base + it * 32 + lane;
    const bool live = i < n;
    k_[it] = live ? key[i] : 0;
    d_[it] = live ? idk[i] : 0;
    ix_[it] = live ? idx[i] : 0;
  }
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int it = 0; it < RT_ITEMS; ++it) {
    const int64_t i = base + it * 32 + lane;
    const bool live = i < n;
    const int d = os_digit(k_[it], d_[it], pass);
    dg[it] = live ? d : -1;
    const unsigned am = __ballot_sync(0xffffffffu, live);
    uint32_t r = 0;
    if (live) {
      const unsigned peers = __match_any_sync(am, d);
      const uint32_t before = cnt[warp][d];
      r = before + __popc(peers & lt);
      __syncwarp(am);
      if ((peers & lt) == 0u) cnt[warp][d] = before + __popc(peers);
    }
    __syncwarp();
    rk[it] = r;
  }
  __syncthreads();
  // per digit: warp offsets within the tile, tile count, look-back
  {
    const int d = threadIdx.x;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < RT_THREADS / 32; ++w) {
      const uint32_t c = cnt[w][d];
      cnt[w][d] = run;
      run += c;
    }
    uint32_t* st = status + (size_t)tile * 256 + d;
    if (tile == 0) {
      st_relaxed(st, OS_PRE | run);
      s_excl[d] = 0;
    } else {
      st_relaxed(st, OS_AGG | run);
      // look back OS_LB predecessors per round trip (independent loads in flight)
      uint32_t excl = 0;
      bool found = false;
      for (int t0 = tile - 1; t0 >= 0 && !found; t0 -= OS_LB) {
        uint32_t v[OS_LB];
#pragma unroll
        for (int u = 0; u < OS_LB; ++u)
          v[u] = (t0 - u >= 0) ? ld_relaxed(status + (size_t)(t0 - u) * 256 + d) : OS_PRE;
#pragma unroll
        for (int u = 0; u < OS_LB; ++u) {
          if (found) break;
          while ((v[u] & ~OS_VAL) == 0u) v[u] = ld_relaxed(status + (size_t)(t0 - u) * 256 + d);
          if (t0 - u >= 0) excl += v[u] & OS_VAL;
          if (v[u] & OS_PRE) found = true;
        }
      }
      st_relaxed(st, OS_PRE | (excl + run));
      s_excl[d] = excl;
    }
    // exclusive scan of the tile counts over digits -> run starts in the tile
    uint32_t x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    if (lane == 31) s_wsum[warp] = x;
    __syncthreads();
    uint32_t pre = 0;
    for (int w = 0; w < warp; ++w) pre += s_wsum[w];
    s_tstart[d] = pre + x - run;
    s_excl[d] += gofs[pass * 256 + d];
  }
  __syncthreads();
  // stage the tile in digit order, then write each digit's run contiguously
#pragma unroll
  for (int it = 0; it < RT_ITEMS; ++it) {
    if (dg[it] < 0) continue;
    const int d = dg[it];
    const uint32_t lp = s_tstart[d] + cnt[warp][d] + rk[it];
    skey[lp] = k_[it];
    sidk[lp] = d_[it];
    six[lp] = ix_[it];
  }
  __syncthreads();
  const int tn = (int)min((int64_t)RT_TILE, n - (int64_t)tile * RT_TILE);
  for (int j = threadIdx.x; j < tn; j += RT_THREADS) {
    const uint64_t kk = skey[j], dd = sidk[j];
    const int d = os_digit(kk, dd, pass);
    const uint32_t pos = s_excl[d] + (uint32_t)j - s_tstart[d];
    okey[pos] = kk;
    oid[pos] = dd;
    oidx[pos] = six[j];
  }
}

__global__ void k_os_out(const uint32_t* __restrict__ ix0, const uint32_t* __restrict__ ix1,
                         int64_t n, const OsMeta* __restrict__ meta, int64_t* __restrict__ perm) {
  pdl_wait();  // the last pass
  const uint32_t* ix = meta->src[OS_PASSES] ? ix1 : ix0;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) perm[i] = ix[i];
}

static size_t os_zeroed_bytes(int64_t ntiles) {
  return ((size_t)OS_PASSES * 256 + (size_t)OS_PASSES * ntiles * 256 + OS_PASSES + 1) * 4;
}

int64_t rank_workspace_bytes(int64_t n) {
  if (n <= COUNT_MAX) return 256;
  if (n <= CHUNK_MAX) return n * (8 + 8 + 4) + 256;
  const int64_t ntiles = (n + RT_TILE - 1) / RT_TILE;
  return 2 * n * (8 + 8 + 4) + (int64_t)os_zeroed_bytes(ntiles) + (int64_t)sizeof(OsMeta) + 1024;
}

int launch_rank(const double* G, const int64_t* ids, int64_t n, int64_t* perm, void* ws,
                int64_t ws_bytes, cudaStream_t st) {
  if (n <= 0) return SS_OK;
  if (n <= COUNT_MAX) {
    count_launch();
    if (n <= 2048)
      SS_CUDA_TRY(pdl_launch(k_rank_count<32>, dim3((unsigned)((n * 32 + 255) / 256)), dim3(256), 0,
                             st, G, ids, (int)n, perm));
    else
      SS_CUDA_TRY(pdl_launch(k_rank_count<8>, dim3((unsigned)((n * 8 + 255) / 256)), dim3(256), 0,
                             st, G, ids, (int)n, perm));
    SS_LAUNCH_CHECK();
    return SS_OK;
  }
  if (n <= CHUNK_MAX) {
    const unsigned nch = (unsigned)((n + CH_N - 1) / CH_N);
    if (!ws || ws_bytes < rank_workspace_bytes(n))
      return set_error(SS_ERR_ARG, "rank workspace too small (%lld < %lld)", (long long)ws_bytes,
                       (long long)rank_workspace_bytes(n));
    uint64_t* sk = reinterpret_cast<uint64_t*>(ws);
    int64_t* sid = reinterpret_cast<int64_t*>(sk + n);
    int32_t* six = reinterpret_cast<int32_t*>(sid + n);
    count_launch();
    SS_CUDA_TRY(pdl_launch(k_rank_chunk, dim3(nch), dim3(CH_N), 0, st, G, ids, (int)n, sk, sid, six));
    SS_LAUNCH_CHECK();
    const size_t smem = (size_t)n * (8 + 8 + 4);
    SS_CUDA_TRY(ensure_dyn_smem(k_rank_merge, smem));
    count_launch();
    SS_CUDA_TRY(pdl_launch(k_rank_merge, dim3(nch), dim3(CH_N), smem, st, (const uint64_t*)sk,
                           (const int64_t*)sid, (const int32_t*)six, (int)n, perm));
    SS_LAUNCH_CHECK();
    return SS_OK;
  }
  if (n >= (int64_t)OS_VAL) return set_error(SS_ERR_UNSUPPORTED, "rank n too large");
  if (ws_bytes < rank_workspace_bytes(n))
    return set_error(SS_ERR_ARG, "rank workspace too small (%lld < %lld)", (long long)ws_bytes,
                     (long long)rank_workspace_bytes(n));
  const int ntiles = (int)((n + RT_TILE - 1) / RT_TILE);
  unsigned char* p = reinterpret_cast<unsigned char*>(ws);
  uint64_t *key0, *key1, *id0, *id1;
  uint32_t *ix0, *ix1;
  key0 = reinterpret_cast<uint64_t*>(p); p += n * 8;
  key1 = reinterpret_cast<uint64_t*>(p); p += n * 8;
  id0 = reinterpret_cast<uint64_t*>(p); p += n * 8;
  id1 = reinterpret_cast<uint64_t*>(p); p += n * 8;
  ix0 = reinterpret_cast<uint32_t*>(p); p += n * 4;
  ix1 = reinterpret_cast<uint32_t*>(p); p += n * 4;
  p = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(p) + 255) & ~(uintptr_t)255);
  uint32_t* ghist = reinterpret_cast<uint32_t*>(p);           // [16][256]
  uint32_t* status = ghist + OS_PASSES * 256;                 // [16][ntiles][256]
  uint32_t* tctr = status + (size_t)OS_PASSES * ntiles * 256;  // [16]
  uint32_t* unsorted = tctr + OS_PASSES;                      // [1]
  OsMeta* meta = reinterpret_cast<OsMeta*>(
      (reinterpret_cast<uintptr_t>(unsorted + 1) + 15) & ~(uintptr_t)15);
  SS_CUDA_TRY(cudaFuncSetAttribute(k_os_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, OS_SMEM));
  SS_CUDA_TRY(cudaMemsetAsync(ghist, 0, os_zeroed_bytes(ntiles), st));
  count_launch();
  k_os_init<<<ntiles, RT_THREADS, 0, st>>>(G, ids, n, key0, id0, ix0, ghist, unsorted);
  SS_LAUNCH_CHECK();
  // scan, passes and output with programmatic dependent launch: each kernel
  // waits for its predecessor in pdl_wait(), and trivial passes overlap
  count_launch();
  SS_CUDA_TRY(pdl_launch(k_os_scan, dim3(1), dim3(256), 0, st, ghist, n, unsorted, meta));
  for (int pass = 0; pass < OS_PASSES; ++pass) {
    count_launch();
    SS_CUDA_TRY(pdl_launch(k_os_pass, dim3(ntiles), dim3(RT_THREADS), OS_SMEM, st, key0, key1, id0,
                           id1, ix0, ix1, n, pass, ghist, status + (size_t)pass * ntiles * 256,
                           tctr + pass, meta));
  }
  count_launch();
  SS_CUDA_TRY(pdl_launch(k_os_out, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, ix0, ix1, n,
                         meta, perm));
  return SS_OK;
}

}  // namespace ss
