// Engine batch formation over the ranked list (SPEC.md:470
// step 3): scan requests in ascending priority and greedily include while the
// projected KV tokens stay <= K and the count <= B.  A not-yet-prefilled
// request projects I + 1 tokens, a running/preempted one I + g + 1, i.e.
// I + g + 1 with g = 0 for pending requests.
//
// Two readings of "greedily include while" are provided:
//   SS_PACK_CUT  (0): stop at the first request that does not fit (the
//                     batch is a prefix of the ranked list);
//   SS_PACK_SKIP (1): skip a request that does not fit and keep scanning
//                     (work-conserving: SPEC.md engine invariant "the batch is
//                     never empty while any request fits").
// A request with I + 1 > K can never run: SPEC.md engine step errors
// ("request cannot fit"); the kernel reports it as count = -1 with the
// offending request index in *out_tokens.
//
// One CTA of 1024 threads walks the ranked list in chunks of 1024: block
// prefix sums of the projected tokens; the cut form is a single pass, the
// skip form resolves the first overflow of each pass and rescans the rest of
// the chunk with the reduced budget (at most B + n/1024 passes in total,
// since every pass either ends the chunk or admits a request).
#include <climits>

#include "ss_common.cuh"
#include "ss_internal.h"

namespace ss {

constexpr int PK_THREADS = 1024;
constexpr int PK_ITEMS = 8;

// exclusive prefix of v over the block; *total = block sum.  All threads call.
__device__ __forceinline__ long long block_excl_scan(long long v, long long* s_warp,
                                                     long long* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long t = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += t;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    long long y = s_warp[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long t = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += t;
    }
    s_warp[lane] = y;
  }
  __syncthreads();
  const long long pre = (warp ? s_warp[warp - 1] : 0) + x - v;
  *total = s_warp[31];
  __syncthreads();
  return pre;
}

__global__ void __launch_bounds__(PK_THREADS)
k_pack_batch(const int64_t* __restrict__ perm, const int32_t* __restrict__ I,
             const int32_t* __restrict__ g, int64_t n, int64_t K, int B, int mode,
             int64_t* __restrict__ out_batch, int32_t* __restrict__ out_count,
             int64_t* __restrict__ out_tokens) {
  __shared__ long long s_warp[32];
  __shared__ long long s_bad;
  __shared__ long long s_used;
  __shared__ int s_first;
  const int tid = threadIdx.x;
  if (tid == 0) s_bad = LLONG_MAX;
  __syncthreads();
  for (int64_t i = tid; i < n; i += PK_THREADS)
    if ((long long)I[i] + 1 > K) atomicMin(&s_bad, (long long)i);
  __syncthreads();
  if (s_bad != LLONG_MAX) {
    if (tid == 0) {
      *out_count = -1;
      *out_tokens = s_bad;
    }
    return;
  }
  long long R = K;  // remaining KV budget (block-uniform)
  int cnt = 0;      // admitted so far (block-uniform)
  if (mode == 0) {
    // cut form: PK_ITEMS consecutive ranked requests per thread, all their
    // loads in flight, one block scan per PK_THREADS * PK_ITEMS requests;
    // projected tokens are >= 1, so the admitted set is a prefix
    for (int64_t base = 0; base < n && cnt < B; base += (int64_t)PK_THREADS * PK_ITEMS) {
      const int64_t i0 = base + (int64_t)tid * PK_ITEMS;
      int64_t rv[PK_ITEMS];
      long long tv[PK_ITEMS];
#pragma unroll
      for (int j = 0; j < PK_ITEMS; ++j) rv[j] = (i0 + j < n) ? perm[i0 + j] : -1;
      long long loc = 0;
#pragma unroll
      for (int j = 0; j < PK_ITEMS; ++j) {
        tv[j] = rv[j] >= 0 ? (long long)I[rv[j]] + (long long)g[rv[j]] + 1 : 0;
        loc += tv[j];
      }
      long long tot;
      if (tid == 0) s_used = 0;  // published by the block scans' barriers
      long long run = block_excl_scan(loc, s_warp, &tot);
      int myok = 0;
      long long last = 0;
#pragma unroll
      for (int j = 0; j < PK_ITEMS; ++j) {
        run += tv[j];
        const bool ok = rv[j] >= 0 && run <= R && (i0 + j - base) < (int64_t)(B - cnt);
        if (ok) {
          out_batch[cnt + (i0 + j - base)] = rv[j];
          ++myok;
          last = run;
        }
      }
      long long nok;
      block_excl_scan(myok, s_warp, &nok);
      // tokens admitted = the prefix at the last admitted request (the
      // largest admitted prefix: prefixes increase)
      if (myok) atomicMax(&s_used, last);
      __syncthreads();
      const long long used = s_used;
      __syncthreads();
      R -= used;
      cnt += (int)nok;
      if (nok < min((int64_t)PK_THREADS * PK_ITEMS, n - base)) break;
    }
  } else
  for (int64_t base = 0; base < n && cnt < B; base += PK_THREADS) {
    const int64_t i = base + tid;
    const bool live = i < n;
    const int64_t r = live ? perm[i] : -1;
    const long long t = live ? (long long)I[r] + (long long)g[r] + 1 : 0;
    if (mode == 0) {
      long long tot;
      const long long pre = block_excl_scan(t, s_warp, &tot);
      const bool ok = live && pre + t <= R && (int)(i - base) < B - cnt;
      const int nok = __syncthreads_count(ok);
      if (ok) out_batch[cnt + (i - base)] = r;
      const int64_t chunk = min((int64_t)PK_THREADS, n - base);
      // ok is a prefix of the chunk: tokens admitted = prefix sum at nok
      if (tid == nok - 1) s_warp[0] = pre + t;
      __syncthreads();
      const long long used = nok ? s_warp[0] : 0;
      __syncthreads();
      R -= used;
      cnt += nok;
      if (nok < chunk) break;
    } else {
      bool done = !live;
      while (true) {
        const bool cand = !done && t <= R;
        long long tot;
        const long long pre = block_excl_scan(cand ? t : 0, s_warp, &tot);
        const bool over = cand && pre + t > R;
        if (tid == 0) s_first = INT_MAX;
        __syncthreads();
        if (over) atomicMin(&s_first, tid);
        __syncthreads();
        const int j = s_first;  // first candidate that overflows (skipped)
        const bool inc = cand && tid < j;
        long long ntot;
        const long long rk = block_excl_scan(inc ? 1 : 0, s_warp, &ntot);
        const bool inc2 = inc && cnt + rk < B;
        if (inc2) out_batch[cnt + rk] = r;
        long long ttot;
        block_excl_scan(inc2 ? t : 0, s_warp, &ttot);
        R -= ttot;
        cnt += (int)min(ntot, (long long)(B - cnt));
        if (tid <= j) done = true;
        if (cnt >= B || j == INT_MAX || __syncthreads_and(done)) break;
      }
    }
  }
  if (tid == 0) {
    *out_count = cnt;
    *out_tokens = K - R;
  }
}

int launch_pack_batch(const int64_t* perm, const int32_t* I, const int32_t* g, int64_t n,
                      int64_t K, int B, int mode, int64_t* out_batch, int32_t* out_count,
                      int64_t* out_tokens, cudaStream_t st) {
  count_launch();
  k_pack_batch<<<1, PK_THREADS, 0, st>>>(perm, I, g, n, K, B, mode, out_batch, out_count,
                                         out_tokens);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

}  // namespace ss
