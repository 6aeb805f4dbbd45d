// Block-wide top-k selection over candidate composites in shared memory,
// shared by the slice/shard merge (k_merge_finish.cu) and the wide-vector
// pass (k_wide.cu).  Composites are unique, so the
// k-th largest is well defined.  nlists = 0 disables the full-list prune
// (for buffers that are not a concatenation of per-list top-k's).
#pragma once
#include "ss_common.cuh"

namespace ss {

// ---------------------------------------------------------------------------
// select the top-k of M candidate composites (cand[0..M) in smem) into
// sel[0..kpad) sorted descending (0-padded), carrying an int32 payload.
// MSB-first 8-bit radix select of the k-th largest when more than k are
// non-zero, then a bitonic sort of the <= k winners.
// ---------------------------------------------------------------------------
// Fast path first: every full input list (k non-zero entries) proves that the
// global k-th best is >= that list's minimum, so candidates below
// tau = max over full lists of their minimum are dropped; when at most
// SORT_MAX candidates survive they are bitonic-sorted directly.
constexpr int SORT_MAX = 512;

static __device__ bool block_select_small(uint64_t* cand, int32_t* cpay, int M, int nlists, int k,
                                   int kpad, uint64_t* sel, int32_t* spay, int* s_misc) {
  __shared__ uint64_t tau_s;
  uint64_t* s_tau = &tau_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  if (tid == 0) { *s_tau = 1ull; s_misc[3] = 0; }
  __syncthreads();
  for (int l = warp; l < nlists; l += nw) {
    uint64_t mn = ~0ull;
    for (int j = lane; j < k; j += 32) mn = min(mn, cand[l * k + j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if (lane == 0 && mn != 0ull) atomicMax(reinterpret_cast<unsigned long long*>(s_tau), mn);
  }
  __syncthreads();
  const uint64_t tau = *s_tau;
  // compact survivors (>= tau, non-zero) into the front of cand (stable
  // order is irrelevant: composites are unique)
  __shared__ uint64_t buf[SORT_MAX];
  __shared__ int32_t pbuf[SORT_MAX];
  for (int i = tid; i < M; i += blockDim.x) {
    const uint64_t c = cand[i];
    if (c >= tau) {
      int p = atomicAdd(&s_misc[3], 1);
      if (p < SORT_MAX) { buf[p] = c; pbuf[p] = cpay[i]; }
    }
  }
  __syncthreads();
  const int m1 = s_misc[3];
  if (m1 > SORT_MAX) return false;
  // rank by counting (composites are unique): no barriers inside, the
  // broadcast LDS of buf[j] is shared by the whole warp
  for (int i = tid; i < kpad; i += blockDim.x) { sel[i] = 0ull; spay[i] = 0; }
  __syncthreads();
  for (int i = tid; i < m1; i += blockDim.x) {
    const uint64_t c = buf[i];
    int r = 0;
    for (int j = 0; j < m1; ++j) r += (buf[j] > c);
    if (r < k) {
      sel[r] = c;
      spay[r] = pbuf[i];
    }
  }
  __syncthreads();
  return true;
}

static __device__ void block_select_topk(uint64_t* cand, int32_t* cpay, int M, int nlists, int k, int kpad,
                                  uint64_t* sel, int32_t* spay, int* hist, int* s_misc) {
  if (block_select_small(cand, cpay, M, nlists, k, kpad, sel, spay, s_misc)) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int nz = 0;
  for (int i = tid; i < M; i += blockDim.x) nz += (cand[i] != 0ull);
  for (int o = 16; o > 0; o >>= 1) nz += __shfl_xor_sync(0xffffffffu, nz, o);
  if (tid == 0) s_misc[0] = 0;
  __syncthreads();
  if (lane == 0) atomicAdd(&s_misc[0], nz);
  __syncthreads();
  const int m0 = s_misc[0];

  uint64_t kth = 1ull;  // select every non-zero when m0 <= k
  if (m0 > k) {
    uint64_t prefix = 0, mask = 0;
    int need = k;
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int d = tid; d < 256; d += blockDim.x) hist[d] = 0;
      __syncthreads();
      for (int i0 = 0; i0 < M; i0 += blockDim.x) {
        int i = i0 + tid;
        bool act = false;
        int d = 0;
        if (i < M) {
          uint64_t c = cand[i];
          act = (c & mask) == prefix;
          d = (int)((c >> shift) & 255ull);
        }
        unsigned am = __ballot_sync(0xffffffffu, act);
        if (act) {
          unsigned peers = __match_any_sync(am, d);
          if ((peers & ((1u << lane) - 1u)) == 0u) atomicAdd(&hist[d], __popc(peers));
        }
      }
      __syncthreads();
      if (warp == 0) {
        // lane l owns digits [255-8l .. 248-8l] (descending)
        int local = 0;
#pragma unroll
        for (int t = 0; t < 8; ++t) local += hist[255 - 8 * lane - t];
        int incl = warp_incl_scan_i32(local, lane);
        int excl = incl - local;
        if (excl < need && incl >= need) {
          int cum = excl;
          for (int t = 0; t < 8; ++t) {
            int d = 255 - 8 * lane - t;
            if (cum + hist[d] >= need) { s_misc[1] = d; s_misc[2] = need - cum; break; }
            cum += hist[d];
          }
        }
      }
      __syncthreads();
      prefix |= (uint64_t)s_misc[1] << shift;
      mask |= 255ull << shift;
      need = s_misc[2];
      __syncthreads();
    }
    kth = prefix;
  }
  for (int i = tid; i < kpad; i += blockDim.x) sel[i] = 0ull;
  if (tid == 0) s_misc[0] = 0;
  __syncthreads();
  for (int i = tid; i < M; i += blockDim.x) {
    uint64_t c = cand[i];
    if (c != 0ull && c >= kth) {
      int p = atomicAdd(&s_misc[0], 1);
      if (p < kpad) {
        sel[p] = c;
        spay[p] = cpay[i];
      }
    }
  }
  __syncthreads();
  for (int size = 2; size <= kpad; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < kpad; i += blockDim.x) {
        int j = i ^ stride;
        if (j > i) {
          bool desc = ((i & size) == 0);
          uint64_t a = sel[i], b = sel[j];
          if ((a < b) == desc) {
            sel[i] = b;
            sel[j] = a;
            int32_t t = spay[i]; spay[i] = spay[j]; spay[j] = t;
          }
        }
      }
      __syncthreads();
    }
  }
}

// Unordered top-k SET (all the histogram needs): tau-prune as above, then the
// k-th largest composite by a 64-step bitwise search where each step is one
// __syncthreads_count over one candidate per thread (composites are unique,
// so {c >= kth} has exactly min(k, m) members).  Falls back to the ordered
// selection when more than blockDim candidates survive the prune.
static __device__ void block_select_set(uint64_t* cand, int32_t* cpay, int M, int nlists, int k, int kpad,
                                 uint64_t* sel, int32_t* spay, int* hist, int* s_misc) {
  __shared__ uint64_t tau_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  if (tid == 0) { tau_s = 1ull; s_misc[3] = 0; }
  __syncthreads();
  for (int l = warp; l < nlists; l += nw) {
    uint64_t mn = ~0ull;
    for (int j = lane; j < k; j += 32) mn = min(mn, cand[l * k + j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if (lane == 0 && mn != 0ull) atomicMax(reinterpret_cast<unsigned long long*>(&tau_s), mn);
  }
  __syncthreads();
  const uint64_t tau = tau_s;
  int nz = 0;
  for (int i = tid; i < M; i += blockDim.x) nz += (cand[i] >= tau);
  for (int o = 16; o > 0; o >>= 1) nz += __shfl_xor_sync(0xffffffffu, nz, o);
  if (lane == 0) atomicAdd(&s_misc[3], nz);
  __syncthreads();
  const int m1 = s_misc[3];
  if (m1 > (int)blockDim.x) {  // rare: the ordered path handles any size
    block_select_topk(cand, cpay, M, nlists, k, kpad, sel, spay, hist, s_misc);
    return;
  }
  // compact the survivors, one per thread
  __shared__ uint64_t one[1024];
  __shared__ int32_t onep[1024];
  if (tid == 0) s_misc[0] = 0;
  __syncthreads();
  for (int i = tid; i < M; i += blockDim.x) {
    const uint64_t c = cand[i];
    if (c >= tau) {
      const int p = atomicAdd(&s_misc[0], 1);
      one[p] = c;
      onep[p] = cpay[i];
    }
  }
  __syncthreads();
  const uint64_t mine = (tid < m1) ? one[tid] : 0ull;
  uint64_t T = 1ull;  // keep everything when m1 <= k
  if (m1 > k) {
    T = 0ull;
    for (int b = 63; b >= 0; --b) {
      const uint64_t t = T | (1ull << b);
      if (__syncthreads_count(mine >= t) >= k) T = t;
    }
  }
  for (int i = tid; i < kpad; i += blockDim.x) { sel[i] = 0ull; spay[i] = 0; }
  if (tid == 0) s_misc[0] = 0;
  __syncthreads();
  if (mine != 0ull && mine >= T) {
    const int p = atomicAdd(&s_misc[0], 1);
    sel[p] = mine;
    spay[p] = onep[tid];
  }
  __syncthreads();
}

}  // namespace ss
