// Per-query bounded min-heap of candidate composites, shared by the CUDA-core
// scan kernel and the tcgen05 GEMM kernel.  Each thread owns one query and
// one heap column in shared memory, laid out [slot][thread] so that a warp's
// accesses never conflict regardless of which heap slot each lane touches.
//
// Invariant: the heap holds the top-`cnt` composites seen so far among rows
// with key >= theta; once full (cnt == k) its root is the k-th best, and the
// scalar s-domain filter `thr_s` is tightened to that root so the hot loop
// rejects almost every row with one compare.
#pragma once
#include "ss_common.cuh"

namespace ss {

struct HeapState {
  int cnt;
  uint64_t root;
  float thr_s;  // conservative filter on s = fl(dot * inv_w)
};

template <int STRIDE>
__device__ __forceinline__ void heap_sift_down(uint64_t* heap, int k, int i, uint64_t x) {
  while (true) {
    int l = 2 * i + 1;
    if (l >= k) break;
    uint64_t cv = heap[l * STRIDE];
    int c = l;
    if (l + 1 < k) {
      uint64_t rv = heap[(l + 1) * STRIDE];
      if (rv < cv) { cv = rv; c = l + 1; }
    }
    if (cv >= x) break;
    heap[i * STRIDE] = cv;
    i = c;
  }
  heap[i * STRIDE] = x;
}

// Offer an exact candidate (already known key >= theta).
template <int STRIDE>
__device__ __forceinline__ void heap_offer(uint64_t* heap, int k, HeapState& st, uint64_t comp,
                                           float iq) {
  if (st.cnt < k) {
    heap[st.cnt * STRIDE] = comp;
    if (++st.cnt == k) {
      for (int i = k / 2 - 1; i >= 0; --i) heap_sift_down<STRIDE>(heap, k, i, heap[i * STRIDE]);
      st.root = heap[0];
      st.thr_s = fmaxf(st.thr_s, s_threshold(comp_key(st.root), iq));
    }
  } else if (comp > st.root) {
    heap_sift_down<STRIDE>(heap, k, 0, comp);
    st.root = heap[0];
    st.thr_s = fmaxf(st.thr_s, s_threshold(comp_key(st.root), iq));
  }
}

// Slow path for a row whose s passed the filter: exact key, theta check, offer.
template <int STRIDE>
__device__ __forceinline__ void heap_consider(uint64_t* heap, int k, HeapState& st, int dot,
                                              float iw, float iq, float theta, int64_t gslot,
                                              int64_t head, int64_t gcap) {
  float key = score_key(dot, iw, iq);
  if (!(key >= theta)) return;
  // `head` is passed pre-reduced mod gcap by the launcher, so no 64-bit modulo
  int64_t rel = gslot - head;
  if (rel < 0) rel += gcap;
  heap_offer<STRIDE>(heap, k, st, make_comp(key, (uint32_t)rel), iq);
}

}  // namespace ss
