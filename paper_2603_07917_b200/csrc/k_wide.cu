// Wide-vector pass of stage 1: exact similarity for feature-hash embeddings
// whose buckets exceed the int8 range (long prompts that repeat a token or a
// bigram more than 127 times; the reference accumulates unbounded +-1 counts,
// _kernels.py:82-95, and scores them in float32).
//
// The tensor-core kernels see such rows as zero rows with a NaN inverse
// norm (never matched) and such queries with a NaN inverse norm; this pass
// restores exactness with CUDA-core integer dot products:
//   * every other query x the bank's wide rows      (k_wide_rows)
//   * every wide query x the whole bank             (k_wide_scan + merge)
// Each produces the exact top-k of its subset of (query, row) pairs as one
// more candidate list per query, merged with the similarity kernel's slice
// lists by the ordinary merge.  Dots are exact in int64 (|x| <= 32767), keys
// fl32(fl32(f32(dot) * inv_w) * inv_q) with f32(dot) correctly rounded --
// the oracle's definition, DESIGN.md section 3.
#include <algorithm>

#include "ss_common.cuh"
#include "ss_internal.h"
#include "topk_select.cuh"

namespace ss {

constexpr int WT = 256;    // threads per CTA
constexpr int WCAP = 768;  // candidate buffer per query (composites): >= 256 + 2 * WT
constexpr int WQ = 4;      // wide queries per k_wide_scan CTA pass
constexpr int WKMAX = 256;

// slots whose wide flag is set -> compact list (order irrelevant)
__global__ void k_wide_list(const uint8_t* __restrict__ flag, int64_t cap, int64_t* __restrict__ out,
                            int* __restrict__ count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool f = flag[i] != 0;
    const unsigned m = __ballot_sync(__activemask(), f);
    if (!m) continue;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(count, __popc(m));
    base = __shfl_sync(__activemask(), base, leader);
    if (f) out[base + __popc(m & ((1u << lane) - 1u))] = i;
  }
}

// query index -> position in the wide-query list (-1: an int8 query)
__global__ void k_wide_qpos(const int64_t* __restrict__ idx, int n, int* __restrict__ qpos) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) qpos[idx[i]] = i;
}

// Running block-wide top-k over appended candidates: every round each thread
// appends at most one candidate per buffer; when a buffer nears WCAP it is
// cut back to its top-k, whose k-th composite then filters later appends.
struct RunTopk {
  uint64_t* cand;  // [WCAP]
  int* cnt;
  uint64_t* floor_c;
};

__device__ __forceinline__ void rt_offer(const RunTopk& r, uint64_t c) {
  if (c > *r.floor_c) r.cand[atomicAdd(r.cnt, 1)] = c;
}

// all threads; leaves the top-k (descending, 0-padded) in sel[0..kpad)
// and its size in *r.cnt
__device__ void rt_compact(const RunTopk& r, int k, int kpad, int32_t* pay, uint64_t* sel,
                           int32_t* spay, int* hist, int* misc) {
  __syncthreads();
  const int m = *r.cnt;
  block_select_topk(r.cand, pay, m, 0, k, kpad, sel, spay, hist, misc);
  __syncthreads();
  int kept = 0;
  for (int i = 0; i < k; ++i) kept += sel[i] != 0ull;
  for (int i = threadIdx.x; i < k; i += blockDim.x) r.cand[i] = sel[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    *r.cnt = kept;
    if (kept == k) *r.floor_c = sel[k - 1];
  }
  __syncthreads();
}

// a candidate list as the merges read it: its m entries first, then zeros;
// ascending, so a full list is a min-heap with its minimum at entry 0 (the
// k-th-best bound k_merge_finish_w takes from entry 0)
__device__ __forceinline__ void write_list(const uint64_t* sel_desc, int m, int k, uint64_t* out) {
  for (int i = threadIdx.x; i < k; i += blockDim.x) out[i] = (i < m) ? sel_desc[m - 1 - i] : 0ull;
}

__device__ __forceinline__ uint64_t wide_comp(long long dot, float iw, float iq, float theta,
                                              int64_t slot, int64_t slot_offset, int64_t hmod,
                                              int64_t gcap) {
  const float key = __fmul_rn(__fmul_rn(__ll2float_rn(dot), iw), iq);
  if (!(key >= theta)) return 0ull;  // NaN (empty / degenerate) never matches
  int64_t rel = slot_offset + slot - hmod;
  if (rel < 0) rel += gcap;
  return make_comp(key, (uint32_t)rel);
}

// Every int8 query x every wide row of the bank (one CTA per query).
__global__ void __launch_bounds__(WT)
k_wide_rows(const int8_t* __restrict__ q, const float* __restrict__ q_inv, int64_t nq,
            const int* __restrict__ qpos, const int16_t* __restrict__ wemb,
            const float* __restrict__ winv, const int64_t* __restrict__ wslots,
            const int* __restrict__ wcount, int dim, int k, int kpad, float theta, int64_t hmod,
            int64_t gcap, int64_t slot_offset, uint64_t* __restrict__ out) {
  __shared__ uint64_t cand[WCAP];
  __shared__ int32_t pay[WCAP];
  __shared__ uint64_t sel[WKMAX];
  __shared__ int32_t spay[WKMAX];
  __shared__ int hist[256], misc[4], cnt;
  __shared__ uint64_t floor_c;
  __shared__ int qv[512];
  const int64_t qi = blockIdx.x;
  if (qpos && qpos[qi] >= 0) return;  // a wide query: the scan path writes its list
  const float iq = q_inv[qi];
  for (int d = threadIdx.x; d < dim; d += blockDim.x) qv[d] = q[qi * dim + d];
  for (int i = threadIdx.x; i < WCAP; i += blockDim.x) pay[i] = 0;
  if (threadIdx.x == 0) { cnt = 0; floor_c = 0ull; }
  __syncthreads();
  const RunTopk rt{cand, &cnt, &floor_c};
  const int nw = *wcount;
  if (iq == iq) {
    for (int base = 0; base < nw; base += blockDim.x) {
      const int i = base + threadIdx.x;
      if (i < nw) {
        const int64_t slot = wslots[i];
        const int16_t* row = wemb + slot * dim;
        long long dot = 0;
        for (int d = 0; d < dim; d += 8) {
          const int4 v = *reinterpret_cast<const int4*>(row + d);
          const int16_t* x = reinterpret_cast<const int16_t*>(&v);
          int part = 0;  // |8 * 127 * 32767| < 2^31
#pragma unroll
          for (int t = 0; t < 8; ++t) part += (int)x[t] * qv[d + t];
          dot += part;
        }
        const uint64_t c = wide_comp(dot, winv[slot], iq, theta, slot, slot_offset, hmod, gcap);
        if (c) rt_offer(rt, c);
      }
      __syncthreads();
      if (cnt > WCAP - (int)blockDim.x) rt_compact(rt, k, kpad, pay, sel, spay, hist, misc);
    }
  }
  rt_compact(rt, k, kpad, pay, sel, spay, hist, misc);
  write_list(sel, cnt, k, out + qi * k);
}

// Wide queries x one row range of the bank (int8 rows of the main plane, the
// wide plane's int16 rows where flagged): per CTA and query the exact top-k
// of its range -> scratch [gridDim.x][n_wq][k] (merged afterwards).
__global__ void __launch_bounds__(WT)
k_wide_scan(const int8_t* __restrict__ emb, const float* __restrict__ inv,
            const uint8_t* __restrict__ wflag, const int16_t* __restrict__ wemb,
            const float* __restrict__ winv, int64_t n_rows, int dim,
            const int16_t* __restrict__ wq, const float* __restrict__ wq_inv, int n_wq, int k,
            int kpad, float theta, int64_t hmod, int64_t gcap, int64_t slot_offset,
            int64_t rows_per_cta, uint64_t* __restrict__ out) {
  __shared__ uint64_t cand[WQ][WCAP];
  __shared__ int32_t pay[WCAP];
  __shared__ uint64_t sel[WKMAX];
  __shared__ int32_t spay[WKMAX];
  __shared__ int hist[256], misc[4], cnt[WQ];
  __shared__ uint64_t floor_c[WQ];
  __shared__ int16_t qv[WQ][512];
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = min(n_rows, r0 + rows_per_cta);
  for (int i = threadIdx.x; i < WCAP; i += blockDim.x) pay[i] = 0;
  for (int w0 = 0; w0 < n_wq; w0 += WQ) {
    const int nwq = min(WQ, n_wq - w0);
    for (int i = threadIdx.x; i < WQ * dim; i += blockDim.x) {
      const int j = i / dim, d = i % dim;
      qv[j][d] = (j < nwq) ? wq[(int64_t)(w0 + j) * dim + d] : (int16_t)0;
    }
    if (threadIdx.x < WQ) { cnt[threadIdx.x] = 0; floor_c[threadIdx.x] = 0ull; }
    __syncthreads();
    float iq[WQ];
#pragma unroll
    for (int j = 0; j < WQ; ++j) iq[j] = (j < nwq) ? wq_inv[w0 + j] : __int_as_float(0x7fc00000);
    for (int64_t base = r0; base < r1; base += blockDim.x) {
      const int64_t r = base + threadIdx.x;
      if (r < r1) {
        long long dot[WQ] = {0, 0, 0, 0};
        float iw;
        if (wflag && wflag[r]) {  // a wide row: int16 x int16
          iw = winv[r];
          const int16_t* row = wemb + r * dim;
          for (int d = 0; d < dim; d += 8) {
            const int4 v = *reinterpret_cast<const int4*>(row + d);
            const int16_t* x = reinterpret_cast<const int16_t*>(&v);
#pragma unroll
            for (int j = 0; j < WQ; ++j) {
              long long p = 0;
#pragma unroll
              for (int t = 0; t < 8; ++t) p += (long long)((int)x[t] * qv[j][d + t]);
              dot[j] += p;
            }
          }
        } else {  // an int8 row: |16 * 127 * 32767| < 2^31 per part
          iw = inv[r];
          const int8_t* row = emb + r * dim;
          if (iw == iw) {
            for (int d = 0; d < dim; d += 16) {
              const int4 v = *reinterpret_cast<const int4*>(row + d);
              const int8_t* x = reinterpret_cast<const int8_t*>(&v);
#pragma unroll
              for (int j = 0; j < WQ; ++j) {
                int p = 0;
#pragma unroll
                for (int t = 0; t < 16; ++t) p += (int)x[t] * qv[j][d + t];
                dot[j] += p;
              }
            }
          }
        }
#pragma unroll
        for (int j = 0; j < WQ; ++j) {
          if (j < nwq) {
            const uint64_t c = wide_comp(dot[j], iw, iq[j], theta, r, slot_offset, hmod, gcap);
            if (c) rt_offer(RunTopk{cand[j], &cnt[j], &floor_c[j]}, c);
          }
        }
      }
      __syncthreads();
      for (int j = 0; j < nwq; ++j)
        if (cnt[j] > WCAP - (int)blockDim.x)
          rt_compact(RunTopk{cand[j], &cnt[j], &floor_c[j]}, k, kpad, pay, sel, spay, hist, misc);
    }
    for (int j = 0; j < nwq; ++j) {
      rt_compact(RunTopk{cand[j], &cnt[j], &floor_c[j]}, k, kpad, pay, sel, spay, hist, misc);
      write_list(sel, cnt[j], k, out + ((int64_t)blockIdx.x * n_wq + w0 + j) * k);
    }
    __syncthreads();
  }
}

// merged wide-query rows (descending, zero-padded) -> their query's list
__global__ void k_wide_scatter(const uint64_t* __restrict__ src, const int64_t* __restrict__ idx,
                               int n, int k, uint64_t* __restrict__ out) {
  __shared__ int m;
  const int w = blockIdx.x;
  if (w >= n) return;
  const uint64_t* row = src + (int64_t)w * k;
  if (threadIdx.x == 0) {
    int c = 0;
    while (c < k && row[c] != 0ull) ++c;
    m = c;
  }
  __syncthreads();
  write_list(row, m, k, out + idx[w] * k);
}

static int wide_scan_ctas(int64_t n_rows, int sms) {
  const int64_t want = (n_rows + 2047) / 2048;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, sms));
}

size_t wide_ws_bytes(const WideQ& wq, int64_t nq, int k, int64_t n_rows, int sms) {
  size_t b = ((size_t)nq * 4 + 255) & ~(size_t)255;  // qpos
  if (wq.n > 0) {
    const int P = wide_scan_ctas(n_rows, sms);
    b += ((size_t)P * wq.n * k * 8 + 255) & ~(size_t)255;  // per-CTA lists
    b += ((size_t)wq.n * k * 12 + 255) & ~(size_t)255;     // merged comp + len
  }
  return b;
}

int launch_wide_pass(const WideBank& wb, const TopkArgs& a, const WideQ& wq, uint64_t* list_out,
                     void* ws, int device, cudaStream_t st) {
  if (a.k > WKMAX) return set_error(SS_ERR_UNSUPPORTED, "wide pass: k > %d", WKMAX);
  if (a.dim > 512 || a.dim % 16) return set_error(SS_ERR_UNSUPPORTED, "wide pass: dim %d", a.dim);
  int kpad = 1;
  while (kpad < a.k) kpad <<= 1;
  const int64_t hmod = a.head % a.gcap;
  SS_CUDA_TRY(cudaMemsetAsync(list_out, 0, (size_t)a.nq * a.k * 8, st));
  char* w = static_cast<char*>(ws);
  int* qpos = nullptr;
  if (wq.n > 0) {
    qpos = reinterpret_cast<int*>(w);
    SS_CUDA_TRY(cudaMemsetAsync(qpos, 0xff, (size_t)a.nq * 4, st));
    count_launch();
    k_wide_qpos<<<(unsigned)((wq.n + 255) / 256), 256, 0, st>>>(wq.idx, (int)wq.n, qpos);
    SS_LAUNCH_CHECK();
  }
  w += ((size_t)a.nq * 4 + 255) & ~(size_t)255;
  if (wb.any) {
    SS_CUDA_TRY(cudaMemsetAsync(wb.list_count, 0, sizeof(int), st));
    count_launch();
    k_wide_list<<<(unsigned)std::min<int64_t>((a.n_rows + 255) / 256, 4 * 148), 256, 0, st>>>(
        wb.plane.flag, a.n_rows, wb.list, wb.list_count);
    SS_LAUNCH_CHECK();
    count_launch();
    k_wide_rows<<<(unsigned)a.nq, WT, 0, st>>>(a.q, a.q_inv, a.nq, qpos, wb.plane.emb,
                                               wb.plane.inv, wb.list, wb.list_count, a.dim, a.k,
                                               kpad, a.theta, hmod, a.gcap, a.slot_offset, list_out);
    SS_LAUNCH_CHECK();
  }
  if (wq.n > 0) {
    const int P = wide_scan_ctas(a.n_rows, sm_count(device));
    uint64_t* lists = reinterpret_cast<uint64_t*>(w);
    w += ((size_t)P * wq.n * a.k * 8 + 255) & ~(size_t)255;
    uint64_t* mc = reinterpret_cast<uint64_t*>(w);
    int32_t* ml = reinterpret_cast<int32_t*>(mc + wq.n * a.k);
    const int64_t rpc = (a.n_rows + P - 1) / P;
    count_launch();
    k_wide_scan<<<(unsigned)P, WT, 0, st>>>(a.emb, a.inv, wb.any ? wb.plane.flag : nullptr,
                                            wb.plane.emb, wb.plane.inv, a.n_rows, a.dim, wq.q,
                                            wq.inv, (int)wq.n, a.k, kpad, a.theta, hmod, a.gcap,
                                            a.slot_offset, rpc, lists);
    SS_LAUNCH_CHECK();
    if (int rc = launch_merge(lists, nullptr, P, wq.n, a.k, mc, ml, wb.bank_lens, a.head, a.gcap,
                              a.slot_offset, st))
      return rc;
    count_launch();
    k_wide_scatter<<<(unsigned)wq.n, 64, 0, st>>>(mc, wq.idx, (int)wq.n, a.k, list_out);
    SS_LAUNCH_CHECK();
  }
  return SS_OK;
}

}  // namespace ss

namespace ss {

// query_similar for one query: every record with key >=
// theta, as (G = -key in f64, id = gcap - 1 - rel) pairs for the rank sort,
// whose ascending (G, id) order is (key desc, insertion_seq desc).  Exact
// integer dots against the int8 plane (and the wide plane where flagged),
// the query given as int16.  Warp-aggregated appends.
__global__ void __launch_bounds__(256)
k_query_all(const int8_t* __restrict__ emb, const float* __restrict__ inv,
            const int64_t* __restrict__ seq, const uint8_t* __restrict__ wflag,
            const int16_t* __restrict__ wemb, const float* __restrict__ winv, int64_t n_rows,
            int dim, const int16_t* __restrict__ q, float iq, float theta, int64_t hmod,
            int64_t gcap, int64_t slot_offset, double* __restrict__ out_G,
            int64_t* __restrict__ out_id, int* __restrict__ count) {
  __shared__ int16_t qv[512];
  for (int d = threadIdx.x; d < dim; d += blockDim.x) qv[d] = q[d];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n_rows;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = base + threadIdx.x;
    uint64_t c = 0ull;
    if (r < n_rows && seq[r] >= 0) {
      long long dot = 0;
      float iw;
      if (wflag && wflag[r]) {
        iw = winv[r];
        const int16_t* row = wemb + r * dim;
        for (int d = 0; d < dim; d += 8) {
          const int4 v = *reinterpret_cast<const int4*>(row + d);
          const int16_t* x = reinterpret_cast<const int16_t*>(&v);
          int p = 0;
#pragma unroll
          for (int t = 0; t < 8; ++t) p += (int)x[t] * (int)qv[d + t];
          dot += p;
        }
      } else {
        iw = inv[r];
        const int8_t* row = emb + r * dim;
        for (int d = 0; d < dim; d += 16) {
          const int4 v = *reinterpret_cast<const int4*>(row + d);
          const int8_t* x = reinterpret_cast<const int8_t*>(&v);
          int p = 0;
#pragma unroll
          for (int t = 0; t < 16; ++t) p += (int)x[t] * (int)qv[d + t];
          dot += p;
        }
      }
      c = wide_comp(dot, iw, iq, theta, r, slot_offset, hmod, gcap);
    }
    const unsigned m = __ballot_sync(0xffffffffu, c != 0ull);
    if (m) {
      const int leader = __ffs(m) - 1;
      int b = 0;
      if (lane == leader) b = atomicAdd(count, __popc(m));
      b = __shfl_sync(0xffffffffu, b, leader);
      if (c) {
        const int p = b + __popc(m & ((1u << lane) - 1u));
        out_G[p] = -(double)comp_key(c);
        out_id[p] = gcap - 1 - (int64_t)comp_rel(c);
      }
    }
  }
}

// sorted (G, id) -> (key, insertion_seq, length) of each match
__global__ void k_query_gather(const double* __restrict__ G, const int64_t* __restrict__ id,
                               const int64_t* __restrict__ perm, int64_t m,
                               const int64_t* __restrict__ seq, const int32_t* __restrict__ lens,
                               int64_t hmod, int64_t gcap, int64_t slot_offset, int64_t cap,
                               float* __restrict__ out_key, int64_t* __restrict__ out_seq,
                               int32_t* __restrict__ out_len) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int64_t j = perm[i];
  const int64_t rel = gcap - 1 - id[j];
  int64_t g = rel + hmod;
  if (g >= gcap) g -= gcap;
  const int64_t slot = g - slot_offset;
  out_key[i] = (float)(-G[j]);
  out_seq[i] = (slot >= 0 && slot < cap) ? seq[slot] : -1;
  out_len[i] = (slot >= 0 && slot < cap) ? lens[slot] : 0;
}

int launch_query_all(const TopkArgs& a, const int64_t* seq, const WideBank& wb, const int16_t* q16,
                     float iq, double* G, int64_t* id, int* count, cudaStream_t st) {
  SS_CUDA_TRY(cudaMemsetAsync(count, 0, sizeof(int), st));
  count_launch();
  const unsigned grid = (unsigned)std::min<int64_t>((a.n_rows + 255) / 256, 148 * 8);
  k_query_all<<<grid, 256, 0, st>>>(a.emb, a.inv, seq, wb.any ? wb.plane.flag : nullptr,
                                    wb.plane.emb, wb.plane.inv, a.n_rows, a.dim, q16, iq, a.theta,
                                    a.head % a.gcap, a.gcap, a.slot_offset, G, id, count);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

int launch_query_gather(const double* G, const int64_t* id, const int64_t* perm, int64_t m,
                        const int64_t* seq, const int32_t* lens, const TopkArgs& a, float* key,
                        int64_t* out_seq, int32_t* out_len, cudaStream_t st) {
  if (m <= 0) return SS_OK;
  count_launch();
  k_query_gather<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(G, id, perm, m, seq, lens,
                                                              a.head % a.gcap, a.gcap,
                                                              a.slot_offset, a.n_rows, key,
                                                              out_seq, out_len);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

}  // namespace ss
