// Native engine round over a GPU-resident request table (the
// callers on both sides of the path, driven as one C-ABI call per iteration).
//
// One call = one iteration of the reference engine's scheduling loop
// restricted to the scheduling state:
//   1. progress: every request of the last batch gains tokens_per_round
//      tokens; those reaching their realised output length complete
//      (k_progress: one CTA walks the batch, binary-searches each id in the
//      id-sorted table, compacts the completions in batch order);
//   2. completions enter the history ring in batch order,
//      gathered straight from the trace arrays (bank_push_gather);
//   3. the table drops them by a stable compaction into its second buffer
//      (k_keep_scan + k_compact_rows), keeping rows in increasing id order;
//   4. up to max_arrivals new requests are appended and predicted by the
//      fused stages 1-3 writing into their table rows (predict_into);
//   5. bucket refreshes (k_refresh), rank of all active requests (ss_rank
//      kernels), batch packing over the ranked list (k_pack_batch), and the
//      next batch's ids (k_batch_ids).
// The host learns one number per call -- the completion count, which sizes
// the ring push, the compaction and the admission.  The Python driver that
// does the same with torch ops is replay_device.DeviceReplay; the parity
// test checks this engine against it round by round.
#include <algorithm>
#include <new>

#include "sagesched.h"
#include "ss_common.cuh"
#include "ss_internal.h"

namespace ss {

constexpr int EG_THREADS = 1024;

__device__ __forceinline__ int block_excl_scan_i32(int v, int* s_warp, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += t;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int y = s_warp[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += t;
    }
    s_warp[lane] = y;
  }
  __syncthreads();
  const int pre = (warp ? s_warp[warp - 1] : 0) + x - v;
  *total = s_warp[31];
  __syncthreads();
  return pre;
}

// 1. progress of the last batch; completions compacted in batch order.  The
// batch carries each request's table row from the pack (the table has not
// moved since); a row whose id does not match falls back to a binary search
// of the id-sorted table.  EG_ITEMS consecutive batch entries per thread
// with their loads in flight, one block scan per EG_THREADS * EG_ITEMS.
constexpr int EG_ITEMS = 8;
__global__ void __launch_bounds__(EG_THREADS)
k_progress(const int64_t* __restrict__ run_ids, const int64_t* __restrict__ run_rows,
           const int32_t* __restrict__ run_count, const int64_t* __restrict__ ids, int64_t n,
           int32_t* __restrict__ g, int tok, const int32_t* __restrict__ true_len,
           int64_t* __restrict__ done_ids, uint8_t* __restrict__ drop, int32_t* __restrict__ n_done) {
  __shared__ int s_warp[32];
  const int cnt = max(*run_count, 0);
  int carry = 0;
  for (int base = 0; base < cnt; base += EG_THREADS * EG_ITEMS) {
    const int i0 = base + threadIdx.x * EG_ITEMS;
    int64_t id[EG_ITEMS], row[EG_ITEMS];
#pragma unroll
    for (int j = 0; j < EG_ITEMS; ++j) {
      const bool v = i0 + j < cnt && n > 0;
      id[j] = v ? run_ids[i0 + j] : -1;
      row[j] = v ? run_rows[i0 + j] : -1;
    }
    int nd = 0;
    bool done[EG_ITEMS];
#pragma unroll
    for (int j = 0; j < EG_ITEMS; ++j) {
      done[j] = false;
      if (id[j] < 0) continue;
      int64_t r = row[j];
      if (r < 0 || r >= n || ids[r] != id[j]) {  // lower_bound in the id-sorted table
        int64_t lo = 0, hi = n;
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (ids[mid] < id[j]) lo = mid + 1; else hi = mid;
        }
        r = (lo < n && ids[lo] == id[j]) ? lo : -1;
      }
      if (r >= 0) {
        const int gn = g[r] + tok;
        g[r] = gn;
        done[j] = gn >= true_len[id[j]];
        if (done[j]) drop[r] = 1;
      }
      nd += done[j];
    }
    int tot;
    int pos = carry + block_excl_scan_i32(nd, s_warp, &tot);
#pragma unroll
    for (int j = 0; j < EG_ITEMS; ++j)
      if (done[j]) done_ids[pos++] = id[j];
    carry += tot;
  }
  if (threadIdx.x == 0) *n_done = carry;
}

// 3a. keep positions (stable) and reset of the drop marks; one CTA
__global__ void __launch_bounds__(EG_THREADS)
k_keep_scan(uint8_t* __restrict__ drop, int64_t n, int64_t* __restrict__ pos) {
  __shared__ int s_warp[32];
  int64_t carry = 0;
  for (int64_t base = 0; base < n; base += EG_THREADS * EG_ITEMS) {
    const int64_t i0 = base + threadIdx.x * EG_ITEMS;  // EG_ITEMS consecutive rows per thread
    bool keep[EG_ITEMS];
    int nk = 0;
#pragma unroll
    for (int j = 0; j < EG_ITEMS; ++j) {
      keep[j] = i0 + j < n && !drop[i0 + j];
      nk += keep[j];
    }
    int tot;
    int64_t p = carry + block_excl_scan_i32(nk, s_warp, &tot);
#pragma unroll
    for (int j = 0; j < EG_ITEMS; ++j) {
      if (i0 + j < n) {
        pos[i0 + j] = keep[j] ? p : -1;
        drop[i0 + j] = 0;
      }
      p += keep[j];
    }
    carry += tot;
  }
}

struct TableBufs {
  int32_t *I, *g, *bucket, *npts;
  int64_t* ids;
  double* G;
  int32_t *pbin, *pcnt;
  int64_t* pD;
};

// 3b. one warp per kept row: scalars + the row's sparse cost law
__global__ void __launch_bounds__(256)
k_compact_rows(TableBufs src, TableBufs dst, const int64_t* __restrict__ pos, int64_t n, int P) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= n) return;
  const int64_t d = pos[r];
  if (d < 0) return;
  if (lane == 0) {
    dst.I[d] = src.I[r];
    dst.g[d] = src.g[r];
    dst.bucket[d] = src.bucket[r];
    dst.npts[d] = src.npts[r];
    dst.ids[d] = src.ids[r];
    dst.G[d] = src.G[r];
  }
  const int np = src.npts[r];  // only the law's points are meaningful
  for (int j = lane; j < np && j < P; j += 32) {
    dst.pbin[d * P + j] = src.pbin[r * P + j];
    dst.pcnt[d * P + j] = src.pcnt[r * P + j];
    dst.pD[d * P + j] = src.pD[r * P + j];
  }
}

// 4a. new rows: ids, input lengths, no progress yet
__global__ void k_admit_rows(TableBufs t, int64_t row0, int64_t n_new, int64_t first_id,
                             const int32_t* __restrict__ tr_I) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_new) return;
  t.ids[row0 + i] = first_id + i;
  t.I[row0 + i] = tr_I[first_id + i];
  t.g[row0 + i] = 0;
  t.bucket[row0 + i] = 0;
}

// 5b. ids of the packed batch (valid below *count)
__global__ void k_batch_ids(const int64_t* __restrict__ batch, const int32_t* __restrict__ count,
                            const int64_t* __restrict__ ids, int64_t n, int64_t* __restrict__ run_ids,
                            int B) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  const int c = *count;
  if (i < c) {
    const int64_t r = batch[i];
    run_ids[i] = (r >= 0 && r < n) ? ids[r] : -1;
  }
}

}  // namespace ss

using namespace ss;

struct ss_table {
  int device = 0;
  int64_t cap = 0;
  int P = 0, B = 0;
  TableBufs buf[2] = {};
  int cur = 0;
  int64_t n_act = 0;
  uint8_t* drop = nullptr;
  int64_t* pos = nullptr;
  int64_t* done_ids = nullptr;
  int32_t* d_ndone = nullptr;
  int32_t* h_ndone = nullptr;  // pinned
  int64_t* perm = nullptr;
  void* rank_ws = nullptr;
  int64_t rank_ws_bytes = 0;
  int64_t* batch = nullptr;
  int32_t* count = nullptr;
  int64_t* tokens = nullptr;
  int64_t* run_ids = nullptr;
  uint8_t* used_fb = nullptr;
};

static void table_free(ss_table* t) {
  for (auto& b : t->buf) {
    cudaFree(b.I); cudaFree(b.g); cudaFree(b.bucket); cudaFree(b.npts); cudaFree(b.ids);
    cudaFree(b.G); cudaFree(b.pbin); cudaFree(b.pcnt); cudaFree(b.pD);
  }
  cudaFree(t->drop); cudaFree(t->pos); cudaFree(t->done_ids); cudaFree(t->d_ndone);
  cudaFreeHost(t->h_ndone);
  cudaFree(t->perm); cudaFree(t->rank_ws); cudaFree(t->batch); cudaFree(t->count);
  cudaFree(t->tokens); cudaFree(t->run_ids); cudaFree(t->used_fb);
}

extern "C" {

int ss_table_create(ss_table_t** out, int32_t device, int64_t capacity, int32_t P,
                    int32_t max_batch) {
  if (!out || capacity < 1 || P < 1 || max_batch < 1 || capacity >= (1LL << 31))
    return set_error(SS_ERR_ARG, "table_create: bad args");
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) return set_error(SS_ERR_CUDA, "table_create: device");
  ss_table* t = new (std::nothrow) ss_table();
  if (!t) return set_error(SS_ERR_ARG, "oom");
  t->device = device;
  t->cap = capacity;
  t->P = P;
  t->B = max_batch;
  bool ok = true;
  auto A = [&](auto** p, size_t bytes) {
    if (ok && cudaMalloc(reinterpret_cast<void**>(p), bytes) != cudaSuccess) ok = false;
  };
  for (auto& b : t->buf) {
    A(&b.I, capacity * 4); A(&b.g, capacity * 4); A(&b.bucket, capacity * 4);
    A(&b.npts, capacity * 4); A(&b.ids, capacity * 8); A(&b.G, capacity * 8);
    A(&b.pbin, capacity * P * 4); A(&b.pcnt, capacity * P * 4); A(&b.pD, capacity * P * 8);
  }
  A(&t->drop, capacity); A(&t->pos, capacity * 8); A(&t->done_ids, (size_t)max_batch * 8);
  A(&t->d_ndone, 4); A(&t->perm, capacity * 8);
  t->rank_ws_bytes = rank_workspace_bytes(capacity);
  A(&t->rank_ws, (size_t)t->rank_ws_bytes);
  A(&t->batch, (size_t)max_batch * 8); A(&t->count, 4); A(&t->tokens, 8);
  A(&t->run_ids, (size_t)max_batch * 8); A(&t->used_fb, capacity);
  if (ok && cudaMallocHost(&t->h_ndone, 4) != cudaSuccess) ok = false;
  if (ok) {
    cudaMemset(t->drop, 0, capacity);
    cudaMemset(t->count, 0, 4);
    ok = cudaDeviceSynchronize() == cudaSuccess;
  }
  cudaSetDevice(prev);
  if (!ok) {
    table_free(t);
    delete t;
    cudaGetLastError();
    return set_error(SS_ERR_CUDA, "table_create: allocation failed");
  }
  *out = t;
  return SS_OK;
}

int ss_table_destroy(ss_table_t* t) {
  if (!t) return SS_OK;
  table_free(t);
  delete t;
  return SS_OK;
}

int ss_table_view(ss_table_t* t, int64_t* n_active, int32_t** I, int32_t** g, int64_t** ids,
                  double** G, int32_t** npts, int64_t** perm, int64_t** run_ids,
                  int32_t** batch_count) {
  if (!t) return set_error(SS_ERR_ARG, "null table");
  const TableBufs& b = t->buf[t->cur];
  if (n_active) *n_active = t->n_act;
  if (I) *I = b.I;
  if (g) *g = b.g;
  if (ids) *ids = b.ids;
  if (G) *G = b.G;
  if (npts) *npts = b.npts;
  if (perm) *perm = t->perm;
  if (run_ids) *run_ids = t->run_ids;
  if (batch_count) *batch_count = t->count;
  return SS_OK;
}

int ss_engine_round(ss_table_t* t, ss_bank_t* h, const int8_t* tr_emb, const float* tr_inv,
                    const int32_t* tr_input_len, const int32_t* tr_true_len, int64_t tr_len,
                    int64_t* next_id, int64_t max_arrivals, int32_t tokens_per_round,
                    int32_t bucket_size, int64_t kv_capacity, int32_t mode, int32_t k,
                    float theta, int32_t min_matches, int32_t max_len, int32_t nbins,
                    int32_t algo, int64_t* n_done_out, int64_t* n_admitted_out, void* stream) {
  if (!t || !h || !next_id || tr_len < 0 || max_arrivals < 0 || tokens_per_round < 0 ||
      bucket_size < 1 || kv_capacity < 1 || nbins > t->P)
    return set_error(SS_ERR_ARG, "engine_round: bad args");
  cudaStream_t st = (cudaStream_t)stream;
  const int P = t->P;
  int64_t n = t->n_act;
  // 1. progress of the last batch
  count_launch();
  k_progress<<<1, EG_THREADS, 0, st>>>(t->run_ids, t->batch, t->count, t->buf[t->cur].ids, n,
                                       t->buf[t->cur].g, tokens_per_round, tr_true_len,
                                       t->done_ids, t->drop, t->d_ndone);
  SS_LAUNCH_CHECK();
  SS_CUDA_TRY(cudaMemcpyAsync(t->h_ndone, t->d_ndone, 4, cudaMemcpyDeviceToHost, st));
  SS_CUDA_TRY(cudaStreamSynchronize(st));  // the one host sync: the completion count
  const int64_t nd = *t->h_ndone;
  if (n_done_out) *n_done_out = nd;
  if (nd > 0) {
    // 2. completions into the ring, in batch order
    if (int rc = bank_push_gather(h, tr_emb, tr_inv, tr_true_len, t->done_ids, nd, st)) return rc;
    // 3. stable compaction into the other buffer
    count_launch();
    k_keep_scan<<<1, EG_THREADS, 0, st>>>(t->drop, n, t->pos);
    SS_LAUNCH_CHECK();
    count_launch();
    k_compact_rows<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(t->buf[t->cur], t->buf[t->cur ^ 1],
                                                            t->pos, n, P);
    SS_LAUNCH_CHECK();
    t->cur ^= 1;
    n -= nd;
  }
  const TableBufs& b = t->buf[t->cur];
  // 4. admissions
  const int64_t lo = *next_id;
  const int64_t n_new = std::max<int64_t>(
      0, std::min<int64_t>({max_arrivals, tr_len - lo, t->cap - n}));
  if (n_new > 0) {
    count_launch();
    k_admit_rows<<<(unsigned)((n_new + 255) / 256), 256, 0, st>>>(b, n, n_new, lo, tr_input_len);
    SS_LAUNCH_CHECK();
    int64_t head_ = 0, size_ = 0, cap_ = 0;
    int32_t dim = 0;
    if (int rc = ss_bank_info(h, &head_, &size_, &cap_, &dim)) return rc;
    if (int rc = predict_into(h, tr_emb + lo * dim, tr_inv + lo, b.I + n, n_new, k, theta,
                              min_matches, max_len, nbins, algo, P, b.npts + n, b.pbin + n * P,
                              b.pcnt + n * P, b.pD + n * P, t->used_fb, b.G + n, st))
      return rc;
    *next_id = lo + n_new;
    n += n_new;
  }
  if (n_admitted_out) *n_admitted_out = n_new;
  t->n_act = n;
  if (n == 0) {
    SS_CUDA_TRY(cudaMemsetAsync(t->count, 0, 4, st));
    return SS_OK;
  }
  // 5. refresh, rank, pack, next batch ids
  if (int rc = launch_refresh(n, b.I, b.g, b.bucket, bucket_size, b.npts, b.pcnt, b.pD, P, b.G,
                              nullptr, 0, st))
    return rc;
  if (int rc = launch_rank(b.G, b.ids, n, t->perm, t->rank_ws, t->rank_ws_bytes, st)) return rc;
  if (int rc = launch_pack_batch(t->perm, b.I, b.g, n, kv_capacity, t->B, mode, t->batch, t->count,
                                 t->tokens, st))
    return rc;
  count_launch();
  k_batch_ids<<<(unsigned)((t->B + 255) / 256), 256, 0, st>>>(t->batch, t->count, b.ids, n,
                                                              t->run_ids, t->B);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

}  // extern "C"
