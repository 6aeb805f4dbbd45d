// Stage 1, small-batch path: vectorised HBM-streaming int8 dot-product scan
// with a fused per-thread top-k (the score matrix is never written).
//
// Reference semantics: query_similar (exact linear scan,
// cos >= theta, desc similarity, tie -> larger insertion_seq) with the
// north-star top-k; scores as DESIGN.md section 3.
//
// Mapping: one thread = one query (its int8 vector lives in registers); a CTA
// holds 128 queries and streams one slice of the bank through shared memory
// in 32-row tiles (cp.async double buffer, broadcast LDS.128 reads), using
// __dp4a for the int8 dot products.  Each slice emits an unsorted partial
// top-k per query; ss_merge_topk merges slices.
#include "ss_common.cuh"
#include "ss_internal.h"
#include "topk_heap.cuh"

namespace ss {

constexpr int SCAN_ROWS = 32;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int D, int SCAN_THREADS>
__global__ void __launch_bounds__(SCAN_THREADS, 2)
k_topk_scan(const int8_t* __restrict__ Q, const float* __restrict__ q_inv, int64_t nq,
            const int8_t* __restrict__ emb, const float* __restrict__ inv, int64_t n_rows,
            int k, float theta, int64_t head, int64_t gcap, int64_t slot_offset,
            int64_t rows_per_slice, uint64_t* __restrict__ partials) {
  constexpr int W = D / 16;  // 16-byte words per row
  extern __shared__ __align__(16) unsigned char smem[];
  int4* s_tile = reinterpret_cast<int4*>(smem);                         // [2][ROWS][W]
  float* s_iw = reinterpret_cast<float*>(smem + 2 * SCAN_ROWS * D);     // [2][ROWS]
  uint64_t* s_heap = reinterpret_cast<uint64_t*>(smem + 2 * SCAN_ROWS * D + 2 * SCAN_ROWS * 4);

  const int tid = threadIdx.x;
  const int64_t q = (int64_t)blockIdx.y * SCAN_THREADS + tid;
  const int slice = blockIdx.x;
  const int64_t r0 = (int64_t)slice * rows_per_slice;
  const int64_t r1 = min(n_rows, r0 + rows_per_slice);

  // query -> registers
  int4 qv[W];
  float iq = __int_as_float(0x7fc00000);
  if (q < nq) {
    const int4* qp = reinterpret_cast<const int4*>(Q + q * D);
#pragma unroll
    for (int w = 0; w < W; ++w) qv[w] = qp[w];
    iq = q_inv[q];
  } else {
#pragma unroll
    for (int w = 0; w < W; ++w) qv[w] = make_int4(0, 0, 0, 0);
  }
  HeapState st;
  st.cnt = 0;
  st.root = 0;
  st.thr_s = (iq == iq) ? s_threshold(theta, iq) : INFINITY;
  uint64_t* heap = s_heap + tid;

  auto load_tile = [&](int buf, int64_t base) {
    // 32 rows x W words = 32*W 16-byte chunks, 128 threads
    for (int c = tid; c < SCAN_ROWS * W; c += SCAN_THREADS) {
      int r = c / W, w = c % W;
      int64_t row = base + r;
      bool ok = row < r1;
      cp_async16(&s_tile[(buf * SCAN_ROWS + r) * W + w],
                 emb + (ok ? row : r0) * D + w * 16, ok);
    }
    if (tid < SCAN_ROWS) {
      int64_t row = base + tid;
      s_iw[buf * SCAN_ROWS + tid] = row < r1 ? inv[row] : __int_as_float(0x7fc00000);
    }
  };

  int buf = 0;
  if (r0 < r1) load_tile(0, r0);
  cp_async_commit();
  for (int64_t base = r0; base < r1; base += SCAN_ROWS) {
    if (base + SCAN_ROWS < r1) load_tile(buf ^ 1, base + SCAN_ROWS);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const int4* tile = s_tile + buf * SCAN_ROWS * W;
    int acc[SCAN_ROWS];
#pragma unroll
    for (int r = 0; r < SCAN_ROWS; ++r) acc[r] = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const int4 a = qv[w];
#pragma unroll
      for (int r = 0; r < SCAN_ROWS; ++r) {
        const int4 b = tile[r * W + w];  // broadcast: every lane reads the same row word
        acc[r] = __dp4a(a.x, b.x, acc[r]);
        acc[r] = __dp4a(a.y, b.y, acc[r]);
        acc[r] = __dp4a(a.z, b.z, acc[r]);
        acc[r] = __dp4a(a.w, b.w, acc[r]);
      }
    }
    if (q < nq) {
#pragma unroll
      for (int r = 0; r < SCAN_ROWS; ++r) {
        float iw = s_iw[buf * SCAN_ROWS + r];
        float s = __fmul_rn(__int2float_rn(acc[r]), iw);
        if (s >= st.thr_s)
          heap_consider<SCAN_THREADS>(heap, k, st, acc[r], iw, iq, theta,
                                      slot_offset + base + r, head, gcap);
      }
    }
    __syncthreads();
    buf ^= 1;
  }
  cp_async_wait<0>();
  if (q < nq) {
    uint64_t* out = partials + ((int64_t)slice * nq + q) * k;
    for (int i = 0; i < k; ++i) out[i] = (i < st.cnt) ? heap[i * SCAN_THREADS] : 0ull;
  }
}

template <int D, int SCAN_THREADS>
static int launch_scan_dt(const TopkArgs& a, uint64_t* partials, int n_slices, cudaStream_t st) {
  size_t smem = (size_t)2 * SCAN_ROWS * D + 2 * SCAN_ROWS * 4 + (size_t)a.k * SCAN_THREADS * 8;
  if (smem > 227 * 1024) return set_error(SS_ERR_UNSUPPORTED, "k=%d too large for scan", a.k);
  SS_CUDA_TRY(cudaFuncSetAttribute(k_topk_scan<D, SCAN_THREADS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int64_t rows_per_slice = (a.n_rows + n_slices - 1) / n_slices;
  rows_per_slice = (rows_per_slice + SCAN_ROWS - 1) / SCAN_ROWS * SCAN_ROWS;
  dim3 grid((unsigned)n_slices, (unsigned)((a.nq + SCAN_THREADS - 1) / SCAN_THREADS));
  count_launch();
  k_topk_scan<D, SCAN_THREADS><<<grid, SCAN_THREADS, smem, st>>>(a.q, a.q_inv, a.nq, a.emb, a.inv, a.n_rows, a.k,
                                                   a.theta, a.head % a.gcap, a.gcap, a.slot_offset,
                                                   rows_per_slice, partials);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

template <int D>
static int launch_scan_d(const TopkArgs& a, uint64_t* partials, int n_slices, cudaStream_t st) {
  return a.k <= 128 ? launch_scan_dt<D, 128>(a, partials, n_slices, st)
                    : launch_scan_dt<D, 64>(a, partials, n_slices, st);
}

static inline int scan_threads(int k) { return k <= 128 ? 128 : 64; }

int topk_scan_slices(const TopkArgs& a, int device) {
  const int SCAN_THREADS = scan_threads(a.k);
  int sms = sm_count(device);
  int64_t qtiles = (a.nq + SCAN_THREADS - 1) / SCAN_THREADS;
  int64_t want = (2 * sms + qtiles - 1) / qtiles;  // ~2 CTAs per SM
  int64_t max_by_rows = (a.n_rows + SCAN_ROWS - 1) / SCAN_ROWS;
  if (want > max_by_rows) want = max_by_rows;
  if (want < 1) want = 1;
  if (want > 512) want = 512;
  return (int)want;
}

int launch_topk_scan(const TopkArgs& a, uint64_t* partials, int n_slices, cudaStream_t st) {
  switch (a.dim) {
    case 128: return launch_scan_d<128>(a, partials, n_slices, st);
    case 256: return launch_scan_d<256>(a, partials, n_slices, st);
    case 384: return launch_scan_d<384>(a, partials, n_slices, st);
    case 512: return launch_scan_d<512>(a, partials, n_slices, st);
    default:
      return set_error(SS_ERR_UNSUPPORTED, "scan path supports dim in {128,256,384,512}, got %d",
                       a.dim);
  }
}

}  // namespace ss
