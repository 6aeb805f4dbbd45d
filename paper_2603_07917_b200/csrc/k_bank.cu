// History bank maintenance: FIFO ring writes and the window-wide fallback
// histogram.  Reference contract: SPEC.md:101-130 (HistoryRecord, push),
// SPEC.md:184-186,223 (fallback = empirical law of the whole window).
#include "ss_common.cuh"
#include "ss_internal.h"

namespace ss {

// one warp per record: 16-byte vector copy of the int8 row, then inverse
// norm (IEEE 1/sqrt, bit-identical to numpy float32), length and seq.
__global__ void __launch_bounds__(256)
k_bank_write(int8_t* __restrict__ emb, float* __restrict__ inv, int32_t* __restrict__ lens,
             int64_t* __restrict__ seq, int dim, const int8_t* __restrict__ src_emb,
             const float* __restrict__ src_inv, const int32_t* __restrict__ src_lens,
             const int64_t* __restrict__ src_seq, const int64_t* __restrict__ src_slot,
             int64_t n, int64_t first_seq, int64_t capacity, int64_t skip,
             int* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const int64_t r = skip + (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= n) return;
  const int64_t s = src_seq ? src_seq[r] : first_seq + r;
  const int64_t slot = src_slot ? src_slot[r] : s % capacity;
  if (slot < 0 || slot >= capacity) {
    if (lane == 0) atomicExch(err, SS_ERR_ARG);
    return;
  }
  const int4* src = reinterpret_cast<const int4*>(src_emb + r * dim);
  int4* dst = reinterpret_cast<int4*>(emb + slot * dim);
  int ss2 = 0;
  for (int w = lane; w < dim / 16; w += 32) {
    int4 v = src[w];
    dst[w] = v;
    const int* vi = reinterpret_cast<const int*>(&v);
#pragma unroll
    for (int t = 0; t < 4; ++t) ss2 = __dp4a(vi[t], vi[t], ss2);
  }
  for (int o = 16; o > 0; o >>= 1) ss2 += __shfl_xor_sync(0xffffffffu, ss2, o);
  if (lane == 0) {
    int L = src_lens[r];
    if (L < 1 || L > 65535) atomicExch(err, SS_ERR_RANGE);
    lens[slot] = L;
    seq[slot] = s;
    float iv;
    if (src_inv) iv = src_inv[r];
    else iv = ss2 ? __fdiv_rn(1.0f, __fsqrt_rn((float)ss2)) : __int_as_float(0x7fc00000);
    inv[slot] = iv;
  }
}

int launch_bank_write(int8_t* emb, float* inv, int32_t* lens, int64_t* seq, int dim,
                      const int8_t* src_emb, const float* src_inv, const int32_t* src_lens,
                      const int64_t* src_seq, const int64_t* src_slot, int64_t n,
                      int64_t first_seq, int64_t capacity, int64_t skip, int* err,
                      cudaStream_t st) {
  int64_t m = n - skip;
  if (m <= 0) return SS_OK;
  count_launch();
  k_bank_write<<<(unsigned)((m + 7) / 8), 256, 0, st>>>(emb, inv, lens, seq, dim, src_emb,
                                                          src_inv, src_lens, src_seq, src_slot,
                                                          n, first_seq, capacity, skip, err);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

// window histogram: per-CTA shared-memory atomics, then one global atomic per
// non-empty bin.  Integer-exact, so the order of accumulation is irrelevant.
__global__ void __launch_bounds__(256)
k_fallback_hist(const int32_t* __restrict__ lens, const int64_t* __restrict__ seq,
                int64_t capacity, int max_len, int nbins, unsigned long long* __restrict__ cnt,
                unsigned long long* __restrict__ sv, unsigned long long* __restrict__ sv2) {
  extern __shared__ unsigned long long s_h[];  // [3][nbins]
  const int w = max_len / nbins;
  for (int b = threadIdx.x; b < 3 * nbins; b += blockDim.x) s_h[b] = 0ull;
  __syncthreads();
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < capacity;
       j += (int64_t)gridDim.x * blockDim.x) {
    if (seq[j] < 0) continue;
    int L = min(lens[j], max_len);
    int b = (L - 1) / w;
    atomicAdd(&s_h[b], 1ull);
    atomicAdd(&s_h[nbins + b], (unsigned long long)L);
    atomicAdd(&s_h[2 * nbins + b], (unsigned long long)L * (unsigned long long)L);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nbins; b += blockDim.x) {
    if (s_h[b]) {
      atomicAdd(&cnt[b], s_h[b]);
      atomicAdd(&sv[b], s_h[nbins + b]);
      atomicAdd(&sv2[b], s_h[2 * nbins + b]);
    }
  }
}

int launch_fallback_hist(const int32_t* lens, const int64_t* seq, int64_t capacity,
                         int max_len, int nbins, int64_t* cnt, int64_t* sv, int64_t* sv2,
                         cudaStream_t st) {
  SS_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * nbins, st));
  SS_CUDA_TRY(cudaMemsetAsync(sv, 0, sizeof(int64_t) * nbins, st));
  SS_CUDA_TRY(cudaMemsetAsync(sv2, 0, sizeof(int64_t) * nbins, st));
  if (capacity <= 0) return SS_OK;
  size_t smem = (size_t)3 * nbins * sizeof(unsigned long long);
  if (smem > 48 * 1024)
    SS_CUDA_TRY(cudaFuncSetAttribute(k_fallback_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int64_t blocks = (capacity + 2047) / 2048;
  if (blocks > 296) blocks = 296;
  count_launch();
  k_fallback_hist<<<(unsigned)blocks, 256, smem, st>>>(
      lens, seq, capacity, max_len, nbins, reinterpret_cast<unsigned long long*>(cnt),
      reinterpret_cast<unsigned long long*>(sv), reinterpret_cast<unsigned long long*>(sv2));
  SS_LAUNCH_CHECK();
  return SS_OK;
}

}  // namespace ss
