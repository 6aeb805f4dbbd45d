// History bank maintenance: FIFO ring writes and the window-wide fallback
// histogram.  Reference contract: SPEC.md:101-130 (HistoryRecord, push),
// SPEC.md:184-186,223 (fallback = empirical law of the whole window).
//
// The bank keeps an exact-length count histogram len_cnt[0..65535] up to date
// on every write (+1 for the new record, -1 for the evicted one; integer
// atomics, so exact), which makes the per-round fallback histogram a scan of
// the count table instead of a scan of the whole window.
#include "ss_common.cuh"
#include "ss_internal.h"

namespace ss {

// one warp per record: 16-byte vector copy of the row, then inverse norm
// (IEEE 1/sqrt of the exact integer sum of squares, bit-identical to numpy
// float32), length and seq.  T = int8: the row goes to the int8 plane.
// T = int16 (feature-hash vectors of long prompts, whose buckets may exceed
// the int8 range, _kernels.py:82-95): a row that fits int8 is narrowed into
// the int8 plane; a row that does not ("wide") leaves a zero row and a NaN
// inverse norm there -- the tensor-core kernels never match it -- and its
// exact int16 vector and inverse norm go to the bank's wide plane, flagged
// per slot, where the CUDA-core wide pass (k_wide.cu) scores it.  Every
// write of a normal row clears the slot's wide flag.
template <typename T>
__global__ void __launch_bounds__(256)
k_bank_write(int8_t* __restrict__ emb, float* __restrict__ inv, int32_t* __restrict__ lens,
             int64_t* __restrict__ seq, int32_t* __restrict__ len_cnt, int dim,
             const T* __restrict__ src_emb, const float* __restrict__ src_inv,
             const int32_t* __restrict__ src_lens, const int64_t* __restrict__ src_seq,
             const int64_t* __restrict__ src_slot, int64_t n, int64_t first_seq,
             int64_t capacity, int64_t skip, int* __restrict__ err,
             const int64_t* __restrict__ src_idx, WidePlane wp) {
  const int lane = threadIdx.x & 31;
  const int64_t r = skip + (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= n) return;
  const int64_t rs = src_idx ? src_idx[r] : r;  // source record (gather)
  const int64_t s = src_seq ? src_seq[r] : first_seq + r;
  const int64_t slot = src_slot ? src_slot[r] : s % capacity;
  if (slot < 0 || slot >= capacity) {
    if (lane == 0) atomicExch(err, SS_ERR_ARG);
    return;
  }
  bool wide = false;
  long long ss2 = 0;
  if constexpr (sizeof(T) == 1) {
    const int4* src = reinterpret_cast<const int4*>(src_emb + rs * dim);
    int4* dst = reinterpret_cast<int4*>(emb + slot * dim);
    int acc = 0;
    for (int w = lane; w < dim / 16; w += 32) {
      int4 v = src[w];
      dst[w] = v;
      const int* vi = reinterpret_cast<const int*>(&v);
#pragma unroll
      for (int t = 0; t < 4; ++t) acc = __dp4a(vi[t], vi[t], acc);
    }
    ss2 = acc;
  } else {
    // 8 int16 per 16-byte load; the row fits int8 iff every |x| <= 127
    const int4* src = reinterpret_cast<const int4*>(src_emb + rs * dim);
    bool fits = true;
    for (int w = lane; w < dim / 8; w += 32) {
      const int4 v = src[w];
      const int16_t* x = reinterpret_cast<const int16_t*>(&v);
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        fits &= (x[t] >= -127 && x[t] <= 127);
        ss2 += (long long)x[t] * x[t];
      }
    }
    wide = !__all_sync(0xffffffffu, fits);
    if (wide && !wp.flag) {  // no wide plane allocated: refuse
      if (lane == 0) atomicExch(err, SS_ERR_RANGE);
      return;
    }
    for (int w = lane; w < dim / 8; w += 32) {
      const int4 v = src[w];
      const int16_t* x = reinterpret_cast<const int16_t*>(&v);
      if (wide) {
        reinterpret_cast<int4*>(wp.emb + slot * dim)[w] = v;
        reinterpret_cast<uint2*>(emb + slot * dim)[w] = make_uint2(0u, 0u);
      } else {
        uint32_t lo = 0, hi = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t) lo |= (uint32_t)(uint8_t)(int8_t)x[t] << (8 * t);
#pragma unroll
        for (int t = 0; t < 4; ++t) hi |= (uint32_t)(uint8_t)(int8_t)x[4 + t] << (8 * t);
        reinterpret_cast<uint2*>(emb + slot * dim)[w] = make_uint2(lo, hi);
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) ss2 += __shfl_xor_sync(0xffffffffu, ss2, o);
  if (lane == 0) {
    if (seq[slot] >= 0) atomicSub(&len_cnt[lens[slot] & 0xffff], 1);  // evicted record
    int L = src_lens[rs];
    if (L < 1 || L > 65535) {
      atomicExch(err, SS_ERR_RANGE);
      L = max(1, min(L, 65535));
    }
    atomicAdd(&len_cnt[L], 1);
    lens[slot] = L;
    seq[slot] = s;
    float iv;
    if (src_inv) iv = src_inv[rs];
    else iv = ss2 ? __fdiv_rn(1.0f, __fsqrt_rn(__ll2float_rn(ss2))) : __int_as_float(0x7fc00000);
    inv[slot] = wide ? __int_as_float(0x7fc00000) : iv;  // the tensor-core kernels skip wide rows
    if (wp.flag) {
      wp.flag[slot] = wide ? 1 : 0;
      if (wide) {
        wp.inv[slot] = iv;
        atomicAdd(wp.count, 1);
      }
    }
  }
}

// The filter bounds of every 16-row group a write touched: (max inverse norm,
// floored at 0; min inverse norm, capped at +inf) over the group's non-NaN
// rows -- exactly the per-16-column bounds the TS kernel's epilogue used to
// reduce from the tile's norms every tile, now computed once per write.  One
// thread per written record recomputes its record's group (records sharing a
// group write the same values).
__global__ void __launch_bounds__(256)
k_bank_bounds(const float* __restrict__ inv, float2* __restrict__ ibnd,
              const int64_t* __restrict__ src_slot, int64_t n, int64_t first_seq, int64_t capacity,
              int64_t skip) {
  const int64_t r = skip + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t slot = src_slot ? src_slot[r] : (first_seq + r) % capacity;
  if (slot < 0 || slot >= capacity) return;  // (k_bank_write flags it)
  const int64_t g = slot >> 4;
  const float4* p = reinterpret_cast<const float4*>(inv + g * 16);
  float hi = 0.f, lo = INFINITY;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const float4 w = p[u];  // NaN (empty, zero or wide row) is ignored by fmaxf / fminf
    hi = fmaxf(hi, fmaxf(fmaxf(w.x, w.y), fmaxf(w.z, w.w)));
    lo = fminf(lo, fminf(fminf(w.x, w.y), fminf(w.z, w.w)));
  }
  ibnd[g] = make_float2(hi, lo);
}

int launch_bank_write(int8_t* emb, float* inv, int32_t* lens, int64_t* seq, int32_t* len_cnt,
                      int dim, const void* src_emb, int src_bytes, const float* src_inv,
                      const int32_t* src_lens, const int64_t* src_seq, const int64_t* src_slot,
                      int64_t n, int64_t first_seq, int64_t capacity, int64_t skip, int* err,
                      cudaStream_t st, const int64_t* src_idx, const WidePlane* wp, float2* ibnd) {
  int64_t m = n - skip;
  if (m <= 0) return SS_OK;
  const WidePlane w = wp ? *wp : WidePlane{};
  count_launch();
  const unsigned grid = (unsigned)((m + 7) / 8);
  if (src_bytes == 2)
    k_bank_write<int16_t><<<grid, 256, 0, st>>>(emb, inv, lens, seq, len_cnt, dim,
                                                static_cast<const int16_t*>(src_emb), src_inv,
                                                src_lens, src_seq, src_slot, n, first_seq, capacity,
                                                skip, err, src_idx, w);
  else
    k_bank_write<int8_t><<<grid, 256, 0, st>>>(emb, inv, lens, seq, len_cnt, dim,
                                               static_cast<const int8_t*>(src_emb), src_inv,
                                               src_lens, src_seq, src_slot, n, first_seq, capacity,
                                               skip, err, src_idx, w);
  SS_LAUNCH_CHECK();
  if (ibnd) {
    count_launch();
    k_bank_bounds<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(inv, ibnd, src_slot, n, first_seq,
                                                              capacity, skip);
    SS_LAUNCH_CHECK();
  }
  return SS_OK;
}

// fallback histogram from the exact-length counts: one CTA walks len_cnt,
// clamps lengths to max_len and accumulates (count, sum v, sum v^2) per bin
// with shared-memory atomics.  Integer-exact.
constexpr int FB_THREADS = 1024;

__global__ void __launch_bounds__(FB_THREADS)
k_fallback_hist(const int32_t* __restrict__ len_cnt, int max_len, int nbins,
                int64_t* __restrict__ cnt, int64_t* __restrict__ sv, int64_t* __restrict__ sv2) {
  extern __shared__ unsigned long long s_h[];  // [3][nbins]
  const int w = max_len / nbins;
  for (int b = threadIdx.x; b < 3 * nbins; b += blockDim.x) s_h[b] = 0ull;
  __syncthreads();
  // 65536 counts = 16 int4 per thread, all loads issued before any use
  const int4* c4 = reinterpret_cast<const int4*>(len_cnt);
  int4 r[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) r[u] = c4[u * FB_THREADS + threadIdx.x];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int base = 4 * (u * FB_THREADS + threadIdx.x);
    const int cs[4] = {r[u].x, r[u].y, r[u].z, r[u].w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int v = base + e;
      const int c = cs[e];
      if (c == 0 || v == 0) continue;
      const unsigned long long L = (unsigned long long)min(v, max_len);
      const int b = (int)(L - 1) / w;
      atomicAdd(&s_h[b], (unsigned long long)c);
      atomicAdd(&s_h[nbins + b], (unsigned long long)c * L);
      atomicAdd(&s_h[2 * nbins + b], (unsigned long long)c * L * L);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nbins; b += blockDim.x) {
    cnt[b] = (int64_t)s_h[b];
    sv[b] = (int64_t)s_h[nbins + b];
    sv2[b] = (int64_t)s_h[2 * nbins + b];
  }
}

int launch_fallback_hist(const int32_t* len_cnt, int max_len, int nbins, int64_t* cnt, int64_t* sv,
                         int64_t* sv2, cudaStream_t st) {
  size_t smem = (size_t)3 * nbins * sizeof(unsigned long long);
  SS_CUDA_TRY(ensure_dyn_smem(k_fallback_hist, smem));
  count_launch();
  k_fallback_hist<<<1, FB_THREADS, smem, st>>>(len_cnt, max_len, nbins, cnt, sv, sv2);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

}  // namespace ss
