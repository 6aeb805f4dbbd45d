// Reference-compatible kernels: the batched, device-side twins of
// servesim._kernels (match_pmfs, gittins_min, embed_accumulate) and
// servesim.cost.cost_distribution.  sm_100a.
#include "ss_common.cuh"
#include "ss_internal.h"

namespace ss {

// ---------------------------------------------------------------------------
// match_pmfs  (reference: servesim/_kernels.py:118-138, numba path)
//   one CTA per query; smem counts[max_len+1] filled with shared-memory
//   atomics; ascending-v compaction by a block-wide ballot scan.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
k_match_pmfs(const float* __restrict__ sims, int64_t nw, const int64_t* __restrict__ lens,
             double theta, int max_len, double* __restrict__ sup, double* __restrict__ mas,
             int64_t* __restrict__ sizes, int64_t out_stride, int* __restrict__ err) {
  extern __shared__ int s_counts[];  // [max_len + 1]
  __shared__ int s_total;
  __shared__ int s_warp[8];
  __shared__ int s_base;
  const int q = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int v = tid; v <= max_len; v += blockDim.x) s_counts[v] = 0;
  if (tid == 0) { s_total = 0; s_base = 0; }
  __syncthreads();
  const float* row = sims + (int64_t)q * nw;
  int local_total = 0;
  for (int64_t j = tid; j < nw; j += blockDim.x) {
    // numba compares the f32 sim with the caller's theta as given: a Python
    // float promotes the comparison to f64 (an np.float32 theta is exact in f64)
    if ((double)row[j] >= theta) {        // _kernels.py:126
      int64_t L = lens[j];
      if (L < 0 || L > max_len) { atomicExch(err, SS_ERR_RANGE); continue; }
      atomicAdd(&s_counts[L], 1);         // _kernels.py:127
      ++local_total;                      // _kernels.py:128
    }
  }
  // block reduce total
  for (int o = 16; o > 0; o >>= 1) local_total += __shfl_xor_sync(0xffffffffu, local_total, o);
  if (lane == 0) atomicAdd(&s_total, local_total);
  __syncthreads();
  const int total = s_total;
  if (total == 0) {
    if (tid == 0) sizes[q] = 0;
    return;
  }
  const double inv = 1.0 / (double)total;  // _kernels.py:131
  // ascending compaction over v = 1..max_len (_kernels.py:132-137)
  for (int v0 = 1; v0 <= max_len; v0 += blockDim.x) {
    int v = v0 + tid;
    int c = (v <= max_len) ? s_counts[v] : 0;
    unsigned ball = __ballot_sync(0xffffffffu, c > 0);
    if (lane == 0) s_warp[warp] = __popc(ball);
    __syncthreads();
    int off = s_base;
    for (int w = 0; w < warp; ++w) off += s_warp[w];
    if (c > 0) {
      int pos = off + __popc(ball & ((1u << lane) - 1u));
      sup[(int64_t)q * out_stride + pos] = (double)v;
      mas[(int64_t)q * out_stride + pos] = __dmul_rn((double)c, inv);
    }
    __syncthreads();
    if (tid == 0) {
      int add = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) add += s_warp[w];
      s_base += add;
    }
    __syncthreads();
  }
  if (tid == 0) sizes[q] = s_base;
}

int launch_match_pmfs(const float* sims, int64_t nq, int64_t nw, const int64_t* lens,
                      double theta, int64_t max_len, double* sup, double* mas,
                      int64_t* sizes, int64_t out_stride, int* err, cudaStream_t st) {
  size_t smem = (size_t)(max_len + 1) * sizeof(int);
  if (smem > 200 * 1024) return set_error(SS_ERR_UNSUPPORTED, "max_len %lld too large", (long long)max_len);
  SS_CUDA_TRY(ensure_dyn_smem(k_match_pmfs, smem));
  count_launch();
  k_match_pmfs<<<(unsigned)nq, 256, smem, st>>>(sims, nw, lens, theta, (int)max_len, sup, mas,
                                                 sizes, out_stride, err);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

// ---------------------------------------------------------------------------
// Gittins over general f64 laws: warp-per-distribution prefix scan.
//   reference form (_kernels.py:110-115):
//     cum_p += m_k; cum_xp += s_k m_k; r_k = (cum_xp + s_k (1 - cum_p)) / cum_p
//   with optional conditioning on attained a:
//     survivors s_k > a, shifted s_k - a, masses renormalised by Z.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_incl_scan_f64(double v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// One law, one warp: min over survivors of (cum_xp + s (1 - cum_p)) / cum_p
// (_kernels.py:104-116; conditioned on attained a and renormalised unless
// ref_mode).  Returns the value on lane 0's `*out_i`.
__device__ __forceinline__ void gittins_warp(const double* s, const double* m, int64_t np, double a,
                                             const double* outlived_i, int ref_mode, double* out_i,
                                             int* err, int lane) {
  // survivors are a suffix (support strictly increasing); find first index
  // with s > a and the survivor mass Z.
  double Z = 0.0;
  int64_t first = np;
  if (a != 0.0 || !ref_mode) {
    for (int64_t b = 0; b < np; b += 32) {
      int64_t k = b + lane;
      bool surv = (k < np) && (s[k] > a);
      unsigned ball = __ballot_sync(0xffffffffu, surv);
      if (ball && first == np) first = b + __ffs(ball) - 1;
      double mz = surv ? m[k] : 0.0;
      for (int o = 16; o > 0; o >>= 1) mz += __shfl_xor_sync(0xffffffffu, mz, o);
      Z += mz;
    }
  } else {
    first = 0;
    Z = 1.0;
  }
  if (first >= np) {  // outlived every hypothesis or empty
    if (lane == 0) *out_i = (np == 0) ? INFINITY : (outlived_i ? *outlived_i : INFINITY);
    return;
  }
  double cp = 0.0, cxp = 0.0, best = INFINITY;
  for (int64_t b = first; b < np; b += 32) {
    int64_t k = b + lane;
    double sk = 0.0, mk = 0.0;
    if (k < np) {
      sk = s[k] - a;
      mk = ref_mode ? m[k] : m[k] / Z;
    }
    double p = warp_incl_scan_f64(mk, lane) + cp;
    double xp = warp_incl_scan_f64(sk * mk, lane) + cxp;
    if (k < np) {
      if (p == 0.0) atomicExch(err, SS_ERR_ZERODIV);
      double r = (xp + sk * (1.0 - p)) / p;
      if (r < best) best = r;
    }
    cp = __shfl_sync(0xffffffffu, p, 31);
    cxp = __shfl_sync(0xffffffffu, xp, 31);
  }
  best = warp_min_f64(best);
  if (lane == 0) *out_i = best;
}

__global__ void __launch_bounds__(256)
k_gittins_dist(const double* __restrict__ support, const double* __restrict__ masses,
               const int64_t* __restrict__ npts, const double* __restrict__ attained,
               const double* __restrict__ outlived, int64_t n, int64_t stride,
               double* __restrict__ out, int* __restrict__ err, int ref_mode) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= n) return;
  gittins_warp(support + i * stride, masses + i * stride, npts[i], attained ? attained[i] : 0.0,
               outlived ? outlived + i : nullptr, ref_mode, out + i, err, lane);
}

// ------------------------------------------------------------ per call ----
// The reference's scalar call (one law per call, host arrays in and out)
// through mapped pinned memory: the kernel pulls the inputs across PCIe with
// every load in flight at once (into shared memory), computes, writes the
// result back into host memory and raises the slot's flag; the caller spins
// on the flag.  No copy-engine transfer and no stream synchronisation.
__device__ __forceinline__ void percall_pull(double* dst, const double* src, int64_t n) {
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) dst[k] = src[k];
}
__device__ __forceinline__ void percall_raise(PerCallHdr* h, uint32_t seq) {
  __threadfence_system();
  *reinterpret_cast<volatile uint32_t*>(&h->flag) = seq;
}

__global__ void __launch_bounds__(128) k_gittins_percall(PerCallHdr* h, uint32_t seq) {
  extern __shared__ double sm[];
  const int64_t n = h->n;
  const double* src = reinterpret_cast<const double*>(h + 1);
  percall_pull(sm, src, 2 * n);
  __shared__ int err;
  __shared__ double res;
  if (threadIdx.x == 0) err = 0;
  __syncthreads();
  if (threadIdx.x < 32) gittins_warp(sm, sm + n, n, 0.0, nullptr, 1, &res, &err, threadIdx.x);
  __syncthreads();
  if (threadIdx.x == 0) {
    h->result = res;
    h->err = err;
    percall_raise(h, seq);
  }
}

__global__ void __launch_bounds__(128) k_cost_percall(PerCallHdr* h, uint32_t seq) {
  const int64_t n = h->n;
  const double in = h->input_len, w_in = h->w_in, w_out = h->w_out;
  const int kind = h->kind;
  const double* src = reinterpret_cast<const double*>(h + 1);
  double* dst = const_cast<double*>(src) + n;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
    const double l = src[k];
    double r;
    if (kind == SS_COST_RESOURCE_BOUND)
      r = __dadd_rn(__dmul_rn(__dmul_rn(l, l), 0.5), __dmul_rn(in, l));  // cost.py:98-99
    else if (kind == SS_COST_OUTPUT_ONLY)
      r = l;                                                               // cost.py:100-101
    else
      r = __dadd_rn(__dmul_rn(w_in, in), __dmul_rn(w_out, l));           // cost.py:102-103
    dst[k] = r;
  }
  __syncthreads();
  if (threadIdx.x == 0) percall_raise(h, seq);
}

int launch_gittins_percall(PerCallHdr* h_dev, int64_t n, uint32_t seq, cudaStream_t st) {
  count_launch();
  k_gittins_percall<<<1, 128, (size_t)2 * n * sizeof(double), st>>>(h_dev, seq);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

int launch_cost_percall(PerCallHdr* h_dev, uint32_t seq, cudaStream_t st) {
  count_launch();
  k_cost_percall<<<1, 128, 0, st>>>(h_dev, seq);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

int launch_gittins_dist(const double* support, const double* masses, const int64_t* npts,
                        const double* attained, const double* outlived, int64_t n, int64_t stride,
                        double* out, int* err, int ref_mode, cudaStream_t st) {
  if (n <= 0) return SS_OK;
  count_launch();
  unsigned grid = (unsigned)((n + 7) / 8);
  k_gittins_dist<<<grid, 256, 0, st>>>(support, masses, npts, attained, outlived, n, stride,
                                       out, err, ref_mode);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

// ---------------------------------------------------------------------------
// embed_accumulate (reference: servesim/_kernels.py:37-102)
//   warp per prompt; lane i hashes token i of a 32-token chunk; the 2-gram
//   hash takes the previous unigram hash from lane i-1 (carry across chunks).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <bool QUANT>
__global__ void __launch_bounds__(128)
k_embed(const int64_t* __restrict__ tokens, const int64_t* __restrict__ offsets, int64_t n,
        uint64_t salt, int dim, double* __restrict__ out_f64, int16_t* __restrict__ out_i16,
        float* __restrict__ out_inv, int* __restrict__ err) {
  extern __shared__ int s_acc[];  // [4][dim]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t p = (int64_t)blockIdx.x * 4 + warp;
  int* acc = s_acc + warp * dim;
  for (int d = lane; d < dim; d += 32) acc[d] = 0;
  __syncwarp();
  if (p < n) {
    const int64_t b = offsets[p], e = offsets[p + 1];
    uint64_t carry = 0;
    const uint64_t PHI = 0x9E3779B97F4A7C15ull, C1 = 0x2545F4914F6CDD1Dull,
                   C2 = 0xD6E8FEB86659FD93ull;
    for (int64_t t0 = b; t0 < e; t0 += 32) {
      int64_t t = t0 + lane;
      bool live = t < e;
      uint64_t u = 0;
      if (live) {
        u = mix64(salt ^ ((uint64_t)tokens[t] * PHI + C1));
        atomicAdd(&acc[(int)(u % (uint64_t)dim)], ((u >> 61) & 1ull) ? -1 : 1);
      }
      uint64_t prev = __shfl_up_sync(0xffffffffu, u, 1);
      if (lane == 0) prev = carry;
      if (live && t > b) {
        uint64_t g = mix64(prev ^ (u * PHI + C2));
        atomicAdd(&acc[(int)(g % (uint64_t)dim)], ((g >> 61) & 1ull) ? -1 : 1);
      }
      carry = __shfl_sync(0xffffffffu, u, 31);
    }
  }
  __syncwarp();
  if (p >= n) return;
  if (!QUANT) {
    for (int d = lane; d < dim; d += 32) out_f64[p * dim + d] = (double)acc[d];
  } else {
    // the exact integer vector as int16 (the bank keeps it in its int8 plane
    // when every bucket fits, in its wide plane otherwise; err[1] counts the
    // rows that do not fit int8); inverse norm of the exact sum of squares
    long long ss2 = 0;
    bool fits = true;
    for (int d = lane; d < dim; d += 32) {
      int v = acc[d];
      if (v > 32767 || v < -32767) atomicExch(err, SS_ERR_RANGE);
      v = max(-32767, min(32767, v));
      fits &= (v >= -127 && v <= 127);
      out_i16[p * dim + d] = (int16_t)v;
      ss2 += (long long)v * v;
    }
    for (int o = 16; o > 0; o >>= 1) ss2 += __shfl_xor_sync(0xffffffffu, ss2, o);
    const bool wide = !__all_sync(0xffffffffu, fits);
    if (lane == 0) {
      out_inv[p] = ss2 ? __fdiv_rn(1.0f, __fsqrt_rn(__ll2float_rn(ss2))) : __int_as_float(0x7fc00000);
      if (wide) atomicAdd(err + 1, 1);
    }
  }
}

int launch_embed(const int64_t* tokens, const int64_t* offsets, int64_t n, uint64_t salt,
                 int dim, double* out_f64, int16_t* out_i16, float* out_inv, int* err,
                 cudaStream_t st) {
  if (n <= 0) return SS_OK;
  size_t smem = (size_t)4 * dim * sizeof(int);
  if (smem > 200 * 1024) return set_error(SS_ERR_UNSUPPORTED, "dim %d too large", dim);
  unsigned grid = (unsigned)((n + 3) / 4);
  count_launch();
  if (out_i16) {
    SS_CUDA_TRY(ensure_dyn_smem(k_embed<true>, smem));
    k_embed<true><<<grid, 128, smem, st>>>(tokens, offsets, n, salt, dim, nullptr, out_i16, out_inv, err);
  } else {
    SS_CUDA_TRY(ensure_dyn_smem(k_embed<false>, smem));
    k_embed<false><<<grid, 128, smem, st>>>(tokens, offsets, n, salt, dim, out_f64, nullptr, nullptr, err);
  }
  SS_LAUNCH_CHECK();
  return SS_OK;
}

// ---------------------------------------------------------------------------
// cost_distribution pushforward (reference: servesim/cost.py:97-118)
// ---------------------------------------------------------------------------
__global__ void k_cost_dist(int kind, double w_in, double w_out, const double* __restrict__ I,
                            const double* __restrict__ ls, const int64_t* __restrict__ npts,
                            int64_t n, int64_t stride, double* __restrict__ out) {
  const int64_t i = blockIdx.y;
  if (i >= n) return;
  const double in = I[i];
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < npts[i];
       k += (int64_t)gridDim.x * blockDim.x) {
    double l = ls[i * stride + k], r;
    if (kind == SS_COST_RESOURCE_BOUND)
      r = __dadd_rn(__dmul_rn(__dmul_rn(l, l), 0.5), __dmul_rn(in, l));  // cost.py:98-99
    else if (kind == SS_COST_OUTPUT_ONLY)
      r = l;                                                               // cost.py:100-101
    else
      r = __dadd_rn(__dmul_rn(w_in, in), __dmul_rn(w_out, l));           // cost.py:102-103
    out[i * stride + k] = r;
  }
}

int launch_cost_dist(int kind, double w_in, double w_out, const double* I, const double* ls,
                     const int64_t* npts, int64_t n, int64_t stride, double* out, cudaStream_t st) {
  if (n <= 0) return SS_OK;
  if (n > 65535) {
    for (int64_t b = 0; b < n; b += 65535) {
      int64_t m = (n - b < 65535) ? n - b : 65535;
      int rc = launch_cost_dist(kind, w_in, w_out, I + b, ls + b * stride, npts + b, m, stride,
                                out + b * stride, st);
      if (rc) return rc;
    }
    return SS_OK;
  }
  count_launch();
  dim3 grid((unsigned)((stride + 127) / 128 < 8 ? (stride + 127) / 128 : 8), (unsigned)n);
  if (grid.x == 0) grid.x = 1;
  k_cost_dist<<<grid, 128, 0, st>>>(kind, w_in, w_out, I, ls, npts, n, stride, out);
  SS_LAUNCH_CHECK();
  return SS_OK;
}


// ---------------------------------------------------------------------------
// host-buffer round inputs read straight from mapped pinned host memory: one
// kernel for up to kGatherSegs (src, dst, bytes) segments instead of one
// copy-engine node each (a small H2D copy node costs ~4 us of the plugin
// call; scripts/probe_e2e.py).  16-byte loads when both ends allow.
// ---------------------------------------------------------------------------
__global__ void k_h2d_gather(GatherSegs g) {
  for (int s = 0; s < g.n; ++s) {
    const unsigned char* src = static_cast<const unsigned char*>(g.src[s]);
    unsigned char* dst = static_cast<unsigned char*>(g.dst[s]);
    const int64_t nb = g.bytes[s];
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    if ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) {
      const int64_t n16 = nb >> 4;
      for (int64_t i = tid; i < n16; i += nt)
        reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
      for (int64_t i = (n16 << 4) + tid; i < nb; i += nt) dst[i] = src[i];
    } else {
      for (int64_t i = tid; i < nb; i += nt) dst[i] = src[i];
    }
  }
}

int launch_h2d_gather(const GatherSegs& g, cudaStream_t st) {
  int64_t total = 0;
  for (int s = 0; s < g.n; ++s) total += g.bytes[s];
  if (total <= 0) return SS_OK;
  int blocks = (int)((total / 16 + 255) / 256);
  blocks = blocks < 1 ? 1 : (blocks > 148 ? 148 : blocks);
  count_launch();
  k_h2d_gather<<<blocks, 256, 0, st>>>(g);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

}  // namespace ss
