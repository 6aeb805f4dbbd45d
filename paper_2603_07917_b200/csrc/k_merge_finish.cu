// Stage 1 merge (slices / shards -> global top-k), and stages 1b-3 fused:
// neighbour-length histogram -> ResourceBound cost law -> Gittins index, plus
// the running-request refresh.  sm_100a.
//
// Reference semantics:
//   predict         SPEC.md:182-194 (>= min_matches neighbours, else fallback)
//   cost            cost.py:97-99 (conditional-mean cost per bin; exact at w=1)
//   gittins         _kernels.py:110-115 in exact integer-count form
//   conditioning    SPEC.md:335-343, outlived rule SPEC.md:373
//   refresh cadence SPEC.md:345-353
#include "ss_common.cuh"
#include "ss_internal.h"
#include "topk_select.cuh"

namespace ss {

constexpr int MF_THREADS = 512;

// load nlists x k candidates of query q; payload = carried length (len) or
// the bank length looked up from the slot (single-GPU / local merge)
__device__ void load_candidates(const uint64_t* comp, const int32_t* len, int nlists, int64_t nq,
                                int k, int64_t q, uint64_t* cand, int32_t* cpay,
                                const int32_t* bank_lens, int64_t head, int64_t gcap,
                                int64_t slot_offset) {
  const int M = nlists * k;
  for (int i = threadIdx.x; i < M; i += blockDim.x) {
    int l = i / k, j = i % k;
    int64_t src = ((int64_t)l * nq + q) * k + j;
    uint64_t c = comp[src];
    cand[i] = c;
    cpay[i] = len ? len[src] : 0;  // bank lengths are gathered for the winners only
  }
  __syncthreads();
}

// winners' lengths from the local bank (single-GPU / local merge)
__device__ void resolve_lens(const uint64_t* sel, int32_t* spay, int k, const int32_t* bank_lens,
                             int64_t head, int64_t gcap, int64_t slot_offset) {
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const uint64_t c = sel[i];
    if (c != 0ull) {
      int64_t g = (int64_t)comp_rel(c) + head % gcap;
      if (g >= gcap) g -= gcap;
      spay[i] = bank_lens[g - slot_offset];
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(MF_THREADS)
k_merge(const uint64_t* __restrict__ comp, const int32_t* __restrict__ len, int nlists,
        int64_t nq, int k, int kpad, uint64_t* __restrict__ out_comp,
        int32_t* __restrict__ out_len, const int32_t* __restrict__ bank_lens, int64_t head,
        int64_t gcap, int64_t slot_offset, PeerOut po) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int M = nlists * k;
  uint64_t* cand = reinterpret_cast<uint64_t*>(smem);      // [M]
  uint64_t* sel = cand + M;                                // [kpad]
  int32_t* cpay = reinterpret_cast<int32_t*>(sel + kpad);  // [M]
  int32_t* spay = cpay + M;                                // [kpad]
  __shared__ int hist[256];
  __shared__ int s_misc[4];
  const int64_t q = blockIdx.x;
  load_candidates(comp, len, nlists, nq, k, q, cand, cpay, bank_lens, head, gcap, slot_offset);
  block_select_topk(cand, cpay, M, nlists, k, kpad, sel, spay, hist, s_misc);
  if (!len) resolve_lens(sel, spay, k, bank_lens, head, gcap, slot_offset);
  int64_t row = q;
  if (po.world > 0) {
    // fused exchange: query q belongs to rank q / nq_local; its merged row is
    // stored straight into that rank's receive buffer (NVLink P2P stores
    // through the IPC-mapped pointer), at [this rank][q % nq_local]
    const int owner = (int)(q / po.nq_local);
    row = (int64_t)po.rank * po.nq_local + (q - (int64_t)owner * po.nq_local);
    out_comp = po.comp[owner];
    out_len = po.len[owner];
  }
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    out_comp[row * k + i] = sel[i];
    out_len[row * k + i] = sel[i] ? spay[i] : 0;
  }
  if (po.world > 0) __threadfence_system();  // peer stores visible before the barrier
}

static size_t merge_smem(int nlists, int k, int kpad) {
  return (size_t)nlists * k * 12 + (size_t)kpad * 12;
}

// ---------------------------------------------------------------------------
// warp-per-query merge (the shard / slice merge for nlists * k <= MW_MAX_M):
// the same result as k_merge -- the top-k composites sorted descending,
// 0-padded, each with its payload (carried length, or the bank length looked
// up for the winners) -- without block barriers.  A block per query spends
// most of its time in __syncthreads at the c4 owner's 8 x 64 candidates per
// query; a warp per query keeps 8192 queries in one short wave.
//   1. candidates + payloads -> per-warp smem; tau = max over full lists of
//      their minimum (the k-th best is >= it, any list order); survivors
//      (>= tau) compacted in place with ballots
//   2. k-th largest: MSB-first 8-bit radix select on the high 32 bits (the
//      key), bitwise on the low 32 bits only if the key is tied at the boundary
//   3. winners ranked by counting (composites are unique) -> output slots
// ---------------------------------------------------------------------------
__device__ __forceinline__ int warp_sum_i32(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int MW_WARPS = 4;
constexpr int MW_MAX_M = 2048;  // 24 KB of candidates per warp

__global__ void __launch_bounds__(MW_WARPS * 32)
k_merge_w(const uint64_t* __restrict__ comp, const int32_t* __restrict__ len, int nlists,
          int64_t nq, int k, uint64_t* __restrict__ out_comp, int32_t* __restrict__ out_len,
          const int32_t* __restrict__ bank_lens, int64_t head, int64_t gcap, int64_t slot_offset,
          PeerOut po, size_t warp_bytes) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t q = (int64_t)blockIdx.x * MW_WARPS + warp;
  pdl_wait();  // the producing kernel's lists
  if (q >= nq) return;  // warp-uniform; no block barriers below
  const int M = nlists * k;
  uint64_t* cand = reinterpret_cast<uint64_t*>(smem + warp * warp_bytes);  // [M]
  int32_t* cpay = reinterpret_cast<int32_t*>(cand + M);                    // [M]
  __shared__ int whist_all[MW_WARPS][256];
  int* whist = whist_all[warp];
  const unsigned lt = (1u << lane) - 1u;

  // 1. load (lists are [nlists][nq][k]); per list its minimum and whether it
  // is full (k non-zero entries) -> tau
  uint64_t tau = 1ull;
  for (int l = 0; l < nlists; ++l) {
    const int64_t src = ((int64_t)l * nq + q) * k;
    uint64_t mn = ~0ull;
    for (int j = lane; j < k; j += 32) {
      const uint64_t c = __ldcs(comp + src + j);
      cand[l * k + j] = c;
      if (len) cpay[l * k + j] = __ldcs(len + src + j);
      mn = min(mn, c);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if (mn != 0ull) tau = max(tau, mn);  // no zero entry: the list is full
  }
  __syncwarp();
  int m1 = 0;
  for (int i0 = 0; i0 < M; i0 += 32) {
    const int i = i0 + lane;
    const uint64_t c = (i < M) ? cand[i] : 0ull;
    const int32_t p = (i < M && len) ? cpay[i] : 0;
    const bool keep = c != 0ull && c >= tau;
    const unsigned b = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    if (keep) {
      cand[m1 + __popc(b & lt)] = c;
      cpay[m1 + __popc(b & lt)] = p;
    }
    m1 += __popc(b);
    __syncwarp();
  }
  // 2. k-th largest: T with |{c >= T}| = min(k, m1)
  uint64_t T = 1ull;
  if (m1 > k) {
    uint32_t th = 0, hmask = 0;
    int need_hi = k;
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int d = lane; d < 256; d += 32) whist[d] = 0;
      __syncwarp();
      for (int i = lane; i < m1; i += 32) {
        const uint32_t h = (uint32_t)(cand[i] >> 32);
        if ((h & hmask) == th) atomicAdd(&whist[(h >> shift) & 255u], 1);
      }
      __syncwarp();
      int local = 0;  // lane owns digits 255-8*lane .. 248-8*lane (descending)
#pragma unroll
      for (int t = 0; t < 8; ++t) local += whist[255 - 8 * lane - t];
      const int incl = warp_incl_scan_i32(local, lane);
      const int excl = incl - local;
      int dsel = -1, nsel = 0;
      if (excl < need_hi && incl >= need_hi) {
        int cum = excl;
        for (int t = 0; t < 8; ++t) {
          const int d = 255 - 8 * lane - t;
          if (cum + whist[d] >= need_hi) { dsel = d; nsel = need_hi - cum; break; }
          cum += whist[d];
        }
      }
      const unsigned who = __ballot_sync(0xffffffffu, dsel >= 0);
      const int src = __ffs(who) - 1;
      dsel = __shfl_sync(0xffffffffu, dsel, src);
      need_hi = __shfl_sync(0xffffffffu, nsel, src);
      th |= (uint32_t)dsel << shift;
      hmask |= 255u << shift;
      __syncwarp();
    }
    int gt = 0, eq = 0;
    for (int i = lane; i < m1; i += 32) {
      const uint32_t h = (uint32_t)(cand[i] >> 32);
      gt += (h > th);
      eq += (h == th);
    }
    gt = warp_sum_i32(gt);
    eq = warp_sum_i32(eq);
    const int need = k - gt;
    uint32_t tl = 0;
    if (eq > need) {  // key tie at the boundary: resolve on rel (insertion order)
      for (int bit = 31; bit >= 0; --bit) {
        const uint32_t t = tl | (1u << bit);
        int cnt = 0;
        for (int i = lane; i < m1; i += 32)
          cnt += ((uint32_t)(cand[i] >> 32) == th) && ((uint32_t)cand[i] >= t);
        if (warp_sum_i32(cnt) >= need) tl = t;
      }
    }
    T = ((uint64_t)th << 32) | tl;
  }
  // winners to the front (unordered), then each one's rank by counting
  int m = 0;
  for (int i0 = 0; i0 < m1; i0 += 32) {
    const int i = i0 + lane;
    const uint64_t c = (i < m1) ? cand[i] : 0ull;
    const int32_t p = (i < m1) ? cpay[i] : 0;
    const bool w = c >= T;
    const unsigned b = __ballot_sync(0xffffffffu, w && i < m1);
    __syncwarp();
    if (w && i < m1) {
      cand[m + __popc(b & lt)] = c;
      cpay[m + __popc(b & lt)] = p;
    }
    m += __popc(b);
    __syncwarp();
  }
  int64_t row = q;
  if (po.world > 0) {  // fused exchange (see k_merge)
    const int owner = (int)(q / po.nq_local);
    row = (int64_t)po.rank * po.nq_local + (q - (int64_t)owner * po.nq_local);
    out_comp = po.comp[owner];
    out_len = po.len[owner];
  }
  // 3. rank r of each winner = #winners above it; slot r of the output row
  for (int i = lane; i < m; i += 32) {
    const uint64_t c = cand[i];
    int r = 0;
    for (int j = 0; j < m; ++j) r += (cand[j] > c);
    int32_t L = cpay[i];
    if (!len) {
      int64_t g = (int64_t)comp_rel(c) + head % gcap;
      if (g >= gcap) g -= gcap;
      L = bank_lens[g - slot_offset];
    }
    out_comp[row * k + r] = c;
    out_len[row * k + r] = L;
  }
  for (int i = m + lane; i < k; i += 32) {
    out_comp[row * k + i] = 0ull;
    out_len[row * k + i] = 0;
  }
  if (po.world > 0) __threadfence_system();  // peer stores visible before the barrier
}

int launch_merge(const uint64_t* comp, const int32_t* len, int nlists, int64_t nq, int k,
                 uint64_t* out_comp, int32_t* out_len, const int32_t* bank_lens, int64_t head,
                 int64_t gcap, int64_t slot_offset, cudaStream_t st, const PeerOut* po) {
  if (nq <= 0) return SS_OK;
  if ((int64_t)nlists * k <= MW_MAX_M) {
    const size_t wb = ((size_t)nlists * k * 12 + 15) & ~(size_t)15;
    const size_t smem = wb * MW_WARPS;
    SS_CUDA_TRY(ensure_dyn_smem(k_merge_w, smem));
    count_launch();
    SS_CUDA_TRY(pdl_launch(k_merge_w, dim3((unsigned)((nq + MW_WARPS - 1) / MW_WARPS)),
                           dim3(MW_WARPS * 32), smem, st, comp, len, nlists, nq, k, out_comp,
                           out_len, bank_lens, head, gcap, slot_offset, po ? *po : PeerOut{}, wb));
    SS_LAUNCH_CHECK();
    return SS_OK;
  }
  int kpad = 1;
  while (kpad < k) kpad <<= 1;
  size_t smem = merge_smem(nlists, k, kpad);
  if (smem > 220 * 1024)
    return set_error(SS_ERR_UNSUPPORTED, "merge of %d lists x k=%d exceeds shared memory", nlists, k);
  SS_CUDA_TRY(cudaFuncSetAttribute(k_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  count_launch();
  k_merge<<<(unsigned)nq, MF_THREADS, smem, st>>>(comp, len, nlists, nq, k, kpad, out_comp, out_len,
                                                 bank_lens, head, gcap, slot_offset,
                                                 po ? *po : PeerOut{});
  SS_LAUNCH_CHECK();
  return SS_OK;
}

__global__ void k_decode(const uint64_t* __restrict__ comp, int64_t n, int64_t head,
                         int64_t capacity, float* __restrict__ key, int64_t* __restrict__ seq,
                         int64_t* __restrict__ slot) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t c = comp[i];
  if (c == 0ull) {
    if (key) key[i] = __int_as_float(0x7fc00000);
    if (seq) seq[i] = -1;
    if (slot) slot[i] = -1;
    return;
  }
  int64_t rel = comp_rel(c);
  if (key) key[i] = comp_key(c);
  if (seq) seq[i] = head - capacity + rel;
  if (slot) slot[i] = (rel + head) % capacity;
}

int launch_decode(const uint64_t* comp, int64_t n, int64_t head, int64_t capacity, float* key,
                  int64_t* seq, int64_t* slot, cudaStream_t st) {
  if (n <= 0) return SS_OK;
  count_launch();
  k_decode<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(comp, n, head, capacity, key, seq, slot);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

// ---------------------------------------------------------------------------
// exact integer-count Gittins over a sorted sparse law (one warp).
//   D_k = sum v^2 + 2 I sum v over bin k  (so c_k s_k = D_k / 2 exactly)
//   attained 2a = A2 = g^2 + 2 I g; survivors D_k > A2 c_k (a suffix)
//   ratio_k = (0.5 P'_k + s'_k (T' - C'_k)) / C'_k,  s'_k = d_k / (2 c_k),
//           = (P'_k c_k + d_k (T' - C'_k)) / (2 c_k C'_k)   (RatioMin::add)
//   d_k = D_k - A2 c_k, P'_k = sum_{j<=k surv} d_j, C'_k = sum c_j, T' = C'_last
// -- the algebra of _kernels.py:110-115 (cum_xp + s (1 - cum_p)) / cum_p with
// masses c/T'.  Integer sums are exact; the fp64 ops are explicit _rn (no FMA
// contraction) in the order of oracle.gittins_points -> bit-identical.
// ---------------------------------------------------------------------------

// exact n1/d1 < n2/d2 for n >= 0, d >= 0 (d = 0: +inf) by products with
// their FMA rounding errors, (p, e) compared lexicographically: p1 < p2
// implies n1 d2 <= n2 d1 exactly, and ties in the exact values pick either
// side with the same quotient.  Division rounds monotonically, so the
// correctly rounded quotient of the pair this minimum keeps equals the
// minimum of the correctly rounded per-point quotients (the reference's
// min over r_k): one divide per law instead of one per point.
__device__ __forceinline__ bool ratio_less(double n1, double d1, double n2, double d2) {
  const double p1 = __dmul_rn(n1, d2), e1 = __fma_rn(n1, d2, -p1);
  const double p2 = __dmul_rn(n2, d1), e2 = __fma_rn(n2, d1, -p2);
  return p1 < p2 || (p1 == p2 && e1 < e2);
}
struct RatioMin {
  double n = 1.0, d = 0.0;  // +inf
  __device__ __forceinline__ void add(long long P, long long C, long long T, long long ck,
                                      long long dk) {
    const double num = __dadd_rn(__dmul_rn((double)P, (double)ck), __dmul_rn((double)dk, (double)(T - C)));
    const double den = __dmul_rn(2.0 * (double)ck, (double)C);
    if (ratio_less(num, den, n, d)) { n = num; d = den; }
  }
  template <int W>  // lanes per group (a power of two <= 32)
  __device__ __forceinline__ void group_reduce() {
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) {
      const double on = __shfl_xor_sync(0xffffffffu, n, o), od = __shfl_xor_sync(0xffffffffu, d, o);
      if (ratio_less(on, od, n, d)) { n = on; d = od; }
    }
  }
  __device__ __forceinline__ double value() const { return d == 0.0 ? INFINITY : __ddiv_rn(n, d); }
};

__device__ double warp_gittins_exact(const int32_t* c, const int64_t* D, int np, long long A2,
                                     int I, int g, int bucket, int lane) {
  int first = np;
  for (int b = 0; b < np; b += 32) {
    int k = b + lane;
    bool s = (k < np) && (D[k] > A2 * (long long)c[k]);
    unsigned ball = __ballot_sync(0xffffffffu, s);
    if (ball) { first = b + __ffs(ball) - 1; break; }
  }
  if (first >= np) {  // outlived every predicted length
    long long gb = (long long)g + bucket;
    return __dadd_rn(__dmul_rn((double)(gb * gb - (long long)g * g), 0.5),
                     __dmul_rn((double)I, (double)bucket));
  }
  long long T = 0;
  for (int k = first + lane; k < np; k += 32) T += c[k];
  for (int o = 16; o > 0; o >>= 1) T += __shfl_xor_sync(0xffffffffu, T, o);
  long long Cc = 0, Pc = 0;
  RatioMin rm;  // min over points of the exact ratio, one divide at the end
  for (int b = first; b < np; b += 32) {
    int k = b + lane;
    long long ck = 0, dk = 0;
    if (k < np) {
      ck = c[k];
      dk = D[k] - A2 * ck;
    }
    long long C = warp_incl_scan_i64(ck, lane) + Cc;
    long long P = warp_incl_scan_i64(dk, lane) + Pc;
    if (k < np) rm.add(P, C, T, ck, dk);
    Cc = __shfl_sync(0xffffffffu, C, 31);
    Pc = __shfl_sync(0xffffffffu, P, 31);
  }
  rm.group_reduce<32>();
  return rm.value();
}

// ---------------------------------------------------------------------------
// finish for one request (whole CTA): histogram of the <= k sorted neighbours
// (shared-memory atomics) or the fallback, ascending ballot-scan compaction
// into the sparse law, then warp-0 Gittins.
// ---------------------------------------------------------------------------
struct FinishSmem {
  int64_t* h_sv;
  int64_t* h_sv2;
  int64_t* l_D;
  int32_t* h_cnt;
  int32_t* l_c;
};

__device__ FinishSmem carve_finish(unsigned char* p, int nbins) {
  FinishSmem f;
  f.h_sv = reinterpret_cast<int64_t*>(p);
  f.h_sv2 = f.h_sv + nbins;
  f.l_D = f.h_sv2 + nbins;
  f.h_cnt = reinterpret_cast<int32_t*>(f.l_D + nbins);
  f.l_c = f.h_cnt + nbins;
  return f;
}
static size_t finish_smem(int nbins) { return (size_t)nbins * (8 * 3 + 4 * 2); }

__device__ void finish_one(const uint64_t* comp, const int32_t* len, int k, int64_t q,
                           int min_matches, int max_len, int nbins, long long Iq,
                           const int64_t* fb_cnt, const int64_t* fb_sv, const int64_t* fb_sv2,
                           int P, int32_t* npts, int32_t* pbin, int32_t* pcnt, int64_t* pD,
                           int64_t* psv, uint8_t* used_fb, double* G, FinishSmem f, int* s_misc,
                           int* s_warp) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = blockDim.x >> 5;
  const int w = max_len / nbins;
  int m = 0;
  for (int i = tid; i < k; i += blockDim.x) m += (comp[i] != 0ull);
  for (int o = 16; o > 0; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
  if (tid == 0) { s_misc[0] = 0; s_misc[1] = 0; }
  __syncthreads();
  if (lane == 0) atomicAdd(&s_misc[0], m);
  __syncthreads();
  const bool fb = s_misc[0] < min_matches;
  if (!fb) {
    for (int b = tid; b < nbins; b += blockDim.x) { f.h_cnt[b] = 0; f.h_sv[b] = 0; f.h_sv2[b] = 0; }
    __syncthreads();
    for (int i = tid; i < k; i += blockDim.x) {
      if (comp[i] == 0ull) continue;
      int L = min(max(len[i], 1), max_len);
      int b = (L - 1) / w;
      atomicAdd(&f.h_cnt[b], 1);
      atomicAdd(reinterpret_cast<unsigned long long*>(&f.h_sv[b]), (unsigned long long)L);
      atomicAdd(reinterpret_cast<unsigned long long*>(&f.h_sv2[b]),
                (unsigned long long)((long long)L * L));
    }
  } else {
    for (int b = tid; b < nbins; b += blockDim.x) {
      f.h_cnt[b] = (int32_t)fb_cnt[b];
      f.h_sv[b] = fb_sv[b];
      f.h_sv2[b] = fb_sv2[b];
    }
  }
  __syncthreads();
  // ascending compaction of non-empty bins
  for (int b0 = 0; b0 < nbins; b0 += blockDim.x) {
    int b = b0 + tid;
    int c = (b < nbins) ? f.h_cnt[b] : 0;
    unsigned ball = __ballot_sync(0xffffffffu, c > 0);
    if (lane == 0) s_warp[warp] = __popc(ball);
    __syncthreads();
    int off = s_misc[1];
    for (int ww = 0; ww < warp; ++ww) off += s_warp[ww];
    if (c > 0) {
      int pos = off + __popc(ball & ((1u << lane) - 1u));
      long long D = f.h_sv2[b] + 2 * Iq * f.h_sv[b];
      f.l_c[pos] = c;
      f.l_D[pos] = D;
      if (pos < P) {
        pbin[q * P + pos] = b;
        pcnt[q * P + pos] = c;
        pD[q * P + pos] = D;
        if (psv) psv[q * P + pos] = f.h_sv[b];
      }
    }
    __syncthreads();
    if (tid == 0) {
      int add = 0;
      for (int ww = 0; ww < nw; ++ww) add += s_warp[ww];
      s_misc[1] += add;
    }
    __syncthreads();
  }
  const int np = s_misc[1];
  if (warp == 0) {
    double g = (np > 0) ? warp_gittins_exact(f.l_c, f.l_D, np, 0, (int)Iq, 0, 0, lane) : INFINITY;
    if (lane == 0) {
      G[q] = g;
      npts[q] = np;
      if (used_fb) used_fb[q] = fb ? 1 : 0;
    }
  }
}

__global__ void __launch_bounds__(MF_THREADS)
k_finish(const uint64_t* __restrict__ comp, const int32_t* __restrict__ len, int64_t nq, int k,
         int min_matches, int max_len, int nbins, const int32_t* __restrict__ I,
         const int64_t* __restrict__ fb_cnt, const int64_t* __restrict__ fb_sv,
         const int64_t* __restrict__ fb_sv2, int P, int32_t* __restrict__ npts,
         int32_t* __restrict__ pbin, int32_t* __restrict__ pcnt, int64_t* __restrict__ pD,
         int64_t* __restrict__ psv, uint8_t* __restrict__ used_fb, double* __restrict__ G) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_misc[4], s_warp[MF_THREADS / 32];
  const int64_t q = blockIdx.x;
  finish_one(comp + q * k, len + q * k, k, q, min_matches, max_len, nbins, I[q], fb_cnt, fb_sv,
             fb_sv2, P, npts, pbin, pcnt, pD, psv, used_fb, G, carve_finish(smem, nbins), s_misc,
             s_warp);
}


// ---------------------------------------------------------------------------
// merge + finish fused (single-GPU round): per request, select the global
// top-k from the similarity kernel's slices, then histogram/cost/Gittins,
// without a global round trip of the neighbour lists in between.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(MF_THREADS)
k_merge_finish(const uint64_t* __restrict__ partials, int nlists, int64_t nq, int k, int kpad,
               const int32_t* __restrict__ bank_lens, int64_t head, int64_t gcap,
               int64_t slot_offset, uint64_t* __restrict__ out_comp,
               int32_t* __restrict__ out_len, int min_matches, int max_len, int nbins,
               const int32_t* __restrict__ I, const int64_t* __restrict__ fb_cnt,
               const int64_t* __restrict__ fb_sv, const int64_t* __restrict__ fb_sv2, int P,
               int32_t* __restrict__ npts, int32_t* __restrict__ pbin, int32_t* __restrict__ pcnt,
               int64_t* __restrict__ pD, int64_t* __restrict__ psv, uint8_t* __restrict__ used_fb,
               double* __restrict__ G) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int M = nlists * k;
  uint64_t* cand = reinterpret_cast<uint64_t*>(smem);      // [M]
  uint64_t* sel = cand + M;                                // [kpad]
  int32_t* cpay = reinterpret_cast<int32_t*>(sel + kpad);  // [M]
  int32_t* spay = cpay + M;                                // [kpad]
  __shared__ int hist[256];
  __shared__ int s_misc[4], s_warp[MF_THREADS / 32];
  const int64_t q = blockIdx.x;
  load_candidates(partials, nullptr, nlists, nq, k, q, cand, cpay, bank_lens, head, gcap,
                  slot_offset);
  block_select_set(cand, cpay, M, nlists, k, kpad, sel, spay, hist, s_misc);  // unordered set
  resolve_lens(sel, spay, k, bank_lens, head, gcap, slot_offset);
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    if (out_comp) out_comp[q * k + i] = sel[i];
    if (out_len) out_len[q * k + i] = sel[i] ? spay[i] : 0;
  }
  finish_one(sel, spay, k, q, min_matches, max_len, nbins, I[q], fb_cnt, fb_sv, fb_sv2, P, npts,
             pbin, pcnt, pD, psv, used_fb, G,
             carve_finish(smem + (((size_t)M * 12 + (size_t)kpad * 12 + 15) & ~(size_t)15), nbins),
             s_misc, s_warp);
}

// ---------------------------------------------------------------------------
// warp-per-request merge + finish (the single-GPU round's default): no block
// barriers, all 32-wide ballots / shuffles, one request per warp, so 1024
// requests are one wave of short warps.
//   1. candidates of all slices -> per-warp smem; tau = max over full lists of
//      their minimum (the global k-th is >= it); survivors compacted in place
//   2. k-th largest composite: bitwise search on the high 32 bits (the key),
//      then on the low 32 bits (rel) only if the key itself is tied
//   3. winners' lengths, histogram (smem atomics) or fallback, ascending
//      ballot compaction of the bins, exact integer Gittins (warp scan)
// ---------------------------------------------------------------------------
constexpr int MFW_WARPS = 4;

// histogram of the m winners' lengths (or the fallback law) -> ascending
// compaction of the non-empty bins into the sparse cost law -> exact Gittins;
// one warp per request (shared by the fused merge+finish and k_finish_w)
__device__ __forceinline__ void warp_finish_tail(
    const int32_t* slen, int m, int64_t q, int k, int min_matches, int max_len, int nbins,
    long long Iq_in, const int64_t* __restrict__ fb_cnt, const int64_t* __restrict__ fb_sv,
    const int64_t* __restrict__ fb_sv2, int P, int32_t* __restrict__ npts,
    int32_t* __restrict__ pbin, int32_t* __restrict__ pcnt, int64_t* __restrict__ pD,
    int64_t* __restrict__ psv, uint8_t* __restrict__ used_fb, double* __restrict__ G,
    FinishSmem f, int lane, double* __restrict__ G2 = nullptr) {
  const unsigned lt = (1u << lane) - 1u;
  // 3b. histogram of the winners (or the fallback law)
  const long long Iq = Iq_in;
  const int w = max_len / nbins;
  const bool fb = m < min_matches;
  // <= k winners of length <= max_len: when k * max_len^2 < 2^32 the sums fit
  // 32-bit shared-memory atomics (native adds instead of 64-bit CAS loops);
  // they live in the first half of the 64-bit arrays' storage
  const bool s32 = !fb && (long long)k * max_len * max_len < (1LL << 32);
  uint32_t* sv32 = reinterpret_cast<uint32_t*>(f.h_sv);
  uint32_t* sv2_32 = reinterpret_cast<uint32_t*>(f.h_sv2);
  if (s32) {
    for (int b = lane; b < nbins; b += 32) { f.h_cnt[b] = 0; sv32[b] = 0u; sv2_32[b] = 0u; }
    __syncwarp();
    for (int i = lane; i < m; i += 32) {
      const int L = min(max(slen[i], 1), max_len);
      const int b = (L - 1) / w;
      atomicAdd(&f.h_cnt[b], 1);
      atomicAdd(&sv32[b], (uint32_t)L);
      atomicAdd(&sv2_32[b], (uint32_t)(L * L));
    }
  } else if (!fb) {
    for (int b = lane; b < nbins; b += 32) { f.h_cnt[b] = 0; f.h_sv[b] = 0; f.h_sv2[b] = 0; }
    __syncwarp();
    for (int i = lane; i < m; i += 32) {
      const int L = min(max(slen[i], 1), max_len);
      const int b = (L - 1) / w;
      atomicAdd(&f.h_cnt[b], 1);
      atomicAdd(reinterpret_cast<unsigned long long*>(&f.h_sv[b]), (unsigned long long)L);
      atomicAdd(reinterpret_cast<unsigned long long*>(&f.h_sv2[b]),
                (unsigned long long)((long long)L * L));
    }
  } else {
    for (int b = lane; b < nbins; b += 32) {
      f.h_cnt[b] = (int32_t)fb_cnt[b];
      f.h_sv[b] = fb_sv[b];
      f.h_sv2[b] = fb_sv2[b];
    }
  }
  __syncwarp();
  int np = 0;
  for (int b0 = 0; b0 < nbins; b0 += 32) {
    const int b = b0 + lane;
    const int c = (b < nbins) ? f.h_cnt[b] : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, c > 0);
    if (c > 0) {
      const int pos = np + __popc(bal & lt);
      const long long sv = s32 ? (long long)sv32[b] : f.h_sv[b];
      const long long sv2 = s32 ? (long long)sv2_32[b] : f.h_sv2[b];
      const long long D = sv2 + 2 * Iq * sv;
      f.l_c[pos] = c;
      f.l_D[pos] = D;
      if (pos < P) {
        pbin[q * P + pos] = b;
        pcnt[q * P + pos] = c;
        pD[q * P + pos] = D;
        if (psv) psv[q * P + pos] = sv;
      }
    }
    np += __popc(bal);
  }
  __syncwarp();
  const double g = (np > 0) ? warp_gittins_exact(f.l_c, f.l_D, np, 0, (int)Iq, 0, 0, lane) : INFINITY;
  if (lane == 0) {
    G[q] = g;
    if (G2) G2[q] = g;  // mirror (e.g. pinned host memory of the plugin call)
    npts[q] = np;
    if (used_fb) used_fb[q] = fb ? 1 : 0;
  }
}




__global__ void __launch_bounds__(MFW_WARPS * 32)
k_merge_finish_w(const uint64_t* __restrict__ partials, int nlists, int64_t nq, int k,
                 const int32_t* __restrict__ bank_lens, int64_t head, int64_t gcap,
                 int64_t slot_offset, uint64_t* __restrict__ out_comp, int32_t* __restrict__ out_len,
                 int min_matches, int max_len, int nbins, const int32_t* __restrict__ I,
                 const int64_t* __restrict__ fb_cnt, const int64_t* __restrict__ fb_sv,
                 const int64_t* __restrict__ fb_sv2, int P, int32_t* __restrict__ npts,
                 int32_t* __restrict__ pbin, int32_t* __restrict__ pcnt, int64_t* __restrict__ pD,
                 int64_t* __restrict__ psv, uint8_t* __restrict__ used_fb, double* __restrict__ G,
                 size_t warp_bytes, double* __restrict__ G2) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t q = (int64_t)blockIdx.x * MFW_WARPS + warp;
  pdl_wait();  // the similarity kernel's partial lists
  if (q >= nq) return;  // warp-uniform; no block barriers below
  const int M = nlists * k;
  unsigned char* base = smem + warp * warp_bytes;
  uint64_t* cand = reinterpret_cast<uint64_t*>(base);       // [M]
  uint64_t* sel = cand + M;                                 // [k]
  int32_t* slen = reinterpret_cast<int32_t*>(sel + k);      // [k]
  FinishSmem f = carve_finish(reinterpret_cast<unsigned char*>(slen + ((k + 3) & ~3)), nbins);
  __shared__ int whist_all[MFW_WARPS][256];
  int* whist = whist_all[warp];
  const unsigned lt = (1u << lane) - 1u;

  // 1. load every slice's list, dropping the zero padding on the fly (a list
  // holds its candidates first, then zeros).  A full list (k candidates) is
  // a min-heap with its minimum at entry 0 (every producer writes its heap
  // array as is), so tau = max over full lists of entry 0 is a lower bound
  // of the global k-th best; candidates below it are dropped afterwards.
  int m1 = 0;
  uint64_t tau = 1ull;
  if ((k & 31) == 0) {  // k multiple of 32: LB lists' loads in flight per batch
    constexpr int LB = 24;
    const int per = k >> 5;
    const uint64_t* src0 = partials + q * k + lane;
    const int64_t lstride = nq * (int64_t)k;
    for (int l0 = 0; l0 < nlists; l0 += LB) {
      const int nl = min(LB, nlists - l0);
      uint64_t root[LB];  // entry 0 of each list of the batch
      for (int jj = 0; jj < per; ++jj) {
        uint64_t v[LB];
#pragma unroll
        for (int u = 0; u < LB; ++u) v[u] = (u < nl) ? __ldcs(src0 + (l0 + u) * lstride + jj * 32) : 0ull;
#pragma unroll
        for (int u = 0; u < LB; ++u) {
          const unsigned b = __ballot_sync(0xffffffffu, v[u] != 0ull);
          if (v[u] != 0ull) cand[m1 + __popc(b & lt)] = v[u];
          m1 += __popc(b);
          if (jj == 0) root[u] = __shfl_sync(0xffffffffu, v[u], 0);
          // entry k-1 present: the list is full, its root bounds the k-th best
          if (jj == per - 1 && (b >> 31) && u < nl) tau = max(tau, root[u]);
        }
        __syncwarp();
      }
    }
  } else {
    int l = 0, j = lane;
    while (j >= k) { j -= k; ++l; }
    for (int i = lane; i < M; i += 32) {
      cand[i] = __ldcs(partials + ((int64_t)l * nq + q) * k + j);
      j += 32;
      while (j >= k) { j -= k; ++l; }
    }
    __syncwarp();
    for (int l2 = 0; l2 < nlists; ++l2) {
      uint64_t mn = ~0ull;
      for (int jx = lane; jx < k; jx += 32) mn = min(mn, cand[l2 * k + jx]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      if (mn != 0ull) tau = max(tau, mn);
    }
    for (int i0 = 0; i0 < M; i0 += 32) {
      const int i = i0 + lane;
      const uint64_t c = (i < M) ? cand[i] : 0ull;
      const bool keep = c != 0ull;
      const unsigned b = __ballot_sync(0xffffffffu, keep);
      __syncwarp();
      if (keep) cand[m1 + __popc(b & lt)] = c;
      m1 += __popc(b);
      __syncwarp();
    }
  }
  __syncwarp();
  if (tau > 1ull) {  // drop candidates below the proven bound (in place, order kept)
    int m2 = 0;
    for (int i0 = 0; i0 < m1; i0 += 32) {
      const int i = i0 + lane;
      const uint64_t c = (i < m1) ? cand[i] : 0ull;
      const bool keep = c >= tau;
      const unsigned b = __ballot_sync(0xffffffffu, keep);
      __syncwarp();
      if (keep) cand[m2 + __popc(b & lt)] = c;
      m2 += __popc(b);
      __syncwarp();
    }
    m1 = m2;
  }
  // 2. k-th largest (unique composites): T such that |{c >= T}| = min(k, m1)
  uint64_t T = 1ull;
  if (m1 > k) {
    // k-th largest high word by an MSB-first 8-bit radix select (4 passes)
    uint32_t th = 0, hmask = 0;
    int need_hi = k;
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int d = lane; d < 256; d += 32) whist[d] = 0;
      __syncwarp();
      for (int i = lane; i < m1; i += 32) {
        const uint32_t h = (uint32_t)(cand[i] >> 32);
        if ((h & hmask) == th) atomicAdd(&whist[(h >> shift) & 255u], 1);
      }
      __syncwarp();
      int local = 0;  // lane owns digits 255-8*lane .. 248-8*lane (descending)
#pragma unroll
      for (int t = 0; t < 8; ++t) local += whist[255 - 8 * lane - t];
      const int incl = warp_incl_scan_i32(local, lane);
      const int excl = incl - local;
      int dsel = -1, nsel = 0;
      if (excl < need_hi && incl >= need_hi) {
        int cum = excl;
        for (int t = 0; t < 8; ++t) {
          const int d = 255 - 8 * lane - t;
          if (cum + whist[d] >= need_hi) { dsel = d; nsel = need_hi - cum; break; }
          cum += whist[d];
        }
      }
      const unsigned who = __ballot_sync(0xffffffffu, dsel >= 0);
      const int src = __ffs(who) - 1;
      dsel = __shfl_sync(0xffffffffu, dsel, src);
      need_hi = __shfl_sync(0xffffffffu, nsel, src);
      th |= (uint32_t)dsel << shift;
      hmask |= 255u << shift;
      __syncwarp();
    }
    int gt = 0, eq = 0;
    for (int i = lane; i < m1; i += 32) {
      const uint32_t h = (uint32_t)(cand[i] >> 32);
      gt += (h > th);
      eq += (h == th);
    }
    gt = warp_sum_i32(gt);
    eq = warp_sum_i32(eq);
    const int need = k - gt;
    uint32_t tl = 0;
    if (eq > need) {  // key tie at the boundary: resolve on rel (insertion order)
      for (int bit = 31; bit >= 0; --bit) {
        const uint32_t t = tl | (1u << bit);
        int cnt = 0;
        for (int i = lane; i < m1; i += 32)
          cnt += ((uint32_t)(cand[i] >> 32) == th) && ((uint32_t)cand[i] >= t);
        if (warp_sum_i32(cnt) >= need) tl = t;
      }
    }
    T = ((uint64_t)th << 32) | tl;
  }
  // 3a. winners (unordered) and their lengths
  int m = 0;
  for (int i0 = 0; i0 < m1; i0 += 32) {
    const int i = i0 + lane;
    const uint64_t c = (i < m1) ? cand[i] : 0ull;
    const bool w = (c != 0ull) && c >= T;
    const unsigned b = __ballot_sync(0xffffffffu, w);
    if (w) {
      const int p = m + __popc(b & lt);
      sel[p] = c;
      int64_t g = (int64_t)comp_rel(c) + head % gcap;
      if (g >= gcap) g -= gcap;
      slen[p] = bank_lens[g - slot_offset];
    }
    m += __popc(b);
  }
  __syncwarp();
  for (int i = lane; i < k; i += 32) {
    if (out_comp) out_comp[q * k + i] = (i < m) ? sel[i] : 0ull;
    if (out_len) out_len[q * k + i] = (i < m) ? slen[i] : 0;
  }
  warp_finish_tail(slen, m, q, k, min_matches, max_len, nbins, I[q], fb_cnt, fb_sv, fb_sv2, P, npts,
                   pbin, pcnt, pD, psv, used_fb, G, f, lane, G2);
}

// finish for neighbour lists already merged (ss_finish: the predictor API and
// the multi-GPU round): one warp per request; the list's non-zero
// composites and their lengths are compacted into per-warp smem, then the
// shared tail (histogram -> cost law -> Gittins)
__global__ void __launch_bounds__(MFW_WARPS * 32)
k_finish_w(const uint64_t* __restrict__ comp, const int32_t* __restrict__ len, int64_t nq, int k,
           int min_matches, int max_len, int nbins, const int32_t* __restrict__ I,
           const int64_t* __restrict__ fb_cnt, const int64_t* __restrict__ fb_sv,
           const int64_t* __restrict__ fb_sv2, int P, int32_t* __restrict__ npts,
           int32_t* __restrict__ pbin, int32_t* __restrict__ pcnt, int64_t* __restrict__ pD,
           int64_t* __restrict__ psv, uint8_t* __restrict__ used_fb, double* __restrict__ G,
           size_t warp_bytes) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t q = (int64_t)blockIdx.x * MFW_WARPS + warp;
  pdl_wait();
  if (q >= nq) return;  // warp-uniform
  unsigned char* base = smem + warp * warp_bytes;
  int32_t* slen = reinterpret_cast<int32_t*>(base);  // [k]
  FinishSmem f = carve_finish(base + (((size_t)k * 4 + 15) & ~(size_t)15), nbins);
  const unsigned lt = (1u << lane) - 1u;
  int m = 0;
  for (int i0 = 0; i0 < k; i0 += 32) {
    const int i = i0 + lane;
    const bool nz = i < k && comp[q * k + i] != 0ull;
    const unsigned b = __ballot_sync(0xffffffffu, nz);
    if (nz) slen[m + __popc(b & lt)] = len[q * k + i];
    m += __popc(b);
  }
  __syncwarp();
  warp_finish_tail(slen, m, q, k, min_matches, max_len, nbins, I[q], fb_cnt, fb_sv, fb_sv2, P, npts,
                   pbin, pcnt, pD, psv, used_fb, G, f, lane);
}

int launch_finish(const uint64_t* comp, const int32_t* len, int64_t nq, int k, int min_matches,
                  int max_len, int nbins, const int32_t* I, const int64_t* fb_cnt,
                  const int64_t* fb_sv, const int64_t* fb_sv2, int P, int32_t* npts,
                  int32_t* pbin, int32_t* pcnt, int64_t* pD, int64_t* psv, uint8_t* used_fb,
                  double* G, cudaStream_t st) {
  if (nq <= 0) return SS_OK;
  {
    const size_t wb = (((size_t)k * 4 + 15) & ~(size_t)15) + ((finish_smem(nbins) + 15) & ~(size_t)15);
    const size_t smem = wb * MFW_WARPS;
    if (smem <= 200 * 1024) {
      SS_CUDA_TRY(ensure_dyn_smem(k_finish_w, smem));
      count_launch();
      SS_CUDA_TRY(pdl_launch(k_finish_w, dim3((unsigned)((nq + MFW_WARPS - 1) / MFW_WARPS)),
                             dim3(MFW_WARPS * 32), smem, st, comp, len, nq, k, min_matches, max_len,
                             nbins, I, fb_cnt, fb_sv, fb_sv2, P, npts, pbin, pcnt, pD, psv, used_fb,
                             G, wb));
      return SS_OK;
    }
  }
  size_t smem = finish_smem(nbins);
  if (smem > 200 * 1024) return set_error(SS_ERR_UNSUPPORTED, "nbins %d too large", nbins);
  SS_CUDA_TRY(ensure_dyn_smem(k_finish, smem));
  count_launch();
  k_finish<<<(unsigned)nq, MF_THREADS, smem, st>>>(comp, len, nq, k, min_matches, max_len, nbins, I,
                                                  fb_cnt, fb_sv, fb_sv2, P, npts, pbin, pcnt, pD,
                                                  psv, used_fb, G);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

int launch_merge_finish(const uint64_t* partials, int nlists, int64_t nq, int k,
                        const int32_t* bank_lens, int64_t head, int64_t gcap, int64_t slot_offset,
                        uint64_t* out_comp, int32_t* out_len, int min_matches, int max_len,
                        int nbins, const int32_t* I, const int64_t* fb_cnt, const int64_t* fb_sv,
                        const int64_t* fb_sv2, int P, int32_t* npts, int32_t* pbin, int32_t* pcnt,
                        int64_t* pD, int64_t* psv, uint8_t* used_fb, double* G, cudaStream_t st,
                        double* G_mirror) {
  if (nq <= 0) return SS_OK;
  {
    const size_t wb = (((size_t)nlists * k * 8 + (size_t)k * 8 + (size_t)((k + 3) & ~3) * 4 + 15) &
                       ~(size_t)15) + ((finish_smem(nbins) + 15) & ~(size_t)15);
    const size_t smem = wb * MFW_WARPS;
    if (smem <= 200 * 1024) {
      SS_CUDA_TRY(ensure_dyn_smem(k_merge_finish_w, smem));
      count_launch();
      SS_CUDA_TRY(pdl_launch(k_merge_finish_w, dim3((unsigned)((nq + MFW_WARPS - 1) / MFW_WARPS)),
                             dim3(MFW_WARPS * 32), smem, st, partials, nlists, nq, k, bank_lens, head,
                             gcap, slot_offset, out_comp, out_len, min_matches, max_len, nbins, I,
                             fb_cnt, fb_sv, fb_sv2, P, npts, pbin, pcnt, pD, psv, used_fb, G, wb,
                             G_mirror));
      SS_LAUNCH_CHECK();
      return SS_OK;
    }
  }
  int kpad = 1;
  while (kpad < k) kpad <<= 1;
  const size_t smem = ((merge_smem(nlists, k, kpad) + 15) & ~(size_t)15) + finish_smem(nbins);
  if (smem > 220 * 1024)
    return set_error(SS_ERR_UNSUPPORTED, "merge+finish of %d lists x k=%d, %d bins exceeds smem",
                     nlists, k, nbins);
  SS_CUDA_TRY(cudaFuncSetAttribute(k_merge_finish, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
  count_launch();
  k_merge_finish<<<(unsigned)nq, MF_THREADS, smem, st>>>(
      partials, nlists, nq, k, kpad, bank_lens, head, gcap, slot_offset, out_comp, out_len,
      min_matches, max_len, nbins, I, fb_cnt, fb_sv, fb_sv2, P, npts, pbin, pcnt, pD, psv, used_fb, G);
  SS_LAUNCH_CHECK();
  if (G_mirror) SS_CUDA_TRY(cudaMemcpyAsync(G_mirror, G, (size_t)nq * 8, cudaMemcpyDefault, st));
  return SS_OK;
}

// ---------------------------------------------------------------------------
// refresh (SPEC.md:345-353 cadence): RF_GL = 8 lanes per request, four
// requests per warp, so the prefix scans are 3 shuffle steps and a ~50-point
// law fills the lanes; one read of the law (its first 64 points stay in
// registers for the second pass), one divide per law (RatioMin).  Same
// arithmetic, in the same order, as warp_gittins_exact / oracle gittins_points:
//   survivors  D_k > A2 c_k (a suffix: bin means increase with the bin)
//   T = sum of surviving c;  C_k, P_k inclusive prefix sums over survivors
//   r_k = (P_k c_k + d_k (T - C_k)) / (2 c_k C_k),  d_k = D_k - A2 c_k,  G = min r_k
//   no survivor -> cost(I, g + bucket) - cost(I, g)
// Loops run to the warp's largest law, masked per group, so every shuffle
// is warp-converged.
// ---------------------------------------------------------------------------
constexpr int RF_GL = 8;
// chunks of RF_GL points kept between the two passes (64 points: a c3 law
// has ~52), 5 blocks per SM (48 registers).  c3 k_refresh on B200
// (profiles/ROUND2.md, r2v-r2zf): 71.5 us with a per-point divide and a
// shuffle-reduced chunk bound; 66.7 us with the cross-multiplied minimum;
// 63.7 us with the bound from redux.sync (a value the compiler knows is
// warp-uniform: the chunk guards become uniform branches, no divergence
// fallbacks around the shuffles, fewer spills) at 5 blocks per SM (6: 64.3,
// 4: 65.6 us); fewer kept chunks measured slower (70-84 us)
#ifndef SS_RF_R
#define SS_RF_R 8
#endif
#ifndef SS_RF_MINB
#define SS_RF_MINB 5
#endif
constexpr int RF_R = SS_RF_R;
constexpr int RF_MINB = SS_RF_MINB;

__device__ __forceinline__ long long grp_incl_scan_i64(long long v, int gl) {
#pragma unroll
  for (int o = 1; o < RF_GL; o <<= 1) {
    const long long t = __shfl_up_sync(0xffffffffu, v, o, RF_GL);
    if (gl >= o) v += t;
  }
  return v;
}
__device__ __forceinline__ int grp_incl_scan_i32(int v, int gl) {
#pragma unroll
  for (int o = 1; o < RF_GL; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o, RF_GL);
    if (gl >= o) v += t;
  }
  return v;
}
__device__ __forceinline__ long long grp_sum_i64(long long v) {
#pragma unroll
  for (int o = RF_GL / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(256, RF_MINB)
k_refresh(int64_t n, const int32_t* __restrict__ I, const int32_t* __restrict__ g_new,
          int32_t* __restrict__ bucket_io, int bucket_size, const int32_t* __restrict__ npts,
          const int32_t* __restrict__ pcnt, const int64_t* __restrict__ pD, int P,
          double* __restrict__ G_io, uint8_t* __restrict__ refreshed, int force) {
  const int lane = threadIdx.x & 31, gl = lane & (RF_GL - 1);
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / RF_GL;
  const bool live = i < n;
  const int g = live ? g_new[i] : 0;
  const int nb = g / bucket_size;
  const bool due = live && (force || nb > bucket_io[i]);
  const int np = due ? npts[i] : 0;
  // warp-wide maximum by redux.sync: a value the compiler knows is uniform,
  // so the chunk guards below are uniform branches
  const int npmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)np);
  const long long Ii = live ? I[i] : 0;
  const long long A2 = (long long)g * g + 2 * Ii * g;
  const int32_t* c = pcnt + (live ? i : 0) * (int64_t)P;
  const int64_t* D = pD + (live ? i : 0) * (int64_t)P;
  // pass 1: the surviving (c_k, d_k = D_k - A2 c_k) -- the first RF_R chunks
  // kept in registers -- and their total count T (one read of the law)
  int cr[RF_R];
  long long dr[RF_R];
  long long T = 0;
#pragma unroll
  for (int j = 0; j < RF_R; ++j) {
    const int k = j * RF_GL + gl;
    int ck = 0;
    long long dk = 0;
    if (k < np) {
      const int cv = c[k];
      const long long dv = D[k] - A2 * cv;
      if (dv > 0) { ck = cv; dk = dv; }
    }
    cr[j] = ck;
    dr[j] = dk;
    T += ck;
  }
  for (int b = RF_R * RF_GL; b < npmax; b += RF_GL) {  // long laws: the rest is re-read below
    const int k = b + gl;
    if (k < np) {
      const int cv = c[k];
      if (D[k] > A2 * cv) T += cv;
    }
  }
  T = grp_sum_i64(T);
  // pass 2: prefix sums and the ratio at every surviving point
  long long Cc = 0, Pc = 0;
  RatioMin rm;
#pragma unroll
  for (int j = 0; j < RF_R; ++j) {
    if (j * RF_GL < npmax) {  // warp-uniform
      const long long C = grp_incl_scan_i32(cr[j], gl) + Cc;
      const long long Pp = grp_incl_scan_i64(dr[j], gl) + Pc;
      if (cr[j] > 0) rm.add(Pp, C, T, cr[j], dr[j]);
      Cc = __shfl_sync(0xffffffffu, C, RF_GL - 1, RF_GL);
      Pc = __shfl_sync(0xffffffffu, Pp, RF_GL - 1, RF_GL);
    }
  }
  for (int b = RF_R * RF_GL; b < npmax; b += RF_GL) {
    const int k = b + gl;
    int ck = 0;
    long long dk = 0;
    if (k < np) {
      const int cv = c[k];
      const long long dv = D[k] - A2 * cv;
      if (dv > 0) { ck = cv; dk = dv; }
    }
    const long long C = grp_incl_scan_i32(ck, gl) + Cc;
    const long long Pp = grp_incl_scan_i64(dk, gl) + Pc;
    if (ck > 0) rm.add(Pp, C, T, ck, dk);
    Cc = __shfl_sync(0xffffffffu, C, RF_GL - 1, RF_GL);
    Pc = __shfl_sync(0xffffffffu, Pp, RF_GL - 1, RF_GL);
  }
  rm.group_reduce<RF_GL>();
  const double best = rm.value();
  if (gl == 0 && live) {
    if (due) {
      double v = best;
      if (T == 0) {  // outlived every predicted length
        const long long gb = (long long)g + bucket_size;
        v = __dadd_rn(__dmul_rn((double)(gb * gb - (long long)g * g), 0.5),
                      __dmul_rn((double)Ii, (double)bucket_size));
      }
      G_io[i] = v;
      bucket_io[i] = nb;
    }
    if (refreshed) refreshed[i] = due ? 1 : 0;
  }
}

int launch_refresh(int64_t n, const int32_t* I, const int32_t* g_new, int32_t* bucket_io,
                   int bucket_size, const int32_t* npts, const int32_t* pcnt, const int64_t* pD,
                   int P, double* G_io, uint8_t* refreshed, int force, cudaStream_t st) {
  if (n <= 0) return SS_OK;
  count_launch();
  const int64_t per_block = 256 / RF_GL;
  k_refresh<<<(unsigned)((n + per_block - 1) / per_block), 256, 0, st>>>(
      n, I, g_new, bucket_io, bucket_size, npts, pcnt, pD, P, G_io, refreshed, force);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

}  // namespace ss
