// Measurement probe (not part of the product library): the dense int8
// tensor-core ceiling of this B200 for the MMA shapes the stage-1 kernels
// issue.  Every CTA (one per SM) keeps its operands resident -- A (128 x dim
// int8) in shared memory or TMEM, B tiles (N x dim int8) in shared memory,
// filled with a hash pattern so the datapath toggles as it does on real
// embeddings -- and one thread issues tcgen05.mma kind::i8 (M = 128, K = 32)
// back to back into two alternating accumulators, committing to an mbarrier
// every tile.  No TMA, no TMEM drains, no epilogue: the time is the tensor
// pipe alone, so 2 * M * N * K * count / time is the int8 dense peak that
// bench.py divides by (roofline.peak of the tcgen05 similarity kernels).
//
// C ABI: mma_peak_run(n_cta, tiles, n, a_in_tmem, stream) launches it; the
// caller times it with CUDA events.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

namespace {

constexpr int BM = 128, BK = 128, UK = 32, DIM = 384, NKB = DIM / BK;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

// MODE (compile time, so the peak loop carries no per-K-block tests -- any
// extra instruction between MMAs lowers the issue rate): 0 = back to back;
// bit 0: commit to bar_c (never completes) after every K-block; bit 1: wait on
// bar_w (already complete) + tcgen05 fence before every K-block; bit 2: the
// same with test_wait; bit 3: poll a shared flag; bit 4: acquire-load poll.
template <int mode>
__global__ void __launch_bounds__(384, 1) k_mma_peak(int tiles, int n, int a_tmem, int nacc, int drain_iters,
                                                     unsigned* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                  // NKB x 16 KB
  uint8_t* sB = sA + NKB * BM * BK;    // NKB x n x 128 B
  __shared__ uint64_t bar, bar_c, bar_w;
  __shared__ uint32_t flag;
  __shared__ uint32_t s_tmem;
  // hash pattern (int8 values spread over the full range)
  const int bytes = NKB * BM * BK + NKB * n * BK;
  for (int i = threadIdx.x * 4; i < bytes; i += blockDim.x * 4) {
    uint32_t h = (uint32_t)(i + 0x9E3779B9u * blockIdx.x);
    h ^= h >> 16; h *= 0x7feb352dU; h ^= h >> 15; h *= 0x846ca68bU; h ^= h >> 16;
    *reinterpret_cast<uint32_t*>(smem + i) = h;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    flag = 1;
    // mode bit 0: commit to bar_c (never completes) after every K-block;
    // bit 1: wait on bar_w (already complete) before every K-block
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1048575;\n" ::"r"(su32(&bar_c)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar_w)));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&bar_w)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic smem writes -> async proxy
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = s_tmem;
  const int acols = nacc * n;  // accumulators, A (TS form) after them
  if (a_tmem && threadIdx.x < 128) {
    // every warp writes its lane quarter of A (96 columns of 4 int8)
    const int w = threadIdx.x >> 5;
    for (int c0 = 0; c0 < DIM / 4; c0 += 8) {
      uint32_t v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = 0x01020304u * (uint32_t)(threadIdx.x + c0 + u);
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(
              tmem + ((uint32_t)(w * 32) << 16) + acols + c0),
          "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
          : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (threadIdx.x >= 128) {
    // drain warps: read the accumulator columns back (tcgen05.ld 32x32b.x32),
    // drain_iters passes over all nacc * n columns, concurrently with the MMAs
    const int w = (threadIdx.x >> 5) & 3;
    unsigned x = 0;
    for (int it = 0; it < drain_iters; ++it) {
      for (int c = 0; c + 32 <= nacc * n; c += 32) {
        uint32_t v[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
            "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
              "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
              "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
              "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(tmem + ((uint32_t)(w * 32) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int u = 0; u < 32; ++u) x ^= v[u];
      }
    }
    if (x == 0x12345678u) sink[0] = x;
  }
  if (threadIdx.x == 0) {
    const uint32_t id = idesc(n);
    for (int t = 0; t < tiles; ++t) {
      const uint32_t d = tmem + (t % nacc) * n;
      for (int kb = 0; kb < NKB; ++kb) {
        if constexpr (mode & 4) {
          asm volatile(
              "{\n.reg .pred p;\nWT_%=:\nmbarrier.test_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra WT_%=;\n}\n" ::"r"(
                  su32(&bar_w))
              : "memory");
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        }
        if constexpr (mode & 8) {  // a plain shared-memory flag, polled
          uint32_t f;
          do {
            asm volatile("ld.volatile.shared.u32 %0, [%1];\n" : "=r"(f) : "r"(su32(&flag)) : "memory");
          } while (f == 0);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        }
        if constexpr (mode & 16) {  // acquire-load poll of the flag
          uint32_t f;
          do {
            asm volatile("ld.acquire.cta.shared.u32 %0, [%1];\n" : "=r"(f) : "r"(su32(&flag)) : "memory");
          } while (f == 0);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        }
        if constexpr (mode & 2) {
          asm volatile(
              "{\n.reg .pred p;\nWW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra WW_%=;\n}\n" ::"r"(
                  su32(&bar_w))
              : "memory");
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        }
#pragma unroll
        for (int kk = 0; kk < BK / UK; ++kk) {
          const uint64_t bd = desc_sw128(su32(sB) + kb * n * BK + kk * UK);
          const uint32_t acc = (kb | kk) != 0;
          if (a_tmem) {
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                "r"(tmem + acols + (kb * (BK / UK) + kk) * (UK / 4)), "l"(bd), "r"(id), "r"(acc)
                : "memory");
          } else {
            const uint64_t ad = desc_sw128(su32(sA) + kb * BM * BK + kk * UK);
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                "l"(ad), "l"(bd), "r"(id), "r"(acc)
                : "memory");
          }
        }
        if constexpr (mode & 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                           su32(&bar_c))
                       : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     su32(&bar))
                 : "memory");
    asm volatile(
        "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(
            su32(&bar))
        : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}

}  // namespace

extern "C" {
// ops per launch = 2 * 128 * n * DIM * tiles * n_cta
int mma_peak_run3(int n_cta, int tiles, int n, int a_in_tmem, int drain_warps, int drain_iters,
                  int mode, void* stream);
int mma_peak_run(int n_cta, int tiles, int n, int a_in_tmem, void* stream) {
  return mma_peak_run3(n_cta, tiles, n, a_in_tmem, 0, 0, 0, stream);
}
int mma_peak_run2(int n_cta, int tiles, int n, int a_in_tmem, int drain_warps, int drain_iters,
                  void* stream) {
  return mma_peak_run3(n_cta, tiles, n, a_in_tmem, drain_warps, drain_iters, 0, stream);
}
// drain_warps (0, 4 or 8) extra warps read the accumulators back drain_iters
// times while the MMAs run: TMEM read bandwidth alone (tiles = 0) and its
// interference with the MMA
int mma_peak_run3(int n_cta, int tiles, int n, int a_in_tmem, int drain_warps, int drain_iters,
                  int mode, void* stream) {
  static unsigned* sink = nullptr;
  if (!sink && cudaMalloc(&sink, 64) != cudaSuccess) return 4;
  // as many accumulators (<= 2) as fit beside A
  const int nacc = (!a_in_tmem || 2 * n + DIM / 4 <= 512) ? 2 : 1;
  if (n < 8 || n > 256 || n % 16 || (a_in_tmem && nacc * n + DIM / 4 > 512)) return 1;
  const size_t smem = 1024 + (size_t)NKB * BM * BK + (size_t)NKB * n * BK;
  auto kern = mode == 0 ? k_mma_peak<0> : mode == 1 ? k_mma_peak<1> : mode == 2 ? k_mma_peak<2> :
              mode == 3 ? k_mma_peak<3> : mode == 4 ? k_mma_peak<4> : mode == 8 ? k_mma_peak<8> :
              mode == 16 ? k_mma_peak<16> : nullptr;
  if (!kern) return 5;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return 2;
  kern<<<n_cta, 128 + 32 * drain_warps, smem, (cudaStream_t)stream>>>(
      tiles, n, a_in_tmem, nacc, drain_warps ? drain_iters : 0, sink);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}
int mma_peak_dim(void) { return DIM; }
}

// ---------------------------------------------------------------------------
// CTA-pair form (cluster of 2, cta_group::2, M = 256): A (128 rows per CTA) in
// each CTA's TMEM, B split across the pair (n/2 rows per CTA's shared memory),
// the leader's thread 0 issues.  sts_warps extra warps per CTA store to a
// scratch shared-memory area as fast as they can while the MMAs run
// (contention of the shared-memory port with the tensor core's B reads, as
// TMA writes and epilogue loads contend in the real kernel).
namespace {
template <int pair>
__global__ void __launch_bounds__(384, 1) k_mma_pair(int tiles, int n, int nacc, int sts_iters,
                                                     unsigned* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  const int nb = pair ? n / 2 : n;     // B rows held by this CTA
  uint8_t* sB = smem;                  // NKB x nb x 128 B
  uint8_t* sX = sB + NKB * nb * BK;    // 16 KB scratch for the store warps
  __shared__ uint64_t bar;
  __shared__ uint32_t s_tmem;
  uint32_t rank = 0;
  if constexpr (pair != 0) asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
  for (int i = threadIdx.x * 4; i < NKB * nb * BK; i += blockDim.x * 4) {
    uint32_t h = (uint32_t)(i + 0x9E3779B9u * (blockIdx.x + 1));
    h ^= h >> 16; h *= 0x7feb352dU; h ^= h >> 15; h *= 0x846ca68bU; h ^= h >> 16;
    *reinterpret_cast<uint32_t*>(smem + i) = h;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) {
    if constexpr (pair != 0) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&s_tmem)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&s_tmem)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  if constexpr (pair != 0)
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  else
    __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = s_tmem;
  const int acols = nacc * n;
  if (threadIdx.x < 128) {
    const int w = threadIdx.x >> 5;
    for (int c0 = 0; c0 < DIM / 4; c0 += 8) {
      uint32_t v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = 0x01020304u * (uint32_t)(threadIdx.x + c0 + u);
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(
              tmem + ((uint32_t)(w * 32) << 16) + acols + c0),
          "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
          : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  if constexpr (pair != 0)
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  else
    __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (threadIdx.x >= 128) {
    // shared-memory store traffic: 16 B per thread per store, a 16 KB window
    uint4* x = reinterpret_cast<uint4*>(sX);
    const int t = threadIdx.x - 128;
    uint4 v = make_uint4(t, t * 3, t * 5, t * 7);
    for (int it = 0; it < sts_iters; ++it) {
#pragma unroll 8
      for (int u = 0; u < 4; ++u) {
        v.x += 1;
        x[(t + u * 256) & 1023] = v;
      }
    }
    if (v.x == 0x12345678u) sink[0] = v.y;
  }
  if (threadIdx.x == 0 && rank == 0) {
    const uint32_t id = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
                        ((uint32_t)((pair ? 2 * BM : BM) >> 4) << 24);
    for (int t = 0; t < tiles; ++t) {
      const uint32_t d = tmem + (t % nacc) * n;
      for (int kb = 0; kb < NKB; ++kb) {
#pragma unroll
        for (int kk = 0; kk < BK / UK; ++kk) {
          const uint64_t bd = desc_sw128(su32(sB) + kb * nb * BK + kk * UK);
          const uint32_t acc = (kb | kk) != 0;
          const uint32_t a = tmem + acols + (kb * (BK / UK) + kk) * (UK / 4);
          if constexpr (pair != 0)
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                "r"(a), "l"(bd), "r"(id), "r"(acc)
                : "memory");
          else
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                "r"(a), "l"(bd), "r"(id), "r"(acc)
                : "memory");
        }
      }
    }
    if constexpr (pair != 0)
      asm volatile(
          "{\n.reg .b16 m;\nmov.b16 m, 3;\n"
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}\n" ::"r"(
              su32(&bar))
          : "memory");
    else
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                       su32(&bar))
                   : "memory");
  }
  if (threadIdx.x == 0)
    asm volatile(
        "{\n.reg .pred p;\nWP:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra WP;\n}\n" ::"r"(
            su32(&bar))
        : "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  if constexpr (pair != 0)
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  else
    __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if constexpr (pair != 0)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}
}  // namespace

extern "C" int mma_pair_run(int n_cta, int tiles, int n, int sts_warps, int sts_iters, int pair,
                            void* stream) {
  static unsigned* sink = nullptr;
  if (!sink && cudaMalloc(&sink, 64) != cudaSuccess) return 4;
  const int nacc = (2 * n + DIM / 4 <= 512) ? 2 : 1;
  if (n % 16 || n > 256) return 1;
  const size_t smem = 1024 + (size_t)NKB * (pair ? n / 2 : n) * BK + 16384;
  auto kern = pair ? k_mma_pair<1> : k_mma_pair<0>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)n_cta);
  cfg.blockDim = dim3(128 + 32 * sts_warps);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = pair ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pair ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tiles, n, nacc, sts_warps ? sts_iters : 0, sink);
  if (e != cudaSuccess) {
    fprintf(stderr, "mma_pair_run: %s\n", cudaGetErrorString(e));
    return 3;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// Issue timing: one CTA, thread 0 issues `count` TS MMAs (N = n) back to back
// and records clock64 after each issue; out[i] = cycles since the first.
namespace {
__global__ void __launch_bounds__(128, 1) k_mma_issue_timing(int count, int n, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t s_tmem;
  __shared__ long long ts[256];
  for (int i = threadIdx.x * 4; i < NKB * n * BK; i += blockDim.x * 4) *reinterpret_cast<uint32_t*>(smem + i) = i * 2654435761u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = s_tmem;
  if (threadIdx.x == 0) {
    const uint32_t id = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
    long long t0 = clock64();
    for (int i = 0; i < count && i < 256; ++i) {
      const uint64_t bd = desc_sw128(su32(smem) + (i % 12 / 4) * n * BK + (i % 4) * UK);
      const int nacc = (2 * n + 96 <= 512) ? 2 : 1;
      const uint32_t d = tmem + ((i / 12) % nacc) * n;
      const uint32_t acc = (i % 12) != 0;
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
          "r"(tmem + nacc * n + (i % 12) * 8), "l"(bd), "r"(id), "r"(acc)
          : "memory");
      ts[i] = clock64() - t0;
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nWI:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra WI;\n}\n" ::"r"(su32(&bar)) : "memory");
    ts[count < 256 ? count : 255] = clock64() - t0;
    for (int i = 0; i <= count && i < 256; ++i) out[i] = ts[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}
}  // namespace

extern "C" int mma_issue_timing(int count, int n, long long* out_dev, void* stream) {
  const size_t smem = 1024 + (size_t)NKB * n * BK;
  if (cudaFuncSetAttribute(k_mma_issue_timing, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return 2;
  k_mma_issue_timing<<<1, 128, smem, (cudaStream_t)stream>>>(count, n, out_dev);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}
