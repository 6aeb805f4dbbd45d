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

__global__ void __launch_bounds__(128, 1) k_mma_peak(int tiles, int n, int a_tmem, int nacc) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                  // NKB x 16 KB
  uint8_t* sB = sA + NKB * BM * BK;    // NKB x n x 128 B
  __shared__ uint64_t bar;
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
  if (a_tmem) {
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
  if (threadIdx.x == 0) {
    const uint32_t id = idesc(n);
    for (int t = 0; t < tiles; ++t) {
      const uint32_t d = tmem + (t % nacc) * n;
      for (int kb = 0; kb < NKB; ++kb) {
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
int mma_peak_run(int n_cta, int tiles, int n, int a_in_tmem, void* stream) {
  // as many accumulators (<= 2) as fit beside A
  const int nacc = (!a_in_tmem || 2 * n + DIM / 4 <= 512) ? 2 : 1;
  if (n < 8 || n > 256 || n % 16 || (a_in_tmem && nacc * n + DIM / 4 > 512)) return 1;
  const size_t smem = 1024 + (size_t)NKB * BM * BK + (size_t)NKB * n * BK;
  if (cudaFuncSetAttribute(k_mma_peak, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return 2;
  k_mma_peak<<<n_cta, 128, smem, (cudaStream_t)stream>>>(tiles, n, a_in_tmem, nacc);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}
int mma_peak_dim(void) { return DIM; }
}
