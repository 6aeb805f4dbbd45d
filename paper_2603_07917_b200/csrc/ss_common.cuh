// Shared device/host helpers for libsagesched (B200, sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include "../../include/sagesched.h"

namespace ss {

// ---------------------------------------------------------------------------
// error plumbing (host): thread-local last-error string, see ss_api.cu
// ---------------------------------------------------------------------------
int set_error(int code, const char* fmt, ...);

#define SS_CUDA_TRY(expr)                                                     \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess)                                                    \
      return ::ss::set_error(SS_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, \
                             #expr, cudaGetErrorString(_e));                  \
  } while (0)

#define SS_LAUNCH_CHECK() SS_CUDA_TRY(cudaGetLastError())

// ---------------------------------------------------------------------------
// orderable encodings
// ---------------------------------------------------------------------------
// fp32 -> u32 whose unsigned order equals the float order (NaN excluded).
__host__ __device__ __forceinline__ uint32_t f32_order(float f) {
#ifdef __CUDA_ARCH__
  uint32_t b = __float_as_uint(f);
#else
  uint32_t b;
  memcpy(&b, &f, 4);
#endif
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__host__ __device__ __forceinline__ float f32_unorder(uint32_t u) {
  uint32_t b = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
#ifdef __CUDA_ARCH__
  return __uint_as_float(b);
#else
  float f;
  memcpy(&f, &b, 4);
  return f;
#endif
}
// fp64 -> u64 order-preserving key (for the rank sort).
__device__ __forceinline__ uint64_t f64_order(double d) {
  uint64_t b = (uint64_t)__double_as_longlong(d);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

// Candidate composite: (orderable key << 32) | rel, rel = (slot - head) mod C
// is monotone in insertion_seq, so descending composite order is
// (key desc, insertion_seq desc) -- SPEC.md:135.  0 is the empty sentinel
// (it would decode to a negative NaN key, which is never produced).
__device__ __forceinline__ uint64_t make_comp(float key, uint32_t rel) {
  return ((uint64_t)f32_order(key) << 32) | rel;
}
__device__ __forceinline__ float comp_key(uint64_t c) { return f32_unorder((uint32_t)(c >> 32)); }
__device__ __forceinline__ uint32_t comp_rel(uint64_t c) { return (uint32_t)c; }

// Conservative s-domain threshold: every row with fl(s*iq) >= K has s >= thr.
__device__ __forceinline__ float s_threshold(float K, float iq) {
  float t = __fdiv_rn(K, iq);
  return t - fabsf(t) * 1.0e-6f - 1.0e-30f;
}

// exact score key = fl32(fl32(f32(dot) * iw) * iq)
__device__ __forceinline__ float score_key(int dot, float iw, float iq) {
  return __fmul_rn(__fmul_rn(__int2float_rn(dot), iw), iq);
}

__device__ __forceinline__ int warp_incl_scan_i32(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}
__device__ __forceinline__ long long warp_incl_scan_i64(long long v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}
__device__ __forceinline__ double warp_min_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Programmatic dependent launch: a kernel launched with pdl_launch() may be
// scheduled while its predecessor on the stream drains; it must call
// pdl_wait() before touching anything the predecessor writes.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

}  // namespace ss

// Internal launchers (host side), implemented per kernel file.
namespace ss {
struct RelMap {          // ring-slot -> rel mapping, global over shards
  int64_t head;          // total pushes so far (next insertion_seq)
  int64_t capacity;      // global ring capacity
  int64_t slot_offset;   // first global slot held by this shard
};
}  // namespace ss
