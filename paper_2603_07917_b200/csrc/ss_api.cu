// C-ABI layer of libsagesched: argument validation, handle/workspace
// management and stage orchestration.  Every function here is declared in
// include/sagesched.h, which cites the reference interface each replaces.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>
#include <math.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <new>

#include "ss_common.cuh"
#include "ss_internal.h"

namespace ss {

static thread_local char g_err[1024] = "";
static std::atomic<int64_t> g_launches{0};

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int sm_count(int device) {
  static int cache[64] = {0};
  if (device < 0 || device >= 64) return 148;
  if (!cache[device]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0)
      v = 148;
    cache[device] = v;
  }
  return cache[device];
}

int pick_slices(int64_t qtiles, int64_t tiles, int sms) {
  if (qtiles < 1 || tiles < 1 || sms < 1) return 1;
  int64_t lo = sms / qtiles;
  if (lo < 1) lo = 1;
  const int64_t hi = std::min<int64_t>(std::max<int64_t>(lo, 64), tiles);
  if (lo >= tiles) return (int)tiles;
  int64_t best = lo;
  double best_eff = 0.0;
  for (int64_t s = lo; s <= hi; ++s) {
    const int64_t ctas = qtiles * s;
    const int64_t waves = (ctas + sms - 1) / sms;
    const double eff = (double)ctas / (double)(waves * sms);
    if (eff >= 0.97) return (int)s;
    if (eff > best_eff + 1e-9) { best_eff = eff; best = s; }
  }
  return (int)best;
}

// per-device sticky error flag for handle-less synchronous entry points,
// followed by one scratch counter (device_err_flag() + 1)
static int* device_err_flag() {
  static std::mutex mu;
  static int* flags[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (!flags[dev]) {
    if (cudaMalloc(&flags[dev], 2 * sizeof(int)) != cudaSuccess) return nullptr;
    cudaMemset(flags[dev], 0, 2 * sizeof(int));
  }
  return flags[dev];
}

static int read_and_clear(int* d_err, cudaStream_t st) {
  int h = 0;
  if (cudaMemcpyAsync(&h, d_err, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return set_error(SS_ERR_CUDA, "error-flag readback failed: %s",
                     cudaGetErrorString(cudaGetLastError()));
  if (h) cudaMemsetAsync(d_err, 0, sizeof(int), st);
  return h;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace ss

using namespace ss;

struct ss_bank {
  int device;
  int64_t cap, gcap, slot_offset;
  int dim;
  int64_t head;
  int8_t* emb = nullptr;
  float* inv = nullptr;
  float2* ibnd = nullptr;  // per 16-row group filter bounds (k_bank_bounds), padded like inv
  int32_t* lens = nullptr;
  int64_t* seq = nullptr;
  int32_t* len_cnt = nullptr;  // exact-length histogram of the window [65536]
  int* d_err = nullptr;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  uint32_t* gslots = nullptr;  // TS kernel pure top-k: per-slice published bounds
  int64_t gslots_cap = 0;
  int8_t* qscratch = nullptr;  // 128 x dim: single-tile query spread (k_topk_tc)
  // wide plane (first int16 push): exact vectors of rows outside int8
  WidePlane wp;
  int64_t* wlist = nullptr;  // [cap] compacted wide slots (per wide pass)
  int* wlist_count = nullptr;
  bool any_wide = false;     // a wide row has been written: rounds run the wide pass
  // side stream of the fused round: the fallback histogram runs concurrently
  // with the similarity kernel (fork/join by events; captured as two graph
  // branches when the caller's stream is being captured)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  uint64_t ws_gen = 0;  // bumped whenever the workspace moves
  // host-buffer round (ss_schedule_round_host) replayed as one CUDA graph
  // once the same call repeats: key = every scalar and pointer baked into it
  struct HostRoundKey {
    int64_t nq, head;
    int32_t k, min_matches, max_len, nbins, algo, any_wide;
    float theta;
    const void* ptr[6];
    uint64_t ws_gen;
    bool operator==(const HostRoundKey& o) const { return memcmp(this, &o, sizeof(*this)) == 0; }
  };
  HostRoundKey last_key{};
  bool have_last = false;
  cudaGraphExec_t host_exec = nullptr;
  HostRoundKey exec_key{};
  cudaStream_t cap_stream = nullptr;
};

// per-slice published bounds for the TS kernel in pure top-k mode (theta <=
// 0).  Grow-on-demand outside graph capture, like the workspace; nullptr
// simply disables the sharing.
static uint32_t* gslots_reserve(ss_bank* h, int64_t nq, float theta) {
  if (!(theta <= 0.f)) return nullptr;
  const int64_t need = 2 * nq * kMaxShareSlices;  // bounds, then the cascade's per-slice counts
  if (need <= h->gslots_cap) return h->gslots;
  if (h->gslots) cudaFree(h->gslots);
  h->gslots = nullptr;
  h->gslots_cap = 0;
  ++h->ws_gen;  // a captured host round baked the old pointer in: re-capture
  if (cudaMalloc(&h->gslots, (size_t)need * sizeof(uint32_t)) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  h->gslots_cap = need;
  return h->gslots;
}

static int ws_reserve(ss_bank* h, size_t bytes) {
  if (bytes <= h->ws_bytes) return SS_OK;
  if (h->ws) cudaFree(h->ws);
  h->ws = nullptr;
  h->ws_bytes = 0;
  size_t want = bytes + bytes / 4;
  SS_CUDA_TRY(cudaMalloc(&h->ws, want));
  h->ws_bytes = want;
  ++h->ws_gen;
  return SS_OK;
}

static inline size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

extern "C" {

const char* ss_last_error(void) { return g_err; }
int ss_version(void) { return 10000; }
int64_t ss_launch_count(void) { return g_launches.load(); }

// ------------------------------------------------------------- compat -----
int ss_match_pmfs(const float* sims, int64_t nq, int64_t nw, const int64_t* lens, double theta,
                  int64_t max_len, double* sup, double* mas, int64_t* sizes, int64_t out_stride,
                  void* stream) {
  if (nq < 0 || nw < 0 || max_len < 1 || out_stride < max_len)
    return set_error(SS_ERR_ARG, "match_pmfs: bad shape (nq=%lld nw=%lld max_len=%lld stride=%lld)",
                     (long long)nq, (long long)nw, (long long)max_len, (long long)out_stride);
  if (nq == 0) return SS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int* err = device_err_flag();
  if (!err) return set_error(SS_ERR_CUDA, "error flag alloc failed");
  int rc = launch_match_pmfs(sims, nq, nw, lens, theta, max_len, sup, mas, sizes, out_stride, err, st);
  if (rc) return rc;
  int e = read_and_clear(err, st);
  if (e == SS_ERR_RANGE) return set_error(SS_ERR_RANGE, "match_pmfs: a matched length lies outside [0, max_len]");
  return e;
}

int ss_gittins_min_batch(const double* support, const double* masses, const int64_t* npts,
                         int64_t n, int64_t stride, double* out, void* stream) {
  if (n < 0 || stride < 0) return set_error(SS_ERR_ARG, "gittins_min_batch: bad shape");
  if (n == 0) return SS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int* err = device_err_flag();
  if (!err) return set_error(SS_ERR_CUDA, "error flag alloc failed");
  int rc = launch_gittins_dist(support, masses, npts, nullptr, nullptr, n, stride, out, err, 1, st);
  if (rc) return rc;
  int e = read_and_clear(err, st);
  if (e == SS_ERR_ZERODIV) return set_error(SS_ERR_ZERODIV, "float division by zero");
  return e;
}

int ss_gittins_dist_batch(const double* support, const double* masses, const int64_t* npts,
                          const double* attained, const double* outlived_index, int64_t n,
                          int64_t stride, double* out, void* stream) {
  if (n < 0 || stride < 0) return set_error(SS_ERR_ARG, "gittins_dist_batch: bad shape");
  int* err = device_err_flag();
  if (!err) return set_error(SS_ERR_CUDA, "error flag alloc failed");
  return launch_gittins_dist(support, masses, npts, attained, outlived_index, n, stride, out, err,
                             0, (cudaStream_t)stream);
}

int ss_embed_accumulate_batch(const int64_t* tokens, const int64_t* offsets, int64_t n,
                              uint64_t salt, int32_t dim, double* out, void* stream) {
  if (n < 0 || dim < 1) return set_error(SS_ERR_ARG, "embed: bad shape");
  return launch_embed(tokens, offsets, n, salt, dim, out, nullptr, nullptr, nullptr,
                      (cudaStream_t)stream);
}

int ss_embed_quantize_batch(const int64_t* tokens, const int64_t* offsets, int64_t n,
                            uint64_t salt, int32_t dim, int16_t* out_emb, float* out_inv_norm,
                            int64_t* n_wide, void* stream) {
  if (n < 0 || dim < 1 || !out_emb || !out_inv_norm) return set_error(SS_ERR_ARG, "embed_quantize: bad args");
  if (n_wide) *n_wide = 0;
  if (n == 0) return SS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int* err = device_err_flag();
  if (!err) return set_error(SS_ERR_CUDA, "error flag alloc failed");
  SS_CUDA_TRY(cudaMemsetAsync(err + 1, 0, sizeof(int), st));
  int rc = launch_embed(tokens, offsets, n, salt, dim, nullptr, out_emb, out_inv_norm, err, st);
  if (rc) return rc;
  int cnt = 0;
  SS_CUDA_TRY(cudaMemcpyAsync(&cnt, err + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  int e = read_and_clear(err, st);  // synchronises
  if (e == SS_ERR_RANGE) return set_error(SS_ERR_RANGE, "embed_quantize: a bucket exceeds the int16 range");
  if (n_wide) *n_wide = cnt;
  return e;
}

int ss_cost_distribution_batch(int32_t kind, double w_in, double w_out, const double* input_len,
                               const double* len_support, const int64_t* npts, int64_t n,
                               int64_t stride, double* out_support, void* stream) {
  if (kind < 0 || kind > 2) return set_error(SS_ERR_ARG, "unknown cost model kind %d", kind);
  if (kind == SS_COST_WEIGHTED_SUM && (w_in <= 0 || w_out <= 0))
    return set_error(SS_ERR_ARG, "weighted-sum weights must be positive");
  return launch_cost_dist(kind, w_in, w_out, input_len, len_support, npts, n, stride, out_support,
                          (cudaStream_t)stream);
}

// ------------------------------------------------- per-call host entry ----
// The reference's scalar call pattern (one law per call, host arrays in and
// out): one packed H2D copy from a library-owned pinned staging buffer, the
// kernel, one D2H, one synchronise -- no allocation per call.  Staging is per
// thread (a handle-less entry point may be called from several threads).
struct HostStaging {
  char* host = nullptr;  // pinned
  char* dev = nullptr;
  size_t bytes = 0;
  int device = -1;
  ~HostStaging() {
    if (host) cudaFreeHost(host);
    if (dev) cudaFree(dev);
  }
  int reserve(size_t need) {
    int d = 0;
    cudaGetDevice(&d);
    if (need <= bytes && d == device) return SS_OK;
    if (host) cudaFreeHost(host);
    if (dev) cudaFree(dev);
    host = nullptr;
    dev = nullptr;
    bytes = 0;
    const size_t want = std::max<size_t>(need, 64 * 1024);
    SS_CUDA_TRY(cudaMallocHost(&host, want));
    SS_CUDA_TRY(cudaMalloc(&dev, want));
    bytes = want;
    device = d;
    return SS_OK;
  }
};
static thread_local HostStaging g_stage;

// Mapped per-call slot and a library stream, per thread (see PerCallHdr).
struct PerCallSlot {
  PerCallHdr* host = nullptr;  // mapped pinned
  PerCallHdr* dev = nullptr;   // its device alias
  cudaStream_t st = nullptr;
  uint32_t seq = 0;
  int device = -1;
  ~PerCallSlot() { release(); }
  void release() {
    if (host) cudaFreeHost(host);
    if (st) cudaStreamDestroy(st);
    host = dev = nullptr;
    st = nullptr;
  }
  int ready() {
    int d = 0;
    cudaGetDevice(&d);
    if (host && d == device) return SS_OK;
    release();
    const size_t bytes = sizeof(PerCallHdr) + (size_t)2 * kPerCallMaxPts * sizeof(double);
    void* p = nullptr;
    SS_CUDA_TRY(cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    host = static_cast<PerCallHdr*>(p);
    memset(host, 0, bytes);
    void* dp = nullptr;
    SS_CUDA_TRY(cudaHostGetDevicePointer(&dp, p, 0));
    dev = static_cast<PerCallHdr*>(dp);
    SS_CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    device = d;
    return SS_OK;
  }
  // spin until the kernel raised the flag for `s` (or the stream failed)
  int wait(uint32_t s) {
    volatile uint32_t* f = &host->flag;
    for (uint32_t spins = 1; *f != s; ++spins) {
      if ((spins & 4095) == 0) {
        cudaError_t e = cudaStreamQuery(st);
        if (e != cudaSuccess && e != cudaErrorNotReady)
          return set_error(SS_ERR_CUDA, "per-call kernel: %s", cudaGetErrorString(e));
        if (e == cudaSuccess && *f != s)
          return set_error(SS_ERR_CUDA, "per-call kernel finished without raising its flag");
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    return SS_OK;
  }
};
static thread_local PerCallSlot g_call;

extern "C" int ss_gittins_min_host(const double* support, const double* masses, int64_t n,
                                   double* out, void* stream) {
  if (n < 0 || !out || (n > 0 && (!support || !masses)))
    return set_error(SS_ERR_ARG, "gittins_min_host: bad args");
  if (n == 0) {
    *out = INFINITY;  // min over no support point
    return SS_OK;
  }
  if (n <= kPerCallMaxPts) {
    // mapped slot: inputs written here, pulled by the kernel; result and
    // flag written back by the kernel (the stream argument orders nothing:
    // inputs and output are host memory)
    if (int rc = g_call.ready()) return rc;
    PerCallHdr* h = g_call.host;
    h->n = n;
    double* data = reinterpret_cast<double*>(h + 1);
    memcpy(data, support, (size_t)n * 8);
    memcpy(data + n, masses, (size_t)n * 8);
    const uint32_t seq = ++g_call.seq;
    std::atomic_thread_fence(std::memory_order_release);
    if (int rc = launch_gittins_percall(g_call.dev, n, seq, g_call.st)) return rc;
    if (int rc = g_call.wait(seq)) return rc;
    if (h->err == SS_ERR_ZERODIV) return set_error(SS_ERR_ZERODIV, "float division by zero");
    *out = h->result;
    return SS_OK;
  }
  // staging: [npts i64][result f64][err i32 + pad][support n][masses n]
  const size_t hdr = 32, need = hdr + (size_t)n * 16;
  if (int rc = g_stage.reserve(need)) return rc;
  char* h = g_stage.host;
  *reinterpret_cast<int64_t*>(h) = n;
  *reinterpret_cast<double*>(h + 8) = 0.0;
  *reinterpret_cast<int*>(h + 16) = 0;
  memcpy(h + hdr, support, (size_t)n * 8);
  memcpy(h + hdr + (size_t)n * 8, masses, (size_t)n * 8);
  cudaStream_t st = (cudaStream_t)stream;
  char* d = g_stage.dev;
  SS_CUDA_TRY(cudaMemcpyAsync(d, h, need, cudaMemcpyHostToDevice, st));
  if (int rc = launch_gittins_dist(reinterpret_cast<const double*>(d + hdr),
                                   reinterpret_cast<const double*>(d + hdr + (size_t)n * 8),
                                   reinterpret_cast<const int64_t*>(d), nullptr, nullptr, 1, n,
                                   reinterpret_cast<double*>(d + 8), reinterpret_cast<int*>(d + 16),
                                   1, st))
    return rc;
  SS_CUDA_TRY(cudaMemcpyAsync(h + 8, d + 8, 12, cudaMemcpyDeviceToHost, st));
  SS_CUDA_TRY(cudaStreamSynchronize(st));
  if (*reinterpret_cast<int*>(h + 16) == SS_ERR_ZERODIV)
    return set_error(SS_ERR_ZERODIV, "float division by zero");
  *out = *reinterpret_cast<double*>(h + 8);
  return SS_OK;
}

extern "C" int ss_cost_distribution_host(int32_t kind, double w_in, double w_out, double input_len,
                                         const double* len_support, int64_t n, double* out_support,
                                         void* stream) {
  if (kind < 0 || kind > 2) return set_error(SS_ERR_ARG, "unknown cost model kind %d", kind);
  if (kind == SS_COST_WEIGHTED_SUM && (w_in <= 0 || w_out <= 0))
    return set_error(SS_ERR_ARG, "weighted-sum weights must be positive");
  if (n < 0 || (n > 0 && (!len_support || !out_support)))
    return set_error(SS_ERR_ARG, "cost_distribution_host: bad args");
  if (n == 0) return SS_OK;
  if (n <= kPerCallMaxPts) {  // mapped slot (see ss_gittins_min_host)
    if (int rc = g_call.ready()) return rc;
    PerCallHdr* h = g_call.host;
    h->n = n;
    h->input_len = input_len;
    h->w_in = w_in;
    h->w_out = w_out;
    h->kind = kind;
    double* data = reinterpret_cast<double*>(h + 1);
    memcpy(data, len_support, (size_t)n * 8);
    const uint32_t seq = ++g_call.seq;
    std::atomic_thread_fence(std::memory_order_release);
    if (int rc = launch_cost_percall(g_call.dev, seq, g_call.st)) return rc;
    if (int rc = g_call.wait(seq)) return rc;
    memcpy(out_support, data + n, (size_t)n * 8);
    return SS_OK;
  }
  // staging: [npts i64][I f64][support n][out n]
  const size_t hdr = 16, need = hdr + (size_t)n * 16;
  if (int rc = g_stage.reserve(need)) return rc;
  char* h = g_stage.host;
  *reinterpret_cast<int64_t*>(h) = n;
  *reinterpret_cast<double*>(h + 8) = input_len;
  memcpy(h + hdr, len_support, (size_t)n * 8);
  cudaStream_t st = (cudaStream_t)stream;
  char* d = g_stage.dev;
  SS_CUDA_TRY(cudaMemcpyAsync(d, h, hdr + (size_t)n * 8, cudaMemcpyHostToDevice, st));
  if (int rc = launch_cost_dist(kind, w_in, w_out, reinterpret_cast<const double*>(d + 8),
                                reinterpret_cast<const double*>(d + hdr),
                                reinterpret_cast<const int64_t*>(d), 1, n,
                                reinterpret_cast<double*>(d + hdr + (size_t)n * 8), st))
    return rc;
  SS_CUDA_TRY(cudaMemcpyAsync(h + hdr + (size_t)n * 8, d + hdr + (size_t)n * 8, (size_t)n * 8,
                              cudaMemcpyDeviceToHost, st));
  SS_CUDA_TRY(cudaStreamSynchronize(st));
  memcpy(out_support, h + hdr + (size_t)n * 8, (size_t)n * 8);
  return SS_OK;
}

// ---------------------------------------------------------------- bank ----
int ss_bank_create(ss_bank_t** out, int32_t device, int64_t capacity, int32_t dim,
                   int64_t global_capacity, int64_t slot_offset) {
  if (!out) return set_error(SS_ERR_ARG, "null out");
  *out = nullptr;
  if (capacity < 1 || dim < 16 || dim % 16 || global_capacity < capacity || slot_offset < 0 ||
      slot_offset + capacity > global_capacity || global_capacity >= (1LL << 32))
    return set_error(SS_ERR_ARG, "bank_create: bad shape (cap=%lld dim=%d gcap=%lld off=%lld)",
                     (long long)capacity, dim, (long long)global_capacity, (long long)slot_offset);
  DeviceGuard g(device);
  ss_bank* h = new (std::nothrow) ss_bank();
  if (!h) return set_error(SS_ERR_ARG, "oom");
  h->device = device;
  h->cap = capacity;
  h->gcap = global_capacity;
  h->slot_offset = slot_offset;
  h->dim = dim;
  h->head = 0;
  int rc = SS_OK;
  auto fail = [&](cudaError_t e) {
    rc = set_error(SS_ERR_CUDA, "bank_create: %s", cudaGetErrorString(e));
  };
  cudaError_t e;
  if ((e = cudaMalloc(&h->emb, (size_t)capacity * dim)) != cudaSuccess) fail(e);
  else if ((e = cudaMalloc(&h->inv, ((size_t)capacity + 256) * 4)) != cudaSuccess) fail(e);
  else if ((e = cudaMalloc(&h->ibnd, (((size_t)capacity + 15) / 16 + 16) * sizeof(float2))) != cudaSuccess)
    fail(e);
  else if ((e = cudaMalloc(&h->lens, (size_t)capacity * 4)) != cudaSuccess) fail(e);
  else if ((e = cudaMalloc(&h->seq, (size_t)capacity * 8)) != cudaSuccess) fail(e);
  else if ((e = cudaMalloc(&h->len_cnt, 65536 * 4)) != cudaSuccess) fail(e);
  else if ((e = cudaMalloc(&h->d_err, sizeof(int))) != cudaSuccess) fail(e);
  else if ((e = cudaMalloc(&h->qscratch, (size_t)128 * dim)) != cudaSuccess) fail(e);
  else if ((e = cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking)) != cudaSuccess) fail(e);
  else if ((e = cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming)) != cudaSuccess) fail(e);
  else if ((e = cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming)) != cudaSuccess) fail(e);
  if (rc == SS_OK) {
    cudaMemset(h->emb, 0, (size_t)capacity * dim);
    cudaMemset(h->inv, 0xff, ((size_t)capacity + 256) * 4);  // NaN: never matches (+1 tile pad)
    {  // every group empty: (0, +inf)
      const size_t ng = ((size_t)capacity + 15) / 16 + 16;
      float2* hb = static_cast<float2*>(malloc(ng * sizeof(float2)));
      if (hb) {
        for (size_t i = 0; i < ng; ++i) hb[i] = make_float2(0.f, INFINITY);
        cudaMemcpy(h->ibnd, hb, ng * sizeof(float2), cudaMemcpyHostToDevice);
        free(hb);
      } else {
        rc = set_error(SS_ERR_ARG, "bank_create: oom");
      }
    }
    cudaMemset(h->lens, 0, (size_t)capacity * 4);
    cudaMemset(h->seq, 0xff, (size_t)capacity * 8);  // -1: empty slot
    cudaMemset(h->len_cnt, 0, 65536 * 4);
    cudaMemset(h->d_err, 0, sizeof(int));
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) fail(e);
  }
  if (rc != SS_OK) {
    ss_bank_destroy(h);
    return rc;
  }
  *out = h;
  return SS_OK;
}

int ss_bank_destroy(ss_bank_t* h) {
  if (!h) return SS_OK;
  DeviceGuard g(h->device);
  cudaFree(h->emb);
  cudaFree(h->inv);
  cudaFree(h->ibnd);
  cudaFree(h->lens);
  cudaFree(h->seq);
  cudaFree(h->len_cnt);
  cudaFree(h->d_err);
  cudaFree(h->ws);
  cudaFree(h->gslots);
  cudaFree(h->qscratch);
  cudaFree(h->wp.emb);
  cudaFree(h->wp.inv);
  cudaFree(h->wp.flag);
  cudaFree(h->wp.count);
  cudaFree(h->wlist);
  cudaFree(h->wlist_count);
  if (h->host_exec) cudaGraphExecDestroy(h->host_exec);
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->side) cudaStreamDestroy(h->side);
  delete h;
  return SS_OK;
}

int ss_bank_push(ss_bank_t* h, const int8_t* emb, const float* inv_norm, const int32_t* lens,
                 int64_t n, void* stream) {
  if (!h || n < 0) return set_error(SS_ERR_ARG, "bank_push: bad args");
  if (h->gcap != h->cap || h->slot_offset != 0)
    return set_error(SS_ERR_ARG, "bank_push on a shard: use ss_bank_write with the global head");
  if (n == 0) return SS_OK;
  int64_t skip = n > h->cap ? n - h->cap : 0;
  int rc = launch_bank_write(h->emb, h->inv, h->lens, h->seq, h->len_cnt, h->dim, emb, 1, inv_norm,
                             lens, nullptr, nullptr, n, h->head, h->cap, skip, h->d_err,
                             (cudaStream_t)stream, nullptr, h->wp.flag ? &h->wp : nullptr, h->ibnd);
  if (rc) return rc;
  h->head += n;
  return SS_OK;
}

int ss_bank_write(ss_bank_t* h, const int8_t* emb, const float* inv_norm, const int32_t* lens,
                  const int64_t* seq, const int64_t* local_slot, int64_t n, void* stream) {
  if (!h || n < 0 || !seq || !local_slot) return set_error(SS_ERR_ARG, "bank_write: bad args");
  return launch_bank_write(h->emb, h->inv, h->lens, h->seq, h->len_cnt, h->dim, emb, 1, inv_norm,
                           lens, seq, local_slot, n, 0, h->cap, 0, h->d_err, (cudaStream_t)stream,
                           nullptr, h->wp.flag ? &h->wp : nullptr, h->ibnd);
}

static int ensure_wide(ss_bank* h) {
  if (h->wp.flag) return SS_OK;
  DeviceGuard g(h->device);
  WidePlane w;
  cudaError_t e = cudaMalloc(&w.emb, (size_t)h->cap * h->dim * 2);
  if (e == cudaSuccess) e = cudaMalloc(&w.inv, (size_t)h->cap * 4);
  if (e == cudaSuccess) e = cudaMalloc(&w.flag, (size_t)h->cap);
  if (e == cudaSuccess) e = cudaMalloc(&w.count, sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&h->wlist, (size_t)h->cap * 8);
  if (e == cudaSuccess) e = cudaMalloc(&h->wlist_count, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(w.flag, 0, (size_t)h->cap);
  if (e == cudaSuccess) e = cudaMemset(w.count, 0, sizeof(int));
  if (e != cudaSuccess) {
    cudaFree(w.emb); cudaFree(w.inv); cudaFree(w.flag); cudaFree(w.count);
    cudaFree(h->wlist); cudaFree(h->wlist_count);
    h->wlist = nullptr;
    h->wlist_count = nullptr;
    return set_error(SS_ERR_CUDA, "wide plane allocation (%lld rows): %s", (long long)h->cap,
                     cudaGetErrorString(e));
  }
  h->wp = w;
  return SS_OK;
}

// after an int16 write: did any wide row land? (rounds then run the wide pass)
static int note_wide(ss_bank* h, cudaStream_t st) {
  int c = 0;
  SS_CUDA_TRY(cudaMemcpyAsync(&c, h->wp.count, sizeof(int), cudaMemcpyDeviceToHost, st));
  SS_CUDA_TRY(cudaStreamSynchronize(st));
  if (c > 0 && !h->any_wide) {
    h->any_wide = true;
    ++h->ws_gen;  // a captured host round lacks the wide pass: re-capture
  }
  return SS_OK;
}

int ss_bank_push16(ss_bank_t* h, const int16_t* emb, const float* inv_norm, const int32_t* lens,
                   int64_t n, void* stream) {
  if (!h || n < 0) return set_error(SS_ERR_ARG, "bank_push16: bad args");
  if (h->gcap != h->cap || h->slot_offset != 0)
    return set_error(SS_ERR_ARG, "bank_push16 on a shard: use ss_bank_write16 with the global head");
  if (n == 0) return SS_OK;
  if (int rc = ensure_wide(h)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t skip = n > h->cap ? n - h->cap : 0;
  int rc = launch_bank_write(h->emb, h->inv, h->lens, h->seq, h->len_cnt, h->dim, emb, 2, inv_norm,
                             lens, nullptr, nullptr, n, h->head, h->cap, skip, h->d_err, st,
                             nullptr, &h->wp, h->ibnd);
  if (rc) return rc;
  h->head += n;
  return note_wide(h, st);
}

int ss_bank_write16(ss_bank_t* h, const int16_t* emb, const float* inv_norm, const int32_t* lens,
                    const int64_t* seq, const int64_t* local_slot, int64_t n, void* stream) {
  if (!h || n < 0 || !seq || !local_slot) return set_error(SS_ERR_ARG, "bank_write16: bad args");
  if (n == 0) return SS_OK;
  if (int rc = ensure_wide(h)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = launch_bank_write(h->emb, h->inv, h->lens, h->seq, h->len_cnt, h->dim, emb, 2, inv_norm,
                             lens, seq, local_slot, n, 0, h->cap, 0, h->d_err, st, nullptr, &h->wp,
                             h->ibnd);
  if (rc) return rc;
  return note_wide(h, st);
}

int ss_bank_set_head(ss_bank_t* h, int64_t global_head) {
  if (!h || global_head < 0) return set_error(SS_ERR_ARG, "bank_set_head: bad args");
  h->head = global_head;
  return SS_OK;
}

int ss_bank_info(ss_bank_t* h, int64_t* head, int64_t* size, int64_t* capacity, int32_t* dim) {
  if (!h) return set_error(SS_ERR_ARG, "null bank");
  if (head) *head = h->head;
  if (size) *size = h->head < h->gcap ? h->head : h->gcap;
  if (capacity) *capacity = h->cap;
  if (dim) *dim = h->dim;
  return SS_OK;
}

int ss_bank_device_ptrs(ss_bank_t* h, int8_t** emb, float** inv_norm, int32_t** lens,
                        int64_t** seq) {
  if (!h) return set_error(SS_ERR_ARG, "null bank");
  if (emb) *emb = h->emb;
  if (inv_norm) *inv_norm = h->inv;
  if (lens) *lens = h->lens;
  if (seq) *seq = h->seq;
  return SS_OK;
}

int ss_bank_sync_check(ss_bank_t* h, void* stream) {
  if (!h) return set_error(SS_ERR_ARG, "null bank");
  DeviceGuard g(h->device);
  int e = read_and_clear(h->d_err, (cudaStream_t)stream);
  if (e == SS_ERR_RANGE) return set_error(SS_ERR_RANGE, "bank: a pushed length lies outside [1, 65535]");
  if (e == SS_ERR_ARG) return set_error(SS_ERR_ARG, "bank: a write targeted a slot outside the shard");
  return e;
}

static int check_bins(int32_t max_len, int32_t nbins) {
  if (max_len < 1 || nbins < 1 || max_len % nbins || nbins > 4096)
    return set_error(SS_ERR_ARG, "max_len (%d) must be a positive multiple of nbins (%d <= 4096)",
                     max_len, nbins);
  return SS_OK;
}

int ss_bank_fallback_hist(ss_bank_t* h, int32_t max_len, int32_t nbins, int64_t* cnt, int64_t* sv,
                          int64_t* sv2, void* stream) {
  if (!h) return set_error(SS_ERR_ARG, "null bank");
  if (int rc = check_bins(max_len, nbins)) return rc;
  return launch_fallback_hist(h->len_cnt, max_len, nbins, cnt, sv, sv2,
                              (cudaStream_t)stream);
}

// ------------------------------------------------------------- predict ----
static int topk_plan(ss_bank* h, const TopkArgs& a, int32_t& algo, int& slices) {
  bool tc_ok = topk_tc_supported(a);
  if (algo == SS_ALGO_AUTO) algo = tc_ok ? SS_ALGO_TCGEN05 : SS_ALGO_SCAN;
  if (algo == SS_ALGO_TCGEN05 && !tc_ok)
    return set_error(SS_ERR_UNSUPPORTED, "tcgen05 path unsupported for dim=%d k=%d", h->dim, a.k);
  if (algo != SS_ALGO_TCGEN05 && algo != SS_ALGO_SCAN)
    return set_error(SS_ERR_ARG, "unknown similarity algo %d", algo);
  slices = (algo == SS_ALGO_TCGEN05) ? topk_tc_slices(a, h->device) : topk_scan_slices(a, h->device);
  while ((int64_t)slices * a.k > 16384 && slices > 1) slices = (slices + 1) / 2;
  return SS_OK;
}

// the wide pass runs when the bank holds (or held) a wide row or the batch
// has wide queries: one more candidate list per query
static bool wide_on(const ss_bank* h, const WideQ& wq) { return h->any_wide || wq.n > 0; }

static WideBank wide_bank(ss_bank* h) {
  WideBank b;
  b.any = h->any_wide;
  b.plane = h->wp;
  b.list = h->wlist;
  b.list_count = h->wlist_count;
  b.bank_lens = h->lens;
  return b;
}

// workspace after the round buffers: [partials: (slices + wide) lists][wide pass scratch]
static size_t topk_ws_need(ss_bank* h, int64_t nq, int32_t k, int32_t algo, const WideQ& wq) {
  TopkArgs a{nullptr, nullptr, nq, h->emb, h->inv, h->cap, h->dim, k, 0.f, h->head, h->gcap,
             h->slot_offset};
  a.inv_padded = true;  // the bank pads inv with one NaN tile
  a.ibnd = h->ibnd;
  int slices = 1;
  if (topk_plan(h, a, algo, slices)) return 0;
  const bool wide = wide_on(h, wq);
  size_t b = align_up((size_t)(slices + (wide ? 1 : 0)) * nq * k * 8);
  if (wide) b += align_up((size_t)nq * 4) + wide_ws_bytes(wq, nq, k, h->cap, sm_count(h->device));
  return b;
}

// q_inv with the wide queries' entries set to NaN (the tensor-core kernels
// must not score their int8 stand-in rows)
__global__ void k_mask_qinv(const float* __restrict__ src, int64_t nq, float* __restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nq;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
__global__ void k_mask_qinv_set(const int64_t* __restrict__ idx, int64_t n, float* __restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[idx[i]] = __int_as_float(0x7fc00000);
}

// stage 1 (+ the wide pass) into `partials` [lists][nq][k]; returns the list count
static int stage1(ss_bank* h, TopkArgs& a, int32_t algo, int slices, const WideQ& wq,
                  uint64_t* partials, char* scratch, cudaStream_t st, int* nlists) {
  const bool wide = wide_on(h, wq);
  *nlists = slices + (wide ? 1 : 0);
  if (wide && wq.n > 0) {
    float* qinv = reinterpret_cast<float*>(scratch);
    scratch += align_up((size_t)a.nq * 4);
    count_launch();
    k_mask_qinv<<<(unsigned)std::min<int64_t>((a.nq + 255) / 256, 1024), 256, 0, st>>>(a.q_inv, a.nq,
                                                                                    qinv);
    count_launch();
    k_mask_qinv_set<<<(unsigned)((wq.n + 255) / 256), 256, 0, st>>>(wq.idx, wq.n, qinv);
    SS_LAUNCH_CHECK();
    a.q_inv = qinv;
  } else if (wide) {
    scratch += align_up((size_t)a.nq * 4);
  }
  int rc = (algo == SS_ALGO_TCGEN05) ? launch_topk_tc(a, partials, slices, st)
                                     : launch_topk_scan(a, partials, slices, st);
  if (rc || !wide) return rc;
  return launch_wide_pass(wide_bank(h), a, wq, partials + (size_t)slices * a.nq * a.k, scratch,
                          h->device, st);
}

static int topk_impl(ss_bank* h, const int8_t* q, const float* q_inv, int64_t nq, int32_t k,
                     float theta, int32_t algo, uint64_t* out_comp, int32_t* out_len,
                     size_t ws_offset, cudaStream_t st, const PeerOut* po = nullptr,
                     const WideQ& wq = WideQ{}) {
  if (k < 1 || k > 256) return set_error(SS_ERR_ARG, "k must lie in [1, 256], got %d", k);
  if (nq < 0) return set_error(SS_ERR_ARG, "nq < 0");
  if (nq == 0) return SS_OK;
  TopkArgs a{q, q_inv, nq, h->emb, h->inv, h->cap, h->dim, k, theta, h->head, h->gcap,
             h->slot_offset};
  a.inv_padded = true;  // the bank pads inv with one NaN tile
  a.ibnd = h->ibnd;
  a.qscratch = h->qscratch;
  int slices = 1;
  if (int rc = topk_plan(h, a, algo, slices)) return rc;
  if (int rc = ws_reserve(h, ws_offset + topk_ws_need(h, nq, k, algo, wq))) return rc;
  a.gslots = gslots_reserve(h, nq, theta);  // after any workspace move
  const bool wide = wide_on(h, wq);
  uint64_t* partials = reinterpret_cast<uint64_t*>((char*)h->ws + ws_offset);
  char* scratch = (char*)partials + align_up((size_t)(slices + (wide ? 1 : 0)) * nq * k * 8);
  int nlists = slices;
  if (int rc = stage1(h, a, algo, slices, wq, partials, scratch, st, &nlists)) return rc;
  return launch_merge(partials, nullptr, nlists, nq, k, out_comp, out_len, h->lens, h->head,
                      h->gcap, h->slot_offset, st, po);
}

int ss_topk(ss_bank_t* h, const int8_t* q, const float* q_inv, int64_t nq, int32_t k, float theta,
            int32_t algo, uint64_t* out_comp, int32_t* out_len, void* stream) {
  if (!h || !out_comp || !out_len) return set_error(SS_ERR_ARG, "topk: null args");
  return topk_impl(h, q, q_inv, nq, k, theta, algo, out_comp, out_len, 0, (cudaStream_t)stream);
}

static int wide_q(int64_t n_wide, const int64_t* idx, const int16_t* wq, const float* winv,
                  WideQ* out) {
  if (n_wide < 0 || (n_wide > 0 && (!idx || !wq || !winv)))
    return set_error(SS_ERR_ARG, "wide queries: bad args (n=%lld)", (long long)n_wide);
  out->n = n_wide;
  out->idx = idx;
  out->q = wq;
  out->inv = winv;
  return SS_OK;
}

int ss_topk_wide(ss_bank_t* h, const int8_t* q, const float* q_inv, int64_t nq, int64_t n_wide,
                 const int64_t* wide_idx, const int16_t* wide_q_emb, const float* wide_q_inv,
                 int32_t k, float theta, int32_t algo, uint64_t* out_comp, int32_t* out_len,
                 void* stream) {
  if (!h || !out_comp || !out_len) return set_error(SS_ERR_ARG, "topk_wide: null args");
  WideQ wq;
  if (int rc = wide_q(n_wide, wide_idx, wide_q_emb, wide_q_inv, &wq)) return rc;
  return topk_impl(h, q, q_inv, nq, k, theta, algo, out_comp, out_len, 0, (cudaStream_t)stream,
                   nullptr, wq);
}

int ss_topk_scatter(ss_bank_t* h, const int8_t* q, const float* q_inv, int64_t nq, int32_t k,
                    float theta, int32_t algo, int32_t world, int32_t rank,
                    uint64_t* const* peer_comp_host, int32_t* const* peer_len_host,
                    void* stream) {
  if (!h || !peer_comp_host || !peer_len_host) return set_error(SS_ERR_ARG, "topk_scatter: null args");
  if (world < 1 || world > SS_MAX_PEERS || rank < 0 || rank >= world || nq % world)
    return set_error(SS_ERR_ARG, "topk_scatter: bad world/rank/nq (%d, %d, %lld)", world, rank,
                     (long long)nq);
  PeerOut po{};
  po.world = world;
  po.rank = rank;
  po.nq_local = nq / world;
  for (int r = 0; r < world; ++r) {
    if (!peer_comp_host[r] || !peer_len_host[r])
      return set_error(SS_ERR_ARG, "topk_scatter: null receive buffer of rank %d", r);
    po.comp[r] = peer_comp_host[r];
    po.len[r] = peer_len_host[r];
  }
  return topk_impl(h, q, q_inv, nq, k, theta, algo, nullptr, nullptr, 0, (cudaStream_t)stream, &po);
}

int ss_topk_gather(ss_bank_t* h, const int8_t* q, const float* q_inv, int64_t nq, int32_t k,
                   float theta, int32_t algo, int32_t world, int32_t rank, uint64_t* owner_comp,
                   int32_t* owner_len, void* stream) {
  if (!h || !owner_comp || !owner_len) return set_error(SS_ERR_ARG, "topk_gather: null args");
  if (world < 1 || rank < 0 || rank >= world || nq < 0)
    return set_error(SS_ERR_ARG, "topk_gather: bad world/rank/nq (%d, %d, %lld)", world, rank,
                     (long long)nq);
  if (nq == 0) return SS_OK;
  // every query belongs to the one owner: owner index q / nq == 0 in the merge
  // kernel's exchange epilogue, row [rank][q] of the owner's buffer
  PeerOut po{};
  po.world = world;
  po.rank = rank;
  po.nq_local = nq;
  po.comp[0] = owner_comp;
  po.len[0] = owner_len;
  return topk_impl(h, q, q_inv, nq, k, theta, algo, nullptr, nullptr, 0, (cudaStream_t)stream, &po);
}

int ss_ipc_malloc(int32_t device, int64_t bytes, void** out) {
  if (!out || bytes <= 0) return set_error(SS_ERR_ARG, "ipc_malloc: bad args");
  int prev = 0;
  SS_CUDA_TRY(cudaGetDevice(&prev));
  SS_CUDA_TRY(cudaSetDevice(device));
  cudaError_t e = cudaMalloc(out, (size_t)bytes);  // plain cudaMalloc: IPC-exportable
  if (e == cudaSuccess) e = cudaMemset(*out, 0, (size_t)bytes);
  cudaSetDevice(prev);  // the caller's current device is left as it was
  if (e != cudaSuccess) return set_error(SS_ERR_CUDA, "ipc_malloc: %s", cudaGetErrorString(e));
  return SS_OK;
}

int ss_ipc_free(void* ptr) {
  if (ptr) SS_CUDA_TRY(cudaFree(ptr));
  return SS_OK;
}

int ss_ipc_handle(const void* ptr, uint8_t* handle_host) {
  if (!ptr || !handle_host) return set_error(SS_ERR_ARG, "ipc_handle: null args");
  static_assert(sizeof(cudaIpcMemHandle_t) == SS_IPC_HANDLE_BYTES, "IPC handle size");
  cudaIpcMemHandle_t hd;
  SS_CUDA_TRY(cudaIpcGetMemHandle(&hd, const_cast<void*>(ptr)));
  memcpy(handle_host, &hd, sizeof(hd));
  return SS_OK;
}

int ss_ipc_open(const uint8_t* handle_host, void** out) {
  if (!handle_host || !out) return set_error(SS_ERR_ARG, "ipc_open: null args");
  cudaIpcMemHandle_t hd;
  memcpy(&hd, handle_host, sizeof(hd));
  SS_CUDA_TRY(cudaIpcOpenMemHandle(out, hd, cudaIpcMemLazyEnablePeerAccess));
  return SS_OK;
}

int ss_ipc_close(void* ptr) {
  if (ptr) SS_CUDA_TRY(cudaIpcCloseMemHandle(ptr));
  return SS_OK;
}

int ss_query_similar(ss_bank_t* h, const int16_t* q, float q_inv, float theta, float* out_key,
                     int64_t* out_seq, int32_t* out_len, int64_t* n_out, void* stream) {
  if (!h || !q || !out_key || !out_seq || !out_len || !n_out)
    return set_error(SS_ERR_ARG, "query_similar: null args");
  *n_out = 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t cap = h->cap;
  // workspace: G f64[cap] | id i64[cap] | perm i64[cap] | count | rank ws
  const size_t oG = 0, oid = align_up((size_t)cap * 8), operm = oid + align_up((size_t)cap * 8),
               ocnt = operm + align_up((size_t)cap * 8), orank = ocnt + 256,
               end = orank + align_up((size_t)rank_workspace_bytes(cap));
  if (int rc = ws_reserve(h, end)) return rc;
  char* w = (char*)h->ws;
  TopkArgs a{nullptr, nullptr, 1, h->emb, h->inv, h->cap, h->dim, 1, theta, h->head, h->gcap,
             h->slot_offset};
  double* G = reinterpret_cast<double*>(w + oG);
  int64_t* id = reinterpret_cast<int64_t*>(w + oid);
  int64_t* perm = reinterpret_cast<int64_t*>(w + operm);
  int* cnt = reinterpret_cast<int*>(w + ocnt);
  if (int rc = launch_query_all(a, h->seq, wide_bank(h), q, q_inv, G, id, cnt, st)) return rc;
  int m = 0;
  SS_CUDA_TRY(cudaMemcpyAsync(&m, cnt, sizeof(int), cudaMemcpyDeviceToHost, st));
  SS_CUDA_TRY(cudaStreamSynchronize(st));
  if (m > 0) {
    if (int rc = launch_rank(G, id, m, perm, w + orank, (int64_t)rank_workspace_bytes(m), st)) return rc;
    if (int rc = launch_query_gather(G, id, perm, m, h->seq, h->lens, a, out_key, out_seq, out_len, st))
      return rc;
    SS_CUDA_TRY(cudaStreamSynchronize(st));
  }
  *n_out = m;
  return SS_OK;
}

int ss_topk_partials(ss_bank_t* h, const int8_t* q, const float* q_inv, int64_t nq, int32_t k,
                     float theta, int32_t algo, uint64_t* partials, int32_t max_slices,
                     int32_t* n_slices, void* stream) {
  if (!h || !partials || !n_slices) return set_error(SS_ERR_ARG, "topk_partials: null args");
  if (k < 1 || k > 256 || nq < 0) return set_error(SS_ERR_ARG, "topk_partials: bad k/nq");
  TopkArgs a{q, q_inv, nq, h->emb, h->inv, h->cap, h->dim, k, theta, h->head, h->gcap,
             h->slot_offset};
  a.inv_padded = true;  // the bank pads inv with one NaN tile
  a.ibnd = h->ibnd;
  a.gslots = gslots_reserve(h, nq, theta);
  a.qscratch = h->qscratch;
  int slices = 1;
  if (int rc = topk_plan(h, a, algo, slices)) return rc;
  if (slices > max_slices) slices = max_slices;
  if (slices < 1) return set_error(SS_ERR_ARG, "topk_partials: max_slices < 1");
  *n_slices = slices;
  if (nq == 0) return SS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  return (algo == SS_ALGO_TCGEN05) ? launch_topk_tc(a, partials, slices, st)
                                   : launch_topk_scan(a, partials, slices, st);
}

int ss_merge_topk(const uint64_t* comp, const int32_t* len, int32_t nlists, int64_t nq, int32_t k,
                  uint64_t* out_comp, int32_t* out_len, void* stream) {
  if (nlists < 1 || k < 1 || k > 256 || nq < 0 || !len)
    return set_error(SS_ERR_ARG, "merge_topk: bad args");
  return launch_merge(comp, len, nlists, nq, k, out_comp, out_len, nullptr, 0, 1, 0,
                      (cudaStream_t)stream);
}

int ss_decode_topk(const uint64_t* comp, int64_t n, int64_t head, int64_t capacity, float* out_key,
                   int64_t* out_seq, int64_t* out_slot, void* stream) {
  if (n < 0 || capacity < 1) return set_error(SS_ERR_ARG, "decode: bad args");
  return launch_decode(comp, n, head, capacity, out_key, out_seq, out_slot, (cudaStream_t)stream);
}

int ss_finish(const uint64_t* comp, const int32_t* len, int64_t nq, int32_t k,
              int32_t min_matches, int32_t max_len, int32_t nbins, const int32_t* input_len,
              const int64_t* fb_cnt, const int64_t* fb_sv, const int64_t* fb_sv2, int32_t P,
              int32_t* npts, int32_t* pbin, int32_t* pcnt, int64_t* pD, int64_t* psv,
              uint8_t* used_fb, double* G, void* stream) {
  if (int rc = check_bins(max_len, nbins)) return rc;
  if (P < nbins) return set_error(SS_ERR_ARG, "P (%d) must be >= nbins (%d)", P, nbins);
  if (k < 1 || min_matches < 0 || nq < 0) return set_error(SS_ERR_ARG, "finish: bad args");
  return launch_finish(comp, len, nq, k, min_matches, max_len, nbins, input_len, fb_cnt, fb_sv,
                       fb_sv2, P, npts, pbin, pcnt, pD, psv, used_fb, G, (cudaStream_t)stream);
}

int ss_refresh(int64_t n, const int32_t* input_len, const int32_t* g_new, int32_t* bucket_io,
               int32_t bucket_size, const int32_t* npts, const int32_t* pcnt, const int64_t* pD,
               int32_t P, double* G_io, uint8_t* refreshed, int32_t force, void* stream) {
  if (n < 0 || bucket_size < 1 || P < 1) return set_error(SS_ERR_ARG, "refresh: bad args");
  return launch_refresh(n, input_len, g_new, bucket_io, bucket_size, npts, pcnt, pD, P, G_io,
                        refreshed, force, (cudaStream_t)stream);
}

int64_t ss_rank_workspace_bytes(int64_t n) { return rank_workspace_bytes(n); }

int ss_rank(const double* G, const int64_t* ids, int64_t n, int64_t* perm, void* workspace,
            int64_t workspace_bytes, void* stream) {
  if (n < 0) return set_error(SS_ERR_ARG, "rank: n < 0");
  return launch_rank(G, ids, n, perm, workspace, workspace_bytes, (cudaStream_t)stream);
}

int ss_pack_batch(const int64_t* perm, const int32_t* input_len, const int32_t* g, int64_t n,
                  int64_t kv_capacity, int32_t max_batch, int32_t mode, int64_t* out_batch,
                  int32_t* out_count, int64_t* out_tokens, void* stream) {
  if (n < 0 || kv_capacity < 1 || max_batch < 1 || (mode != SS_PACK_CUT && mode != SS_PACK_SKIP))
    return set_error(SS_ERR_ARG, "pack_batch: bad args (n=%lld K=%lld B=%d mode=%d)",
                     (long long)n, (long long)kv_capacity, max_batch, mode);
  if (!perm && n > 0) return set_error(SS_ERR_ARG, "pack_batch: perm is null");
  return launch_pack_batch(perm, input_len, g, n, kv_capacity, max_batch, mode, out_batch,
                           out_count, out_tokens, (cudaStream_t)stream);
}

// ----------------------------------------------------------- fused round --
// workspace layout: [topk partials ...][comp nq*k][len nq*k][fb 3*nbins][rank ws][host-round bufs]
struct RoundLayout {
  size_t comp, len, fb, rank, end;
};
static RoundLayout round_layout(int64_t nq, int k, int nbins) {
  RoundLayout L;
  size_t o = 0;
  L.comp = o; o += align_up((size_t)nq * k * 8);
  L.len = o; o += align_up((size_t)nq * k * 4);
  L.fb = o; o += align_up((size_t)3 * nbins * 8);
  L.rank = o; o += align_up((size_t)rank_workspace_bytes(nq));
  L.end = o;
  return L;
}

static int round_impl(ss_bank* h, const int8_t* q, const float* q_inv, const int32_t* input_len,
                      const int64_t* ids, int64_t nq, int32_t k, float theta, int32_t min_matches,
                      int32_t max_len, int32_t nbins, int32_t algo, int32_t P, int32_t* npts,
                      int32_t* pbin, int32_t* pcnt, int64_t* pD, uint8_t* used_fb, double* G,
                      int64_t* perm, size_t extra_front, cudaStream_t st, bool do_rank = true,
                      double* G_mirror = nullptr, const WideQ& wq = WideQ{}) {
  if (int rc = check_bins(max_len, nbins)) return rc;
  if (P < nbins) return set_error(SS_ERR_ARG, "P (%d) must be >= nbins (%d)", P, nbins);
  if (h->head <= 0) return set_error(SS_ERR_EMPTY, "cold start: the history window is empty");
  if (nq == 0) return SS_OK;
  RoundLayout L = round_layout(nq, k, nbins);
  size_t base = extra_front;
  if (int rc = ws_reserve(h, base + L.end + topk_ws_need(h, nq, k, algo, wq))) return rc;
  char* ws = (char*)h->ws + base;
  uint64_t* comp = reinterpret_cast<uint64_t*>(ws + L.comp);
  int32_t* len = reinterpret_cast<int32_t*>(ws + L.len);
  int64_t* fb = reinterpret_cast<int64_t*>(ws + L.fb);
  // stage 1: similarity kernel writes per-slice partial top-k lists, which
  // live after the round buffers; merge + stages 1b-3 run fused per request
  if (k < 1 || k > 256) return set_error(SS_ERR_ARG, "k must lie in [1, 256], got %d", k);
  TopkArgs a{q, q_inv, nq, h->emb, h->inv, h->cap, h->dim, k, theta, h->head, h->gcap,
             h->slot_offset};
  a.inv_padded = true;  // the bank pads inv with one NaN tile
  a.ibnd = h->ibnd;
  a.gslots = gslots_reserve(h, nq, theta);
  a.qscratch = h->qscratch;
  int slices = 1;
  if (int rc = topk_plan(h, a, algo, slices)) return rc;
  uint64_t* partials = reinterpret_cast<uint64_t*>((char*)h->ws + base + L.end);
  char* scratch = (char*)partials + align_up((size_t)(slices + (wide_on(h, wq) ? 1 : 0)) * nq * k * 8);
  // fork: the window's fallback law (1 CTA) overlaps the similarity kernel,
  // which leaves SMs free (slices x query tiles <= the SM count)
  SS_CUDA_TRY(cudaEventRecord(h->ev_fork, st));
  SS_CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev_fork, 0));
  int rc = launch_fallback_hist(h->len_cnt, max_len, nbins, fb, fb + nbins, fb + 2 * nbins, h->side);
  if (rc) return rc;
  SS_CUDA_TRY(cudaEventRecord(h->ev_join, h->side));
  int nlists = slices;
  rc = stage1(h, a, algo, slices, wq, partials, scratch, st, &nlists);
  SS_CUDA_TRY(cudaStreamWaitEvent(st, h->ev_join, 0));  // join before any early return
  if (rc) return rc;
  rc = launch_merge_finish(partials, nlists, nq, k, h->lens, h->head, h->gcap, h->slot_offset, comp,
                           len, min_matches, max_len, nbins, input_len, fb, fb + nbins,
                           fb + 2 * nbins, P, npts, pbin, pcnt, pD, nullptr, used_fb, G, st,
                           G_mirror);
  if (rc) return rc;
  if (!do_rank) return SS_OK;
  return launch_rank(G, ids, nq, perm, ws + L.rank, (int64_t)rank_workspace_bytes(nq), st);
}



int ss_schedule_round(ss_bank_t* h, const int8_t* q, const float* q_inv, const int32_t* input_len,
                      const int64_t* ids, int64_t nq, int32_t k, float theta, int32_t min_matches,
                      int32_t max_len, int32_t nbins, int32_t algo, int32_t P, int32_t* npts,
                      int32_t* pbin, int32_t* pcnt, int64_t* pD, uint8_t* used_fb, double* G,
                      int64_t* perm, void* stream) {
  if (!h) return set_error(SS_ERR_ARG, "null bank");
  return round_impl(h, q, q_inv, input_len, ids, nq, k, theta, min_matches, max_len, nbins, algo, P,
                    npts, pbin, pcnt, pD, used_fb, G, perm, 0, (cudaStream_t)stream);
}

int ss_schedule_round_wide(ss_bank_t* h, const int8_t* q, const float* q_inv,
                           const int32_t* input_len, const int64_t* ids, int64_t nq, int64_t n_wide,
                           const int64_t* wide_idx, const int16_t* wide_q_emb,
                           const float* wide_q_inv, int32_t k, float theta, int32_t min_matches,
                           int32_t max_len, int32_t nbins, int32_t algo, int32_t P, int32_t* npts,
                           int32_t* pbin, int32_t* pcnt, int64_t* pD, uint8_t* used_fb, double* G,
                           int64_t* perm, void* stream) {
  if (!h) return set_error(SS_ERR_ARG, "null bank");
  WideQ wq;
  if (int rc = wide_q(n_wide, wide_idx, wide_q_emb, wide_q_inv, &wq)) return rc;
  return round_impl(h, q, q_inv, input_len, ids, nq, k, theta, min_matches, max_len, nbins, algo, P,
                    npts, pbin, pcnt, pD, used_fb, G, perm, 0, (cudaStream_t)stream, true, nullptr,
                    wq);
}

static bool is_pinned(const void* p) {
  if (!p) return true;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// device address of pinned (page-locked, mapped) host memory; nullptr otherwise
static void* mapped_ptr(void* p) {
  if (!p) return nullptr;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

// H2D of the inputs, the fused round, D2H of G and perm -- all enqueued on st
static int host_round_enqueue(ss_bank* h, const int8_t* q_host, const float* q_inv_host,
                              const int32_t* input_len_host, const int64_t* ids_host, int64_t nq,
                              int32_t k, float theta, int32_t min_matches, int32_t max_len,
                              int32_t nbins, int32_t algo, double* G_host, int64_t* perm_host,
                              cudaStream_t st) {
  const int P = nbins;
  // front region: device copies of the inputs and the per-request state
  size_t o = 0;
  size_t oq = o; o += align_up((size_t)nq * h->dim);
  size_t oqi = o; o += align_up((size_t)nq * 4);
  size_t oI = o; o += align_up((size_t)nq * 4);
  size_t oid = o; o += align_up((size_t)nq * 8);
  size_t onp = o; o += align_up((size_t)nq * 4);
  size_t opb = o; o += align_up((size_t)nq * P * 4);
  size_t opc = o; o += align_up((size_t)nq * P * 4);
  size_t opD = o; o += align_up((size_t)nq * P * 8);
  size_t ofb = o; o += align_up((size_t)nq);
  size_t oG = o; o += align_up((size_t)nq * 8);
  size_t operm = o; o += align_up((size_t)nq * 8);
  RoundLayout L = round_layout(nq, k, nbins);
  if (int rc = ws_reserve(h, o + L.end + topk_ws_need(h, nq, k, algo, WideQ{}))) return rc;
  char* w = (char*)h->ws;
  // inputs: when every host buffer is pinned (mapped), one kernel reads them
  // straight from host memory (one launch instead of four copy-engine nodes:
  // the call is 8 us shorter per round at c2, scripts/time_e2e.py); pageable
  // buffers go through cudaMemcpyAsync
  const void* q_m = mapped_ptr(const_cast<int8_t*>(q_host));
  const void* qi_m = mapped_ptr(const_cast<float*>(q_inv_host));
  const void* I_m = mapped_ptr(const_cast<int32_t*>(input_len_host));
  const void* id_m = ids_host ? mapped_ptr(const_cast<int64_t*>(ids_host)) : nullptr;
  if (q_m && qi_m && I_m && (id_m || !ids_host)) {
    GatherSegs g{};
    g.src[0] = q_m; g.dst[0] = w + oq; g.bytes[0] = nq * h->dim;
    g.src[1] = qi_m; g.dst[1] = w + oqi; g.bytes[1] = nq * 4;
    g.src[2] = I_m; g.dst[2] = w + oI; g.bytes[2] = nq * 4;
    g.n = 3;
    if (ids_host) { g.src[3] = id_m; g.dst[3] = w + oid; g.bytes[3] = nq * 8; g.n = 4; }
    if (int rc = launch_h2d_gather(g, st)) return rc;
  } else {
    SS_CUDA_TRY(cudaMemcpyAsync(w + oq, q_host, (size_t)nq * h->dim, cudaMemcpyHostToDevice, st));
    SS_CUDA_TRY(cudaMemcpyAsync(w + oqi, q_inv_host, (size_t)nq * 4, cudaMemcpyHostToDevice, st));
    SS_CUDA_TRY(cudaMemcpyAsync(w + oI, input_len_host, (size_t)nq * 4, cudaMemcpyHostToDevice, st));
    if (ids_host)
      SS_CUDA_TRY(cudaMemcpyAsync(w + oid, ids_host, (size_t)nq * 8, cudaMemcpyHostToDevice, st));
  }
  // pinned perm buffer: the rank kernel stores the order straight into host
  // memory (one D2H copy node fewer per round)
  int64_t* perm_dev = static_cast<int64_t*>(mapped_ptr(perm_host));
  double* G_dev = static_cast<double*>(mapped_ptr(G_host));  // finish mirrors G into it
  int rc = round_impl(h, (const int8_t*)(w + oq), (const float*)(w + oqi), (const int32_t*)(w + oI),
                      ids_host ? (const int64_t*)(w + oid) : nullptr, nq, k, theta, min_matches,
                      max_len, nbins, algo, P, (int32_t*)(w + onp), (int32_t*)(w + opb),
                      (int32_t*)(w + opc), (int64_t*)(w + opD), (uint8_t*)(w + ofb),
                      (double*)(w + oG), perm_dev ? perm_dev : (int64_t*)(w + operm), o, st, true,
                      G_dev);
  if (rc) return rc;
  w = (char*)h->ws;
  if (G_host && !G_dev) SS_CUDA_TRY(cudaMemcpyAsync(G_host, w + oG, (size_t)nq * 8, cudaMemcpyDeviceToHost, st));
  if (perm_host && !perm_dev)
    SS_CUDA_TRY(cudaMemcpyAsync(perm_host, w + operm, (size_t)nq * 8, cudaMemcpyDeviceToHost, st));
  return SS_OK;
}

int ss_schedule_round_host(ss_bank_t* h, const int8_t* q_host, const float* q_inv_host,
                           const int32_t* input_len_host, const int64_t* ids_host, int64_t nq,
                           int32_t k, float theta, int32_t min_matches, int32_t max_len,
                           int32_t nbins, int32_t algo, double* G_host, int64_t* perm_host,
                           void* stream) {
  if (!h || nq < 0) return set_error(SS_ERR_ARG, "round_host: bad args");
  if (nq == 0) return SS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  ss_bank::HostRoundKey key;
  memset(&key, 0, sizeof(key));
  key.nq = nq; key.head = h->head; key.k = k; key.min_matches = min_matches;
  key.max_len = max_len; key.nbins = nbins; key.algo = algo; key.theta = theta;
  key.any_wide = h->any_wide;
  const void* ptrs[6] = {q_host, q_inv_host, input_len_host, ids_host, G_host, perm_host};
  memcpy(key.ptr, ptrs, sizeof(ptrs));
  key.ws_gen = h->ws_gen;
  // 3rd+ identical call: one graph launch (H2D + round + D2H nodes)
  if (h->host_exec && key == h->exec_key) {
    SS_CUDA_TRY(cudaGraphLaunch(h->host_exec, st));
    SS_CUDA_TRY(cudaStreamSynchronize(st));
    return SS_OK;
  }
  const bool repeat = h->have_last && key == h->last_key;
  if (int rc = host_round_enqueue(h, q_host, q_inv_host, input_len_host, ids_host, nq, k, theta,
                                  min_matches, max_len, nbins, algo, G_host, perm_host, st))
    return rc;
  SS_CUDA_TRY(cudaStreamSynchronize(st));
  key.ws_gen = h->ws_gen;  // the eager call may have grown the workspace
  h->last_key = key;
  h->have_last = true;
  // the same call twice in a row (the workspace now fits it): capture it on a
  // private stream so later calls replay one graph.  Pageable host buffers
  // stay on the eager path.
  if (repeat && is_pinned(q_host) && is_pinned(q_inv_host) && is_pinned(input_len_host) &&
      is_pinned(ids_host) && is_pinned(G_host) && is_pinned(perm_host)) {
    if (!h->cap_stream && cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking) != cudaSuccess) {
      cudaGetLastError();
      return SS_OK;
    }
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      cudaGetLastError();
      return SS_OK;
    }
    const uint64_t gen0 = h->ws_gen;
    int rc = host_round_enqueue(h, q_host, q_inv_host, input_len_host, ids_host, nq, k, theta,
                                min_matches, max_len, nbins, algo, G_host, perm_host, h->cap_stream);
    cudaError_t e = cudaStreamEndCapture(h->cap_stream, &g);
    if (rc == SS_OK && e == cudaSuccess && g && h->ws_gen == gen0) {
      cudaGraphExec_t ex = nullptr;
      if (cudaGraphInstantiate(&ex, g, 0) == cudaSuccess) {
        if (h->host_exec) cudaGraphExecDestroy(h->host_exec);
        h->host_exec = ex;
        h->exec_key = key;
      }
    }
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();  // a failed capture leaves the eager path in place
  }
  return SS_OK;
}

}  // extern "C"

namespace ss {
int predict_into(ss_bank* h, const int8_t* q, const float* q_inv, const int32_t* input_len,
                 int64_t nq, int32_t k, float theta, int32_t min_matches, int32_t max_len,
                 int32_t nbins, int32_t algo, int32_t P, int32_t* npts, int32_t* pbin,
                 int32_t* pcnt, int64_t* pD, uint8_t* used_fb, double* G, cudaStream_t st) {
  return round_impl(h, q, q_inv, input_len, nullptr, nq, k, theta, min_matches, max_len, nbins,
                    algo, P, npts, pbin, pcnt, pD, used_fb, G, nullptr, 0, st, false);
}
int bank_push_gather(ss_bank* h, const int8_t* src_emb, const float* src_inv,
                     const int32_t* src_lens, const int64_t* src_idx, int64_t n, cudaStream_t st) {
  if (h->gcap != h->cap || h->slot_offset != 0)
    return set_error(SS_ERR_ARG, "push on a shard: use ss_bank_write with the global head");
  if (n <= 0) return SS_OK;
  const int64_t skip = n > h->cap ? n - h->cap : 0;
  int rc = launch_bank_write(h->emb, h->inv, h->lens, h->seq, h->len_cnt, h->dim, src_emb, 1,
                             src_inv, src_lens, nullptr, nullptr, n, h->head, h->cap, skip,
                             h->d_err, st, src_idx, h->wp.flag ? &h->wp : nullptr, h->ibnd);
  if (rc) return rc;
  h->head += n;
  return SS_OK;
}
}  // namespace ss

