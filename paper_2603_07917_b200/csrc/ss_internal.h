// Internal (non-ABI) declarations shared between the kernel files and the
// C-ABI layer in ss_api.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

struct ss_bank;  // the C-ABI bank handle (include/sagesched.h: ss_bank_t)

namespace ss {

void count_launch();

// opt `kern` in to `dyn` bytes of dynamic shared memory when its static
// shared memory plus `dyn` exceeds the 48 KB default (the default limit
// covers both)
template <typename... KArgs>
inline cudaError_t ensure_dyn_smem(void (*kern)(KArgs...), size_t dyn) {
  if (dyn == 0) return cudaSuccess;
  cudaFuncAttributes fa{};
  if (cudaError_t e = cudaFuncGetAttributes(&fa, kern)) return e;
  if (fa.sharedSizeBytes + dyn <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
}

// launch `kern` with the programmatic-stream-serialization attribute (PDL):
// its launch overlaps the tail of the previous kernel on the stream; the
// kernel calls pdl_wait() before reading that kernel's outputs
template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
int set_error(int code, const char* fmt, ...);
int sm_count(int device);
// bank slices per query tile for a grid of qtiles x slices CTAs (one CTA per
// SM at a time): the fewest slices >= sms / qtiles whose grid fills its last
// wave to >= 97% (or the best fill up to 64 slices), capped by the tile count
int pick_slices(int64_t qtiles, int64_t tiles, int sms);

int launch_match_pmfs(const float* sims, int64_t nq, int64_t nw, const int64_t* lens,
                      double theta, int64_t max_len, double* sup, double* mas,
                      int64_t* sizes, int64_t out_stride, int* err, cudaStream_t st);
// Per-call slot in mapped pinned memory (64-byte header, then the data):
// the host writes n (and the cost parameters) and the inputs, launches, and
// spins until the kernel sets flag to the call's sequence number.
struct PerCallHdr {
  uint32_t flag;
  int32_t err;
  double result;
  int64_t n;
  double input_len;
  double w_in, w_out;
  int32_t kind;
  int32_t pad[3];
};
static_assert(sizeof(PerCallHdr) == 64, "per-call header is 64 bytes");
constexpr int64_t kPerCallMaxPts = 2048;  // 2 x 2048 doubles of inputs = 32 KB of shared memory
int launch_gittins_percall(PerCallHdr* h_dev, int64_t n, uint32_t seq, cudaStream_t st);
int launch_cost_percall(PerCallHdr* h_dev, uint32_t seq, cudaStream_t st);
constexpr int kGatherSegs = 4;
struct GatherSegs {  // (src, dst, bytes) triples, by value as a kernel parameter
  const void* src[kGatherSegs];
  void* dst[kGatherSegs];
  int64_t bytes[kGatherSegs];
  int n;
};
int launch_h2d_gather(const GatherSegs& g, cudaStream_t st);
int launch_gittins_dist(const double* support, const double* masses, const int64_t* npts,
                        const double* attained, const double* outlived, int64_t n,
                        int64_t stride, double* out, int* err, int ref_mode, cudaStream_t st);
int launch_embed(const int64_t* tokens, const int64_t* offsets, int64_t n, uint64_t salt,
                 int dim, double* out_f64, int16_t* out_i16, float* out_inv, int* err,
                 cudaStream_t st);
int launch_cost_dist(int kind, double w_in, double w_out, const double* I, const double* ls,
                     const int64_t* npts, int64_t n, int64_t stride, double* out,
                     cudaStream_t st);

// The bank's wide plane (lazily allocated on the first int16 push): exact
// int16 vectors of rows whose feature-hash buckets exceed int8, per slot.
struct WidePlane {
  int16_t* emb = nullptr;   // [cap, dim]
  float* inv = nullptr;     // [cap] true inverse norm of a wide row
  uint8_t* flag = nullptr;  // [cap] 1 = the slot holds a wide row
  int* count = nullptr;     // device counter of wide rows written (host reads it after a push)
};

// bank maintenance (k_bank.cu); src_bytes = 1 (int8 rows) or 2 (int16 rows)
int launch_bank_write(int8_t* emb, float* inv, int32_t* lens, int64_t* seq, int32_t* len_cnt,
                      int dim, const void* src_emb, int src_bytes, const float* src_inv,
                      const int32_t* src_lens, const int64_t* src_seq, const int64_t* src_slot,
                      int64_t n, int64_t first_seq, int64_t capacity, int64_t skip, int* err,
                      cudaStream_t st, const int64_t* src_idx = nullptr,
                      const WidePlane* wp = nullptr, float2* ibnd = nullptr);
int launch_fallback_hist(const int32_t* len_cnt, int max_len, int nbins, int64_t* cnt,
                         int64_t* sv, int64_t* sv2, cudaStream_t st);

// wide queries of a batch (feature-hash vectors outside int8): their indices
// in the batch, exact int16 vectors and inverse norms (k_wide.cu)
struct WideQ {
  int64_t n = 0;
  const int64_t* idx = nullptr;  // [n] query indices
  const int16_t* q = nullptr;    // [n, dim]
  const float* inv = nullptr;    // [n]
};
// the bank's side of the wide pass
struct WideBank {
  bool any = false;          // the bank has received a wide row
  WidePlane plane;
  int64_t* list = nullptr;   // [cap] scratch: compacted wide slots
  int* list_count = nullptr;
  const int32_t* bank_lens = nullptr;
};

// similarity + top-k
struct TopkArgs {
  const int8_t* q;
  const float* q_inv;
  int64_t nq;
  const int8_t* emb;
  const float* inv;
  int64_t n_rows;        // local slots scanned [0, n_rows)
  int dim;
  int k;
  float theta;
  int64_t head, gcap, slot_offset;  // rel = (slot_offset + j - head) mod gcap
  // inv is followed by at least one tile (256 floats) of NaN padding, so a
  // whole tile's inverse norms may be bulk-copied (the bank allocates it so)
  bool inv_padded = false;
  // per 16-row group of the bank: (max inverse norm or 0, min inverse norm or
  // +inf) over its non-NaN rows, kept by every bank write (k_bank_bounds) and
  // padded like inv; the TS kernel's per-16-column filter bounds
  const float2* ibnd = nullptr;
  // optional [kMaxShareSlices][nq] scratch for the TS kernel's pure top-k
  // mode: every slice publishes the R-th best key it holds per query, and
  // every slice filters with the minimum over slices (a lower bound of the
  // global k-th key once all have published)
  uint32_t* gslots = nullptr;
  // optional 128 x dim scratch: a single query tile is re-laid out across the
  // four TMEM lane quarters (k_topk_tc `spread`)
  int8_t* qscratch = nullptr;
};
constexpr int kMaxShareSlices = 160;
// pure top-k cascade (launch_topk_ts / launch_topk_tc): the threshold pass's
// theta -- the paper's similarity threshold
constexpr float kCascadeTheta = 0.8f;
int launch_topk_scan(const TopkArgs& a, uint64_t* partials, int n_slices, cudaStream_t st);
int topk_scan_slices(const TopkArgs& a, int device);
int launch_topk_tc(const TopkArgs& a, uint64_t* partials, int n_slices, cudaStream_t st);
int topk_tc_slices(const TopkArgs& a, int device);
bool topk_tc_supported(const TopkArgs& a);
// tcgen05 kernel with the query block in TMEM (k_topk_sm100_ts.cu); one
// partial list per CTA slice
bool topk_ts_supported(const TopkArgs& a);
int topk_ts_lists(const TopkArgs& a, int device);
int launch_topk_ts(const TopkArgs& a, uint64_t* partials, int n_lists, cudaStream_t st);

// the wide pass (k_wide.cu): one more candidate list per query, written to
// list_out [nq][k]; ws of wide_ws_bytes()
size_t wide_ws_bytes(const WideQ& wq, int64_t nq, int k, int64_t n_rows, int sms);
int launch_wide_pass(const WideBank& wb, const TopkArgs& a, const WideQ& wq, uint64_t* list_out,
                     void* ws, int device, cudaStream_t st);

// query_similar of one query over the whole bank (k_wide.cu)
int launch_query_all(const TopkArgs& a, const int64_t* seq, const WideBank& wb, const int16_t* q16,
                     float iq, double* G, int64_t* id, int* count, cudaStream_t st);
int launch_query_gather(const double* G, const int64_t* id, const int64_t* perm, int64_t m,
                        const int64_t* seq, const int32_t* lens, const TopkArgs& a, float* key,
                        int64_t* out_seq, int32_t* out_len, cudaStream_t st);

// Receive buffers of every rank for the fused merge + exchange (k_merge with
// po.world > 0): rank r's [world][nq_local][k] rows, IPC-mapped into this process.
#define SS_MAX_PEERS 8
struct PeerOut {
  uint64_t* comp[SS_MAX_PEERS];
  int32_t* len[SS_MAX_PEERS];
  int64_t nq_local;
  int world;  // 0: plain local output
  int rank;
};
int launch_merge(const uint64_t* comp, const int32_t* len, int nlists, int64_t nq, int k,
                 uint64_t* out_comp, int32_t* out_len, const int32_t* bank_lens,
                 int64_t head, int64_t gcap, int64_t slot_offset, cudaStream_t st,
                 const PeerOut* po = nullptr);
int launch_decode(const uint64_t* comp, int64_t n, int64_t head, int64_t capacity,
                  float* key, int64_t* seq, int64_t* slot, cudaStream_t st);
int launch_finish(const uint64_t* comp, const int32_t* len, int64_t nq, int k,
                  int min_matches, int max_len, int nbins, const int32_t* I,
                  const int64_t* fb_cnt, const int64_t* fb_sv, const int64_t* fb_sv2, int P,
                  int32_t* npts, int32_t* pbin, int32_t* pcnt, int64_t* pD, int64_t* psv,
                  uint8_t* used_fb, double* G, cudaStream_t st);
int launch_merge_finish(const uint64_t* partials, int nlists, int64_t nq, int k,
                        const int32_t* bank_lens, int64_t head, int64_t gcap, int64_t slot_offset,
                        uint64_t* out_comp, int32_t* out_len, int min_matches, int max_len,
                        int nbins, const int32_t* I, const int64_t* fb_cnt, const int64_t* fb_sv,
                        const int64_t* fb_sv2, int P, int32_t* npts, int32_t* pbin, int32_t* pcnt,
                        int64_t* pD, int64_t* psv, uint8_t* used_fb, double* G, cudaStream_t st,
                        double* G_mirror = nullptr);
int launch_refresh(int64_t n, const int32_t* I, const int32_t* g_new, int32_t* bucket_io,
                   int bucket_size, const int32_t* npts, const int32_t* pcnt,
                   const int64_t* pD, int P, double* G_io, uint8_t* refreshed, int force,
                   cudaStream_t st);

// fused stages 1-3 for a batch of pending requests into caller arrays (the
// fused round without its rank), on bank h (ss_api.cu)
int predict_into(ss_bank* h, const int8_t* q, const float* q_inv, const int32_t* input_len,
                 int64_t nq, int32_t k, float theta, int32_t min_matches, int32_t max_len,
                 int32_t nbins, int32_t algo, int32_t P, int32_t* npts, int32_t* pbin,
                 int32_t* pcnt, int64_t* pD, uint8_t* used_fb, double* G, cudaStream_t st);
// ring push of src rows src_idx[0..n) (gather) at the bank head (ss_api.cu)
int bank_push_gather(::ss_bank* h, const int8_t* src_emb, const float* src_inv,
                     const int32_t* src_lens, const int64_t* src_idx, int64_t n, cudaStream_t st);

// batch formation (k_pack.cu)
int launch_pack_batch(const int64_t* perm, const int32_t* I, const int32_t* g, int64_t n,
                      int64_t K, int B, int mode, int64_t* out_batch, int32_t* out_count,
                      int64_t* out_tokens, cudaStream_t st);

// rank
int64_t rank_workspace_bytes(int64_t n);
int launch_rank(const double* G, const int64_t* ids, int64_t n, int64_t* perm,
                void* ws, int64_t ws_bytes, cudaStream_t st);

}  // namespace ss
