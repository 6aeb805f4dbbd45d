/*
 * sagesched.h -- C ABI of libsagesched, the B200-native (sm_100a) drop-in for
 * SageSched's per-scheduling-round hot path (arxiv 2603.07917):
 *   predict (history-bank similarity -> top-k -> length histogram)
 *   -> cost (O^2/2 + I*O) -> Gittins index -> rank.
 *
 * Conventions:
 *   - plain pointers and sizes only; every array pointer is DEVICE memory
 *     unless the parameter name ends in `_host`;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream);
 *   - every entry point returns 0 (SS_OK) or an SS_ERR_* code, and
 *     ss_last_error() returns a thread-local message for the last failure;
 *   - a bank handle is not thread-safe: one scheduling thread per handle,
 *     mirroring the reference's single-writer window.
 *
 * Each entry point names the reference interface it replaces (file:line into
 * /root/reference).  The Python host mirror is paper_2603_07917_b200/.
 */
#ifndef SAGESCHED_H_
#define SAGESCHED_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- status */
#define SS_OK 0
#define SS_ERR_ARG 1         /* bad argument (ValueError in the reference)      */
#define SS_ERR_RANGE 2       /* length outside [lo, max_len] (UB in numba)      */
#define SS_ERR_EMPTY 3       /* empty window / distribution (cold start)        */
#define SS_ERR_CUDA 4        /* CUDA runtime failure                            */
#define SS_ERR_ZERODIV 5     /* leading zero mass: ZeroDivisionError, _kernels.py:113 */
#define SS_ERR_UNSUPPORTED 6 /* shape/arch not supported by this build          */

/* similarity algorithms for ss_topk */
#define SS_ALGO_AUTO 0
#define SS_ALGO_SCAN 1   /* CUDA-core int8 dp4a streaming scan + fused top-k    */
#define SS_ALGO_TCGEN05 2 /* tcgen05/TMEM int8 GEMM fed by TMA + fused top-k   */

/* cost kinds (cost.py:31-52, names cost.py:121-135) */
#define SS_COST_RESOURCE_BOUND 0
#define SS_COST_OUTPUT_ONLY 1
#define SS_COST_WEIGHTED_SUM 2

typedef struct ss_bank ss_bank_t;

const char* ss_last_error(void);
int ss_version(void);
/* Number of kernels this library has launched in this process (evidence for
 * bench.py's gpu_launches). */
int64_t ss_launch_count(void);

/* ------------------------------------------------ reference _kernels.py --- */
/* servesim._kernels.match_pmfs (_kernels.py:118-138): threshold match ->
 * exact integer-length pmf.  sims f32[nq,nw], lens i64[nw] in [0,max_len];
 * sup/mas f64[nq,out_stride], sizes i64[nq].  Bit-compatible with the numba
 * path (mass = c * (1.0/total)); theta is compared in f64 as numba does for a
 * Python-float theta (exact for an np.float32 one).  Out-of-range lens ->
 * SS_ERR_RANGE. Synchronises. */
int ss_match_pmfs(const float* sims, int64_t nq, int64_t nw, const int64_t* lens,
                  double theta, int64_t max_len, double* sup, double* mas,
                  int64_t* sizes, int64_t out_stride, void* stream);

/* servesim._kernels.gittins_min (_kernels.py:104-116), batched: one
 * warp-per-distribution prefix scan.  support/masses f64[n,stride], npts
 * i64[n]; out f64[n].  Leading zero mass -> SS_ERR_ZERODIV. Synchronises. */
int ss_gittins_min_batch(const double* support, const double* masses,
                         const int64_t* npts, int64_t n, int64_t stride,
                         double* out, void* stream);

/* gittins_index(condition_on_attained(d, a)) for general f64 laws
 * (outlived rule SPEC.md:373 supplied as outlived_index[i]).
 * attained may be NULL (a = 0).  Async. */
int ss_gittins_dist_batch(const double* support, const double* masses,
                          const int64_t* npts, const double* attained,
                          const double* outlived_index, int64_t n,
                          int64_t stride, double* out, void* stream);

/* servesim._kernels.embed_accumulate (_kernels.py:70-102), batched over
 * prompts: tokens i64 (concatenated), offsets i64[n+1]; out f64[n,dim]. Async. */
int ss_embed_accumulate_batch(const int64_t* tokens, const int64_t* offsets,
                              int64_t n, uint64_t salt, int32_t dim,
                              double* out, void* stream);

/* Same hash (_kernels.py:82-95), emitted as the exact integer vector in int16
 * plus its fp32 inverse norm (IEEE 1/sqrt of the exact int64 sum of squares)
 * for the bank.  Buckets beyond int8 (long prompts that
 * repeat a token or bigram > 127 times) are kept exactly; *n_wide (host
 * pointer, may be NULL) receives how many rows do not fit int8.  |bucket| >
 * 32767 -> SS_ERR_RANGE.  Synchronises. */
int ss_embed_quantize_batch(const int64_t* tokens, const int64_t* offsets, int64_t n,
                            uint64_t salt, int32_t dim, int16_t* out_emb, float* out_inv_norm,
                            int64_t* n_wide, void* stream);

/* --------------------------------------------------- reference cost.py --- */
/* cost.cost_distribution (cost.py:97-118), batched: len_support f64[n,stride]
 * -> out_support f64[n,stride]; input_len f64[n] (>= 1 else SS_ERR_ARG). Async. */
int ss_cost_distribution_batch(int32_t kind, double w_in, double w_out,
                               const double* input_len, const double* len_support,
                               const int64_t* npts, int64_t n, int64_t stride,
                               double* out_support, void* stream);
/* Per-call forms of gittins_min (_kernels.py:104-116) and cost_distribution
 * (cost.py:107-118) for the reference's scalar call pattern: HOST arrays in
 * and out, no allocation per call.  Up to 2048 points the inputs go into a
 * per-thread mapped pinned slot that the kernel reads across PCIe and
 * answers through (result + a completion flag the caller spins on: no
 * copy-engine transfer, no stream synchronise); the call runs on the
 * library's own per-thread stream and `stream` may be NULL (inputs and
 * outputs are host memory, so it orders nothing).  Longer laws take one
 * packed H2D copy, the kernel, one D2H and a synchronise on `stream`.  (A
 * batched engine uses the *_batch forms or the fused round.)
 * gittins_min_host with a leading zero mass -> SS_ERR_ZERODIV, as numba
 * raises; n = 0 -> +inf. */
int ss_gittins_min_host(const double* support, const double* masses, int64_t n, double* out,
                        void* stream);
int ss_cost_distribution_host(int32_t kind, double w_in, double w_out, double input_len,
                              const double* len_support, int64_t n, double* out_support,
                              void* stream);

/* ------------------------------------- history bank ----- */
/* FIFO ring of (int8 embedding[dim], fp32 inverse norm, output length,
 * insertion_seq).  A handle holds one shard [slot_offset, slot_offset+capacity)
 * of a global ring of global_capacity slots (== capacity on one GPU). */
int ss_bank_create(ss_bank_t** out, int32_t device, int64_t capacity, int32_t dim,
                   int64_t global_capacity, int64_t slot_offset);
int ss_bank_destroy(ss_bank_t* h);
/* push n records at the ring head: slot = seq mod capacity,
 * evicting the oldest.  inv_norm may be NULL (computed on device, IEEE
 * 1/sqrt).  lens must lie in [1, 65535].  Async. */
int ss_bank_push(ss_bank_t* h, const int8_t* emb, const float* inv_norm,
                 const int32_t* lens, int64_t n, void* stream);
/* push of int16 feature-hash rows (ss_embed_quantize_batch output): a row
 * that fits int8 enters the int8 plane like ss_bank_push; a "wide" row keeps
 * its exact int16 vector in the bank's wide plane (allocated on first use,
 * 2 * dim bytes per slot), scored exactly by the CUDA-core wide pass of every
 * later top-k / round (one more candidate list per query).  Synchronises. */
int ss_bank_push16(ss_bank_t* h, const int16_t* emb, const float* inv_norm,
                   const int32_t* lens, int64_t n, void* stream);
/* ss_bank_write with int16 rows (the sharded host's form of ss_bank_push16). */
int ss_bank_write16(ss_bank_t* h, const int16_t* emb, const float* inv_norm,
                    const int32_t* lens, const int64_t* seq, const int64_t* local_slot,
                    int64_t n, void* stream);
/* scatter-write records at explicit LOCAL slots with explicit seqs (used by
 * the sharded host, which owns the global ring head).  Async. */
int ss_bank_write(ss_bank_t* h, const int8_t* emb, const float* inv_norm,
                  const int32_t* lens, const int64_t* seq, const int64_t* local_slot,
                  int64_t n, void* stream);
int ss_bank_set_head(ss_bank_t* h, int64_t global_head);
int ss_bank_info(ss_bank_t* h, int64_t* head, int64_t* size, int64_t* capacity,
                 int32_t* dim);
int ss_bank_device_ptrs(ss_bank_t* h, int8_t** emb, float** inv_norm,
                        int32_t** lens, int64_t** seq);
/* synchronise `stream` and return (then clear) the bank's sticky device
 * error: SS_ERR_RANGE for a pushed length outside [1, 65535], SS_ERR_ARG for
 * a write outside the shard. */
int ss_bank_sync_check(ss_bank_t* h, void* stream);
/* window-wide binned length histogram (the predictor fallback,
 * SPEC.md:184-186,223): cnt/sv/sv2 i64[nbins], bin = (len-1)/(max_len/nbins).
 * Lengths > max_len are clamped to max_len.  Async. */
int ss_bank_fallback_hist(ss_bank_t* h, int32_t max_len, int32_t nbins,
                          int64_t* cnt, int64_t* sv, int64_t* sv2, void* stream);

/* ------------------------------------------------ predict stages -------- */
/* Stage 1 (query_similar SPEC.md:132-140 + top-k): for each query, the
 * top-k bank rows by (key desc, insertion_seq desc) among key >= theta,
 * key = fl32(fl32(f32(dot(q,w)) * inv_w) * inv_q).  Score matrix never
 * written.  out_comp u64[nq,k] sorted desc, 0 = empty; out_len i32[nq,k].
 * Composite = (orderable(key) << 32) | rel, rel = (slot - head) mod C. Async. */
int ss_topk(ss_bank_t* h, const int8_t* q, const float* q_inv, int64_t nq,
            int32_t k, float theta, int32_t algo, uint64_t* out_comp,
            int32_t* out_len, void* stream);
/* ss_topk for a batch holding wide queries (feature-hash vectors outside
 * int8): rows wide_idx[0..n_wide) of the batch are scored with their exact
 * int16 vectors wide_q_emb [n_wide, dim] and inverse norms wide_q_inv (their
 * q / q_inv entries are ignored), everything else as ss_topk.  Async. */
int ss_topk_wide(ss_bank_t* h, const int8_t* q, const float* q_inv, int64_t nq, int64_t n_wide,
                 const int64_t* wide_idx, const int16_t* wide_q_emb, const float* wide_q_inv,
                 int32_t k, float theta, int32_t algo, uint64_t* out_comp, int32_t* out_len,
                 void* stream);
/* query_similar in full: EVERY record of the window with
 * key >= theta (theta = -1: the whole window), ordered by key desc, then
 * insertion_seq desc.  One query, given as its exact integer vector in int16
 * (int8 vectors widened), with its inverse norm.  out_* hold the window's
 * capacity; *n_out (host) = number of records returned.  Synchronises. */
int ss_query_similar(ss_bank_t* h, const int16_t* q, float q_inv, float theta, float* out_key,
                     int64_t* out_seq, int32_t* out_len, int64_t* n_out, void* stream);
/* The similarity kernel alone (no merge): writes the unsorted per-slice
 * partial top-k lists u64[n_slices][nq][k] into `partials` (capacity
 * max_slices slices) and the slice count into *n_slices.  Used to time the
 * dominant kernel for the roofline and by the sharded host.  Async. */
int ss_topk_partials(ss_bank_t* h, const int8_t* q, const float* q_inv, int64_t nq,
                     int32_t k, float theta, int32_t algo, uint64_t* partials,
                     int32_t max_slices, int32_t* n_slices, void* stream);
/* merge nlists per-shard candidate lists (layout [nlists][nq][k]) into the
 * global top-k (the multi-GPU gather/merge step).  Async. */
int ss_merge_topk(const uint64_t* comp, const int32_t* len, int32_t nlists,
                  int64_t nq, int32_t k, uint64_t* out_comp, int32_t* out_len,
                  void* stream);
/* Fused merge + exchange of the multi-GPU round with per-rank queues
 * (SURVEY 8(e) stage 3, replacing the candidate all_to_all that would follow
 * a per-shard run of the reference's similarity step -- SPEC.md:132-140
 * query_similar, computed in float32 as _kernels.py:172 does): the local
 * top-k of nq = world * nq_local queries (rank-major: rows
 * [r*nq_local, (r+1)*nq_local) are rank r's queue) against this rank's
 * shard, whose merge kernel stores each merged row straight into the
 * owner's receive buffer -- peer_comp_host[r] / peer_len_host[r] (device
 * pointers, IPC-mapped for r != rank) laid out [world][nq_local][k] -- at
 * row [rank][q % nq_local], as NVLink P2P stores.  The caller orders the
 * peers' reads after a barrier (e.g. a 1-element NCCL all_reduce) and then
 * merges its receive buffer with ss_merge_topk.  world <= 8 (one
 * NVLink/NVSwitch node); nq % world == 0.  Async. */
#define SS_IPC_HANDLE_BYTES 64
int ss_topk_scatter(ss_bank_t* h, const int8_t* q, const float* q_inv, int64_t nq,
                    int32_t k, float theta, int32_t algo, int32_t world, int32_t rank,
                    uint64_t* const* peer_comp_host, int32_t* const* peer_len_host,
                    void* stream);
/* The single-owner form (north star: "the rest runs on the rank owning the
 * queue"; SPEC.md:468-470 ranks every pending request in one order): all nq
 * queries belong to one owner rank, whose receive buffer owner_comp /
 * owner_len (IPC-mapped here unless rank == owner) is laid out [world][nq][k];
 * this rank's merged local top-k rows are stored at [rank][q] -- the
 * all-gather of k candidates per query, done by the merge kernel's own NVLink
 * stores.  Async. */
int ss_topk_gather(ss_bank_t* h, const int8_t* q, const float* q_inv, int64_t nq, int32_t k,
                   float theta, int32_t algo, int32_t world, int32_t rank,
                   uint64_t* owner_comp, int32_t* owner_len, void* stream);
/* IPC-exportable device buffers for ss_topk_scatter: cudaMalloc'd (zeroed) on
 * `device`, exported as a 64-byte handle, opened (peer-mapped) by the other
 * ranks of the node.  Synchronous. */
int ss_ipc_malloc(int32_t device, int64_t bytes, void** out);
int ss_ipc_free(void* ptr);
int ss_ipc_handle(const void* ptr, uint8_t* handle_host);
int ss_ipc_open(const uint8_t* handle_host, void** out);
int ss_ipc_close(void* ptr);
/* decode composites: key f32, seq = head - capacity + rel, global slot. Async. */
int ss_decode_topk(const uint64_t* comp, int64_t n, int64_t head, int64_t capacity,
                   float* out_key, int64_t* out_seq, int64_t* out_slot, void* stream);

/* Stages 1b-3 fused (predict SPEC.md:182-194 -> cost cost.py:97-118 ->
 * gittins SPEC.md:325-333): histogram of the surviving neighbours (or the
 * fallback when fewer than min_matches survive), ResourceBound
 * conditional-mean cost per bin, Gittins index in exact integer form.
 * Writes the request's sparse cost law (P >= nbins points) for later
 * refreshes: npts i32[nq], pbin i32[nq,P], pcnt i32[nq,P], pD i64[nq,P]
 * (D = sum v^2 + 2 I sum v), psv i64[nq,P] (sum v; may be NULL), used_fb
 * u8[nq] (may be NULL), G f64[nq]. Async. */
int ss_finish(const uint64_t* comp, const int32_t* len, int64_t nq, int32_t k,
              int32_t min_matches, int32_t max_len, int32_t nbins,
              const int32_t* input_len, const int64_t* fb_cnt, const int64_t* fb_sv,
              const int64_t* fb_sv2, int32_t P, int32_t* npts, int32_t* pbin,
              int32_t* pcnt, int64_t* pD, int64_t* psv, uint8_t* used_fb, double* G,
              void* stream);

/* Running-request refresh: for each request
 * i, if force or floor(g_new/bucket) > bucket_io[i]: G_io[i] = Gittins of
 * its law conditioned on attained cost(I, g_new); bucket_io updated.
 * refreshed u8[n] may be NULL.  Async. */
int ss_refresh(int64_t n, const int32_t* input_len, const int32_t* g_new,
               int32_t* bucket_io, int32_t bucket_size, const int32_t* npts,
               const int32_t* pcnt, const int64_t* pD, int32_t P, double* G_io,
               uint8_t* refreshed, int32_t force, void* stream);

/* Stage 4: perm i64[n] = indices sorted by ascending
 * (G, id) -- i.e. descending north-star index 1/G.  Device radix sort.
 * workspace: ss_rank_workspace_bytes(n) bytes of device memory. Async. */
int64_t ss_rank_workspace_bytes(int64_t n);
int ss_rank(const double* G, const int64_t* ids, int64_t n, int64_t* perm,
            void* workspace, int64_t workspace_bytes, void* stream);

/* ---------------------------------------------------- batch formation -- */
/* Engine step 3, the caller right after
 * ss_rank: walk perm (ascending priority) and admit request r while the
 * projected KV tokens sum(I[r] + g[r] + 1) <= kv_capacity and the count
 * <= max_batch (SPEC.md:501 defaults K = 8192, B = 64).  mode SS_PACK_CUT
 * stops at the first request that does not fit; SS_PACK_SKIP skips it and
 * keeps scanning.  out_batch i64[max_batch] receives the admitted request
 * indices in priority order, *out_count their number and *out_tokens the KV
 * tokens they project.  A request with I + 1 > kv_capacity anywhere in [0, n)
 * ("request cannot fit", SPEC.md engine errors) gives *out_count = -1 and
 * *out_tokens = its index.  I, g i32[n] indexed by request; device pointers;
 * async (graph-capturable). */
#define SS_PACK_CUT 0
#define SS_PACK_SKIP 1
int ss_pack_batch(const int64_t* perm, const int32_t* input_len, const int32_t* g,
                  int64_t n, int64_t kv_capacity, int32_t max_batch, int32_t mode,
                  int64_t* out_batch, int32_t* out_count, int64_t* out_tokens,
                  void* stream);

/* -------------------------------------------------------- engine round -- */
/* A GPU-resident table of active requests (ids ascending, two buffers for the
 * stable compaction) and one C call per engine iteration (SPEC.md:462-470,
 * scheduling state only): the last batch gains tokens_per_round tokens;
 * requests reaching tr_true_len complete and enter the bank ring in batch
 * order; up to max_arrivals trace requests from *next_id on
 * are admitted and predicted (fused stages 1-3); bucket refreshes
 * (SPEC.md:345-353); all active requests are ranked and the
 * next batch packed (ss_pack_batch semantics, max_batch from the table).
 * Trace arrays are device pointers indexed by request id (ids = arrival
 * order).  Synchronises once (the completion count).  *next_id advances by
 * the admitted count; *n_done_out / *n_admitted_out report the round. */
typedef struct ss_table ss_table_t;
int ss_table_create(ss_table_t** out, int32_t device, int64_t capacity, int32_t P,
                    int32_t max_batch);
int ss_table_destroy(ss_table_t* t);
/* device pointers of the live buffer (rows [0, n_active)) for inspection */
int ss_table_view(ss_table_t* t, int64_t* n_active, int32_t** input_len, int32_t** g,
                  int64_t** ids, double** G, int32_t** npts, int64_t** perm,
                  int64_t** run_ids, int32_t** batch_count);
int ss_engine_round(ss_table_t* t, ss_bank_t* h, const int8_t* tr_emb, const float* tr_inv,
                    const int32_t* tr_input_len, const int32_t* tr_true_len, int64_t tr_len,
                    int64_t* next_id, int64_t max_arrivals, int32_t tokens_per_round,
                    int32_t bucket_size, int64_t kv_capacity, int32_t mode, int32_t k,
                    float theta, int32_t min_matches, int32_t max_len, int32_t nbins,
                    int32_t algo, int64_t* n_done_out, int64_t* n_admitted_out, void* stream);

/* ----------------------------------------------- fused scheduling round -- */
/* One round for a batch of nq pending requests on a single-GPU bank:
 * ss_topk -> ss_bank_fallback_hist -> ss_finish -> ss_rank.  All device
 * pointers; state arrays as in ss_finish; perm i64[nq].  Uses handle-owned
 * workspace, so it can be captured in a CUDA graph after one warm-up call. */
int ss_schedule_round(ss_bank_t* h, const int8_t* q, const float* q_inv,
                      const int32_t* input_len, const int64_t* ids, int64_t nq,
                      int32_t k, float theta, int32_t min_matches, int32_t max_len,
                      int32_t nbins, int32_t algo, int32_t P, int32_t* npts,
                      int32_t* pbin, int32_t* pcnt, int64_t* pD, uint8_t* used_fb,
                      double* G, int64_t* perm, void* stream);
/* ss_schedule_round with wide queries (see ss_topk_wide). */
int ss_schedule_round_wide(ss_bank_t* h, const int8_t* q, const float* q_inv,
                           const int32_t* input_len, const int64_t* ids, int64_t nq, int64_t n_wide,
                           const int64_t* wide_idx, const int16_t* wide_q_emb,
                           const float* wide_q_inv, int32_t k, float theta, int32_t min_matches,
                           int32_t max_len, int32_t nbins, int32_t algo, int32_t P, int32_t* npts,
                           int32_t* pbin, int32_t* pcnt, int64_t* pD, uint8_t* used_fb, double* G,
                           int64_t* perm, void* stream);
/* Same round from HOST buffers (the plugin call a scheduler makes): copies
 * q/q_inv/input_len/ids host->device, runs the round, copies G and perm
 * device->host, and synchronises the stream. */
int ss_schedule_round_host(ss_bank_t* h, const int8_t* q_host, const float* q_inv_host,
                           const int32_t* input_len_host, const int64_t* ids_host,
                           int64_t nq, int32_t k, float theta, int32_t min_matches,
                           int32_t max_len, int32_t nbins, int32_t algo,
                           double* G_host, int64_t* perm_host, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SAGESCHED_H_ */
