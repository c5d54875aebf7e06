/*
 * flatknn.h -- C ABI of the B200-native exact flat k-NN engine (libflatknn.so).
 *
 * Drop-in boundary for the reference's exhaustive-search hot path
 * (arxiv/paper_2401_08281 reference, package `annkit`, /root/reference/pkg):
 *
 *   reference interface                                   replaced by
 *   ----------------------------------------------------  -------------------------
 *   FlatIndex.__init__(d, metric)      flat.py:21-26      fk_create
 *   FlatIndex._add(x, ids)             flat.py:28-32      fk_add
 *     (norms einsum at add             flat.py:31)
 *   FlatIndex._search(q, k)            flat.py:58-62      fk_search
 *     flat_search_blas                 flat.py:94-118
 *     topk_rows / _monotone_key        core.py:193-236
 *     _finish (position -> id)         flat.py:68-73
 *   FlatIndex.ntotal                   core.py:118,143    fk_ntotal
 *   (Faiss-style reset; none in ref)   SURVEY 8(b)        fk_reset
 *   FlatIndex.reconstruct_batch        flat.py:43-44      fk_reconstruct
 *   FlatIndex.remove_ids               flat.py:46-56      fk_remove_ids
 *   FlatIndex._positions (id -> pos)   flat.py:34-41      fk_positions
 *   refine_search re-ranking           core.py:368-394    fk_refine
 *   _kernels function table errors     _kernels/__init__.py:37-41 -> fk_last_error
 *   (none: SPEC.md:115 non-goal)       SURVEY 8(e)        fk_merge_shards, fk_xchg_*
 *
 * Conventions: plain pointers and sizes only.  Every entry point returns 0 on
 * success or a negative FK_E* code; fk_last_error() then returns a message
 * (thread-local).  `stream` is a cudaStream_t (NULL = legacy default stream).
 * `on_device` != 0 means every data pointer of that call is CUDA device memory
 * on the index's device; otherwise they are host pointers (pinned memory gives
 * asynchronous copies; pageable memory works but copies synchronously).
 * Results are written in the reference's order: best first, ties broken by the
 * smaller storage position, k > ntotal padded with id -1 and +inf (L2) / -inf
 * (IP).
 */
#ifndef FLATKNN_H_
#define FLATKNN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fk_index fk_index;

/* metric codes: same values as annkit _pykernels.M_IP / M_L2 (_pykernels.py:14-15) */
#define FK_METRIC_IP 0
#define FK_METRIC_L2 1

/* storage / input dtypes */
#define FK_F32 0  /* storage: fp32 as an exact tf32 hi/lo split (k <= 16, or 33 <~ k <= 128,
                     over >= 256k rows: one scaled-fp16 filter pass + certified exact fp32
                     rescoring; otherwise 3xTF32; fp32-faithful either way) */
#define FK_F16 1  /* storage: fp16 (RNE from f32), tensor-core kind::f16      */
#define FK_BF16 2 /* storage: bf16 (RNE from f32), tensor-core kind::f16      */

/* error codes */
#define FK_OK 0
#define FK_E_INVALID -1     /* bad argument (ValueError in the Python mirror)  */
#define FK_E_CUDA -2        /* CUDA runtime / driver failure                  */
#define FK_E_NOMEM -3       /* device allocation failed                       */
#define FK_E_UNSUPPORTED -4 /* valid but not supported (NotImplementedError)  */
#define FK_E_NOTFOUND -5    /* unknown id (KeyError, flat.py:40-41)            */

/* Create an empty index on CUDA device `device` (flat.py:21-26). */
int fk_create(int device, int d, int metric, int storage, fk_index** out);

/* Append n vectors (row-major n x d of `dtype`) with int64 ids (flat.py:28-32;
 * ids == NULL -> sequential ntotal..ntotal+n-1, core.py:128-131).  Ids are
 * validated (>= 0) by the caller, as core.py:139-141 does.  Base norms are
 * computed on device from the stored (rounded) values. */
int fk_add(fk_index* h, const void* x, int64_t n, int dtype, const int64_t* ids, int on_device,
           void* stream);

/* Exact top-k for nq queries (row-major nq x d of `dtype`); FlatIndex._search
 * dispatch: nq >= FK_OPT_BLAS_THRESHOLD -> the fused GEMM + top-k path
 * (flat_search_blas semantics), else the direct per-pair path (flat_search).
 * D: nq x k float32 distances (L2: squared, clamped at 0; IP: inner product).
 * I: nq x k int64 ids (-1 for padding).
 * P: optional (may be NULL) nq x k int64 storage positions (-1 for padding),
 *    needed to order ties across shards (fk_merge_shards). */
int fk_search(fk_index* h, const void* q, int64_t nq, int dtype, int k, float* D, int64_t* I, int64_t* P,
              int on_device, void* stream);

/* Merge per-shard results into the single-index answer.  Inputs are
 * nshard x nq x k arrays (shard-major) of distances, GLOBAL storage positions
 * and ids, each shard's rows already best-first.  Output ordered by
 * (distance, global position) exactly like a single unsharded index.  All
 * pointers are device pointers on the current device. */
int fk_merge_shards(int metric, int nshard, int64_t nq, int k, const float* D_in, const int64_t* P_in,
                    const int64_t* I_in, float* D_out, int64_t* I_out, void* stream);

/* Peer-memory exchange for the row-sharded index (the fused alternative to
 * NCCL all-gather + fk_merge_shards).  Every rank exports one
 * device block (CUDA IPC handle of fk_xchg_handle_bytes() bytes) holding its
 * per-search lists and two counters; after fk_xchg_connect with every rank's
 * handle, a search is: fk_xchg_acquire (wait until the peers finished reading
 * this rank's previous lists) -> local search -> fk_xchg_put (distances,
 * GLOBAL positions, ids) -> fk_xchg_merge (publish, wait for every peer,
 * merge by (distance, global position) reading the peers' lists directly ->
 * the single-index answer on every rank).  All on `stream`, no host sync;
 * bounded device waits, fk_xchg_status reports a timeout. */
typedef struct fk_xchg fk_xchg;
int fk_xchg_handle_bytes(void);
int fk_xchg_create(int device, int rank, int world, int64_t nq_cap, int k_cap, fk_xchg** out, void* handle_out);
int fk_xchg_connect(fk_xchg* x, const void* all_handles);
int fk_xchg_acquire(fk_xchg* x, void* stream);
int fk_xchg_put(fk_xchg* x, int64_t nq, int k, const float* D, const int64_t* P, const int64_t* I, void* stream);
int fk_xchg_merge(fk_xchg* x, int metric, int64_t nq, int k, float* D_out, int64_t* I_out, void* stream);
int fk_xchg_status(fk_xchg* x);
void fk_xchg_destroy(fk_xchg* x);

/* Copy the stored vectors of the given storage positions back as float32
 * (flat.py:43-44 reconstruct_batch; the Python mirror maps ids->positions). */
int fk_reconstruct(fk_index* h, const int64_t* positions, int64_t n, float* out, int on_device, void* stream);

/* Remove every stored vector whose id is in ids[0..n) (flat.py:46-56),
 * compacting storage in place and preserving order.  *removed = count.
 * Runs on the device (sorted kill list, keep mask, ordered compaction); only
 * the removed count comes back to the host. */
int fk_remove_ids(fk_index* h, const int64_t* ids, int64_t n, int on_device, int64_t* removed, void* stream);

/* ids[0..n) -> storage positions (flat.py:34-41 `_positions`): a duplicated
 * id maps to its LAST position, as the reference's {id: i} dict does.
 * FK_E_NOTFOUND (KeyError) names the first unknown id.  The sorted id table
 * lives on the device and is rebuilt lazily after add / remove / reset. */
int fk_positions(fk_index* h, const int64_t* ids, int64_t n, int64_t* pos, int on_device, void* stream);

/* refine_search (core.py:368-394) with this index as `exact`: q [nq][d]
 * float32 queries, cand [nq][L] shortlist ids from the fast index (-1 =
 * empty, skipped; unknown ids -> FK_E_NOTFOUND like reconstruct_batch).
 * Each candidate gets the direct distance of its stored vector (fp64
 * accumulation, one rounding to fp32) under `metric` (the FAST index's,
 * core.py:375); D/I [nq][k] = the first k by (value best first, id), padded
 * with -1 and +inf (L2) / -inf (IP).  L <= 14464 (shortlist held in smem). */
int fk_refine(fk_index* h, int metric, const float* q, int64_t nq, const int64_t* cand, int L, int k, float* D,
              int64_t* I, int on_device, void* stream);

/* Drop all vectors, keep the device allocation (Faiss Index::reset). */
int fk_reset(fk_index* h);

int64_t fk_ntotal(const fk_index* h);
int fk_dim(const fk_index* h);

/* Copy the ids table (ntotal int64) to host memory. */
int fk_get_ids(fk_index* h, int64_t* out_host);

void fk_destroy(fk_index* h);

const char* fk_last_error(void);

/* Instrumentation: when enabled (on > 0; the events of `on` searches, at
 * least 64, are created here, up front), fk_search records CUDA events around
 * each of its kernels on the launch stream (no host synchronisation).  fk_kernel_times
 * waits for them and returns the mean durations (ms) per search since its
 * previous call: [0] query prep, [1] fused GEMM+top-k, [2] merge; *nlaunch =
 * total kernel launches of those searches.  Then it resets the accumulators. */
int fk_set_profiling(fk_index* h, int on);
int fk_kernel_times(fk_index* h, float* ms3, int* nlaunch);

/* Timed-loop gate (bench instrumentation, no reference counterpart): enqueue
 * a one-thread kernel on `stream` that waits until *host_flag (pinned host
 * memory) is nonzero or timeout_s seconds pass, so a timed loop can enqueue
 * all its work before the GPU starts and host jitter cannot idle the GPU. */
int fk_gate(const int* host_flag, double timeout_s, void* stream);

/* Range search (replaces annkit flat.py:121-144 `flat_range_search`, reached
 * through Index.range_search core.py:152-155 / FlatIndex._range_search):
 * every stored vector with direct distance <= radius (L2) or inner product
 * >= radius (IP), per query sorted best first with ties by smaller id
 * (flat.py:137).  Writes lims [nq + 1] (CSR offsets, host or device) and the
 * entry count to *total, and returns the entries in a per-call result object
 * *out (caller-owned: fk_range_fetch copies them, fk_range_free releases it),
 * so concurrent range searches on one index never mix their results. */
typedef struct fk_range_result fk_range_result;
int fk_range_search(fk_index* h, const void* q, int64_t nq, int dtype, float radius, int64_t* lims, int64_t* total,
                    fk_range_result** out, int on_device, void* stream);
/* Copy ids [total] (int64) and distances [total] (f32); capacity = entries
 * the output arrays hold (FK_E_INVALID when smaller than total). */
int fk_range_fetch(fk_range_result* r, int64_t* ids, float* dist, int64_t capacity, int on_device, void* stream);
int64_t fk_range_total(const fk_range_result* r);
void fk_range_free(fk_range_result* r);

/* Per-index options.
 * FK_OPT_PLAN_ROWS: database rows the fp32 algorithm choice is made for
 * (0 = the index's own ntotal).  A shard of a row-sharded index passes the
 * global row count so every shard runs the algorithm the unsharded search
 * would (ShardedFlatIndex does). */
#define FK_OPT_PLAN_ROWS 1
/* FK_OPT_BLAS_THRESHOLD: batches of fewer queries take the direct path
 * (exact per-pair distances, flat.py:58-62 -> flat_search flat.py:76-91);
 * default 20 = annkit config.blas_threshold (config.py:9); 0 disables it. */
#define FK_OPT_BLAS_THRESHOLD 2
int fk_set_option(fk_index* h, int option, int64_t value);

/* k-means assignment in fp64 (replaces annkit quantize.py:38-62 `_assign`,
 * the Lloyd-iteration / IVF-training consumer of the flat path).
 * Device pointers: x [n][d] f32, c [nc][d] f64, cnorm [nc] f64, optional
 * cand [n][kc] (candidate centroid ids per row, e.g. the GPU flat-search
 * shortlist; NULL = ids 0..kc-1) and approx [n][kc] (their fp32 distances,
 * best first) -> assign [n] i64, err [n] f64 (max(|x|^2 + |c|^2 - 2 x.c, 0)),
 * uncertain [n] (1 = shortlist gap below margin*(|x|^2 + cmax): rescore the
 * row over all centroids).  by_ip: argmax inner product (spherical). */
int fk_kmeans_rescore(const float* x, int64_t n, int d, const double* c, const double* cnorm, int64_t nc,
                      const int64_t* cand, int kc, int by_ip, const float* approx, double margin, double cmax,
                      int64_t* assign, double* err, int* uncertain, void* stream);

/* Tuning / introspection of the last search plan, FK_PLAN_INTS ints: grid,
 * N-chunks (split-N), tiles per chunk, work units, smem pipeline stages,
 * query-operand mode, dynamic smem bytes, 100*queue+epilogue warps, TMEM
 * accumulator buffers, epilogue warps, (reserved). */
#define FK_PLAN_INTS 12
int fk_last_plan(fk_index* h, int* out);

#ifdef __cplusplus
}
#endif

#endif /* FLATKNN_H_ */
