// libflatknn.so -- C ABI (include/flatknn.h) over the sm_100a flat k-NN kernels.
//
// Host side of the drop-in for the reference FlatIndex hot path
// (/root/reference/pkg/src/annkit/flat.py:14-118, core.py:107-236).
// Owns device storage (operand layout + norms + ids), plans the persistent
// fused GEMM+top-k launch (split-N work units ordered for L2 reuse), encodes
// the TMA tensor maps and runs prep -> fused -> merge on the caller's stream.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_set>
#include <vector>

#include "fk_host.cuh"
#include "flatknn_kernels.cuh"
#include "storage_kernels.cuh"
#include "filter16_kernels.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

using namespace fk;
using fkh::set_err;
using fkh::SMEM_LIMIT;

namespace fkh {
namespace {
thread_local std::string g_err;
}
int set_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}
const char* last_error() { return g_err.c_str(); }
}  // namespace fkh

namespace {

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                      CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                      CUtensorMapFloatOOBfill);

PFN_encodeTiled_t get_encode() {
  static PFN_encodeTiled_t fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(p);
  });
  return fn;
}

// 2-D row-major [rows][cols] tensor, box = 128 bytes of K x 128 rows, SW128.
int make_map(CUtensorMap* m, const void* base, int elem_bytes, uint64_t cols, uint64_t rows, uint32_t box_rows = 128) {
  PFN_encodeTiled_t enc = get_encode();
  if (!enc) return set_err(FK_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  const CUtensorMapDataType dt = elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT16;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * (cuuint64_t)elem_bytes};
  cuuint32_t box[2] = {(cuuint32_t)(128 / elem_bytes), box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(FK_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return FK_OK;
}

constexpr int FK_MAX_K = 2048;
// fp32 searches with k <= 16 over at least this many rows run the 1-pass TF32
// filter + exact rescoring (kmode 4) on the hi half of the split storage;
// smaller searches are dominated by the rescoring merge and keep 3xTF32
constexpr int64_t FP32_1X_MIN_ROWS = 262144;
constexpr size_t L2_CHUNK_BYTES = 48ull << 20;  // streamed base per N-chunk (2 chunks in flight << 126 MB L2)
constexpr size_t PARTIAL_BYTES = 4ull << 30;    // split-N partial top-k lists
constexpr int DIRECT_CHUNK = 8192;   // direct path: rows per first-level selection slice
constexpr int MERGE_SMC = 16384;    // large-k merge: survivors gathered in smem (128 KB) + 2048 winners
constexpr int SMEM_RESERVE = 1024 /*align*/ + 512 /*barriers + tmem slot*/;

// Rounding-band coefficient of the 1-pass filter (times |q| max|x|, L2; IP
// half): 2 x (filter-value error bound) with a 2^-10 margin -- scaled fp16
// (MODE 5): 2 x 2 x (2^-10 + 2^-27) -> 2^-8; tf32 truncation (MODE 4):
// 2 x 2 x (2^-9 + 2^-20) -> 2^-7.  FK_BAND scales it (experiments, >= 1).
float f1p_band(int kmode) {
  float b = (kmode == 5 ? 0.00390625f : 0.0078125f) * (1.f + 0.0009765625f);
  if (const char* e = getenv("FK_BAND")) b *= std::max(1.f, (float)atof(e));
  return b;
}

// smallest database (global rows) served by the 1-pass path (FK_FP32_1PASS_MINROWS)
int64_t fp32_1pass_min_rows() {
  if (const char* e = getenv("FK_FP32_1PASS_MINROWS")) return atoll(e);
  return FP32_1X_MIN_ROWS;
}

// largest k served by the 1-pass filter + rescoring path (FK_FP32_1PASS_MAXK)
int fp32_1pass_max_k() {
  if (const char* e = getenv("FK_FP32_1PASS_MAXK")) return atoi(e);
  return 128;
}
// sample rows of the large-k bound pass (the 32nd of 8 ntotal / k rows sits
// near the 4k-th overall); 0 when it would cost more than a quarter pass
int64_t est_rows(int64_t rows, int k) {
  const int64_t m = ((rows * 8) / k + BN - 1) / BN * BN;
  return (m >= 32 * BN && m * 4 <= rows) ? m : 0;
}
// 1-pass filter + rescoring for fp32 storage: k <= 16 (register queues), or
// 16 < k <= FK_FP32_1PASS_MAXK when the sampled bound pass is affordable
// (measured on 1M x 128, 10k queries: k = 64 6.9 vs 12.0 ms 3xTF32, k = 100
// 6.8 vs 11.2; without the bound pass k = 32 loses, 11.7 vs 10.0; k = 1024
// loses to the rescoring gather, 31 vs 12.8)
// rows: the global row count (plan rows of a shard), local: this index's
// own rows (where the bound pass samples)
bool fp32_1pass_ok(int k, int64_t rows, int64_t local) {
  if (rows < fp32_1pass_min_rows() || k > fp32_1pass_max_k()) return false;
  return k <= 16 || est_rows(local, k) > 0;
}
int elem_bytes_of(int storage) { return storage == FK_F32 ? 4 : 2; }
int chunk_elems_of(int storage) { return storage == FK_F32 ? 32 : 64; }
int split_of(int storage) { return storage == FK_F32 ? 2 : 1; }

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  int ensure(size_t want) {
    if (want <= bytes) return FK_OK;
    // growth is rare: wait for every stream that may still read the old buffer
    if (p) cudaDeviceSynchronize();
    release();
    size_t b = std::max<size_t>(want, 256);
    cudaError_t e = cudaMalloc(&p, b);
    if (e != cudaSuccess) {
      p = nullptr;
      return set_err(FK_E_NOMEM, "cudaMalloc(%zu) failed: %s", b, cudaGetErrorString(e));
    }
    bytes = b;
    return FK_OK;
  }
};

}  // namespace

struct fk_index {
  int device = 0, d = 0, dp = 0, metric = FK_METRIC_L2, storage = FK_F32;
  int fold = 0;  // bf16 L2 with d+3 <= dp: norms folded into the GEMM operands (MODE 3 kernels)
  int split = 1;  // fp32: 2 = 3xTF32 hi/lo split (MODE 0), 1 = raw fp32 + TF32 filter + exact rescoring (MODE 4)
  int64_t ntotal = 0, cap = 0;
  void* s0 = nullptr;        // stored operand (hi / f16 / bf16) [cap][dp]
  void* s1 = nullptr;        // lo part (fp32 mode) [cap][dp]
  float* norms = nullptr;    // [cap]
  float* xn_max = nullptr;   // device scalar: max stored norm
  int64_t* ids = nullptr;    // [cap]
  DevBuf q_in, q0, q1, qn, pkey, ppos, thr, pcnt, cbuf, fail, outD, outI, outP, stage_in, stage_ids;
  // range search: candidates, exact pass, sort scratch and the CSR result
  DevBuf rfail, rcomp, rflag, glock, gkeys;
  unsigned int* inexact = nullptr;  // device {base, queries}: a value with a nonzero lo part was stored/staged  // fp32 MODE 4: per-query certification flags, exact-fallback composites
  DevBuf rcand, rcount, rdist, rkid, rkrd, rkeep, rrowc, rsel, rnsel, rtmp, rkid2, rkrd2, rv1, rv2, rlims;
  // every call that touches the handle's scratch or storage waits for the
  // previous such call's stream work (stream-ordered reuse: concurrent
  // searches on different streams stay correct) and records this event
  // sorted (id, position) table for id -> position lookups (flat.py:34-41),
  // rebuilt lazily after add / remove / reset
  DevBuf idt_keys, idt_pos, idt_tmp, idt_miss, rm_kill, rm_flags, rm_keep;
  int64_t idt_n = -1;
  // fp32 MODE 5 filter operands: scaled fp16 copy of the base [cap][dp16]
  // (rows [0, f16_rows) converted; built lazily at search time), its scale
  // state (F16State), the staged queries' fp16 rows and 2^-s per query
  DevBuf x16, f16st, q16, qinv;
  DevBuf ovf;  // F1P overflow lists: [nq][ovf_cap] keys, positions, [nq] counts
  int r_ovf_cap = 0;
  int dp16 = 0;
  int64_t f16_rows = 0;
  cudaEvent_t scratch_ev = nullptr;
  bool scratch_used = false;
  int64_t plan_rows = 0;  // FK_OPT_PLAN_ROWS (0: ntotal)
  int64_t blas_threshold = 20;  // FK_OPT_BLAS_THRESHOLD (reference config.py:9)
  float r_radius = 0.f;
  int r_kfinal = 0;  // MODE 4 search: the caller's k (lists keep k' >= k)
  bool r_union = false;  // MODE 4 search: maintain the per-query running union bound
  bool r_prepass = false;  // bound pass: publish thr_key only (no overflow lists or row flags; the union only when asked)
  DevBuf rflag_pre;
  unsigned long long r_cap = 0;
  long long est_fallbacks = 0;  // large-k searches whose estimated bound failed certification
  std::mutex mu;
  int num_sms = 148;
  int profiling = 0;
  // profiling: one quad of events per search (prep / fused / merge), read
  // lazily by fk_kernel_times so the timed loop never synchronises the host
  std::vector<std::array<cudaEvent_t, 4>> ev_pool;
  size_t ev_used = 0;
  int nlaunch = 0;        // launches of the last search
  long long nlaunch_acc = 0;  // launches since the last fk_kernel_times
  int plan[FK_PLAN_INTS] = {0};
  float* dbg_ip = nullptr;  // test hook (FK_DEBUG_IP)
  unsigned long long* trace = nullptr;  // debug timeline hook
};

// Entries of one range search (owned by the caller until fk_range_free).
struct fk_range_result {
  int device = 0;
  int64_t total = 0;
  // stream-ordered allocations from the device's default memory pool (a
  // per-call cudaMalloc/cudaFree pair costs more than the search's kernels)
  void* ids = nullptr;
  void* dist = nullptr;
  cudaStream_t stream = nullptr;
};

namespace {

cudaEvent_t* next_events(fk_index* h) {
  if (h->ev_used == h->ev_pool.size()) {
    std::array<cudaEvent_t, 4> q{};
    for (auto& e : q)
      if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    h->ev_pool.push_back(q);
  }
  return h->ev_pool[h->ev_used++].data();
}

size_t row_bytes(const fk_index* h) { return (size_t)h->dp * elem_bytes_of(h->storage); }

// Stream ordering of the handle's scratch (see fk_index::scratch_ev).
int scratch_begin(fk_index* h, cudaStream_t st) {
  if (h->scratch_used) CK(cudaStreamWaitEvent(st, h->scratch_ev, 0));
  return FK_OK;
}
int scratch_end(fk_index* h, cudaStream_t st) {
  CK(cudaEventRecord(h->scratch_ev, st));
  h->scratch_used = true;
  return FK_OK;
}

int grow(fk_index* h, int64_t need, cudaStream_t st) {
  if (need <= h->cap) return FK_OK;
  int64_t nc = std::max<int64_t>(need, h->cap * 2);
  nc = std::max<int64_t>(nc, 1024);
  nc = (nc + BN - 1) / BN * BN;
  const size_t rb = row_bytes(h);
  void *n0 = nullptr, *n1 = nullptr;
  float* nn = nullptr;
  int64_t* ni = nullptr;
  cudaError_t e = cudaMalloc(&n0, nc * rb);
  if (e == cudaSuccess && h->split == 2) e = cudaMalloc(&n1, nc * rb);
  if (e == cudaSuccess) e = cudaMalloc((void**)&nn, nc * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc((void**)&ni, nc * sizeof(int64_t));
  if (e != cudaSuccess) {
    cudaFree(n0);
    cudaFree(n1);
    cudaFree(nn);
    cudaFree(ni);
    return set_err(FK_E_NOMEM, "device allocation of %lld rows failed: %s", (long long)nc, cudaGetErrorString(e));
  }
  CK(cudaMemsetAsync(nn, 0, nc * sizeof(float), st));
  if (h->ntotal > 0) {
    CK(cudaMemcpyAsync(n0, h->s0, h->ntotal * rb, cudaMemcpyDeviceToDevice, st));
    if (n1) CK(cudaMemcpyAsync(n1, h->s1, h->ntotal * rb, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(nn, h->norms, h->ntotal * sizeof(float), cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(ni, h->ids, h->ntotal * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  }
  CK(cudaDeviceSynchronize());  // in-flight searches on any stream may read the old storage
  cudaFree(h->s0);
  cudaFree(h->s1);
  cudaFree(h->norms);
  cudaFree(h->ids);
  h->s0 = n0;
  h->s1 = n1;
  h->norms = nn;
  h->ids = ni;
  h->cap = nc;
  return FK_OK;
}

// kernel operand mode of an index: 0 fp32 hi/lo (3xTF32), 4 fp32 raw (TF32
// filter + exact rescoring), 1 fp16, 2 bf16 (3 = bf16 with folded norms)
int kmode_of(const fk_index* h) {
  if (h->storage == FK_F32) return h->split == 2 ? 0 : 4;
  return h->storage == FK_F16 ? 1 : 2;
}

int launch_prep(int kmode, const void* x, int dtype, int64_t n, int d, int dp, void* o0, void* o1, float* norms,
                int64_t row0, cudaStream_t st, int fold = 0, unsigned int* inexact = nullptr) {
  if (n <= 0) return FK_OK;
  const int wpb = 8;
  const unsigned grid = (unsigned)((n + wpb - 1) / wpb);
  if (kmode == 0)
    prep_rows_kernel<0><<<grid, wpb * 32, 0, st>>>(x, dtype, n, d, dp, o0, o1, norms, row0, 0, inexact);
  else if (kmode == 4)
    prep_rows_kernel<4><<<grid, wpb * 32, 0, st>>>(x, dtype, n, d, dp, o0, o1, norms, row0, 0);
  else if (kmode == 1)
    prep_rows_kernel<1><<<grid, wpb * 32, 0, st>>>(x, dtype, n, d, dp, o0, o1, norms, row0, 0);
  else
    prep_rows_kernel<2><<<grid, wpb * 32, 0, st>>>(x, dtype, n, d, dp, o0, o1, norms, row0, fold);
  CKL();
  return FK_OK;
}

size_t dtype_bytes(int dtype) { return dtype == FK_F32 ? 4 : 2; }

int launch_fused(int epi, int kmode, bool fold, bool ip, int kq, const CUtensorMap& a0, const CUtensorMap& a1,
                 const CUtensorMap& b0, const CUtensorMap& b1, const SearchParams& sp, int grid, int smem,
                 cudaStream_t st) {
  using fkh::launch_fused_mode;
  switch (kmode) {
    case 0: return launch_fused_mode<0>(epi, ip, kq, a0, a1, b0, b1, sp, grid, smem, st);
    case 4: return launch_fused_mode<4>(epi, ip, kq, a0, a1, b0, b1, sp, grid, smem, st);
    case 5: return launch_fused_mode<5>(epi, ip, kq, a0, a1, b0, b1, sp, grid, smem, st);
    case 1: return launch_fused_mode<1>(epi, ip, kq, a0, a1, b0, b1, sp, grid, smem, st);
    default:
      if (fold && !ip) return launch_fused_mode<3>(epi, ip, kq, a0, a1, b0, b1, sp, grid, smem, st);
      return launch_fused_mode<2>(epi, ip, kq, a0, a1, b0, b1, sp, grid, smem, st);
  }
}

// Split-N plan: choose the number of N-chunks S so that num_m*S work units
// spread evenly over the persistent grid (each unit = one 128-query tile x
// one contiguous range of base tiles).  Units are ordered chunk-major, so the
// CTAs resident at any moment stream the same ~2 chunks of the base through
// L2 (the base is read from HBM about once per wave).
// min_S bounds a chunk to an L2-resident window (units of one chunk start
// together; over a long chunk they drift apart and re-read it from HBM);
// max_S bounds the partial-list memory.
void plan_split(int num_m, int n_tiles, int num_sms, int min_S, int max_S, int* S_out, int* chunk_out) {
  double best_cost = 1e300;
  int bestS = 1, bestC = n_tiles;
  const double ovh = 1.5;  // per-unit cost in tile-equivalents (A reload, pipeline fill, flush)
  const int smax = std::max(1, std::min(max_S, n_tiles));
  for (int S = std::max(1, std::min(min_S, smax)); S <= smax; ++S) {
    const int chunk = (n_tiles + S - 1) / S;
    const int s_eff = (n_tiles + chunk - 1) / chunk;
    if (s_eff != S) continue;
    const long units = (long)num_m * S;
    const long grid = std::min<long>(units, num_sms);
    const long waves = (units + grid - 1) / grid;
    const double cost = (double)waves * (chunk + ovh) * ((double)num_sms / grid) + 1e-4 * S;
    if (cost < best_cost) {
      best_cost = cost;
      bestS = S;
      bestC = chunk;
    }
  }
  *S_out = bestS;
  *chunk_out = bestC;
}

}  // namespace

// =====================================================================  C ABI
extern "C" {

const char* fk_last_error(void) { return fkh::last_error(); }

int fk_create(int device, int d, int metric, int storage, fk_index** out) {
  if (!out) return set_err(FK_E_INVALID, "out is NULL");
  *out = nullptr;
  if (d < 1) return set_err(FK_E_INVALID, "d must be >= 1");
  if (metric != FK_METRIC_L2 && metric != FK_METRIC_IP)
    return set_err(FK_E_UNSUPPORTED, "metric %d not supported by the GPU flat index (L2=1, IP=0)", metric);
  if (storage != FK_F32 && storage != FK_F16 && storage != FK_BF16)
    return set_err(FK_E_INVALID, "unknown storage %d", storage);
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return set_err(FK_E_INVALID, "device %d out of range (%d devices)", device, ndev);
  CK(cudaSetDevice(device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return set_err(FK_E_UNSUPPORTED, "device %d is sm_%d%d; this build targets sm_100a (B200)", device, prop.major,
                   prop.minor);
  fk_index* h = new fk_index();
  h->device = device;
  h->d = d;
  const int ce = chunk_elems_of(storage);
  h->dp = (d + ce - 1) / ce * ce;
  h->dp16 = (d + 63) / 64 * 64;
  h->metric = metric;
  h->storage = storage;
  // bf16 L2 with >= 3 free padding columns: fold the norms into the operands
  // (FK_NO_FOLD=1 keeps the separate norm tile; tests compare both layouts)
  h->fold = storage == FK_BF16 && metric == FK_METRIC_L2 && d + 3 <= h->dp;
  // fp32: raw storage + 1-pass TF32 filter with exact fp32 rescoring of the
  // survivors (FK_FP32_ALGO=1, experimental) or the 3xTF32 hi/lo split (default)
  h->split = 1;
  if (storage == FK_F32) {
    h->split = 2;
    if (const char* e = getenv("FK_FP32_ALGO"); e && atoi(e) == 1) h->split = 1;
  }
  if (const char* e = getenv("FK_NO_FOLD"); e && atoi(e)) h->fold = 0;
  h->num_sms = prop.multiProcessorCount;
  {  // range results come from the default pool: keep freed blocks cached
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  // {base, queries} exactness flags of the tf32 split (MODE 0/4) and of the
  // scaled fp16 filter operands (MODE 5)
  if (cudaMalloc((void**)&h->inexact, 4 * sizeof(unsigned int)) != cudaSuccess ||
      cudaMemset(h->inexact, 0, 4 * sizeof(unsigned int)) != cudaSuccess ||
      cudaMalloc((void**)&h->xn_max, sizeof(float)) != cudaSuccess || cudaMemset(h->xn_max, 0, sizeof(float)) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->scratch_ev, cudaEventDisableTiming) != cudaSuccess) {
    cudaFree(h->inexact);
    cudaFree(h->xn_max);
    delete h;
    return set_err(FK_E_NOMEM, "cudaMalloc failed");
  }
  if (const char* e = getenv("FK_NUM_SMS")) h->num_sms = std::max(1, std::min(atoi(e), h->num_sms));
  *out = h;
  return FK_OK;
}

void fk_destroy(fk_index* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  cudaFree(h->s0);
  cudaFree(h->s1);
  cudaFree(h->norms);
  cudaFree(h->ids);
  for (DevBuf* b : {&h->q_in, &h->q0, &h->q1, &h->qn, &h->pkey, &h->ppos, &h->thr, &h->pcnt, &h->cbuf, &h->fail,
                    &h->outD, &h->outI, &h->outP, &h->stage_in, &h->stage_ids, &h->rfail, &h->rcomp, &h->rflag,
                    &h->glock, &h->gkeys, &h->rcand, &h->rcount, &h->rdist, &h->rkid, &h->rkrd, &h->rkeep,
                    &h->rrowc, &h->rsel, &h->rnsel, &h->rtmp, &h->rkid2, &h->rkrd2, &h->rv1, &h->rv2, &h->rlims,
                    &h->idt_keys, &h->idt_pos, &h->idt_tmp, &h->idt_miss, &h->rm_kill, &h->rm_flags, &h->rm_keep,
                    &h->x16, &h->f16st, &h->q16, &h->qinv, &h->ovf, &h->rflag_pre})
    b->release();
  if (h->scratch_ev) cudaEventDestroy(h->scratch_ev);
  cudaFree(h->xn_max);
  cudaFree(h->inexact);
  for (auto& q : h->ev_pool)
    for (auto& e : q) cudaEventDestroy(e);
  delete h;
}

int64_t fk_ntotal(const fk_index* h) { return h ? h->ntotal : -1; }
int fk_dim(const fk_index* h) { return h ? h->d : -1; }

int fk_reset(fk_index* h) {
  if (!h) return set_err(FK_E_INVALID, "NULL index");
  std::lock_guard<std::mutex> g(h->mu);
  CK(cudaSetDevice(h->device));
  // a search still in flight on another stream reads the scalars reset below
  if (h->scratch_used) CK(cudaEventSynchronize(h->scratch_ev));
  CK(cudaMemset(h->xn_max, 0, sizeof(float)));
  CK(cudaMemset(h->inexact, 0, 4 * sizeof(unsigned int)));
  if (h->f16st.p) CK(cudaMemset(h->f16st.p, 0, sizeof(F16State)));
  h->ntotal = 0;
  h->idt_n = -1;
  h->f16_rows = 0;
  return FK_OK;
}

int fk_add(fk_index* h, const void* x, int64_t n, int dtype, const int64_t* ids, int on_device, void* stream) {
  if (!h) return set_err(FK_E_INVALID, "NULL index");
  if (n < 0) return set_err(FK_E_INVALID, "n must be >= 0");
  if (dtype != FK_F32 && dtype != FK_F16 && dtype != FK_BF16) return set_err(FK_E_INVALID, "bad dtype %d", dtype);
  if (n == 0) return FK_OK;
  if (!x) return set_err(FK_E_INVALID, "x is NULL");
  if (h->ntotal + n >= (int64_t)0xFFFFFFFFll)
    return set_err(FK_E_UNSUPPORTED, "a single index holds < 2^32 vectors (positions are 32-bit, core.py:219)");
  std::lock_guard<std::mutex> g(h->mu);
  CK(cudaSetDevice(h->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = scratch_begin(h, st);
  if (rc) return rc;
  if ((rc = grow(h, h->ntotal + n, st))) return rc;
  const size_t eb = dtype_bytes(dtype);
  const size_t in_row = (size_t)h->d * eb;
  // stage host input in <= 256 MB slices
  const int64_t slice = on_device ? n : std::max<int64_t>(1, (int64_t)((256ull << 20) / in_row));
  for (int64_t r0 = 0; r0 < n; r0 += slice) {
    const int64_t m = std::min(slice, n - r0);
    const void* src = static_cast<const uint8_t*>(x) + (size_t)r0 * in_row;
    if (!on_device) {
      if ((rc = h->stage_in.ensure(m * in_row))) return rc;
      CK(cudaMemcpyAsync(h->stage_in.p, src, m * in_row, cudaMemcpyHostToDevice, st));
      src = h->stage_in.p;
    }
    if ((rc = launch_prep(kmode_of(h), src, dtype, m, h->d, h->dp, h->s0, h->s1, h->norms, h->ntotal + r0, st,
                          h->fold ? 1 : 0, h->inexact)))
      return rc;
    if (!on_device) CK(cudaStreamSynchronize(st));  // stage buffer reused by the next slice
  }
  if (ids) {
    CK(cudaMemcpyAsync(h->ids + h->ntotal, ids, n * sizeof(int64_t),
                       on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  } else {
    iota_ids_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(h->ids + h->ntotal, h->ntotal, n);
    CKL();
  }
  norm_max_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, st>>>(
      h->norms + h->ntotal, n, reinterpret_cast<unsigned int*>(h->xn_max));
  CKL();
  if ((rc = scratch_end(h, st))) return rc;
  if (!on_device) CK(cudaStreamSynchronize(st));
  h->ntotal += n;
  h->idt_n = -1;
  return FK_OK;
}

}  // extern "C"

namespace {

struct Plan {
  int a_kt = 0;  // a_mode 3: K-chunks of the query operand kept in TMEM
  int kq, epi, nh, num_m, n_tiles, S, chunk_tiles, probe_tiles, num_units, grid, a_mode, stages, smem, S_tot, cap,
      xn_slots,
      acc_stages, n_issuers, cluster, num_mu, bn, kmode;
};

// Tile / split-N / pipeline plan for one fused pass over base rows [0, nb_pass).
// kmode: kernel operand mode of this pass (-1: the index's own); fp32
// storage runs either 3xTF32 (kmode 0, hi+lo streamed) or the 1-pass TF32
// filter (kmode 4, hi or raw streamed)
int make_plan(fk_index* h, int64_t nq, int64_t nb_pass, int k, int kq, int force_S, Plan* pl, int kmode = -1) {
  Plan P{};
  P.kq = kq;
  if (kmode < 0) kmode = kmode_of(h);
  P.kmode = kmode;
  // operand layout of this pass: 16-bit (fp16/bf16 storage, or the scaled
  // fp16 filter copy of fp32 rows, MODE 5) or fp32/tf32
  const bool h16 = h->storage != FK_F32 || kmode == 5;
  const int dpk = kmode == 5 ? h->dp16 : h->dp;
  // 16-bit operands: 2 epilogue warps per TMEM lane quarter (the epilogue, not
  // the MMA, paces a 16-bit tile); fp32 3xTF32 is MMA-paced -> 1 per quarter
  P.epi = h16 ? 8 : 4;
  // 32-deep queues of the fp32 filter (12 < k <= 16): one group per quarter
  // (two spill: cfg2 shape, k = 16: 5.7 ms vs 8.4)
  if (kmode == 5 && kq == 32) P.epi = 4;
  if (const char* e = getenv(kmode == 5 ? "FK_EPI5" : "FK_EPI"); e && kq >= 0) P.epi = atoi(e) == 8 ? 8 : 4;
  P.nh = P.epi / 4;
  // Long 16-bit searches with a light epilogue (folded norms or IP): ONE
  // epilogue group.  Under the board's power cap fewer busy warps buy clock:
  // cfg5 (100M rows) 281 -> 252 ms, 16M rows 39.0 -> 36.5 ms; at 1M rows
  // (not capped) two groups stay 7-10 % faster.  Threshold in nq * rows * dp.
  if (h16 && kmode != 5 && kq > 0 && (h->fold || h->metric == FK_METRIC_IP) &&
      (double)nq * (double)nb_pass * (double)dpk >= 4e12 && !getenv("FK_EPI")) {
    P.epi = 4;
    P.nh = 1;
  }
  P.num_m = (int)((nq + BM - 1) / BM);
  const int split = kmode == 0 ? 2 : 1;
  const int num_kb = dpk / (h16 ? 64 : 32);
  const int a_bytes = split * num_kb * (int)CHUNK_BYTES;
  const int a_tmem_cols = h16 ? dpk / 2 : split * dpk;
  // Query operand placement and tile width:
  //  * 16-bit with two epilogue groups: the accumulator ring wants 4 buffers
  //    (an even count, see below), so A goes to smem (SS MMA) when it fits;
  //  * A in TMEM (TS MMA) beside >= 2 x 128 accumulator columns;
  //  * a large 16-bit A (257-384 TMEM columns, e.g. d=768) is split (a_mode
  //    3): its first 8 K-chunks (256 columns) in TMEM beside TWO 128-column
  //    accumulators, the rest resident in smem (SS MMAs for those K-steps);
  //    one accumulator would drain the MMA pipe at every tile (cfg4 shape:
  //    MMA-only 118 cycles per MMA).  FK_AMODE3=0: the old plan (A wholly in
  //    TMEM beside ONE accumulator, 3.5 % faster than 2 x 64-column
  //    accumulators; FK_BN=64 keeps that one);
  //  * otherwise A in smem, or streamed with every stage (a_mode 2).
  P.bn = 128;
  bool single_acc = getenv("FK_ACC") && atoi(getenv("FK_ACC")) == 1;
  if (h16 && P.nh == 2 && a_bytes <= 64 * 1024) P.a_mode = 1;
  else if (kmode == 4 && a_bytes <= 64 * 1024) P.a_mode = 1;  // 1-pass fp32: 4 accumulators (+2.5 %)
  else if (a_tmem_cols <= 256) P.a_mode = 0;
  else if (a_tmem_cols <= 384) {
    if (h16 && !(getenv("FK_AMODE3") && atoi(getenv("FK_AMODE3")) == 0) && !getenv("FK_BN")) {
      P.a_mode = 3;
      P.a_kt = 8;  // 8 x 32 TMEM columns (64 16-bit K per chunk)
    } else {
      P.a_mode = 0;
      single_acc = true;
    }
  } else P.a_mode = 1;
  // split operand: ONE epilogue group keeps up with the d = 768 MMA (cfg4
  // shape: 28.2 vs 31.0 ms with two, and half the partial lists); range
  // search keeps the default width
  if (P.a_mode == 3 && kq >= 0 && !getenv("FK_EPI")) {
    P.epi = 4;
    P.nh = 1;
  }
  if (const char* e = getenv("FK_FORCE_AMODE")) P.a_mode = std::max(0, std::min(2, atoi(e)));
  if (const char* e = getenv("FK_BN")) {
    P.bn = atoi(e) == 64 ? 64 : 128;
    if (P.bn == 64 && !(getenv("FK_ACC") && atoi(getenv("FK_ACC")) == 1)) single_acc = false;
  }
  // single accumulator: A may take up to 512 - TBN columns; the MMA then
  // waits for each tile's readout (one issuer, one epilogue group)
  if (P.a_mode == 0 && a_tmem_cols > 512 - (single_acc ? 1 : 2) * P.bn) P.a_mode = 1;
  if (P.a_mode != 0) P.bn = 128;
  if (P.bn == 64) {  // 64-column kernels exist only for the default epilogue width
    P.epi = h16 ? 8 : 4;
    P.nh = P.epi / 4;
  }
  const int bn = P.bn;
  const int b_chunk = bn * 128;
  P.n_tiles = (int)((nb_pass + bn - 1) / bn);
  // cluster mode (FK_CLUSTER=2): CTA pairs take query tiles 2*mu, 2*mu+1 of
  // the same chunk and share each base tile (half loaded by each, multicast)
  P.cluster = 1;
  if (const char* e = getenv("FK_CLUSTER")) P.cluster = atoi(e) == 2 ? 2 : 1;
  if (P.num_m < 2 || h->num_sms < 2) P.cluster = 1;
  // (the 1-pass fp32 search certifies far fewer queries in pair mode: not used)
  if (kmode == 4) P.cluster = 1;
  if (kmode == 5 && !getenv("FK_CLUSTER5")) P.cluster = 1;
  P.num_mu = (P.num_m + P.cluster - 1) / P.cluster;
  // chunk <= L2_CHUNK_BYTES of streamed base; partial lists <= PARTIAL_BYTES
  const size_t tile_bytes = (size_t)bn * dpk * (h16 ? 2 : 4) * split;
  // (very large k: partial lists are k deep, so merge cost grows with S -> 4x window)
  size_t l2_chunk = L2_CHUNK_BYTES;
  if (const char* e = getenv("FK_L2_CHUNK_MB")) l2_chunk = (size_t)std::max(1, atoi(e)) << 20;
  const int max_chunk = std::max<int>(16, (int)(l2_chunk * (k >= 512 ? 4 : 1) / tile_bytes));
  const int min_S = (P.n_tiles + max_chunk - 1) / max_chunk;
  const size_t list_bytes = (size_t)nq * P.nh * std::max(k, 1) * 8;  // one chunk's partial lists
  int max_S = (int)std::max<size_t>(1, std::min<size_t>(PARTIAL_BYTES / list_bytes, 1 << 20));
  // 1-pass lists: every query's S x NH lists (+ its overflow list) must fit the
  // rescoring merge's survivor buffer, else the query falls back to a scan
  if ((kmode == 4 || kmode == 5) && kq > 0) max_S = std::max(1, std::min(max_S, (MERGE_SMC - 64) / (P.nh * std::max(k, 1))));
  plan_split(P.num_mu, P.n_tiles, h->num_sms / P.cluster, min_S, max_S, &P.S, &P.chunk_tiles);
  int fs = force_S;
  if (const char* e = getenv("FK_FORCE_S"); e && !force_S) fs = atoi(e);
  if (fs > 0) {
    P.S = std::max(1, std::min(fs, std::min(max_S, P.n_tiles)));
    P.chunk_tiles = (P.n_tiles + P.S - 1) / P.S;
    P.S = (P.n_tiles + P.chunk_tiles - 1) / P.chunk_tiles;
  }
  // Probe chunk (register-queue lists): a short chunk 0 per query tile lets the
  // first units finish early and publish the running-union bound while the
  // long chunks are still in their insertion-heavy start (FK_PROBE = tiles)
  P.probe_tiles = 0;
  {
    int probe = 0;
    if (const char* e = getenv("FK_PROBE")) probe = std::max(0, atoi(e));
    if (probe > 0 && kq > 0 && P.S >= 2 && P.n_tiles > 4 * probe) {
      P.probe_tiles = probe;
      P.chunk_tiles = (P.n_tiles - probe + P.S - 1) / P.S;
      P.S = 1 + (P.n_tiles - probe + P.chunk_tiles - 1) / P.chunk_tiles;
    }
  }
  P.num_units = P.num_mu * P.S;  // per CTA pair in cluster mode
  P.grid = P.cluster * std::min(P.num_units, h->num_sms / P.cluster);
  const int hist_bytes = kq == 0 ? P.epi * 1024 : 0;
  // norm-tile ring: 4 slots when smem is tight (fp32), 8 otherwise
  // (even: one sub-ring per producer/issuer pair)
  P.xn_slots = (h->metric == FK_METRIC_IP || h->fold) ? 0 : (!h16 && P.a_mode != 2) ? 4 : 8;
  const int xn_bytes = P.xn_slots * bn * 4;
  auto stage_bytes_for = [&](int mode) { return split * b_chunk + (mode == 2 ? split * (int)CHUNK_BYTES : 0); };
  // smem-resident query chunks: all (a_mode 1) or those past the TMEM part (a_mode 3)
  const int a_tail_bytes = split * (num_kb - P.a_kt) * (int)CHUNK_BYTES;
  auto a_smem_for = [&](int mode) { return mode == 1 ? a_bytes : (mode == 3 ? a_tail_bytes : 0); };
  auto stages_for = [&](int mode) {
    const int avail = SMEM_LIMIT - SMEM_RESERVE - hist_bytes - xn_bytes - a_smem_for(mode);
    return avail / stage_bytes_for(mode);
  };
  P.stages = stages_for(P.a_mode);
  if (P.a_mode == 1 && P.stages < 3) {
    P.a_mode = 2;
    P.stages = stages_for(2);
  }
  P.stages = std::min(P.stages, MAX_STAGES);
  if (const char* e = getenv("FK_STAGES")) P.stages = std::max(2, std::min(P.stages, atoi(e)));
  if (P.stages < 2) return set_err(FK_E_UNSUPPORTED, "pipeline does not fit in shared memory");
  // TMEM: 512 columns = acc_stages x 128-column accumulators (+ the query operand in a_mode 0)
  P.acc_stages = std::min(4, (512 - (P.a_mode == 0 ? a_tmem_cols : (P.a_mode == 3 ? P.a_kt * 32 : 0))) / bn);
  if (const char* e = getenv("FK_ACC")) P.acc_stages = std::max(1, std::min(P.acc_stages, atoi(e)));
  if (single_acc) P.acc_stages = 1;
  P.n_issuers = P.stages >= 4 ? 2 : 1;  // each issuer needs a sub-ring of >= 2 slots
  if (const char* e = getenv("FK_ISSUERS")) P.n_issuers = (atoi(e) == 1 || P.stages < 4) ? 1 : 2;
  // Tiles alternate between the 2 MMA issuers and between the NH epilogue
  // groups; each party must wait on EVERY phase of the buffers it uses (an
  // mbarrier parity wait cannot skip a phase), so buffer = tile % acc_stages
  // must map each party onto its own buffers: acc_stages % parties == 0.
  if (P.acc_stages == 1) {  // one buffer: one issuer and one epilogue group wait on every phase
    P.n_issuers = 1;
    P.epi = 4;
    P.nh = 1;
  }
  if ((P.n_issuers == 2 || P.nh == 2) && (P.acc_stages & 1)) P.acc_stages -= 1;
  P.smem = SMEM_RESERVE + hist_bytes + xn_bytes + a_smem_for(P.a_mode) + P.stages * stage_bytes_for(P.a_mode);
  P.S_tot = P.S * P.nh;
  P.cap = kq == 0 ? (std::max(2 * k, k + 256) + 31) / 32 * 32 : 0;  // >= k + one tile (128) of slack
  *pl = P;
  return FK_OK;
}

// One fused GEMM + top-k pass over base rows [0, nb_pass) for the prepared
// queries; partial lists land in h->pkey/ppos (+pcnt), bounds in h->thr.
int run_fused(fk_index* h, const Plan& P, int64_t nq, int64_t nb_pass, int k, bool ip, cudaStream_t st) {
  int rc;
  if ((rc = h->pkey.ensure((size_t)nq * P.S_tot * k * sizeof(uint32_t)))) return rc;
  if ((rc = h->ppos.ensure((size_t)nq * P.S_tot * k * sizeof(uint32_t)))) return rc;
  if (P.kq == 0) {
    if ((rc = h->pcnt.ensure((size_t)nq * P.S_tot * sizeof(int)))) return rc;
    if ((rc = h->cbuf.ensure((size_t)P.grid * P.epi * 32 * P.cap * sizeof(uint64_t)))) return rc;
  }
  CUtensorMap ta0, ta1, tb0, tb1;
  const bool f16 = P.kmode == 5;  // scaled fp16 filter copies of the fp32 rows
  const bool h16 = h->storage != FK_F32 || f16;
  const int eb = h16 ? 2 : 4;
  const int dpk = f16 ? h->dp16 : h->dp;
  const void* qop = f16 ? h->q16.p : h->q0.p;
  const void* bop = f16 ? h->x16.p : h->s0;
  if ((rc = make_map(&ta0, qop, eb, dpk, nq))) return rc;
  const uint32_t b_rows = P.cluster == 2 ? P.bn / 2 : P.bn;  // cluster mode: each CTA loads half a tile
  if ((rc = make_map(&tb0, bop, eb, dpk, nb_pass, b_rows))) return rc;
  if (P.kmode == 0) {
    if ((rc = make_map(&ta1, h->q1.p, eb, h->dp, nq))) return rc;
    if ((rc = make_map(&tb1, h->s1, eb, h->dp, nb_pass, b_rows))) return rc;
  } else {
    ta1 = ta0;
    tb1 = tb0;
  }
  SearchParams sp;
  std::memset(&sp, 0, sizeof(sp));
  sp.qnorm = static_cast<const float*>(h->qn.p);
  sp.xnorm = h->norms;
  sp.xn_max = h->xn_max;
  sp.part_key = static_cast<uint32_t*>(h->pkey.p);
  sp.part_pos = static_cast<uint32_t*>(h->ppos.p);
  sp.thr_key = static_cast<uint32_t*>(h->thr.p);
  sp.part_cnt = static_cast<int*>(h->pcnt.p);
  sp.cbuf = static_cast<uint64_t*>(h->cbuf.p);
  sp.cap = P.cap;
  sp.dbg_ip = h->dbg_ip;
  sp.trace = h->trace;
  sp.qa0 = qop;
  sp.qa1 = h->q1.p;
  sp.nq = (int)nq;
  sp.nb = (int)nb_pass;
  sp.k = k;
  sp.num_m = P.num_m;
  sp.n_tiles = P.n_tiles;
  sp.chunk_tiles = P.chunk_tiles;
  sp.probe_tiles = P.probe_tiles;
  sp.S = P.S;
  sp.num_units = P.num_units;
  sp.num_kb = dpk / (h16 ? 64 : 32);
  sp.a_mode = P.a_mode;
  sp.a_kt = P.a_kt;
  sp.stages = P.stages;
  sp.xn_slots = P.xn_slots;
  sp.acc_stages = P.acc_stages;
  {
    const int bk = h16 ? 64 : 32, kstep = h16 ? 16 : 8;
    const int last = h->d + (h->fold ? 3 : 0) - (sp.num_kb - 1) * bk;  // K elements in the last chunk (1..bk)
    sp.kk_last = (last + kstep - 1) / kstep;
  }
  sp.n_issuers = P.n_issuers;
  sp.n_producers = P.n_issuers == 2 ? 2 : 1;
  if (const char* e = getenv("FK_PRODUCERS")) sp.n_producers = (atoi(e) == 1 || P.n_issuers == 1) ? 1 : 2;
  sp.cluster = P.cluster;
  sp.bn = P.bn;
  sp.xbase = h->s0;
  sp.kfinal = h->r_kfinal > 0 ? h->r_kfinal : k;
  sp.pub_mask = 15;
  if (const char* e = getenv("FK_PUB")) sp.pub_mask = std::max(0, atoi(e));
  sp.rflag = static_cast<unsigned int*>(h->rflag.p);
  if (h->r_prepass) {
    // bound pre-pass: its rows are searched again by the main pass, so it
    // must not feed the union (duplicates) or flag rows; only thr_key counts
    if ((rc = h->rflag_pre.ensure((size_t)nq * sizeof(unsigned int)))) return rc;
    sp.rflag = static_cast<unsigned int*>(h->rflag_pre.p);
  } else if (h->r_ovf_cap > 0) {
    sp.ovf_cap = h->r_ovf_cap;
    sp.ovf_key = static_cast<uint32_t*>(h->ovf.p);
    sp.ovf_pos = sp.ovf_key + (size_t)nq * sp.ovf_cap;
    sp.ovf_cnt = sp.ovf_pos + (size_t)nq * sp.ovf_cap;
  }
  // exactness flags: tf32 split {base, queries}; MODE 5 its own pair
  sp.inexact = f16 ? h->inexact + 2 : (h->split == 2 ? h->inexact : nullptr);  // raw storage: full band
  sp.qinv = static_cast<const float*>(h->qinv.p);
  sp.band_l2 = f1p_band(P.kmode);
  sp.xinv = f16 ? &static_cast<const F16State*>(h->f16st.p)->xinv : nullptr;
  sp.glock = h->r_union ? static_cast<unsigned int*>(h->glock.p) : nullptr;
  sp.gkeys = h->r_union ? static_cast<uint32_t*>(h->gkeys.p) : nullptr;
  sp.radius = h->r_radius;
  sp.rcand = static_cast<unsigned long long*>(h->rcand.p);
  sp.rcount = static_cast<unsigned long long*>(h->rcount.p);
  sp.rcap = h->r_cap;
  sp.num_mu = P.num_mu;
  if (const char* e = getenv("FK_DEBUG_FLAGS")) sp.dbg_flags = atoi(e);
  // streamed base tiles are re-read by every query tile of the chunk: keep
  // them (evict_last beats evict_first by 5-9 % on cfg2/3/5, FK_B_POLICY)
  sp.b_policy = 2;
  if (const char* e = getenv("FK_B_POLICY")) sp.b_policy = atoi(e);
  rc = launch_fused(P.epi, P.kmode, h->fold != 0, ip, P.kq, ta0, ta1, tb0, tb1, sp, P.grid, P.smem, st);
  if (rc == FK_OK) h->nlaunch++;
  return rc;
}

int launch_merge(fk_index* h, const Plan& P, int64_t nq, int k, bool ip, float* dD, int64_t* dI, int64_t* dP,
                 int* fail, cudaStream_t st) {
  const uint32_t* pk = static_cast<const uint32_t*>(h->pkey.p);
  const uint32_t* pp = static_cast<const uint32_t*>(h->ppos.p);
  if (P.kq == 0 || P.S_tot > 128) {  // bounded merge (any number of lists)
    // survivors buffer sized to the expected survivor count (~k..2k, the
    // radix-select fallback covers overflow) so several CTAs share an SM;
    // winners: k padded to a power of two for the bitonic sort
    // k >= 512 (S lists of k each: ~S*k/2 survivors): an 8k-entry buffer and
    // 512 threads per query (cfg3 k=1024: merge 2.07 -> 1.33 ms; smaller k:
    // 4k entries and 256 threads stay best, cfg4 k=100)
    const bool big_k = k >= 512;
    int smc = std::min(MERGE_SMC, std::max(1024, (big_k ? 8 : 4) * k));
    if (nq <= 4 * (int64_t)h->num_sms)  // small batch: every list entry fits (no global-memory select)
      smc = std::min(MERGE_SMC, std::max<int>(smc, P.S_tot * k));
    if (const char* e = getenv("FK_MERGE_SMC")) smc = std::max(1, std::min(MERGE_SMC, atoi(e)));
    int p2 = 1;
    while (p2 < k) p2 <<= 1;
    const size_t msmem = (size_t)(smc + p2) * 8;
    static std::atomic<uint64_t> merge_cfg{0};
    int rc = fkh::once_per_device(merge_cfg, []() -> int {
      CK(cudaFuncSetAttribute(merge_large_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (MERGE_SMC + FK_MAX_K) * 8));
      CK(cudaFuncSetAttribute(merge_large_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (MERGE_SMC + FK_MAX_K) * 8));
      return FK_OK;
    });
    if (rc) return rc;
    const int* pc = P.kq == 0 ? static_cast<const int*>(h->pcnt.p) : nullptr;  // queue lists: k entries each
    const uint32_t* thr = static_cast<const uint32_t*>(h->thr.p);
    int mthreads = big_k ? 512 : 256;
    if (const char* e = getenv("FK_MERGE_THREADS")) mthreads = std::max(32, std::min(1024, atoi(e))) / 32 * 32;
    if (ip)
      merge_large_kernel<true><<<(unsigned)nq, mthreads, msmem, st>>>(pk, pp, pc, P.S_tot, (int)nq, k, thr, h->ids, dD,
                                                                       dI, dP, smc, fail);
    else
      merge_large_kernel<false><<<(unsigned)nq, mthreads, msmem, st>>>(pk, pp, pc, P.S_tot, (int)nq, k, thr, h->ids,
                                                                        dD, dI, dP, smc, fail);
  } else {
    const int wpb = 8;
    const unsigned mgrid = (unsigned)((nq + wpb - 1) / wpb);
    if (ip)
      merge_kernel<true><<<mgrid, wpb * 32, 0, st>>>(pk, pp, P.S_tot, (int)nq, k, h->ids, dD, dI, dP);
    else
      merge_kernel<false><<<mgrid, wpb * 32, 0, st>>>(pk, pp, P.S_tot, (int)nq, k, h->ids, dD, dI, dP);
  }
  CKL();
  h->nlaunch++;
  return FK_OK;
}

// Queries -> device operand layout + norms (shared by search and range search).
int stage_queries(fk_index* h, const void* q, int64_t nq, int dtype, int on_device, cudaStream_t st,
                  bool f16 = false) {
  int rc;
  const size_t in_row = (size_t)h->d * dtype_bytes(dtype);
  const void* qsrc = q;
  if (!on_device) {
    if ((rc = h->q_in.ensure(nq * in_row))) return rc;
    CK(cudaMemcpyAsync(h->q_in.p, q, nq * in_row, cudaMemcpyHostToDevice, st));
    qsrc = h->q_in.p;
  }
  const size_t qrow = row_bytes(h);
  if ((rc = h->q0.ensure(nq * qrow))) return rc;
  if (h->split == 2 && (rc = h->q1.ensure(nq * qrow))) return rc;
  if ((rc = h->qn.ensure(nq * sizeof(float)))) return rc;
  if (h->inexact) CK(cudaMemsetAsync(h->inexact + 1, 0, sizeof(unsigned int), st));
  if (f16) {  // MODE 5: scaled fp16 filter rows + 2^-s per query (filter16_kernels.cuh)
    if ((rc = h->q16.ensure((size_t)nq * h->dp16 * 2))) return rc;
    if ((rc = h->qinv.ensure((size_t)nq * sizeof(float)))) return rc;
    CK(cudaMemsetAsync(h->inexact + 3, 0, sizeof(unsigned int), st));
    f16_query_kernel<<<(unsigned)((nq + 7) / 8), 256, 0, st>>>(qsrc, dtype, nq, h->d, h->dp16,
                                                                 static_cast<__half*>(h->q16.p),
                                                                 static_cast<float*>(h->qinv.p), h->inexact + 3);
    CKL();
    h->nlaunch++;
  }
  return launch_prep(kmode_of(h), qsrc, dtype, nq, h->d, h->dp, h->q0.p, h->q1.p, static_cast<float*>(h->qn.p), 0, st,
                     h->fold ? 2 : 0, h->inexact ? h->inexact + 1 : nullptr);
}

// MODE 5: bring the scaled fp16 copy of the base up to date (rows added
// since the last conversion; every row when the base scale changed or the
// copy was invalidated).  The scale decision happens on the device.
int ensure_f16_base(fk_index* h, cudaStream_t st) {
  int rc;
  if (h->split != 2 || !h->s1) return set_err(FK_E_UNSUPPORTED, "the fp16 filter needs the hi/lo fp32 storage");
  const size_t need = (size_t)h->cap * h->dp16 * 2;
  if (h->x16.bytes < need) {
    if ((rc = h->x16.ensure(need))) return rc;
    h->f16_rows = 0;
  }
  if (!h->f16st.p) {
    if ((rc = h->f16st.ensure(sizeof(F16State)))) return rc;
    CK(cudaMemsetAsync(h->f16st.p, 0, sizeof(F16State), st));
    h->f16_rows = 0;
  }
  if (h->f16_rows == h->ntotal) return FK_OK;
  auto fs = static_cast<F16State*>(h->f16st.p);
  const auto hi = static_cast<const float*>(h->s0);
  const auto lo = static_cast<const float*>(h->s1);
  const size_t e0 = (size_t)h->f16_rows * h->dp, e1 = (size_t)h->ntotal * h->dp;
  const unsigned ga = (unsigned)std::min<size_t>((e1 - e0 + 255) / 256, (size_t)h->num_sms * 8);
  absmax_rows_kernel<<<ga, 256, 0, st>>>(hi, lo, e0, e1, &fs->absmax);
  CKL();
  f16_scale_kernel<<<1, 32, 0, st>>>(fs, (long long)h->f16_rows, h->inexact + 2);
  CKL();
  const unsigned gc = (unsigned)std::min<int64_t>((h->ntotal + 7) / 8, (int64_t)h->num_sms * 16);
  f16_base_kernel<<<gc, 256, 0, st>>>(hi, lo, h->f16_rows, h->ntotal, h->d, h->dp, h->dp16,
                                      static_cast<__half*>(h->x16.p), fs, h->inexact + 2);
  CKL();
  h->nlaunch += 3;
  h->f16_rows = h->ntotal;
  return FK_OK;
}

// Bound pre-pass: a short fused pass over the first rows of the base (every
// query) publishes each query's k-th (+ band) to thr_key before the main
// pass, so the first wave of units filters with a useful bound instead of
// inserting ~k ln(n/k) candidates per row.  Any k entries give a valid upper
// bound, so the rows may be any subset; the main pass searches them again.
// FK_PREPASS = rows (default 0 = off: on cfg2 16k / 32k rows cost 0.26 /
// 0.40 ms more than they save -- the running-union bound already makes the
// later waves cheap).
// One bound-only fused pass over base rows [0, rows): lists of `k` entries
// (queue bucket kq), publishing (kfinal-th + band) per query to thr_key; no
// union, overflow lists or row flags (its rows are searched again).
int run_bound_pass(fk_index* h, int64_t nq, int64_t rows, int k, int kq, int kfinal, bool ip, int kmode,
                   cudaStream_t st, bool use_union = false) {
  Plan pp;
  int rc;
  if ((rc = make_plan(h, nq, rows, k, kq, 0, &pp, kmode))) return rc;
  const bool su = h->r_union;
  const int so = h->r_ovf_cap, sk = h->r_kfinal;
  h->r_prepass = true;
  h->r_union = use_union;  // union of disjoint sample rows: valid when the main pass does not read it
  h->r_ovf_cap = 0;
  h->r_kfinal = kfinal;
  rc = run_fused(h, pp, nq, rows, k, ip, st);
  h->r_prepass = false;
  h->r_union = su;
  h->r_ovf_cap = so;
  h->r_kfinal = sk;
  return rc;
}

int run_prepass(fk_index* h, int64_t nq, int k, int kq, bool ip, int kmode, cudaStream_t st) {
  if (kq <= 0) return FK_OK;
  int64_t rows = 0;
  if (const char* e = getenv("FK_PREPASS")) rows = std::max<int64_t>(0, atoll(e));
  rows = rows / BN * BN;
  if (rows <= 0 || h->ntotal < 16 * rows) return FK_OK;
  return run_bound_pass(h, nq, rows, k, kq, h->r_kfinal > 0 ? h->r_kfinal : k, ip, kmode, st);
}

// fp32 MODE 4 search: fused pass with a 1-pass TF32 GEMM keeping k' >= k
// entries per list in tf32 order, then merge_rescore_kernel (certify + exact
// values + exact top-k); uncertified queries get the exact fallback.
int search_mode4(fk_index* h, int64_t nq, int k, bool ip, float* dD, int64_t* dI, int64_t* dP, cudaEvent_t* ev,
                 cudaStream_t st, Plan* plan_out, int kmode = 4) {
  int rc;
  if (kmode == 5 && (rc = ensure_f16_base(h, st))) return rc;
  // k' >= k entries per list, the slack absorbs the tf32 band around the k-th
  // (register queues of 16 with the per-query overflow lists: measured
  // cfg2 3.7 ms fused vs 5.6 with 32-deep queues, 0 of 10k uncertified).
  // The slack k' - k must stay >= 4: every entry a full queue drops within
  // the band goes to the 64-entry overflow list, and with k' = k (k = 16) it
  // overflows for every query -> the whole-base exact fallback (cfg2 shape,
  // k = 16: 3277 ms; k = 14: 54 ms, 204 ms at 1k queries).  12 < k <= 16
  // take 32-deep queues (5.7 ms at k = 16, 0 uncertified).
  int kp = k <= 4 ? 8 : k <= 12 ? 16 : k <= 16 ? 32 : std::min(k + std::max(64, k / 4), FK_MAX_K);
  if (const char* e = getenv("FK_KP")) kp = std::max(k, std::min(atoi(e), FK_MAX_K));
  const int kq = kp <= 8 ? 8 : kp <= 16 ? 16 : kp <= 32 ? 32 : 0;
  Plan pl;
  if ((rc = make_plan(h, nq, h->ntotal, kp, kq, 0, &pl, kmode))) return rc;
  *plan_out = pl;
  if ((rc = h->thr.ensure((size_t)nq * sizeof(uint32_t)))) return rc;
  CK(cudaMemsetAsync(h->thr.p, 0xFF, (size_t)nq * sizeof(uint32_t), st));
  if ((rc = h->rflag.ensure((size_t)nq * sizeof(unsigned int)))) return rc;
  CK(cudaMemsetAsync(h->rflag.p, 0, (size_t)nq * sizeof(unsigned int), st));
  const bool gunion = pl.num_units >= 4 * pl.grid && !getenv("FK_NO_UNION");
  if (gunion) {
    if ((rc = h->glock.ensure((size_t)nq * sizeof(unsigned int))) || (rc = h->gkeys.ensure((size_t)nq * 32 * 4)))
      return rc;
    CK(cudaMemsetAsync(h->glock.p, 0, (size_t)nq * sizeof(unsigned int), st));
    CK(cudaMemsetAsync(h->gkeys.p, 0xFF, (size_t)nq * 32 * 4, st));
  }
  h->r_union = gunion;
  h->r_kfinal = k;
  // overflow lists for band members dropped by full register queues
  int ovf_cap = kq > 0 ? 64 : 0;
  if (const char* e = getenv("FK_OVF")) ovf_cap = kq > 0 ? std::max(0, atoi(e)) : 0;
  uint32_t *okey = nullptr, *opos = nullptr;
  unsigned int* ocnt = nullptr;
  if (ovf_cap > 0) {
    if ((rc = h->ovf.ensure((size_t)nq * (2 * ovf_cap + 1) * 4))) return rc;
    okey = static_cast<uint32_t*>(h->ovf.p);
    opos = okey + (size_t)nq * ovf_cap;
    ocnt = opos + (size_t)nq * ovf_cap;
    CK(cudaMemsetAsync(ocnt, 0, (size_t)nq * 4, st));
  }
  h->r_ovf_cap = ovf_cap;
  if (ev) CK(cudaEventRecord(ev[1], st));
  if ((rc = run_prepass(h, nq, kp, kq, ip, kmode, st))) return rc;
  if (kq == 0 && !getenv("FK_NO_EST")) {
    // large k: seed each query's bound with (32nd filter value of a sample of
    // m = 8 ntotal / k rows) + band -- near the 4k-th overall for unordered
    // data -- so the lists the merge gathers stay ~4k deep; the merge
    // certifies bound > t_k + band per query (else the exact fallback)
    const int64_t m_est = est_rows(h->ntotal, k);
    // (the sample's units and epilogue groups each see part of it: their
    // lists merge into the per-query union, whose 32nd + band is published;
    // the KQ = 0 main pass never reads the union)
    if (m_est > 0) {
      if ((rc = h->glock.ensure((size_t)nq * sizeof(unsigned int))) || (rc = h->gkeys.ensure((size_t)nq * 32 * 4)))
        return rc;
      CK(cudaMemsetAsync(h->glock.p, 0, (size_t)nq * sizeof(unsigned int), st));
      CK(cudaMemsetAsync(h->gkeys.p, 0xFF, (size_t)nq * 32 * 4, st));
      if ((rc = run_bound_pass(h, nq, m_est, 32, 32, 32, ip, kmode, st, true))) return rc;
    }
  }
  rc = run_fused(h, pl, nq, h->ntotal, kp, ip, st);
  h->r_kfinal = 0;
  h->r_union = false;
  h->r_ovf_cap = 0;
  if (rc) return rc;
  if (ev) CK(cudaEventRecord(ev[2], st));
  if ((rc = h->rfail.ensure((size_t)(2 * nq + 1) * sizeof(int)))) return rc;
  int* fcount = static_cast<int*>(h->rfail.p) + 2 * nq;  // device list of uncertified queries
  int* flist = static_cast<int*>(h->rfail.p) + nq;
  CK(cudaMemsetAsync(fcount, 0, sizeof(int), st));
  // survivor buffer: 24 k' by default; a small batch (one query tile split
  // over every SM: S_tot k' entries per query) gets room for all of its list
  // and overflow entries -- few CTAs, and an overflow would send the query to
  // the exact fallback (a scan of the whole base per query)
  // (any batch size: when every list entry could survive -- e.g. 32-deep
  // queues over many lists -- an overflow would send the query to the exact
  // fallback; a larger buffer only costs merge occupancy)
  int smc = std::min(MERGE_SMC, std::max(1024, 24 * kp));
  smc = std::min(MERGE_SMC, std::max<int>(smc, pl.S_tot * kp + ovf_cap));
  int p2 = 1;
  while (p2 < k) p2 <<= 1;
  static std::atomic<uint64_t> cfg{0};
  if ((rc = fkh::once_per_device(cfg, []() -> int {
         CK(cudaFuncSetAttribute(merge_rescore_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (MERGE_SMC + FK_MAX_K) * 8));
         CK(cudaFuncSetAttribute(merge_rescore_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (MERGE_SMC + FK_MAX_K) * 8));
         return FK_OK;
       })))
    return rc;
  const size_t msmem = (size_t)(smc + p2) * 8;
  const auto pk = static_cast<const uint32_t*>(h->pkey.p);
  const auto pp = static_cast<const uint32_t*>(h->ppos.p);
  const int* pc = kq == 0 ? static_cast<const int*>(h->pcnt.p) : nullptr;
  const auto thr = static_cast<const uint32_t*>(h->thr.p);
  const auto q0 = static_cast<const float*>(h->q0.p);
  const auto xb = static_cast<const float*>(h->s0);
  // split storage: the exact operands are hi + lo (exact in fp32)
  const auto q1 = h->split == 2 ? static_cast<const float*>(h->q1.p) : nullptr;
  const auto xl = h->split == 2 ? static_cast<const float*>(h->s1) : nullptr;
  const auto qn = static_cast<const float*>(h->qn.p);
  int* fail = static_cast<int*>(h->rfail.p);
  // the filter pass's exactness flags and rounding-band coefficient (L2; IP half)
  const unsigned int* inexact = kmode == 5 ? h->inexact + 2 : (h->split == 2 ? h->inexact : nullptr);
  const float band_l2 = f1p_band(kmode);
  // register-queue lists of a few hundred entries per query: the
  // warp-per-query merge (same certification, band and exact values)
  const bool warp_merge = kq > 0 && (size_t)pl.S_tot * kp <= 1024 && k <= 32 &&
                          !(getenv("FK_MERGE_WARP") && atoi(getenv("FK_MERGE_WARP")) == 0);
  const auto rfl = static_cast<const unsigned int*>(h->rflag.p);
  if (warp_merge && ip)
    merge_rescore_warp_kernel<true><<<(unsigned)((nq + 7) / 8), 256, 0, st>>>(
        pk, pp, pl.S_tot, (int)nq, kp, k, thr, q0, q1, xb, xl, qn, h->norms, h->xn_max, h->dp, h->ids, dD, dI, dP,
        fail, fcount, flist, rfl, inexact, band_l2, okey, opos, ocnt, ovf_cap);
  else if (warp_merge)
    merge_rescore_warp_kernel<false><<<(unsigned)((nq + 7) / 8), 256, 0, st>>>(
        pk, pp, pl.S_tot, (int)nq, kp, k, thr, q0, q1, xb, xl, qn, h->norms, h->xn_max, h->dp, h->ids, dD, dI, dP,
        fail, fcount, flist, rfl, inexact, band_l2, okey, opos, ocnt, ovf_cap);
  else if (ip)
    merge_rescore_kernel<true><<<(unsigned)nq, 256, msmem, st>>>(pk, pp, pc, pl.S_tot, (int)nq, kp, k, thr, q0, q1, xb, xl, qn,
                                                                  h->norms, h->xn_max, h->dp, h->ids, dD, dI, dP, smc,
                                                                  fail, fcount, flist,
                                                                  static_cast<const unsigned int*>(h->rflag.p),
                                                                  inexact, band_l2, okey, opos, ocnt, ovf_cap);
  else
    merge_rescore_kernel<false><<<(unsigned)nq, 256, msmem, st>>>(pk, pp, pc, pl.S_tot, (int)nq, kp, k, thr, q0, q1, xb, xl, qn,
                                                                   h->norms, h->xn_max, h->dp, h->ids, dD, dI, dP, smc,
                                                                   fail, fcount, flist,
                                                                  static_cast<const unsigned int*>(h->rflag.p),
                                                                  inexact, band_l2, okey, opos, ocnt, ovf_cap);
  CKL();
  h->nlaunch++;
  if (getenv("FK_DIAG")) {  // diagnostics: how many queries failed certification
    int nf = 0;
    CK(cudaMemcpyAsync(&nf, fcount, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    long long osum = 0, orows = 0, omax = 0;
    if (ocnt) {
      std::vector<unsigned int> oc(nq);
      CK(cudaMemcpy(oc.data(), ocnt, nq * 4, cudaMemcpyDeviceToHost));
      for (auto c : oc) {
        osum += c;
        orows += c > 0;
        omax = std::max<long long>(omax, c);
      }
    }
    std::vector<int> fv(nq);
    CK(cudaMemcpy(fv.data(), fail, nq * sizeof(int), cudaMemcpyDeviceToHost));
    int why[5] = {0, 0, 0, 0, 0};
    for (int v : fv) why[std::max(0, std::min(4, v))]++;
    fprintf(stderr,
            "[fk] mode%d k=%d k'=%d nq=%lld uncertified=%d (smem %d, band %d, <k %d, flag %d) overflow rows=%lld "
            "entries=%lld max=%lld\n",
            kmode, k, kp, (long long)nq, nf, why[1], why[2], why[3], why[4], orows, osum, omax);
  }
  // uncertified queries: exact fallback on the device (no host sync); up to
  // one wave of CTAs, each scanning the base for its failed queries, with a
  // scratch slot of one exact composite per row (<= 2 GB of slots)
  const int nslots = (int)std::max<int64_t>(
      1, std::min<int64_t>({nq, (int64_t)h->num_sms, (2048ll << 20) / (h->ntotal * 8)}));
  if ((rc = h->rcomp.ensure((size_t)nslots * h->ntotal * 8))) return rc;
  static std::atomic<uint64_t> fcfg{0};
  if ((rc = fkh::once_per_device(fcfg, []() -> int {
         CK(cudaFuncSetAttribute(fallback_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, FK_MAX_K * 8));
         CK(cudaFuncSetAttribute(fallback_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, FK_MAX_K * 8));
         return FK_OK;
       })))
    return rc;
  auto comp = static_cast<uint64_t*>(h->rcomp.p);
  const size_t ssm = (size_t)p2 * 8;
  const unsigned dgrid = 2u * (unsigned)h->num_sms;
  if (ip)
    fallback_dist_kernel<true><<<dgrid, 256, 0, st>>>(fcount, flist, nslots, q0, q1, qn, xb, xl, h->norms, h->ntotal,
                                                      h->dp, comp);
  else
    fallback_dist_kernel<false><<<dgrid, 256, 0, st>>>(fcount, flist, nslots, q0, q1, qn, xb, xl, h->norms,
                                                       h->ntotal, h->dp, comp);
  CKL();
  if (ip)
    fallback_select_kernel<true><<<nslots, 1024, ssm, st>>>(fcount, flist, nslots, h->ntotal, k, h->ids, dD, dI, dP,
                                                            comp);
  else
    fallback_select_kernel<false><<<nslots, 1024, ssm, st>>>(fcount, flist, nslots, h->ntotal, k, h->ids, dD, dI, dP,
                                                             comp);
  CKL();
  h->nlaunch += 2;
  if (ip)
    fallback_kernel<true><<<nslots, 256, ssm, st>>>(fcount, flist, q0, q1, qn, xb, xl, h->norms, h->ntotal, h->dp, k,
                                                    h->ids, dD, dI, dP, comp);
  else
    fallback_kernel<false><<<nslots, 256, ssm, st>>>(fcount, flist, q0, q1, qn, xb, xl, h->norms, h->ntotal, h->dp, k,
                                                     h->ids, dD, dI, dP, comp);
  CKL();
  h->nlaunch++;
  return FK_OK;
}

// Direct path (flat.py:58-62 -> flat_search flat.py:76-91) for batches
// below the BLAS threshold: exact direct distances of every (query, row),
// then a per-query top-k selection.  Queries are staged already.
int search_direct(fk_index* h, int64_t nq, int k, bool ip, float* dD, int64_t* dI, int64_t* dP, cudaEvent_t* ev,
                  cudaStream_t st) {
  int rc;
  const int64_t n = h->ntotal;
  if (n > (int64_t)INT32_MAX) return set_err(FK_E_UNSUPPORTED, "direct path over more than 2^31 rows");
  const int64_t group = std::max<int64_t>(1, std::min<int64_t>(nq, (2048ll << 20) / (n * 8)));
  if ((rc = h->rcomp.ensure((size_t)group * n * 8))) return rc;
  auto comp = static_cast<uint64_t*>(h->rcomp.p);
  int p2 = 1;
  while (p2 < k) p2 <<= 1;
  const size_t qrow = row_bytes(h);
  const int mode = h->storage == FK_F32 ? (h->split == 2 ? 0 : 4) : (h->storage == FK_F16 ? 1 : 2);
  if (ev) CK(cudaEventRecord(ev[1], st));
  for (int64_t g0 = 0; g0 < nq; g0 += group) {
    const int gq = (int)std::min(group, nq - g0);
    const void* qa = static_cast<const uint8_t*>(h->q0.p) + (size_t)g0 * qrow;
    const void* qb = h->split == 2 ? static_cast<const uint8_t*>(h->q1.p) + (size_t)g0 * qrow : nullptr;
    const unsigned grid = (unsigned)((n + 7) / 8);
    const size_t qsm = (size_t)gq * h->d * sizeof(double);
    // several queries: the 8-query batched reduction (19 queries on 1M rows
    // 2.55 -> 1.53 ms); one query keeps the plain butterfly (0.36 vs 0.45 ms)
    if (gq >= 2 && h->d <= 256 && qsm <= 48 * 1024 && !(getenv("FK_DIRECT_WARP1") && atoi(getenv("FK_DIRECT_WARP1")))) {
      const unsigned grid = (unsigned)std::min<int64_t>((n + 7) / 8, (int64_t)h->num_sms * 16);
      if (mode == 0)
        direct_dist_warp8_kernel<0><<<grid, 256, qsm, st>>>(qa, qb, gq, h->s0, h->s1, n, h->d, h->dp, ip, 0, comp);
      else if (mode == 4)
        direct_dist_warp8_kernel<4><<<grid, 256, qsm, st>>>(qa, nullptr, gq, h->s0, nullptr, n, h->d, h->dp, ip, 0, comp);
      else if (mode == 1)
        direct_dist_warp8_kernel<1><<<grid, 256, qsm, st>>>(qa, nullptr, gq, h->s0, nullptr, n, h->d, h->dp, ip, 0, comp);
      else
        direct_dist_warp8_kernel<2><<<grid, 256, qsm, st>>>(qa, nullptr, gq, h->s0, nullptr, n, h->d, h->dp, ip, h->fold,
                                                            comp);
    } else if (mode == 0)
      direct_dist_kernel<0><<<grid, 256, 0, st>>>(qa, qb, gq, h->s0, h->s1, n, h->d, h->dp, ip, 0, comp);
    else if (mode == 4)
      direct_dist_kernel<4><<<grid, 256, 0, st>>>(qa, nullptr, gq, h->s0, nullptr, n, h->d, h->dp, ip, 0, comp);
    else if (mode == 1)
      direct_dist_kernel<1><<<grid, 256, 0, st>>>(qa, nullptr, gq, h->s0, nullptr, n, h->d, h->dp, ip, 0, comp);
    else
      direct_dist_kernel<2><<<grid, 256, 0, st>>>(qa, nullptr, gq, h->s0, nullptr, n, h->d, h->dp, ip, h->fold, comp);
    CKL();
    if (ev && g0 == 0) CK(cudaEventRecord(ev[2], st));
    // two-level selection when the rows outnumber the slices' k-lists
    const uint64_t* sel_in = comp;
    int64_t sel_n = n;
    const int64_t nch = (n + DIRECT_CHUNK - 1) / DIRECT_CHUNK;
    if (nch > 1 && nch * k < n) {
      if ((rc = h->rkid.ensure((size_t)gq * nch * k * 8))) return rc;
      auto part = static_cast<uint64_t*>(h->rkid.p);
      direct_chunk_topk_kernel<<<dim3((unsigned)nch, (unsigned)gq), 256, 0, st>>>(comp, n, DIRECT_CHUNK, k, part);
      CKL();
      h->nlaunch++;
      sel_in = part;
      sel_n = nch * k;
    }
    if (ip)
      direct_select_kernel<true><<<gq, 256, (size_t)p2 * 8, st>>>(sel_in, sel_n, (int)g0, k, h->ids, dD, dI, dP);
    else
      direct_select_kernel<false><<<gq, 256, (size_t)p2 * 8, st>>>(sel_in, sel_n, (int)g0, k, h->ids, dD, dI, dP);
    CKL();
    h->nlaunch += 2;
  }
  return FK_OK;
}

__global__ void gather_range_kernel(const unsigned int* __restrict__ order, const unsigned long long* __restrict__ key_id,
                                    const float* __restrict__ dist, int64_t n, int64_t* __restrict__ ids_out,
                                    float* __restrict__ dist_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const unsigned int j = order[i];
    ids_out[i] = static_cast<int64_t>(key_id[j]);
    dist_out[i] = dist[j];
  }
}
__global__ void gather_u64_kernel(const unsigned int* __restrict__ idx, const unsigned long long* __restrict__ src,
                                  int64_t n, unsigned long long* __restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}
__global__ void iota_u32_kernel(unsigned int* out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (unsigned int)i;
}
__global__ void counts_to_i64_kernel(const unsigned int* __restrict__ c, int64_t nq, int64_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= nq) out[i] = i < nq ? (int64_t)c[i] : 0;
}

}  // namespace

extern "C" {

int fk_range_search(fk_index* h, const void* q, int64_t nq, int dtype, float radius, int64_t* lims, int64_t* total,
                    fk_range_result** out, int on_device, void* stream) {
  if (!h) return set_err(FK_E_INVALID, "NULL index");
  if (nq < 0) return set_err(FK_E_INVALID, "nq must be >= 0");
  if (dtype != FK_F32 && dtype != FK_F16 && dtype != FK_BF16) return set_err(FK_E_INVALID, "bad dtype %d", dtype);
  if (!lims || !total || !out) return set_err(FK_E_INVALID, "NULL output pointer");
  *out = nullptr;
  if (nq > (int64_t)INT32_MAX / 2) return set_err(FK_E_UNSUPPORTED, "nq too large for one call");
  if (nq > 0 && !q) return set_err(FK_E_INVALID, "NULL query pointer");
  std::lock_guard<std::mutex> g(h->mu);
  CK(cudaSetDevice(h->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool ip = h->metric == FK_METRIC_IP;
  int rc;
  if ((rc = scratch_begin(h, st))) return rc;
  // the entries go to a per-call result object (no state left in the handle
  // between the two calls: concurrent range searches cannot mix results)
  fk_range_result* res = new fk_range_result();
  res->device = h->device;
  struct Guard {
    fk_range_result*& r;
    ~Guard() { fk_range_free(r); }
  } guard{res};
  if ((rc = h->rlims.ensure((size_t)(nq + 1) * sizeof(int64_t)))) return rc;
  int64_t* dlims = static_cast<int64_t*>(h->rlims.p);
  if (nq == 0 || h->ntotal == 0) {  // flat.py:124-125: empty lists
    CK(cudaMemsetAsync(dlims, 0, (size_t)(nq + 1) * sizeof(int64_t), st));
  } else {
    if ((rc = stage_queries(h, q, nq, dtype, on_device, st))) return rc;
    Plan pl;
    if ((rc = make_plan(h, nq, h->ntotal, 1, -1, 0, &pl))) return rc;
    h->r_radius = radius;
    if ((rc = h->thr.ensure((size_t)nq * sizeof(uint32_t)))) return rc;
    if ((rc = h->rcount.ensure(sizeof(unsigned long long)))) return rc;
    unsigned long long want = std::max<unsigned long long>(h->r_cap, std::max<int64_t>(1 << 20, nq * 64));
    unsigned long long n = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
      if ((rc = h->rcand.ensure(want * sizeof(unsigned long long)))) return rc;
      h->r_cap = want;
      CK(cudaMemsetAsync(h->rcount.p, 0, sizeof(unsigned long long), st));
      if ((rc = run_fused(h, pl, nq, h->ntotal, 1, ip, st))) return rc;
      CK(cudaMemcpyAsync(&n, h->rcount.p, sizeof(n), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (n <= h->r_cap) break;
      want = n;  // every candidate was counted: one rerun with room for all of them
    }
    if (n > 0xFFFFFFFFull) return set_err(FK_E_UNSUPPORTED, "range search with %llu candidates", n);
    // exact direct distances + radius test + sort keys
    if ((rc = h->rdist.ensure(n * sizeof(float) + 16))) return rc;
    if ((rc = h->rkid.ensure(n * 8 + 16)) || (rc = h->rkrd.ensure(n * 8 + 16))) return rc;
    if ((rc = h->rkeep.ensure(n * 4 + 16)) || (rc = h->rrowc.ensure((size_t)nq * 4))) return rc;
    CK(cudaMemsetAsync(h->rrowc.p, 0, (size_t)nq * 4, st));
    auto rd = static_cast<float*>(h->rdist.p);
    auto kid = static_cast<unsigned long long*>(h->rkid.p);
    auto krd = static_cast<unsigned long long*>(h->rkrd.p);
    auto keep = static_cast<unsigned int*>(h->rkeep.p);
    auto rowc = static_cast<unsigned int*>(h->rrowc.p);
    const auto cand = static_cast<const unsigned long long*>(h->rcand.p);
    if (n > 0) {
      const unsigned grid = (unsigned)((n + 7) / 8);
      if (h->storage == FK_F32 && h->split == 2)
        range_exact_kernel<0><<<grid, 256, 0, st>>>(cand, n, h->q0.p, h->q1.p, h->s0, h->s1, h->d, h->dp, ip, 0, radius,
                                                    h->ids, rd, kid, krd, keep, rowc);
      else if (h->storage == FK_F32)
        range_exact_kernel<4><<<grid, 256, 0, st>>>(cand, n, h->q0.p, nullptr, h->s0, nullptr, h->d, h->dp, ip, 0,
                                                    radius, h->ids, rd, kid, krd, keep, rowc);
      else if (h->storage == FK_F16)
        range_exact_kernel<1><<<grid, 256, 0, st>>>(cand, n, h->q0.p, nullptr, h->s0, nullptr, h->d, h->dp, ip, 0,
                                                    radius, h->ids, rd, kid, krd, keep, rowc);
      else
        range_exact_kernel<2><<<grid, 256, 0, st>>>(cand, n, h->q0.p, nullptr, h->s0, nullptr, h->d, h->dp, ip,
                                                    h->fold, radius, h->ids, rd, kid, krd, keep, rowc);
      CKL();
    }
    // survivors -> (row, value, id) order: stable LSD radix passes (id, then row|value)
    if ((rc = h->rv1.ensure(n * 4 + 16)) || (rc = h->rv2.ensure(n * 4 + 16)) || (rc = h->rsel.ensure(n * 4 + 16)) ||
        (rc = h->rnsel.ensure(16)) || (rc = h->rkid2.ensure(n * 8 + 16)) || (rc = h->rkrd2.ensure(n * 8 + 16)))
      return rc;
    auto v1 = static_cast<unsigned int*>(h->rv1.p);
    auto v2 = static_cast<unsigned int*>(h->rv2.p);
    auto sel = static_cast<unsigned int*>(h->rsel.p);
    auto kid2 = static_cast<unsigned long long*>(h->rkid2.p);
    auto krd2 = static_cast<unsigned long long*>(h->rkrd2.p);
    int64_t nsel = 0;
    if (n > 0) {
      iota_u32_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(v1, (int64_t)n);
      size_t tb = 0;
      CK(cub::DeviceSelect::Flagged(nullptr, tb, v1, keep, sel, static_cast<int64_t*>(h->rnsel.p), (int64_t)n, st));
      if ((rc = h->rtmp.ensure(tb))) return rc;
      CK(cub::DeviceSelect::Flagged(h->rtmp.p, tb, v1, keep, sel, static_cast<int64_t*>(h->rnsel.p), (int64_t)n, st));
      CK(cudaMemcpyAsync(&nsel, h->rnsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
    if (nsel > 0) {
      const unsigned g = (unsigned)((nsel + 255) / 256);
      int row_bits = 1;
      while ((1ll << row_bits) < nq) ++row_bits;
      gather_u64_kernel<<<g, 256, 0, st>>>(sel, kid, nsel, kid2);  // ids of the survivors
      CKL();
      size_t tb1 = 0, tb2 = 0;
      CK(cub::DeviceRadixSort::SortPairs(nullptr, tb1, kid2, krd2, sel, v1, nsel, 0, 64, st));
      CK(cub::DeviceRadixSort::SortPairs(nullptr, tb2, kid2, krd2, v1, v2, nsel, 0, 32 + row_bits, st));
      if ((rc = h->rtmp.ensure(std::max(tb1, tb2)))) return rc;
      // pass 1: by user id (flat.py:137, the secondary key)
      CK(cub::DeviceRadixSort::SortPairs(h->rtmp.p, tb1, kid2, krd2, sel, v1, nsel, 0, 64, st));
      // pass 2 (stable): by (row, best-first value)
      gather_u64_kernel<<<g, 256, 0, st>>>(v1, krd, nsel, kid2);
      CKL();
      CK(cub::DeviceRadixSort::SortPairs(h->rtmp.p, tb2, kid2, krd2, v1, v2, nsel, 0, 32 + row_bits, st));
      res->stream = st;
      CK(cudaMallocAsync(&res->ids, (size_t)nsel * 8, st));
      CK(cudaMallocAsync(&res->dist, (size_t)nsel * 4, st));
      gather_range_kernel<<<g, 256, 0, st>>>(v2, kid, rd, nsel, static_cast<int64_t*>(res->ids),
                                             static_cast<float*>(res->dist));
      CKL();
    }
    res->total = nsel;
    // lims = exclusive scan of the per-row survivor counts (nq + 1 entries)
    if ((rc = h->rv1.ensure((size_t)(nq + 1) * 8))) return rc;
    auto cnt64 = static_cast<int64_t*>(h->rv1.p);
    counts_to_i64_kernel<<<(unsigned)((nq + 256) / 256), 256, 0, st>>>(rowc, nq, cnt64);
    CKL();
    size_t tbs = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tbs, cnt64, dlims, nq + 1, st));
    if ((rc = h->rtmp.ensure(tbs))) return rc;
    CK(cub::DeviceScan::ExclusiveSum(h->rtmp.p, tbs, cnt64, dlims, nq + 1, st));
  }
  CK(cudaMemcpyAsync(lims, dlims, (size_t)(nq + 1) * sizeof(int64_t),
                     on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
  if ((rc = scratch_end(h, st))) return rc;
  CK(cudaStreamSynchronize(st));
  *total = res->total;
  *out = res;
  res = nullptr;  // ownership passes to the caller
  return FK_OK;
}

int fk_range_fetch(fk_range_result* r, int64_t* ids, float* dist, int64_t capacity, int on_device, void* stream) {
  if (!r) return set_err(FK_E_INVALID, "NULL range result");
  if (r->total == 0) return FK_OK;
  if (!ids || !dist) return set_err(FK_E_INVALID, "NULL output pointer");
  if (capacity < r->total)
    return set_err(FK_E_INVALID, "output capacity %lld < %lld range entries", (long long)capacity,
                   (long long)r->total);
  CK(cudaSetDevice(r->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  CK(cudaMemcpyAsync(ids, r->ids, (size_t)r->total * sizeof(int64_t), kind, st));
  CK(cudaMemcpyAsync(dist, r->dist, (size_t)r->total * sizeof(float), kind, st));
  CK(cudaStreamSynchronize(st));
  return FK_OK;
}

int64_t fk_range_total(const fk_range_result* r) { return r ? r->total : -1; }

void fk_range_free(fk_range_result* r) {
  if (!r) return;
  cudaSetDevice(r->device);
  // ordered after every use on the search's stream (fk_range_fetch copies on
  // its own stream and synchronizes before returning)
  if (r->ids) cudaFreeAsync(r->ids, r->stream);
  if (r->dist) cudaFreeAsync(r->dist, r->stream);
  delete r;
}

int fk_set_option(fk_index* h, int option, int64_t value) {
  if (!h) return set_err(FK_E_INVALID, "NULL index");
  std::lock_guard<std::mutex> g(h->mu);
  switch (option) {
    case FK_OPT_PLAN_ROWS:
      if (value < 0) return set_err(FK_E_INVALID, "plan rows must be >= 0");
      h->plan_rows = value;
      return FK_OK;
    case FK_OPT_BLAS_THRESHOLD:
      if (value < 0) return set_err(FK_E_INVALID, "blas threshold must be >= 0");
      h->blas_threshold = value;
      return FK_OK;
  }
  return set_err(FK_E_INVALID, "unknown option %d", option);
}

int fk_search(fk_index* h, const void* q, int64_t nq, int dtype, int k, float* D, int64_t* I, int64_t* P,
              int on_device, void* stream) {
  if (!h) return set_err(FK_E_INVALID, "NULL index");
  if (k < 1) return set_err(FK_E_INVALID, "k must be >= 1");
  if (nq < 0) return set_err(FK_E_INVALID, "nq must be >= 0");
  if (dtype != FK_F32 && dtype != FK_F16 && dtype != FK_BF16) return set_err(FK_E_INVALID, "bad dtype %d", dtype);
  if (nq == 0) return FK_OK;
  if (!q || !D || !I) return set_err(FK_E_INVALID, "NULL query/output pointer");
  if (nq > (int64_t)INT32_MAX / 2) return set_err(FK_E_UNSUPPORTED, "nq too large for one call");
  if (k > FK_MAX_K) return set_err(FK_E_UNSUPPORTED, "k=%d exceeds the maximum supported k (%d)", k, FK_MAX_K);
  std::lock_guard<std::mutex> g(h->mu);
  CK(cudaSetDevice(h->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool ip = h->metric == FK_METRIC_IP;
  const size_t nout = (size_t)nq * k;
  int rc;
  if ((rc = scratch_begin(h, st))) return rc;
  h->nlaunch = 0;
  cudaEvent_t* ev = nullptr;
  if (h->profiling && h->ntotal > 0 && !(ev = next_events(h))) return set_err(FK_E_CUDA, "cudaEventCreate failed");

  float* dD = D;
  int64_t* dI = I;
  int64_t* dP = P;
  if (!on_device) {
    if ((rc = h->outD.ensure(nout * sizeof(float)))) return rc;
    if ((rc = h->outI.ensure(nout * sizeof(int64_t)))) return rc;
    dD = static_cast<float*>(h->outD.p);
    dI = static_cast<int64_t*>(h->outI.p);
    if (P) {
      if ((rc = h->outP.ensure(nout * sizeof(int64_t)))) return rc;
      dP = static_cast<int64_t*>(h->outP.p);
    }
  }

  if (h->ntotal == 0) {  // flat.py:70-71: all-sentinel rows
    fill_sentinel_kernel<<<(unsigned)((nout + 255) / 256), 256, 0, st>>>(dD, dI, dP, nout,
                                                                         ip ? -INFINITY : INFINITY);
    CKL();
    h->nlaunch = 1;
  } else if (nq < h->blas_threshold) {  // flat.py:58-62: small batches take the direct path
    if (ev) CK(cudaEventRecord(ev[0], st));
    if ((rc = stage_queries(h, q, nq, dtype, on_device, st))) return rc;
    h->nlaunch++;
    if ((rc = search_direct(h, nq, k, ip, dD, dI, dP, ev, st))) return rc;
    if (ev) CK(cudaEventRecord(ev[3], st));
    std::memset(h->plan, 0, sizeof(h->plan));
    h->plan[11] = -1;  // direct path
  } else if (h->storage == FK_F32 &&
             (h->split == 1 ||
              (fp32_1pass_ok(k, h->plan_rows > 0 ? h->plan_rows : h->ntotal, h->ntotal) &&
               !getenv("FK_FP32_3X")))) {
    // filter pass: scaled fp16 (MODE 5, default with the hi/lo storage) or
    // tf32 (MODE 4; FK_FP32_FILTER=tf32, or raw fp32 storage)
    const char* ff = getenv("FK_FP32_FILTER");
    const int fmode = (h->split == 2 && !(ff && std::strcmp(ff, "tf32") == 0)) ? 5 : 4;
    if (ev) CK(cudaEventRecord(ev[0], st));
    if ((rc = stage_queries(h, q, nq, dtype, on_device, st, fmode == 5))) return rc;
    h->nlaunch++;
    Plan pl;
    if ((rc = search_mode4(h, nq, k, ip, dD, dI, dP, ev, st, &pl, fmode))) return rc;
    if (ev) CK(cudaEventRecord(ev[3], st));
    h->plan[0] = pl.grid;
    h->plan[1] = pl.S;
    h->plan[2] = pl.chunk_tiles;
    h->plan[3] = pl.num_units;
    h->plan[4] = pl.stages;
    h->plan[5] = pl.a_mode;
    h->plan[6] = pl.smem;
    h->plan[7] = pl.kq * 100 + pl.epi;
    h->plan[8] = pl.acc_stages;
    h->plan[9] = pl.epi;
    h->plan[10] = pl.bn;
    h->plan[11] = pl.kmode;
  } else {
    const int kq = k <= 8 ? 8 : k <= 16 ? 16 : k <= 32 ? 32 : 0;  // 0: large-k buffers

    // ---- queries -> device operand layout + norms
    if (ev) CK(cudaEventRecord(ev[0], st));
    if ((rc = stage_queries(h, q, nq, dtype, on_device, st))) return rc;
    h->nlaunch++;

    Plan pl;
    if ((rc = make_plan(h, nq, h->ntotal, k, kq, 0, &pl))) return rc;
    // Large k: estimate each query's bound from a prefix sample -- the exact
    // 32nd best of m = ntotal*8/k rows sits near the 4k-th overall (it falls
    // below the true k-th only if >= 32 of the m rows beat it: Poisson(8) >= 32,
    // p ~ 1e-9 for i.i.d. order).  The merge certifies every query (>= k
    // survivors under the bound => exact); any failure reruns without it.
    int64_t m_est = 0;
    if (kq == 0 && !getenv("FK_NO_EST")) {
      m_est = ((h->ntotal * 8) / k + BN - 1) / BN * BN;
      // at least 32 tiles, while that sample still estimates a rank >= 2k
      // (256 <= rows/k < 512; 300k rows, k = 1000, 100 queries: 6.2 -> 0.74 ms)
      if (m_est < 32 * BN && (int64_t)32 * BN * k <= h->ntotal * 16) m_est = 32 * BN;
      // small k (33..~63): 8 rows/k would exceed an eighth of the rows; an
      // eighth (at most 256 tiles) still estimates a rank >= 256 >= 2k
      if (m_est * 8 > h->ntotal && k <= 128 && !getenv("FK_EST_SMALLK0"))
        m_est = std::min<int64_t>(h->ntotal / 8, 256 * BN) / BN * BN;
      if (m_est < 32 * BN || m_est * 8 > h->ntotal) m_est = 0;
    }
    if ((rc = h->thr.ensure((size_t)nq * sizeof(uint32_t)))) return rc;
    if ((rc = h->fail.ensure(sizeof(int)))) return rc;
    // k <= 32: per-query running union of the finished units' top-k (exact
    // values here, so its k-th is a valid shared bound)
    // (only when later waves of units can profit: >= 4 units per CTA)
    h->r_union = kq > 0 && pl.num_units >= 4 * pl.grid && !getenv("FK_NO_UNION");
    if (h->r_union) {
      if ((rc = h->glock.ensure((size_t)nq * sizeof(unsigned int))) || (rc = h->gkeys.ensure((size_t)nq * 32 * 4)))
        return rc;
      CK(cudaMemsetAsync(h->glock.p, 0, (size_t)nq * sizeof(unsigned int), st));
      CK(cudaMemsetAsync(h->gkeys.p, 0xFF, (size_t)nq * 32 * 4, st));
    }
    for (int attempt = 0; attempt < 2; ++attempt) {
      const bool est = attempt == 0 && m_est > 0;
      CK(cudaMemsetAsync(h->thr.p, 0xFF, (size_t)nq * sizeof(uint32_t), st));
      if (ev) CK(cudaEventRecord(ev[1], st));
      if (est) {
        // Few query tiles: split the sample over the SMs and keep the
        // per-query running union of the units' 32-lists -- its 32nd is the
        // bound one list over the whole sample gives (d = 768 fp32, 129
        // queries, k = 33: 3.31 -> 0.85 ms; one CTA per query tile before)
        Plan pe;
        // (at most 8 units per query tile: every unit merges into the union
        // under a per-query lock at its end)
        const bool split = pl.num_m < h->num_sms / 2 && !getenv("FK_EST_S1");
        const int s_est = split ? std::max(1, std::min(8, h->num_sms / std::max(1, pl.num_m))) : 1;
        if ((rc = make_plan(h, nq, m_est, 32, 32, s_est, &pe))) return rc;
        const bool su = h->r_union;
        if (split && pe.S > 1) {
          if ((rc = h->glock.ensure((size_t)nq * sizeof(unsigned int))) || (rc = h->gkeys.ensure((size_t)nq * 32 * 4)))
            return rc;
          CK(cudaMemsetAsync(h->glock.p, 0, (size_t)nq * sizeof(unsigned int), st));
          CK(cudaMemsetAsync(h->gkeys.p, 0xFF, (size_t)nq * 32 * 4, st));
          h->r_union = true;
        }
        rc = run_fused(h, pe, nq, m_est, 32, ip, st);
        h->r_union = su;
        if (rc) return rc;
        CK(cudaMemsetAsync(h->fail.p, 0, sizeof(int), st));
      }
      if (kq > 0 && (rc = run_prepass(h, nq, k, kq, ip, pl.kmode, st))) return rc;
      if ((rc = run_fused(h, pl, nq, h->ntotal, k, ip, st))) return rc;
      if (ev) CK(cudaEventRecord(ev[2], st));
      if ((rc = launch_merge(h, pl, nq, k, ip, dD, dI, dP, est ? static_cast<int*>(h->fail.p) : nullptr, st)))
        return rc;
      if (!est) break;
      int nfail = 0;
      CK(cudaMemcpyAsync(&nfail, h->fail.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      h->est_fallbacks += nfail > 0;
      if (nfail == 0) break;  // every query certified: exact
    }
    h->r_union = false;
    if (ev) CK(cudaEventRecord(ev[3], st));
    h->plan[0] = pl.grid;
    h->plan[1] = pl.S;
    h->plan[2] = pl.chunk_tiles;
    h->plan[3] = pl.num_units;
    h->plan[4] = pl.stages;
    h->plan[5] = pl.a_mode;
    h->plan[6] = pl.smem;
    h->plan[7] = kq * 100 + pl.epi;
    h->plan[8] = pl.acc_stages;
    h->plan[9] = pl.epi;
    h->plan[10] = pl.bn;
    h->plan[11] = pl.kmode;
  }

  if (!on_device) {
    CK(cudaMemcpyAsync(D, dD, nout * sizeof(float), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(I, dI, nout * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    if (P) CK(cudaMemcpyAsync(P, dP, nout * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  }
  if ((rc = scratch_end(h, st))) return rc;
  if (!on_device) CK(cudaStreamSynchronize(st));
  h->nlaunch_acc += h->nlaunch;
  return FK_OK;
}

int fk_merge_shards(int metric, int nshard, int64_t nq, int k, const float* D_in, const int64_t* P_in,
                    const int64_t* I_in, float* D_out, int64_t* I_out, void* stream) {
  if (nshard < 1 || nshard > 64) return set_err(FK_E_INVALID, "nshard must be in [1, 64]");
  if (k < 1 || nq < 0) return set_err(FK_E_INVALID, "bad k / nq");
  if (nq == 0) return FK_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int wpb = 8;
  const unsigned grid = (unsigned)((nq + wpb - 1) / wpb);
  if (metric == FK_METRIC_IP)
    shard_merge_kernel<true><<<grid, wpb * 32, 0, st>>>(nshard, (int)nq, k, D_in, P_in, I_in, D_out, I_out);
  else
    shard_merge_kernel<false><<<grid, wpb * 32, 0, st>>>(nshard, (int)nq, k, D_in, P_in, I_in, D_out, I_out);
  CKL();
  return FK_OK;
}

int fk_reconstruct(fk_index* h, const int64_t* positions, int64_t n, float* out, int on_device, void* stream) {
  if (!h) return set_err(FK_E_INVALID, "NULL index");
  if (n <= 0) return FK_OK;
  std::lock_guard<std::mutex> g(h->mu);
  CK(cudaSetDevice(h->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc;
  const int64_t* dpos = positions;
  float* dout = out;
  if (!on_device) {
    std::vector<int64_t> chk(positions, positions + n);
    for (int64_t p : chk)
      if (p < 0 || p >= h->ntotal) return set_err(FK_E_INVALID, "position %lld out of range", (long long)p);
    if ((rc = h->stage_ids.ensure(n * sizeof(int64_t)))) return rc;
    if ((rc = h->stage_in.ensure(n * (size_t)h->d * sizeof(float)))) return rc;
    CK(cudaMemcpyAsync(h->stage_ids.p, positions, n * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    dpos = static_cast<const int64_t*>(h->stage_ids.p);
    dout = static_cast<float*>(h->stage_in.p);
  }
  const unsigned grid = (unsigned)((n + 7) / 8);
  if (h->storage == FK_F32 && h->split == 2)
    reconstruct_kernel<0><<<grid, 256, 0, st>>>(h->s0, h->s1, h->dp, h->d, dpos, n, dout, 1.f);
  else if (h->storage == FK_F32)
    reconstruct_kernel<4><<<grid, 256, 0, st>>>(h->s0, h->s1, h->dp, h->d, dpos, n, dout, 1.f);
  else if (h->storage == FK_F16)
    reconstruct_kernel<1><<<grid, 256, 0, st>>>(h->s0, h->s1, h->dp, h->d, dpos, n, dout, 1.f);
  else
    reconstruct_kernel<2><<<grid, 256, 0, st>>>(h->s0, h->s1, h->dp, h->d, dpos, n, dout, h->fold ? -0.5f : 1.f);
  CKL();
  if (!on_device) {
    CK(cudaMemcpyAsync(out, dout, n * (size_t)h->d * sizeof(float), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  return FK_OK;
}

int fk_get_ids(fk_index* h, int64_t* out_host) {
  if (!h) return set_err(FK_E_INVALID, "NULL index");
  std::lock_guard<std::mutex> g(h->mu);
  CK(cudaSetDevice(h->device));
  if (h->ntotal) CK(cudaMemcpy(out_host, h->ids, h->ntotal * sizeof(int64_t), cudaMemcpyDeviceToHost));
  return FK_OK;
}

int fk_remove_ids(fk_index* h, const int64_t* ids, int64_t n, int on_device, int64_t* removed, void* stream) {
  if (!h) return set_err(FK_E_INVALID, "NULL index");
  if (removed) *removed = 0;
  if (n <= 0 || h->ntotal == 0) return FK_OK;
  std::lock_guard<std::mutex> g(h->mu);
  CK(cudaSetDevice(h->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = scratch_begin(h, st);
  if (rc) return rc;
  const int64_t nt = h->ntotal;
  // kill list -> device, sorted (np.isin, flat.py:47)
  if ((rc = h->rm_kill.ensure((size_t)n * 16))) return rc;
  int64_t* kill = static_cast<int64_t*>(h->rm_kill.p);
  int64_t* kill_sorted = kill + n;
  CK(cudaMemcpyAsync(kill, ids, n * sizeof(int64_t), on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                     st));
  size_t tb_sort = 0, tb_sel = 0;
  CK(cub::DeviceRadixSort::SortKeys(nullptr, tb_sort, kill, kill_sorted, n, 0, 64, st));
  CK(cub::DeviceSelect::Flagged(nullptr, tb_sel, cub::CountingInputIterator<int64_t>(0), (const uint8_t*)nullptr,
                                (int64_t*)nullptr, (int64_t*)nullptr, nt, st));
  if ((rc = h->idt_tmp.ensure(std::max(tb_sort, tb_sel)))) return rc;
  CK(cub::DeviceRadixSort::SortKeys(h->idt_tmp.p, tb_sort, kill, kill_sorted, n, 0, 64, st));
  // keep mask over storage, then the ordered keep list (flat.py:49-53)
  if ((rc = h->rm_flags.ensure((size_t)nt + 16))) return rc;
  if ((rc = h->rm_keep.ensure((size_t)(nt + 1) * sizeof(int64_t)))) return rc;
  auto flags = static_cast<uint8_t*>(h->rm_flags.p);
  auto keep = static_cast<int64_t*>(h->rm_keep.p);
  int64_t* nsel = keep + nt;
  keep_flags_kernel<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(h->ids, nt, kill_sorted, n, flags);
  CKL();
  CK(cub::DeviceSelect::Flagged(h->idt_tmp.p, tb_sel, cub::CountingInputIterator<int64_t>(0), flags, keep, nsel, nt,
                                st));
  int64_t nk = 0;
  CK(cudaMemcpyAsync(&nk, nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const int64_t nrem = nt - nk;
  if (removed) *removed = nrem;
  if (nrem > 0 && nk > 0) {
    // compact every column in place, order preserved: keep[i] >= i, so a
    // slice [c0, c0 + m) gathered through scratch only reads rows >= c0
    // that later slices have not overwritten yet
    const size_t rb = row_bytes(h);
    struct Col {
      void* p;
      size_t rb;
    } cols[4] = {{h->s0, rb}, {h->s1, rb}, {h->norms, sizeof(float)}, {h->ids, sizeof(int64_t)}};
    const int64_t slice = std::max<int64_t>(1, (int64_t)((256ull << 20) / rb));
    if ((rc = h->stage_in.ensure((size_t)std::min(slice, nk) * rb))) return rc;
    for (auto& c : cols) {
      if (!c.p) continue;
      const int64_t cs = std::max<int64_t>(1, (int64_t)((256ull << 20) / c.rb));
      for (int64_t c0 = 0; c0 < nk; c0 += cs) {
        const int64_t m = std::min(cs, nk - c0);
        gather_rows_kernel<<<(unsigned)m, 128, 0, st>>>(static_cast<const uint8_t*>(c.p),
                                                         static_cast<uint8_t*>(h->stage_in.p), c.rb, keep + c0, m);
        CKL();
        CK(cudaMemcpyAsync(static_cast<uint8_t*>(c.p) + (size_t)c0 * c.rb, h->stage_in.p, m * c.rb,
                           cudaMemcpyDeviceToDevice, st));
      }
    }
  }
  if (nrem > 0) {
    // the filter bound needs max stored norm: recompute over the survivors
    CK(cudaMemsetAsync(h->xn_max, 0, sizeof(float), st));
    if (nk > 0) {
      norm_max_kernel<<<(unsigned)std::min<int64_t>((nk + 255) / 256, 1024), 256, 0, st>>>(
          h->norms, nk, reinterpret_cast<unsigned int*>(h->xn_max));
      CKL();
    }
    h->ntotal = nk;
    h->idt_n = -1;
    h->f16_rows = 0;  // the fp16 filter copy (and its scale) is rebuilt from the survivors
    if (h->f16st.p) CK(cudaMemsetAsync(h->f16st.p, 0, sizeof(F16State), st));
  }
  if ((rc = scratch_end(h, st))) return rc;
  CK(cudaStreamSynchronize(st));
  return FK_OK;
}

}  // extern "C"

namespace {

// Build (lazily) the stably sorted (id, position) table.
int ensure_id_table(fk_index* h, cudaStream_t st) {
  const int64_t n = h->ntotal;
  if (h->idt_n == n) return FK_OK;
  int rc;
  if ((rc = h->idt_keys.ensure((size_t)n * 8))) return rc;
  if ((rc = h->idt_pos.ensure((size_t)n * 16))) return rc;
  auto keys = static_cast<int64_t*>(h->idt_keys.p);
  auto pos = static_cast<int64_t*>(h->idt_pos.p);
  int64_t* iota = pos + n;
  iota_ids_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(iota, 0, n);
  CKL();
  size_t tb = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, h->ids, keys, iota, pos, n, 0, 64, st));
  if ((rc = h->idt_tmp.ensure(tb))) return rc;
  CK(cub::DeviceRadixSort::SortPairs(h->idt_tmp.p, tb, h->ids, keys, iota, pos, n, 0, 64, st));
  h->idt_n = n;
  return FK_OK;
}

// ids [m] (device) -> positions [m] (device); FK_E_NOTFOUND naming the first
// unknown id.  Caller holds the lock and has ordered the stream.
int lookup_positions(fk_index* h, const int64_t* ids, int64_t m, int skip_negative, int64_t* pos, cudaStream_t st) {
  int rc;
  if ((rc = ensure_id_table(h, st))) return rc;
  if ((rc = h->idt_miss.ensure(sizeof(unsigned long long)))) return rc;
  auto miss = static_cast<unsigned long long*>(h->idt_miss.p);
  CK(cudaMemsetAsync(miss, 0xFF, sizeof(unsigned long long), st));
  lookup_positions_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(
      static_cast<const int64_t*>(h->idt_keys.p), static_cast<const int64_t*>(h->idt_pos.p), h->ntotal, ids, m,
      skip_negative, pos, miss);
  CKL();
  unsigned long long first = 0;
  CK(cudaMemcpyAsync(&first, miss, sizeof first, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (first != ~0ull) {
    int64_t bad = 0;
    CK(cudaMemcpy(&bad, ids + first, sizeof bad, cudaMemcpyDeviceToHost));
    return set_err(FK_E_NOTFOUND, "unknown id %lld", (long long)bad);
  }
  return FK_OK;
}

}  // namespace

extern "C" {

int fk_positions(fk_index* h, const int64_t* ids, int64_t n, int64_t* pos, int on_device, void* stream) {
  if (!h) return set_err(FK_E_INVALID, "NULL index");
  if (n <= 0) return FK_OK;
  if (!ids || !pos) return set_err(FK_E_INVALID, "NULL argument");
  std::lock_guard<std::mutex> g(h->mu);
  CK(cudaSetDevice(h->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = scratch_begin(h, st);
  if (rc) return rc;
  const int64_t* dids = ids;
  int64_t* dpos = pos;
  if (!on_device) {
    if ((rc = h->stage_ids.ensure((size_t)n * 16))) return rc;
    auto sp = static_cast<int64_t*>(h->stage_ids.p);
    CK(cudaMemcpyAsync(sp, ids, n * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    dids = sp;
    dpos = sp + n;
  }
  rc = lookup_positions(h, dids, n, 0, dpos, st);
  if (rc == FK_OK && !on_device) {
    CK(cudaMemcpyAsync(pos, dpos, n * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  const int rc2 = scratch_end(h, st);
  return rc ? rc : rc2;
}

int fk_refine(fk_index* h, int metric, const float* q, int64_t nq, const int64_t* cand, int L, int k, float* D,
              int64_t* I, int on_device, void* stream) {
  if (!h) return set_err(FK_E_INVALID, "NULL index");
  if (k < 1) return set_err(FK_E_INVALID, "k must be >= 1");
  if (L < k) return set_err(FK_E_INVALID, "shortlist must be >= k");
  if (metric != FK_METRIC_L2 && metric != FK_METRIC_IP) return set_err(FK_E_UNSUPPORTED, "metric %d", metric);
  if (nq <= 0) return FK_OK;
  if (!q || !cand || !D || !I) return set_err(FK_E_INVALID, "NULL argument");
  const size_t smem = (size_t)L * 16;
  if (smem > (size_t)SMEM_LIMIT) return set_err(FK_E_UNSUPPORTED, "shortlist %d above %d", L, SMEM_LIMIT / 16);
  std::lock_guard<std::mutex> g(h->mu);
  CK(cudaSetDevice(h->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = scratch_begin(h, st);
  if (rc) return rc;
  const size_t nc = (size_t)nq * L;
  const float* dq = q;
  const int64_t* dc = cand;
  float* dD = D;
  int64_t* dI = I;
  if (!on_device) {
    if ((rc = h->stage_in.ensure((size_t)nq * h->d * 4 + (size_t)nq * k * 4))) return rc;
    if ((rc = h->rkeep.ensure(nc * 8 + (size_t)nq * k * 8))) return rc;
    auto sq = static_cast<float*>(h->stage_in.p);
    auto sc = static_cast<int64_t*>(h->rkeep.p);
    CK(cudaMemcpyAsync(sq, q, (size_t)nq * h->d * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(sc, cand, nc * 8, cudaMemcpyHostToDevice, st));
    dq = sq;
    dc = sc;
    dD = sq + (size_t)nq * h->d;
    dI = sc + nc;
  }
  if ((rc = h->stage_ids.ensure(nc * 8))) return rc;
  auto cpos = static_cast<int64_t*>(h->stage_ids.p);
  if ((rc = lookup_positions(h, dc, (int64_t)nc, 1, cpos, st))) {
    scratch_end(h, st);
    return rc;
  }
  static std::atomic<uint64_t> cfg[5];
  const int mode = h->storage == FK_F32 ? (h->split == 2 ? 0 : 4) : (h->storage == FK_F16 ? 1 : 2);
  const double scale = h->fold ? -0.5 : 1.0;
  const int ip = metric == FK_METRIC_IP;
#define FK_REFINE(M)                                                                                       \
  do {                                                                                                     \
    if ((rc = fkh::once_per_device(cfg[M], [] {                                                            \
           CK(cudaFuncSetAttribute(refine_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT)); \
           return FK_OK;                                                                                   \
         })))                                                                                              \
      return rc;                                                                                           \
    refine_kernel<M><<<(unsigned)nq, 256, smem, st>>>(dq, h->d, dc, cpos, L, k, h->s0, h->s1, h->dp, scale, ip, \
                                                      dD, dI);                                             \
  } while (0)
  if (mode == 0) FK_REFINE(0);
  else if (mode == 4) FK_REFINE(4);
  else if (mode == 1) FK_REFINE(1);
  else FK_REFINE(2);
#undef FK_REFINE
  CKL();
  if (!on_device) {
    CK(cudaMemcpyAsync(D, dD, (size_t)nq * k * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(I, dI, (size_t)nq * k * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  return scratch_end(h, st);
}

int fk_set_profiling(fk_index* h, int on) {
  if (!h) return set_err(FK_E_INVALID, "NULL index");
  std::lock_guard<std::mutex> g(h->mu);
  if (on > 0) {
    // create the event pool up front (on = searches to reserve): event
    // creation inside a timed loop costs driver calls that can stall it
    CK(cudaSetDevice(h->device));
    const size_t want = h->ev_used + (size_t)std::max(on, 64);
    while (h->ev_pool.size() < want) {
      std::array<cudaEvent_t, 4> q{};
      for (auto& e : q) CK(cudaEventCreate(&e));
      h->ev_pool.push_back(q);
    }
  }
  h->profiling = on > 0;
  return FK_OK;
}

// Device-side gate for timed loops: one thread spins until *flag (pinned
// host memory, read through UVA) becomes nonzero or timeout_s passes.
__global__ void gate_kernel(const volatile int* flag, unsigned long long timeout_ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (*flag == 0) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) break;
    __nanosleep(1000);
  }
}

int fk_gate(const int* host_flag, double timeout_s, void* stream) {
  if (!host_flag) return set_err(FK_E_INVALID, "NULL flag");
  gate_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(host_flag, (unsigned long long)(timeout_s * 1e9));
  CKL();
  return FK_OK;
}

int fk_kernel_times(fk_index* h, float* ms3, int* nlaunch) {
  if (!h) return set_err(FK_E_INVALID, "NULL index");
  std::lock_guard<std::mutex> g(h->mu);
  CK(cudaSetDevice(h->device));
  double acc[3] = {0, 0, 0};
  for (size_t i = 0; i < h->ev_used; ++i) {
    auto& q = h->ev_pool[i];
    CK(cudaEventSynchronize(q[3]));
    for (int j = 0; j < 3; ++j) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, q[j], q[j + 1]));
      acc[j] += ms;
    }
  }
  if (ms3)
    for (int j = 0; j < 3; ++j) ms3[j] = h->ev_used ? (float)(acc[j] / h->ev_used) : 0.f;
  if (nlaunch) *nlaunch = (int)h->nlaunch_acc;
  h->ev_used = 0;
  h->nlaunch_acc = 0;
  return FK_OK;
}

int fk_kmeans_rescore(const float* x, int64_t n, int d, const double* c, const double* cnorm, int64_t nc,
                      const int64_t* cand, int kc, int by_ip, const float* approx, double margin, double cmax,
                      int64_t* assign, double* err, int* uncertain, void* stream) {
  if (n < 0 || d < 1 || nc < 1 || kc < 1) return set_err(FK_E_INVALID, "bad sizes");
  if (!x || !c || !cnorm || !assign || !err) return set_err(FK_E_INVALID, "NULL argument");
  if (n == 0) return FK_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int wpb = 8;
  kmeans_rescore_kernel<<<(unsigned)((n + wpb - 1) / wpb), wpb * 32, 0, st>>>(
      x, n, d, c, cnorm, nc, cand, kc, by_ip, approx, margin, cmax, assign, err, uncertain);
  CKL();
  return FK_OK;
}

int fk_last_plan(fk_index* h, int* out) {
  if (!h || !out) return set_err(FK_E_INVALID, "NULL argument");
  std::memcpy(out, h->plan, sizeof(h->plan));
  return FK_OK;
}

// Test hook (not in the public header): route raw inner products of the next
// searches to a caller-owned device buffer [nq][ntotal] (NULL disables).
int fk_debug_set_trace(fk_index* h, unsigned long long* dev_buf) {
  if (!h) return set_err(FK_E_INVALID, "NULL index");
  h->trace = dev_buf;
  return FK_OK;
}

int fk_debug_set_ip_dump(fk_index* h, float* dev_buf) {
  if (!h) return set_err(FK_E_INVALID, "NULL index");
  h->dbg_ip = dev_buf;
  return FK_OK;
}

}  // extern "C"
