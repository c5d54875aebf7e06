// Host-side helpers shared by the translation units of libflatknn.so:
// thread-local error reporting, CUDA check macros, per-device one-time
// kernel attribute setup, and the fused-kernel launch entry points (one
// translation unit per operand MODE, compiled in parallel).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "../../include/flatknn.h"
#include "fused_kernel.cuh"

namespace fkh {

// Sets the thread-local message returned by fk_last_error and returns code.
int set_err(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));

#define CK(expr)                                                                                         \
  do {                                                                                                   \
    cudaError_t e_ = (expr);                                                                             \
    if (e_ != cudaSuccess)                                                                               \
      return ::fkh::set_err(e_ == cudaErrorMemoryAllocation ? FK_E_NOMEM : FK_E_CUDA,                    \
                            "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

#define CKL()                                                                                            \
  do {                                                                                                   \
    cudaError_t e_ = cudaGetLastError();                                                                 \
    if (e_ != cudaSuccess)                                                                               \
      return ::fkh::set_err(FK_E_CUDA, "kernel launch failed: %s (%s:%d)", cudaGetErrorString(e_),       \
                            __FILE__, __LINE__);                                                         \
  } while (0)

constexpr int SMEM_LIMIT = 232448 - 1024;  // sm_100 227 KB per block, minus the static barrier block

// Function attributes (max dynamic smem) are per device context: run
// `configure` once per (call site, device).  Thread-safe; a failed attempt
// is retried by the next caller.
template <class F>
int once_per_device(std::atomic<uint64_t>& done, F configure) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return FK_OK;
  const int rc = configure();
  if (rc == FK_OK) done.fetch_or(bit, std::memory_order_acq_rel);
  return rc;
}

// fused_knn_kernel<MODE, KQ, IP, EPI, TBN> launch for one operand MODE
// (defined in fused_m<MODE>.cu); epi 4/8, kq 8/16/32 (queue), 0 (large k),
// -1 (range), sp.bn 64/128, sp.cluster 1/2.
template <int MODE>
int launch_fused_mode(int epi, bool ip, int kq, const CUtensorMap& a0, const CUtensorMap& a1,
                      const CUtensorMap& b0, const CUtensorMap& b1, const fk::SearchParams& sp, int grid, int smem,
                      cudaStream_t st);

}  // namespace fkh
