// Device-side storage operations of the flat index: the id -> position
// table (flat.py:34-41), remove_ids compaction (flat.py:46-56) and the
// refine_search re-ranking (core.py:368-394).  Everything stays on the GPU:
// no id list is copied to the host.
#pragma once
#include <cuda_fp16.h>
#include <cuda_bf16.h>

#include <cstdint>

#include "fused_kernel.cuh"

namespace fk {

// First index j in sorted a[0..n) with a[j] > v.
__device__ __forceinline__ int64_t upper_bound_i64(const int64_t* __restrict__ a, int64_t n, int64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (a[m] <= v) lo = m + 1;
    else hi = m;
  }
  return lo;
}

// id -> storage position through the stably sorted (id, position) table.
// The reference's `_pos_of_id = {int(v): i for i, v in enumerate(ids)}`
// (flat.py:36-37) keeps the LAST position of a duplicated id, hence
// upper_bound - 1.  skip_negative: ids < 0 (search padding) map to -1
// without counting as missing; otherwise the smallest index of an unknown id
// goes to *first_missing (KeyError, flat.py:40-41).
__global__ void lookup_positions_kernel(const int64_t* __restrict__ sorted_ids, const int64_t* __restrict__ sorted_pos,
                                        int64_t n, const int64_t* __restrict__ ids, int64_t m, int skip_negative,
                                        int64_t* __restrict__ pos, unsigned long long* __restrict__ first_missing) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int64_t v = ids[i];
  if (skip_negative && v < 0) {
    pos[i] = -1;
    return;
  }
  const int64_t j = upper_bound_i64(sorted_ids, n, v);
  if (j > 0 && sorted_ids[j - 1] == v) {
    pos[i] = sorted_pos[j - 1];
  } else {
    pos[i] = -1;
    atomicMin(first_missing, static_cast<unsigned long long>(i));
  }
}

// remove_ids mask (flat.py:47 `np.isin(self.ids, ids)`): keep[i] = ids[i]
// not in the sorted kill list.
__global__ void keep_flags_kernel(const int64_t* __restrict__ ids, int64_t n, const int64_t* __restrict__ kill_sorted,
                                  int64_t m, uint8_t* __restrict__ keep) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t v = ids[i];
  const int64_t j = upper_bound_i64(kill_sorted, m, v);
  keep[i] = (j > 0 && kill_sorted[j - 1] == v) ? 0 : 1;
}

// Value of a stored element as the reference's float32 vector
// (`reconstruct_batch`): fp32 split hi + lo (exact), raw fp32, fp16, bf16
// (fold mode stores -2x: scale -0.5, exact).
template <int MODE>
__device__ __forceinline__ double refine_stored(const void* a, const void* b, size_t off, double scale) {
  if (MODE == 0) return (double)(static_cast<const float*>(a)[off] + static_cast<const float*>(b)[off]);
  if (MODE == 4) return (double)static_cast<const float*>(a)[off];
  if (MODE == 1) return (double)__half2float(static_cast<const __half*>(a)[off]);
  return (double)__bfloat162float(static_cast<const __nv_bfloat16*>(a)[off]) * scale;
}

// refine_search (core.py:368-394), one CTA per query: the L shortlist
// candidates (ids, -1 skipped; positions from the id table) get the DIRECT
// distance of the reconstructed vector (pairwise_distances -> dist_one,
// _ckernels.pyx:49-57: L2 sum (q - x)^2, IP sum q x) accumulated in fp64 and
// rounded once to fp32; the first k by (best value, candidate id, shortlist
// slot) -- Python's stable `sorted(key=(value, id))` -- are written best
// first, the rest padded with -1 / +inf (L2) or -inf (IP) (core.py:379-381).
// Selection is an exact rank count over the shortlist held in smem.
template <int MODE>
__global__ void __launch_bounds__(256) refine_kernel(const float* __restrict__ q, int d,
                                                     const int64_t* __restrict__ cand,
                                                     const int64_t* __restrict__ cpos, int L, int k,
                                                     const void* __restrict__ s0, const void* __restrict__ s1,
                                                     int dp, double scale, int is_ip, float* __restrict__ D,
                                                     int64_t* __restrict__ I) {
  extern __shared__ __align__(16) uint8_t fk_refine_smem[];
  int64_t* cid = reinterpret_cast<int64_t*>(fk_refine_smem);  // [L] (-1: empty)
  uint32_t* key = reinterpret_cast<uint32_t*>(cid + L);        // [L]
  float* val = reinterpret_cast<float*>(key + L);              // [L]
  __shared__ int n_valid;
  const int qi = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const float* qr = q + (size_t)qi * d;
  if (threadIdx.x == 0) n_valid = 0;
  __syncthreads();
  for (int j = warp; j < L; j += nw) {
    const int64_t p = cpos[(size_t)qi * L + j];
    double acc = 0.0;
    if (p >= 0) {
      for (int c = lane; c < d; c += 32) {
        const double x = refine_stored<MODE>(s0, s1, (size_t)p * dp + c, scale);
        const double qv = (double)qr[c];
        if (is_ip) {
          acc = fma(qv, x, acc);
        } else {
          const double t = qv - x;
          acc = fma(t, t, acc);
        }
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, off);
    if (lane == 0) {
      const float v = static_cast<float>(acc);
      cid[j] = p >= 0 ? cand[(size_t)qi * L + j] : -1;
      key[j] = dist_key(v, is_ip != 0);
      val[j] = v;
      if (p >= 0) atomicAdd(&n_valid, 1);
    }
  }
  __syncthreads();
  const int nv = n_valid;
  for (int j = threadIdx.x; j < L; j += blockDim.x) {
    const int64_t idj = cid[j];
    if (idj < 0) continue;
    const uint32_t kj = key[j];
    int r = 0;
    for (int i = 0; i < L; ++i) {
      const int64_t idi = cid[i];
      const uint32_t ki = key[i];
      r += (idi >= 0) & ((ki < kj) | ((ki == kj) & ((idi < idj) | ((idi == idj) & (i < j)))));
    }
    if (r < k) {
      D[(size_t)qi * k + r] = val[j];
      I[(size_t)qi * k + r] = idj;
    }
  }
  const float pad = is_ip ? -__int_as_float(0x7f800000) : __int_as_float(0x7f800000);
  for (int s = nv + threadIdx.x; s < k; s += blockDim.x) {
    D[(size_t)qi * k + s] = pad;
    I[(size_t)qi * k + s] = -1;
  }
}

}  // namespace fk
