// fp32 MODE 5 operands: a 16-bit copy of fp32 rows for the filter pass of
// the certified 1-pass search (fused_kernel.cuh, merge_rescore_kernel).
//
// x~ = fp16_rne(x * 2^s) with a power-of-two scale s -- one per query row,
// one for the whole base -- chosen so the scaled max |x| lies in
// [2^13, 2^14): every normal element then keeps 11 significant bits
// (|x~ 2^-s - x| <= 2^-11 |x|, the same precision as a tf32 operand), an
// element that lands in the fp16 subnormal range errs by <= 2^-25 2^-s
// <= 2^-38 max|x| absolutely, and nothing overflows.  Products of two fp16
// values are exact in fp32 and the tensor core runs kind::f16 at twice the
// tf32 rate on half the bytes.  The epilogue multiplies the accumulator back
// by 2^-(s_q + s_x) (exact) before the filter, so t is a 1-pass estimate of
// the inner product with |t - ip| <= (2^-10 + 2^-27) |q||x| + accumulation.
#pragma once
#include <cuda_fp16.h>

#include <cstdint>

namespace fk {

constexpr int F16_TOP = 13;    // scaled max |x| in [2^13, 2^14)
constexpr int F16_SMAX = 60;   // |s| beyond this: the scale is flagged unusable

// Base scale state (device): running max finite |x|, the scale exponent of
// the converted copy, its inverse 2^-s (NaN = unusable -> every query takes
// the exact fallback) and whether the last update forces a full rebuild.
struct F16State {
  unsigned int absmax;  // float bits of max finite |x| (non-negative: uint order == float order)
  int s;
  float xinv;
  int rebuild;
};

__device__ __forceinline__ int f16_scale_exp(float m, bool* ok) {
  if (!(m > 0.f)) {  // all zero (or nothing finite): any scale is exact
    *ok = true;
    return 0;
  }
  const int s = F16_TOP - ilogbf(m);
  *ok = s >= -F16_SMAX && s <= F16_SMAX;
  return max(-F16_SMAX, min(F16_SMAX, s));
}

// max finite |hi + lo| over the stored elements [e0, e1) (padding is zero)
__global__ void absmax_rows_kernel(const float* __restrict__ s0, const float* __restrict__ s1, size_t e0, size_t e1,
                                   unsigned int* __restrict__ absmax) {
  float m = 0.f;
  for (size_t i = e0 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < e1; i += (size_t)gridDim.x * blockDim.x) {
    const float v = fabsf(s0[i] + s1[i]);  // hi + lo == x exactly
    if (v <= 3.402823466e38f) m = fmaxf(m, v);  // finite only
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, off));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(absmax, __float_as_uint(m));
}

// New base scale from the running max; a changed scale (or an empty copy)
// rebuilds every row and restarts the base's exactness flag.
__global__ void f16_scale_kernel(F16State* st, long long converted_rows, unsigned int* inexact_base) {
  if (threadIdx.x != 0) return;
  bool ok;
  const int s = f16_scale_exp(__uint_as_float(st->absmax), &ok);
  const int rebuild = (converted_rows == 0 || s != st->s) ? 1 : 0;
  st->rebuild = rebuild;
  st->s = s;
  st->xinv = ok ? ldexpf(1.f, -s) : __int_as_float(0x7FC00000);
  if (rebuild) *inexact_base = 0u;
}

// Stored fp32 rows (hi + lo) -> scaled fp16 rows [n][dp16]; rows below
// r_keep are already converted with the current scale unless st->rebuild.
// inexact_base: set when some element is not exactly x~ 2^-s (then the
// band keeps its rounding term; all-exact data collapses it).
__global__ void f16_base_kernel(const float* __restrict__ s0, const float* __restrict__ s1, int64_t r_keep, int64_t n,
                                int d, int dp, int dp16, __half* __restrict__ out, const F16State* __restrict__ st,
                                unsigned int* __restrict__ inexact_base) {
  const int lane = threadIdx.x & 31;
  const int64_t r0 = (st->rebuild ? 0 : r_keep);
  const int s = st->s;
  bool inexact = false;
  for (int64_t r = r0 + (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n;
       r += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    for (int c = lane; c < dp16; c += 32) {
      const float v = c < d ? s0[(size_t)r * dp + c] + s1[(size_t)r * dp + c] : 0.f;
      const float sv = ldexpf(v, s);
      const __half h = __float2half_rn(sv);
      out[(size_t)r * dp16 + c] = h;
      if (__half2float(h) != sv && !isnan(v)) inexact = true;
    }
  }
  if (__any_sync(0xFFFFFFFFu, inexact) && lane == 0) atomicOr(inexact_base, 1u);
}

// Query rows (any input dtype) -> scaled fp16 rows [n][dp16] + 2^-s per row
// (NaN when the row's scale is unusable: that query takes the exact fallback).
__global__ void f16_query_kernel(const void* __restrict__ x, int dtype, int64_t n, int d, int dp16,
                                 __half* __restrict__ out, float* __restrict__ qinv,
                                 unsigned int* __restrict__ inexact_q) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  auto load = [&](int c) -> float {
    if (dtype == 0) return static_cast<const float*>(x)[(size_t)r * d + c];
    if (dtype == 1) return __half2float(static_cast<const __half*>(x)[(size_t)r * d + c]);
    return __bfloat162float(static_cast<const __nv_bfloat16*>(x)[(size_t)r * d + c]);
  };
  float m = 0.f;
  for (int c = lane; c < d; c += 32) {
    const float v = fabsf(load(c));
    if (v <= 3.402823466e38f) m = fmaxf(m, v);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, off));
  bool ok;
  const int s = f16_scale_exp(m, &ok);
  bool inexact = false;
  for (int c = lane; c < dp16; c += 32) {
    const float v = c < d ? load(c) : 0.f;
    const float sv = ldexpf(v, s);
    const __half h = __float2half_rn(sv);
    out[(size_t)r * dp16 + c] = h;
    if (__half2float(h) != sv && !isnan(v)) inexact = true;
  }
  if (lane == 0) qinv[r] = ok ? ldexpf(1.f, -s) : __int_as_float(0x7FC00000);
  if (__any_sync(0xFFFFFFFFu, inexact) && lane == 0) atomicOr(inexact_q, 1u);
}

}  // namespace fk
