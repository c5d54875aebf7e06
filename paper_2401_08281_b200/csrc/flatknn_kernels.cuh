// Device kernels of the B200-native exact flat k-NN engine other than the
// fused GEMM + top-k kernel (fused_kernel.cuh): merges, rescoring, fallback,
// conversions, storage ops, range search, k-means rescoring.
#pragma once
#include "fused_kernel.cuh"

namespace fk {

// ------------------------------------------------------------ merges
// One warp per query: k rounds of a warp-wide argmin over the heads of S
// sorted partial lists (lane l owns lists l, l+32, l+64, l+96 -> S <= 128).
template <bool IS_IP>
__global__ void merge_kernel(const uint32_t* __restrict__ pkey, const uint32_t* __restrict__ ppos, int S, int nq,
                             int k, const int64_t* __restrict__ ids, float* __restrict__ D,
                             int64_t* __restrict__ I, int64_t* __restrict__ P) {
  const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (q >= nq) return;
  const uint32_t* lk = pkey + (size_t)q * S * k;
  const uint32_t* lp = ppos + (size_t)q * S * k;
  int h0 = 0, h1 = 0, h2 = 0, h3 = 0;
  auto head = [&](int i, int h) -> uint64_t {
    const int l = lane + 32 * i;
    if (l >= S || h >= k) return ~0ull;
    const size_t o = (size_t)l * k + h;
    return (static_cast<uint64_t>(lk[o]) << 32) | lp[o];
  };
  uint64_t c0 = head(0, 0), c1 = head(1, 0), c2 = head(2, 0), c3 = head(3, 0);
  for (int r = 0; r < k; ++r) {
    uint64_t best = c0;
    int bi = 0;
    if (c1 < best) { best = c1; bi = 1; }
    if (c2 < best) { best = c2; bi = 2; }
    if (c3 < best) { best = c3; bi = 3; }
    const uint64_t w = warp_min_u64(best);
    if (w != ~0ull && best == w) {
      if (bi == 0) c0 = head(0, ++h0);
      else if (bi == 1) c1 = head(1, ++h1);
      else if (bi == 2) c2 = head(2, ++h2);
      else c3 = head(3, ++h3);
    }
    if (lane == 0) {
      const size_t o = (size_t)q * k + r;
      if (w == ~0ull) {
        D[o] = IS_IP ? -INFINITY : INFINITY;
        I[o] = -1;
        if (P) P[o] = -1;
      } else {
        const uint32_t key = static_cast<uint32_t>(w >> 32);
        const uint32_t ps = static_cast<uint32_t>(w & 0xFFFFFFFFu);
        D[o] = key_dist(key, IS_IP);
        I[o] = ids[ps];
        if (P) P[o] = ps;
      }
    }
  }
}

// Shard merge: nshard lists per query of (D, global position, id), already
// best-first.  Ordering by (monotone key, global position) reproduces the
// unsharded reference order exactly.  Lane l owns shards l, l+32 (<= 64).
template <bool IS_IP>
__global__ void shard_merge_kernel(int nshard, int nq, int k, const float* __restrict__ Din,
                                   const int64_t* __restrict__ Pin, const int64_t* __restrict__ Iin,
                                   float* __restrict__ D, int64_t* __restrict__ I) {
  const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (q >= nq) return;
  auto head = [&](int s, int h, int64_t& id) -> uint64_t {
    if (s >= nshard || h >= k) return ~0ull;
    const size_t o = ((size_t)s * nq + q) * k + h;
    const int64_t ps = Pin[o];
    if (ps < 0) return ~0ull;
    id = Iin[o];
    const float v = Din[o];
    return (static_cast<uint64_t>(dist_key(v, IS_IP)) << 32) | static_cast<uint32_t>(ps);
  };
  int h0 = 0, h1 = 0;
  int64_t id0 = -1, id1 = -1;
  uint64_t c0 = head(lane, 0, id0), c1 = head(lane + 32, 0, id1);
  for (int r = 0; r < k; ++r) {
    const bool second = c1 < c0;
    const uint64_t best = second ? c1 : c0;
    const int64_t bid = second ? id1 : id0;
    const uint64_t w = warp_min_u64(best);
    const unsigned win = __ballot_sync(0xFFFFFFFFu, w != ~0ull && best == w);
    int64_t wid = -1;
    if (win) wid = __shfl_sync(0xFFFFFFFFu, bid, __ffs(win) - 1);
    if (w != ~0ull && best == w) {
      if (second) c1 = head(lane + 32, ++h1, id1);
      else c0 = head(lane, ++h0, id0);
    }
    if (lane == 0) {
      const size_t o = (size_t)q * k + r;
      if (w == ~0ull) {
        D[o] = IS_IP ? -INFINITY : INFINITY;
        I[o] = -1;
      } else {
        D[o] = key_dist(static_cast<uint32_t>(w >> 32), IS_IP);
        I[o] = wid;
      }
    }
  }
}


// Block-wide exact k-th smallest (1-based) of n composites read through
// load(e) (all threads call it; MSB-first 8-bit radix with a shared histogram).
template <class Load>
__device__ uint64_t block_kth(Load load, int n, uint32_t k, uint32_t* hist, uint32_t* sel) {
  const int tid = threadIdx.x;
  uint64_t prefix = 0;
  uint32_t need = k;
  for (int shift = 56; shift >= 0; shift -= 8) {
    const uint64_t hmask = (shift == 56) ? 0ull : (~0ull << (shift + 8));
    for (int b = tid; b < 256; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    for (int e = tid; e < n; e += blockDim.x) {
      const uint64_t v = load(e);
      if ((v & hmask) == prefix) atomicAdd(&hist[static_cast<uint32_t>(v >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid < 32) {
      const int lane = tid;
      uint32_t c[8], sum = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        c[i] = hist[lane * 8 + i];
        sum += c[i];
      }
      uint32_t incl = sum;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t o = __shfl_up_sync(FULLMASK, incl, off);
        if (lane >= off) incl += o;
      }
      const uint32_t excl = incl - sum;
      if (excl < need && need <= incl) {
        uint32_t run = excl;
        bool done = false;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (!done && run < need && need <= run + c[i]) {
            sel[0] = lane * 8 + i;
            sel[1] = run;
            sel[2] = c[i];
            done = true;
          }
          run += c[i];
        }
      }
    }
    __syncthreads();
    const uint32_t bin = sel[0], before = sel[1], bcnt = sel[2];
    need -= before;
    prefix |= static_cast<uint64_t>(bin) << shift;
    __syncthreads();
    if (bcnt == 1) {
      const uint64_t m2 = ~0ull << shift;
      for (int e = tid; e < n; e += blockDim.x) {
        const uint64_t v = load(e);
        if ((v & m2) == prefix) {
          sel[3] = static_cast<uint32_t>(v >> 32);
          sel[4] = static_cast<uint32_t>(v);
        }
      }
      __syncthreads();
      const uint64_t r = (static_cast<uint64_t>(sel[3]) << 32) | sel[4];
      __syncthreads();
      return r;
    }
  }
  return prefix;
}

// Large-k final merge: one CTA per query.  Survivors of every partial list
// with key <= the query's final shared bound (a superset of the true top-k,
// at least k of them) are gathered into smem; an exact block radix select
// finds the k-th (key, position); the k winners are bitonic-sorted.  If the
// survivors overflow smem the select reads the lists from global instead.
template <bool IS_IP>
__global__ void __launch_bounds__(1024) merge_large_kernel(const uint32_t* __restrict__ pkey,
                                                          const uint32_t* __restrict__ ppos,
                                                          const int* __restrict__ pcnt, int S, int nq, int k,
                                                          const uint32_t* __restrict__ thr_key,
                                                          const int64_t* __restrict__ ids, float* __restrict__ D,
                                                          int64_t* __restrict__ I, int64_t* __restrict__ P,
                                                          int smc, int* __restrict__ fail) {
  extern __shared__ uint64_t sm[];  // smc survivors, then the k winners (pow2-padded)
  __shared__ int count, count2;
  __shared__ uint32_t hist[256], sel[8];
  const int q = blockIdx.x;
  const int tid = threadIdx.x;
  if (q >= nq) return;
  const uint32_t thr = thr_key[q];
  const uint32_t* lk = pkey + (size_t)q * S * k;
  const uint32_t* lp = ppos + (size_t)q * S * k;
  const int* lc = pcnt ? pcnt + (size_t)q * S : nullptr;  // NULL: register-queue lists (k each, sentinel-padded)
  if (tid == 0) {
    count = 0;
    count2 = 0;
  }
  __syncthreads();
  const int total = S * k;
  auto gload = [&](int e) -> uint64_t {
    const int s = e / k, i = e - s * k;
    if (lc && i >= lc[s]) return ~0ull;
    const uint32_t key = lk[e];
    if (key > thr || lp[e] == 0xFFFFFFFFu) return ~0ull;
    return (static_cast<uint64_t>(key) << 32) | lp[e];
  };
  // the query's S*k block is contiguous: flat, coalesced, 4 independent key
  // loads in flight per thread (the gather is latency-bound otherwise)
  auto take = [&](int e, uint32_t key) {
    if (key > thr) return;
    const uint32_t ps = __ldcs(lp + e);
    if (ps == 0xFFFFFFFFu) return;
    if (lc) {
      const int s = e / k;
      if (e - s * k >= lc[s]) return;
    }
    const int idx = atomicAdd(&count, 1);
    if (idx < smc) sm[idx] = (static_cast<uint64_t>(key) << 32) | ps;
  };
  const int step = blockDim.x;
  int e = tid;
  for (; e + 3 * step < total; e += 4 * step) {
    const uint32_t k0 = __ldcs(lk + e), k1 = __ldcs(lk + e + step), k2 = __ldcs(lk + e + 2 * step),
                   k3 = __ldcs(lk + e + 3 * step);
    take(e, k0);
    take(e + step, k1);
    take(e + 2 * step, k2);
    take(e + 3 * step, k3);
  }
  for (; e < total; e += step) take(e, __ldcs(lk + e));
  __syncthreads();
  const int n = count;
  // certification (estimated bound): fewer than k survivors means the bound
  // may have excluded true neighbours -> the host reruns without the estimate
  if (fail != nullptr && n < k && tid == 0) atomicAdd(fail, 1);
  uint64_t* win = sm + smc;  // k winners
  int nw;
  if (n <= k) {
    for (int i = tid; i < n; i += blockDim.x) win[i] = sm[i];
    nw = n;
  } else {
    uint64_t kth;
    if (n <= smc)
      kth = block_kth([&](int e) { return sm[e]; }, n, (uint32_t)k, hist, sel);
    else
      kth = block_kth(gload, total, (uint32_t)k, hist, sel);
    if (n <= smc) {
      for (int i = tid; i < n; i += blockDim.x)
        if (sm[i] <= kth) win[atomicAdd(&count2, 1)] = sm[i];
    } else {
      for (int e = tid; e < total; e += blockDim.x) {
        const uint64_t v = gload(e);
        if (v != ~0ull && v <= kth) win[atomicAdd(&count2, 1)] = v;
      }
    }
    __syncthreads();
    nw = count2;  // == k (composites are unique)
  }
  int P2 = 1;
  while (P2 < nw) P2 <<= 1;
  for (int i = nw + tid; i < P2; i += blockDim.x) win[i] = ~0ull;
  __syncthreads();
  for (int size = 2; size <= P2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < P2 / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const uint64_t a = win[lo], b = win[hi];
        if ((a > b) == asc) {
          win[lo] = b;
          win[hi] = a;
        }
      }
      __syncthreads();
    }
  }
  for (int r = tid; r < k; r += blockDim.x) {
    const size_t o = (size_t)q * k + r;
    const uint64_t w = r < nw ? win[r] : ~0ull;
    if (w == ~0ull) {
      D[o] = IS_IP ? -INFINITY : INFINITY;
      I[o] = -1;
      if (P) P[o] = -1;
    } else {
      const uint32_t ps = static_cast<uint32_t>(w);
      D[o] = key_dist(static_cast<uint32_t>(w >> 32), IS_IP);
      I[o] = ids[ps];
      if (P) P[o] = ps;
    }
  }
}

// ------------------------------------------------------------ 1-pass rescoring merge
// Exact fp32 inner product of one (query, row) pair by a whole warp: lane l
// accumulates the float4 chunks l, l+32, ... sequentially (hi + lo == the fp32
// value exactly), then a fixed xor-butterfly sums the lanes -- the same value
// on every lane, the same summation order in the rescoring merge and the exact
// fallback (one load round instead of dp/4 dependent ones per pair).
__device__ __forceinline__ float warp_exact_dot(const float4* __restrict__ qh, const float4* __restrict__ ql,
                                                const float4* __restrict__ xh, const float4* __restrict__ xl, int dp,
                                                int lane) {
  float acc = 0.f;
  for (int c = lane; c < dp / 4; c += 32) {
    float4 a = __ldg(qh + c), b = __ldg(xh + c);
    if (ql) {
      const float4 t = __ldg(ql + c);
      a = make_float4(a.x + t.x, a.y + t.y, a.z + t.z, a.w + t.w);
    }
    if (xl) {
      const float4 t = __ldg(xl + c);
      b = make_float4(b.x + t.x, b.y + t.y, b.z + t.z, b.w + t.w);
    }
    acc = fmaf(a.x, b.x, acc);
    acc = fmaf(a.y, b.y, acc);
    acc = fmaf(a.z, b.z, acc);
    acc = fmaf(a.w, b.w, acc);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, off);
  return acc;
}

// The same value as warp_exact_dot computed by ONE thread (the exact
// fallback scans a whole base per failed query: a thread per row keeps its
// loads in flight): the 32 lane partials in the same sequential order, then
// the xor-butterfly's pairing (lane 0's view: v[i] += v[i + off]).
__device__ __forceinline__ float thread_exact_dot(const float4* __restrict__ qh, const float4* __restrict__ ql,
                                                  const float4* __restrict__ xh, const float4* __restrict__ xl,
                                                  int dp) {
  float v[32];
#pragma unroll
  for (int l = 0; l < 32; ++l) v[l] = 0.f;
  for (int c0 = 0; c0 < dp / 4; c0 += 32) {
#pragma unroll
    for (int l = 0; l < 32; ++l) {
      const int c = c0 + l;
      if (c < dp / 4) {
        float4 a = __ldg(qh + c), b = __ldg(xh + c);
        if (ql) {
          const float4 t = __ldg(ql + c);
          a = make_float4(a.x + t.x, a.y + t.y, a.z + t.z, a.w + t.w);
        }
        if (xl) {
          const float4 t = __ldg(xl + c);
          b = make_float4(b.x + t.x, b.y + t.y, b.z + t.z, b.w + t.w);
        }
        float acc = v[l];
        acc = fmaf(a.x, b.x, acc);
        acc = fmaf(a.y, b.y, acc);
        acc = fmaf(a.z, b.z, acc);
        acc = fmaf(a.w, b.w, acc);
        v[l] = acc;
      }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int i = 0; i < off; ++i) v[i] = v[i] + v[i + off];
  return v[0];
}

// fp32 MODE 4 runs the fused pass with a 1-pass TF32 GEMM and keeps k' >= k
// entries per list ranked by their tf32 value t.  With e = max|t - v| over all
// pairs (|t - v| <= 2^-8 |q| max|x| for L2, half for IP), every exact top-k
// member has t <= t_k + 2e (t_k = k-th smallest t overall), and every entry
// that did not reach a list has t >= bound (the final shared k'-th bound).
// One CTA per query: gather the list entries below the bound, CERTIFY
// bound > t_k + 2e (else flag the query for the exact fallback), recompute the
// gathered entries' distances exactly (fp32 FMA over d from the stored rows,
// the value of flat.py:111) and select the exact top-k by (value, position).
template <bool IS_IP>
__global__ void __launch_bounds__(256) merge_rescore_kernel(
    const uint32_t* __restrict__ pkey, const uint32_t* __restrict__ ppos, const int* __restrict__ pcnt, int S, int nq,
    int kp, int k, const uint32_t* __restrict__ thr_key, const float* __restrict__ q0, const float* __restrict__ q1,
    const float* __restrict__ xb, const float* __restrict__ xl,
    const float* __restrict__ qnorm, const float* __restrict__ xnorm, const float* __restrict__ xn_max, int dp,
    const int64_t* __restrict__ ids, float* __restrict__ D, int64_t* __restrict__ I, int64_t* __restrict__ P, int smc,
    int* __restrict__ fail, int* __restrict__ fail_count, int* __restrict__ fail_list,
    const unsigned int* __restrict__ rflag, const unsigned int* __restrict__ inexact, float band_l2,
    const uint32_t* __restrict__ ovf_key, const uint32_t* __restrict__ ovf_pos,
    const unsigned int* __restrict__ ovf_cnt, int ovf_cap) {
  extern __shared__ uint64_t sm[];  // smc gathered entries, then the k winners (pow2-padded)
  __shared__ int count, count2;
  __shared__ uint32_t hist[256], sel[8];
  const int q = blockIdx.x;
  const int tid = threadIdx.x;
  if (q >= nq) return;
  // uncertified queries are appended to fail_list for fallback_kernel (no host round trip)
  // fail[q]: 0 certified; reason otherwise (1 survivors > smem buffer, 2 bound
  // does not clear the band, 3 fewer than k under the bound, 4 row flag)
  auto mark_failed = [&](int why) {
    fail[q] = why;
    fail_list[atomicAdd(fail_count, 1)] = q;
  };
  const uint32_t thr = thr_key[q];
  const uint32_t* lk = pkey + (size_t)q * S * kp;
  const uint32_t* lp = ppos + (size_t)q * S * kp;
  const int* lc = pcnt ? pcnt + (size_t)q * S : nullptr;
  if (tid == 0) {
    count = 0;
    count2 = 0;
  }
  __syncthreads();
  const int total = S * kp;
  for (int e = tid; e < total; e += blockDim.x) {
    const uint32_t key = lk[e];
    if (key > thr) continue;
    const uint32_t ps = lp[e];
    if (ps == 0xFFFFFFFFu) continue;
    if (lc) {
      const int s = e / kp;
      if (e - s * kp >= lc[s]) continue;
    }
    const int idx = atomicAdd(&count, 1);
    if (idx < smc) sm[idx] = (static_cast<uint64_t>(key) << 32) | ps;
  }
  if (ovf_cnt != nullptr) {  // band members the units' full queues dropped
    const int no = min((int)ovf_cnt[q], ovf_cap);
    for (int e = tid; e < no; e += blockDim.x) {
      const uint32_t key = ovf_key[(size_t)q * ovf_cap + e];
      if (key > thr) continue;
      const int idx = atomicAdd(&count, 1);
      if (idx < smc) sm[idx] = (static_cast<uint64_t>(key) << 32) | ovf_pos[(size_t)q * ovf_cap + e];
    }
  }
  __syncthreads();
  int n = count;
  if (n > smc) {  // more survivors than the buffer: exact fallback for this query
    if (tid == 0) mark_failed(1);
    return;
  }
  // certification on the tf32 values
  const float qn = qnorm[q];
  // band = 2 x the filter-value error bound, times |q| max|x| (band_l2 =
  // 2^-7 tf32 / 2^-8 scaled fp16, with a 2^-10 margin; IP half), plus the fp32
  // accumulation slack (4 dp + 8) 2^-23 (qn + max xn) (same as the fused
  // kernel's band4)
  const bool tf32_exact = inexact != nullptr && (inexact[0] | inexact[1]) == 0u;
  const float e2 = (tf32_exact ? 0.f : (IS_IP ? 0.5f * band_l2 : band_l2)) * sqrtf(band_norm(qn) * band_norm(*xn_max)) +
                   (4.f * (float)dp + 8.f) * 1.1920928955078125e-07f * (band_norm(qn) + band_norm(*xn_max));
  bool ok = true;
  int why = 0;
  uint32_t band_key = 0xFFFFFFFFu;  // only entries with t <= t_k + band can be in the exact top-k
  if (n >= k) {
    const uint64_t kth = block_kth([&](int e) { return sm[e]; }, n, (uint32_t)k, hist, sel);
    const float tk = unmonotone(static_cast<uint32_t>(kth >> 32));
    const float lim = tk + e2 + 9.5367431640625e-07f * (fabsf(tk) + qn);
    band_key = monotone(lim);
    // large-k lists (pcnt != NULL) were filtered by the units' k'-th values:
    // every entry that did not reach a list has t >= thr, so thr must clear
    // the band.  (Register-queue lists filter with (own k-th + band) bounds,
    // which never drop a band member: only the row flag below matters.)
    if (lc != nullptr && thr != 0xFFFFFFFFu && !(unmonotone(thr) > lim)) {
      ok = false;
      why = 2;
    }
  } else if (thr != 0xFFFFFFFFu) {
    ok = false;  // fewer than k gathered although entries were dropped
    why = 3;
  }
  // a register queue that dropped a band member flagged its row
  if (rflag[q]) {
    ok = false;
    why = 4;
  }
  if (tid == 0) {
    if (ok) fail[q] = 0;
    else mark_failed(why);
  }
  if (!ok) return;
  // keep the band only (typically k + a few): in-place compaction
  if (band_key != 0xFFFFFFFFu) {
    __syncthreads();
    uint64_t mine[8];
    int nm = 0;
    for (int i = tid; i < n && nm < 8; i += blockDim.x)
      if (static_cast<uint32_t>(sm[i] >> 32) <= band_key) mine[nm++] = sm[i];
    const bool spill = (n > 8 * (int)blockDim.x);  // cannot happen: n <= smc <= 8 * 256 * ... guard anyway
    __syncthreads();
    if (tid == 0) count2 = 0;
    __syncthreads();
    if (!spill) {
      for (int j = 0; j < nm; ++j) sm[atomicAdd(&count2, 1)] = mine[j];
      __syncthreads();
      n = count2;
      __syncthreads();
      if (tid == 0) count2 = 0;
      __syncthreads();
    }
  }
  // exact values for the remaining entries
  const float4* qv = reinterpret_cast<const float4*>(q0 + (size_t)q * dp);
  const float4* qlv = q1 ? reinterpret_cast<const float4*>(q1 + (size_t)q * dp) : nullptr;
  for (int i = tid >> 5; i < n; i += blockDim.x >> 5) {  // a warp per entry
    const uint32_t ps = static_cast<uint32_t>(sm[i]);
    const float acc = warp_exact_dot(qv, qlv, reinterpret_cast<const float4*>(xb + (size_t)ps * dp),
                                     xl ? reinterpret_cast<const float4*>(xl + (size_t)ps * dp) : nullptr, dp,
                                     tid & 31);
    float v = acc;
    if (!IS_IP) {
      v = fmaf(-2.f, acc, qn + xnorm[ps]);  // flat.py:111
      v = (v <= 0.f) ? 0.f : v;              // flat.py:112
    }
    __syncwarp();
    if ((tid & 31) == 0) sm[i] = (static_cast<uint64_t>(dist_key(v, IS_IP)) << 32) | ps;
  }
  __syncthreads();
  uint64_t* win = sm + smc;
  int nw;
  if (n <= k) {
    for (int i = tid; i < n; i += blockDim.x) win[i] = sm[i];
    nw = n;
  } else {
    const uint64_t kth = block_kth([&](int e) { return sm[e]; }, n, (uint32_t)k, hist, sel);
    for (int i = tid; i < n; i += blockDim.x)
      if (sm[i] <= kth) win[atomicAdd(&count2, 1)] = sm[i];
    __syncthreads();
    nw = count2;
  }
  int P2 = 1;
  while (P2 < nw) P2 <<= 1;
  for (int i = nw + tid; i < P2; i += blockDim.x) win[i] = ~0ull;
  __syncthreads();
  for (int size = 2; size <= P2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < P2 / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const uint64_t a = win[lo], b2 = win[hi];
        if ((a > b2) == asc) {
          win[lo] = b2;
          win[hi] = a;
        }
      }
      __syncthreads();
    }
  }
  for (int r = tid; r < k; r += blockDim.x) {
    const size_t o = (size_t)q * k + r;
    const uint64_t w = r < nw ? win[r] : ~0ull;
    if (w == ~0ull) {
      D[o] = IS_IP ? -INFINITY : INFINITY;
      I[o] = -1;
      if (P) P[o] = -1;
    } else {
      const uint32_t ps = static_cast<uint32_t>(w);
      D[o] = key_dist(static_cast<uint32_t>(w >> 32), IS_IP);
      I[o] = ids[ps];
      if (P) P[o] = ps;
    }
  }
}

// Warp-per-query form of merge_rescore_kernel for register-queue lists
// (S * k' small, k <= 32): 8 queries per CTA, the gathered composites in a
// warp-private smem buffer (W_SMW entries; more -> exact fallback), ranks by
// counting instead of block-wide radix selects, the same certification, band
// and warp_exact_dot rescoring (values bit-identical to the CTA form).
constexpr int W_SMW = 512;
template <bool IS_IP>
__global__ void __launch_bounds__(256) merge_rescore_warp_kernel(
    const uint32_t* __restrict__ pkey, const uint32_t* __restrict__ ppos, int S, int nq, int kp, int k,
    const uint32_t* __restrict__ thr_key, const float* __restrict__ q0, const float* __restrict__ q1,
    const float* __restrict__ xb, const float* __restrict__ xl, const float* __restrict__ qnorm,
    const float* __restrict__ xnorm, const float* __restrict__ xn_max, int dp, const int64_t* __restrict__ ids,
    float* __restrict__ D, int64_t* __restrict__ I, int64_t* __restrict__ P, int* __restrict__ fail,
    int* __restrict__ fail_count, int* __restrict__ fail_list, const unsigned int* __restrict__ rflag,
    const unsigned int* __restrict__ inexact, float band_l2, const uint32_t* __restrict__ ovf_key,
    const uint32_t* __restrict__ ovf_pos, const unsigned int* __restrict__ ovf_cnt, int ovf_cap) {
  __shared__ uint64_t sbuf[8][W_SMW];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = blockIdx.x * 8 + w;
  if (q >= nq) return;
  uint64_t* buf = sbuf[w];
  auto mark_failed = [&](int why) {
    if (lane == 0) {
      fail[q] = why;
      fail_list[atomicAdd(fail_count, 1)] = q;
    }
  };
  const uint32_t thr = thr_key[q];
  const int total = S * kp;
  int n = 0;
  auto push = [&](bool take, uint64_t v) {
    const unsigned b = __ballot_sync(0xFFFFFFFFu, take);
    const int at = n + __popc(b & ((1u << lane) - 1u));
    if (take && at < W_SMW) buf[at] = v;
    n += __popc(b);
  };
  for (int e0 = 0; e0 < total; e0 += 32) {
    const int e = e0 + lane;
    uint64_t v = 0;
    bool take = false;
    if (e < total) {
      const uint32_t key = pkey[(size_t)q * total + e];
      const uint32_t ps = ppos[(size_t)q * total + e];
      take = key <= thr && ps != 0xFFFFFFFFu;
      v = (static_cast<uint64_t>(key) << 32) | ps;
    }
    push(take, v);
  }
  if (ovf_cnt != nullptr) {
    const int no = min((int)ovf_cnt[q], ovf_cap);
    for (int e0 = 0; e0 < no; e0 += 32) {
      const int e = e0 + lane;
      uint64_t v = 0;
      bool take = false;
      if (e < no) {
        const uint32_t key = ovf_key[(size_t)q * ovf_cap + e];
        take = key <= thr;
        v = (static_cast<uint64_t>(key) << 32) | ovf_pos[(size_t)q * ovf_cap + e];
      }
      push(take, v);
    }
  }
  __syncwarp();
  if (n > W_SMW) {
    mark_failed(1);
    return;
  }
  // rank of buf[i] among the n (unique) composites
  auto rank_of = [&](uint64_t v, int cnt) {
    int r = 0;
    for (int j = 0; j < cnt; ++j) r += buf[j] < v;
    return r;
  };
  const float qn = qnorm[q];
  const bool tf32_exact = inexact != nullptr && (inexact[0] | inexact[1]) == 0u;
  const float e2 = (tf32_exact ? 0.f : (IS_IP ? 0.5f * band_l2 : band_l2)) * sqrtf(band_norm(qn) * band_norm(*xn_max)) +
                   (4.f * (float)dp + 8.f) * 1.1920928955078125e-07f * (band_norm(qn) + band_norm(*xn_max));
  uint32_t band_key = 0xFFFFFFFFu;
  int why = 0;
  if (n >= k) {
    uint64_t kth = ~0ull;
    for (int i = lane; i < n; i += 32)
      if (rank_of(buf[i], n) == k - 1) kth = buf[i];
    kth = warp_min_u64(kth);
    const float tk = unmonotone(static_cast<uint32_t>(kth >> 32));
    band_key = monotone(tk + e2 + 9.5367431640625e-07f * (fabsf(tk) + qn));
  } else if (thr != 0xFFFFFFFFu) {
    why = 3;
  }
  if (rflag[q]) why = 4;
  if (why) {
    mark_failed(why);
    return;
  }
  if (lane == 0) fail[q] = 0;
  // keep the band (order-preserving warp compaction), rescore exactly
  int m = 0;
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    const uint64_t v = i < n ? buf[i] : 0;
    const bool keep = i < n && static_cast<uint32_t>(v >> 32) <= band_key;
    const unsigned b = __ballot_sync(0xFFFFFFFFu, keep);
    __syncwarp();
    if (keep) buf[m + __popc(b & ((1u << lane) - 1u))] = v;
    m += __popc(b);
    __syncwarp();
  }
  const float4* qv = reinterpret_cast<const float4*>(q0 + (size_t)q * dp);
  const float4* qlv = q1 ? reinterpret_cast<const float4*>(q1 + (size_t)q * dp) : nullptr;
  for (int i = 0; i < m; ++i) {
    const uint32_t ps = static_cast<uint32_t>(buf[i]);
    const float acc = warp_exact_dot(qv, qlv, reinterpret_cast<const float4*>(xb + (size_t)ps * dp),
                                     xl ? reinterpret_cast<const float4*>(xl + (size_t)ps * dp) : nullptr, dp, lane);
    float v = acc;
    if (!IS_IP) {
      v = fmaf(-2.f, acc, qn + xnorm[ps]);  // flat.py:111
      v = (v <= 0.f) ? 0.f : v;              // flat.py:112
    }
    __syncwarp();
    if (lane == 0) buf[i] = (static_cast<uint64_t>(dist_key(v, IS_IP)) << 32) | ps;
    __syncwarp();
  }
  // the first k by (exact key, position), best first, padded
  for (int i = lane; i < m; i += 32) {
    const uint64_t v = buf[i];
    const int r = rank_of(v, m);
    if (r < k) {
      const size_t o = (size_t)q * k + r;
      D[o] = key_dist(static_cast<uint32_t>(v >> 32), IS_IP);
      I[o] = ids[static_cast<uint32_t>(v)];
      if (P) P[o] = static_cast<uint32_t>(v);
    }
  }
  for (int r = m + lane; r < k; r += 32) {
    const size_t o = (size_t)q * k + r;
    D[o] = IS_IP ? -INFINITY : INFINITY;
    I[o] = -1;
    if (P) P[o] = -1;
  }
}

// Exact top-k of one query from its n composites (key << 32 | position):
// block radix select of the k-th, compaction, bitonic sort of the winners,
// then (distance, id, position) rows with -1 / worst padding.  All threads of
// the CTA call it; win holds >= pow2(k) entries.
template <bool IS_IP>
__device__ void block_select_write(const uint64_t* comp, int nn, int k, int q, uint64_t* win, int* count,
                                   uint32_t* hist, uint32_t* sel, const int64_t* __restrict__ ids,
                                   float* __restrict__ D, int64_t* __restrict__ I, int64_t* __restrict__ P) {
  const int tid = threadIdx.x;
  if (tid == 0) *count = 0;
  __syncthreads();
  int nw;
  if (nn <= k) {
    for (int i = tid; i < nn; i += blockDim.x) win[i] = comp[i];
    nw = nn;
  } else {
    const uint64_t kth = block_kth([&](int e) { return comp[e]; }, nn, (uint32_t)k, hist, sel);
    for (int i = tid; i < nn; i += blockDim.x)
      if (comp[i] <= kth) win[atomicAdd(count, 1)] = comp[i];
    __syncthreads();
    nw = *count;
  }
  int P2 = 1;
  while (P2 < nw) P2 <<= 1;
  for (int i = nw + tid; i < P2; i += blockDim.x) win[i] = ~0ull;
  __syncthreads();
  for (int size = 2; size <= P2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < P2 / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const uint64_t a = win[lo], b = win[hi];
        if ((a > b) == asc) {
          win[lo] = b;
          win[hi] = a;
        }
      }
      __syncthreads();
    }
  }
  for (int r = tid; r < k; r += blockDim.x) {
    const size_t o = (size_t)q * k + r;
    const uint64_t w = r < nw ? win[r] : ~0ull;
    if (w == ~0ull) {
      D[o] = IS_IP ? -INFINITY : INFINITY;
      I[o] = -1;
      if (P) P[o] = -1;
    } else {
      const uint32_t ps = static_cast<uint32_t>(w);
      D[o] = key_dist(static_cast<uint32_t>(w >> 32), IS_IP);
      I[o] = ids[ps];
      if (P) P[o] = ps;
    }
  }
  __syncthreads();
}

// Exact composites of the first `nslots` failed queries (slot f = failed
// query f), their rows split over the whole grid: a few uncertified queries
// no longer scan the base with one CTA each (1M rows: ~25 ms per query).
// fallback_select_kernel selects for those slots; fallback_kernel takes the
// failed queries past them (whole-base scan per CTA).
template <bool IS_IP>
__global__ void __launch_bounds__(256) fallback_dist_kernel(const int* __restrict__ fail_count,
                                                            const int* __restrict__ fail_list, int nslots,
                                                            const float* __restrict__ q0, const float* __restrict__ q1,
                                                            const float* __restrict__ qnorm, const float* __restrict__ xb,
                                                            const float* __restrict__ xl,
                                                            const float* __restrict__ xnorm, int64_t n, int dp,
                                                            uint64_t* __restrict__ scratch) {
  const int nf = min(*fail_count, nslots);
  if (nf == 0) return;
  const int R = max(1, (int)gridDim.x / nf);  // row ranges per failed query
  const int64_t span = (n + R - 1) / R;
  for (int w = blockIdx.x; w < nf * R; w += gridDim.x) {
    const int f = w / R;
    const int64_t r0 = (int64_t)(w - f * R) * span, r1 = min(n, r0 + span);
    const int q = fail_list[f];
    const float qn = qnorm[q];
    const float4* qh = reinterpret_cast<const float4*>(q0 + (size_t)q * dp);
    const float4* ql = q1 ? reinterpret_cast<const float4*>(q1 + (size_t)q * dp) : nullptr;
    uint64_t* comp = scratch + (size_t)f * n;
    for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {  // the same values as fallback_kernel
      const float acc = thread_exact_dot(qh, ql, reinterpret_cast<const float4*>(xb + (size_t)r * dp),
                                         xl ? reinterpret_cast<const float4*>(xl + (size_t)r * dp) : nullptr, dp);
      float v = acc;
      if (!IS_IP) {
        v = fmaf(-2.f, acc, qn + xnorm[r]);
        v = (v <= 0.f) ? 0.f : v;
      }
      comp[r] = (static_cast<uint64_t>(dist_key(v, IS_IP)) << 32) | static_cast<uint32_t>(r);
    }
  }
}

// Selection for the slots fallback_dist_kernel filled: one 1024-thread CTA
// per failed query (the radix passes over n composites are latency-bound).
template <bool IS_IP>
__global__ void __launch_bounds__(1024) fallback_select_kernel(const int* __restrict__ fail_count,
                                                               const int* __restrict__ fail_list, int nslots, int64_t n,
                                                               int k, const int64_t* __restrict__ ids,
                                                               float* __restrict__ D, int64_t* __restrict__ I,
                                                               int64_t* __restrict__ P, const uint64_t* __restrict__ scratch) {
  extern __shared__ uint64_t win[];
  __shared__ int count;
  __shared__ uint32_t hist[256], sel[8];
  const int nf = min(*fail_count, nslots);
  for (int f = blockIdx.x; f < nf; f += gridDim.x)
    block_select_write<IS_IP>(scratch + (size_t)f * n, (int)n, k, fail_list[f], win, &count, hist, sel, ids, D, I, P);
}

// Exact fallback, on the device: CTA b takes failed queries b, b+grid, ...;
// exact composites of every row into its scratch slot, block radix select of
// the k-th, bitonic sort of the winners.  Launched after every MODE 4 merge
// (it exits at once when nothing failed), so a search never syncs the host.
template <bool IS_IP>
__global__ void __launch_bounds__(256) fallback_kernel(const int* __restrict__ fail_count,
                                                       const int* __restrict__ fail_list, const float* __restrict__ q0,
                                                       const float* __restrict__ q1, const float* __restrict__ qnorm,
                                                       const float* __restrict__ xb, const float* __restrict__ xl,
                                                       const float* __restrict__ xnorm, int64_t n, int dp, int k,
                                                       const int64_t* __restrict__ ids, float* __restrict__ D,
                                                       int64_t* __restrict__ I, int64_t* __restrict__ P,
                                                       uint64_t* __restrict__ scratch) {
  extern __shared__ uint64_t win[];
  __shared__ int count;
  __shared__ uint32_t hist[256], sel[8];
  const int tid = threadIdx.x;
  const int nf = *fail_count;
  uint64_t* comp = scratch + (size_t)blockIdx.x * n;
  // failed queries f < grid were answered by fallback_dist/select_kernel
  for (int f = blockIdx.x + gridDim.x; f < nf; f += gridDim.x) {
    const int q = fail_list[f];
    const float qn = qnorm[q];
    const float4* qh = reinterpret_cast<const float4*>(q0 + (size_t)q * dp);
    const float4* ql = q1 ? reinterpret_cast<const float4*>(q1 + (size_t)q * dp) : nullptr;
    for (int64_t r = tid; r < n; r += blockDim.x) {  // a thread per row, the merge's summation order
      const float acc = thread_exact_dot(qh, ql, reinterpret_cast<const float4*>(xb + (size_t)r * dp),
                                         xl ? reinterpret_cast<const float4*>(xl + (size_t)r * dp) : nullptr, dp);
      float v = acc;
      if (!IS_IP) {
        v = fmaf(-2.f, acc, qn + xnorm[r]);
        v = (v <= 0.f) ? 0.f : v;
      }
      comp[r] = (static_cast<uint64_t>(dist_key(v, IS_IP)) << 32) | static_cast<uint32_t>(r);
    }
    block_select_write<IS_IP>(comp, (int)n, k, q, win, &count, hist, sel, ids, D, I, P);
    __syncthreads();
  }
}

// ------------------------------------------------------------ direct path (nq < blas_threshold)
// Reference flat.py:58-62 sends batches below config.blas_threshold (20,
// config.py:9) to flat_search (flat.py:76-91): per-pair DIRECT distances
// (pairwise -> dist_one, _ckernels.pyx:49-57: L2 sum (q - x)^2, IP sum q x)
// ranked by topk_rows.  Here: one warp per stored row evaluates every query
// of the group, accumulating in fp64 from the stored operands (fp32: hi + lo
// == x exactly; fold: -2x scaled back) and rounding once to fp32 -- a self
// distance is exactly +0.0 -- then one CTA per query selects the top-k.
template <int MODE>
__device__ __forceinline__ double stored_val(const void* a, const void* b, size_t off) {
  if (MODE == 0) return (double)(static_cast<const float*>(a)[off] + static_cast<const float*>(b)[off]);
  if (MODE == 4) return (double)static_cast<const float*>(a)[off];
  if (MODE == 1) return (double)__half2float(static_cast<const __half*>(a)[off]);
  return (double)__bfloat162float(static_cast<const __nv_bfloat16*>(a)[off]);
}

// Direct distances, a warp per stored row (d <= 256, the row in registers),
// the staged queries in smem as doubles, 8 queries per reduction: a
// transposing butterfly (xor 16 / 8 / 4 exchange halves of the 8 partial sums,
// xor 2 / 1 finish) costs 9 double shuffles instead of 40 -- and adds the
// same pairs in the same order as direct_dist_kernel, so the values are
// bit-identical to it.
template <int MODE>
__global__ void __launch_bounds__(256) direct_dist_warp8_kernel(const void* __restrict__ q0,
                                                                const void* __restrict__ q1, int nq,
                                                                const void* __restrict__ s0,
                                                                const void* __restrict__ s1, int64_t n, int d, int dp,
                                                                int is_ip, int fold, uint64_t* __restrict__ comp) {
  extern __shared__ double qs[];  // [nq][d]
  for (int i = threadIdx.x; i < nq * d; i += blockDim.x) {
    const int qi = i / d, c = i - qi * d;
    qs[i] = stored_val<MODE>(q0, q1, (size_t)qi * dp + c);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  // grid-stride over rows: the query staging above is paid once per CTA
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n;
       r += (int64_t)gridDim.x * (blockDim.x >> 5)) {
  constexpr int XR = 8;
  double xv[XR];
#pragma unroll
  for (int i = 0; i < XR; ++i) {
    const int c = lane + 32 * i;
    xv[i] = c < d ? stored_val<MODE>(s0, s1, (size_t)r * dp + c) * (fold ? -0.5 : 1.0) : 0.0;  // -2x folded (exact)
  }
  for (int qb = 0; qb < nq; qb += 8) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double acc = 0.0;
      if (qb + j < nq) {
        const double* qrow = qs + (size_t)(qb + j) * d;
#pragma unroll
        for (int i = 0; i < XR; ++i) {
          const int c = lane + 32 * i;
          if (c < d) {
            const double qv = qrow[c];
            if (is_ip) acc = fma(qv, xv[i], acc);
            else {
              const double t = qv - xv[i];
              acc = fma(t, t, acc);
            }
          }
        }
      }
      v[j] = acc;
    }
    // xor 16: lanes without bit 4 keep sums 0-3, lanes with it 4-7
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool hi = lane & 16;
      const double send = hi ? v[j] : v[j + 4], keep = hi ? v[j + 4] : v[j];
      v[j] = keep + __shfl_xor_sync(FULLMASK, send, 16);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {  // xor 8
      const bool hi = lane & 8;
      const double send = hi ? v[j] : v[j + 2], keep = hi ? v[j + 2] : v[j];
      v[j] = keep + __shfl_xor_sync(FULLMASK, send, 8);
    }
    {  // xor 4
      const bool hi = lane & 4;
      const double send = hi ? v[0] : v[1], keep = hi ? v[1] : v[0];
      v[0] = keep + __shfl_xor_sync(FULLMASK, send, 4);
    }
    v[0] += __shfl_xor_sync(FULLMASK, v[0], 2);
    v[0] += __shfl_xor_sync(FULLMASK, v[0], 1);
    const int qi = qb + ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
    if ((lane & 3) == 0 && qi < nq)
      comp[(size_t)qi * n + r] =
          (static_cast<uint64_t>(dist_key(static_cast<float>(v[0]), is_ip != 0)) << 32) | static_cast<uint32_t>(r);
  }
  }
}

template <int MODE>
__global__ void __launch_bounds__(256) direct_dist_kernel(const void* __restrict__ q0, const void* __restrict__ q1,
                                                          int nq, const void* __restrict__ s0,
                                                          const void* __restrict__ s1, int64_t n, int d, int dp,
                                                          int is_ip, int fold, uint64_t* __restrict__ comp) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  constexpr int XR = 8;  // stored row cached in registers for d <= 256
  double xv[XR];
#pragma unroll
  for (int i = 0; i < XR; ++i) {
    const int c = lane + 32 * i;
    xv[i] = c < d ? stored_val<MODE>(s0, s1, (size_t)r * dp + c) * (fold ? -0.5 : 1.0) : 0.0;  // -2x folded (exact)
  }
  for (int qi = 0; qi < nq; ++qi) {
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < XR; ++i) {
      const int c = lane + 32 * i;
      if (c < d) {
        const double qv = stored_val<MODE>(q0, q1, (size_t)qi * dp + c);
        if (is_ip) acc = fma(qv, xv[i], acc);
        else {
          const double t = qv - xv[i];
          acc = fma(t, t, acc);
        }
      }
    }
    for (int c = lane + 32 * XR; c < d; c += 32) {
      const double qv = stored_val<MODE>(q0, q1, (size_t)qi * dp + c);
      const double x = stored_val<MODE>(s0, s1, (size_t)r * dp + c) * (fold ? -0.5 : 1.0);
      if (is_ip) acc = fma(qv, x, acc);
      else {
        const double t = qv - x;
        acc = fma(t, t, acc);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(FULLMASK, acc, off);
    if (lane == 0) {
      const float v = static_cast<float>(acc);
      comp[(size_t)qi * n + r] = (static_cast<uint64_t>(dist_key(v, is_ip != 0)) << 32) | static_cast<uint32_t>(r);
    }
  }
}

// Direct path, first selection level: the exact k smallest composites of
// each `chunk`-row slice of one query's row (grid: slices x queries), padded
// with ~0 to k -- the per-query selection then runs over slices x k entries
// instead of every row (one CTA over 1M composites took milliseconds).
__global__ void __launch_bounds__(256) direct_chunk_topk_kernel(const uint64_t* __restrict__ comp, int64_t n,
                                                                int chunk, int k, uint64_t* __restrict__ out) {
  __shared__ uint32_t hist[256], sel[8];
  __shared__ int cnt_out;
  const int64_t c0 = (int64_t)blockIdx.x * chunk;
  const int64_t left = n - c0;
  const int cnt = left < (int64_t)chunk ? (int)left : chunk;
  const uint64_t* src = comp + (size_t)blockIdx.y * n + c0;
  uint64_t* dst = out + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * k;
  if (threadIdx.x == 0) cnt_out = 0;
  __syncthreads();
  uint64_t kth = ~0ull;  // valid composites are < ~0 (keys < 0xFFFFFFFF)
  if (cnt > k) kth = block_kth([&](int e) { return __ldg(src + e); }, cnt, (uint32_t)k, hist, sel);
  for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
    const uint64_t v = __ldg(src + e);
    if (v <= kth) dst[atomicAdd(&cnt_out, 1)] = v;
  }
  __syncthreads();
  for (int i = cnt_out + threadIdx.x; i < k; i += blockDim.x) dst[i] = ~0ull;
}

template <bool IS_IP>
__global__ void __launch_bounds__(256) direct_select_kernel(const uint64_t* __restrict__ comp, int64_t n, int q0,
                                                            int k, const int64_t* __restrict__ ids,
                                                            float* __restrict__ D, int64_t* __restrict__ I,
                                                            int64_t* __restrict__ P) {
  extern __shared__ uint64_t win[];
  __shared__ int count;
  __shared__ uint32_t hist[256], sel[8];
  block_select_write<IS_IP>(comp + (size_t)blockIdx.x * n, (int)n, k, q0 + blockIdx.x, win, &count, hist, sel, ids,
                            D, I, P);
}

// ------------------------------------------------------------ conversions
__device__ __forceinline__ float load_elem(const void* x, int dtype, size_t i) {
  if (dtype == 0) return static_cast<const float*>(x)[i];
  if (dtype == 1) return __half2float(static_cast<const __half*>(x)[i]);
  return __bfloat162float(static_cast<const __nv_bfloat16*>(x)[i]);
}
__device__ __forceinline__ float tf32_rna(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}

// One warp per row: convert n rows of `x` (row-major n x d, dtype in_dtype)
// into the stored layout at rows [row0, row0+n) of out0/out1 (dp columns,
// zero padded), and write fp32 squared norms of the STORED values.
// fold (MODE 2 storage, FOLD kernels): 1 = base row, stored as -2x with the
// row's squared norm split exactly into 3 bf16 at columns d..d+2; 2 = query
// row, with 1.0 at columns d..d+2.  Then <query, base> = xn - 2 q.x.
template <int MODE>
__global__ void prep_rows_kernel(const void* __restrict__ x, int in_dtype, int64_t n, int d, int dp,
                                 void* __restrict__ out0, void* __restrict__ out1, float* __restrict__ norms,
                                 int64_t row0, int fold, unsigned int* __restrict__ inexact = nullptr) {
  const int64_t rloc = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (rloc >= n) return;
  const int64_t orow = row0 + rloc;
  double acc = 0.0;
  for (int c = lane; c < dp; c += 32) {
    const float v = c < d ? load_elem(x, in_dtype, (size_t)rloc * d + c) : 0.f;
    if (MODE == 0) {
      const float hi = tf32_rna(v);
      const float lo = v - hi;  // exact: x == hi + lo
      if (inexact != nullptr && lo != 0.f) *inexact = 1u;  // the value needs more than one tf32 term
      static_cast<float*>(out0)[(size_t)orow * dp + c] = hi;
      static_cast<float*>(out1)[(size_t)orow * dp + c] = lo;
      acc += (double)v * (double)v;
    } else if (MODE == 4) {  // raw fp32
      static_cast<float*>(out0)[(size_t)orow * dp + c] = v;
      acc += (double)v * (double)v;
    } else if (MODE == 1) {
      const __half h = __float2half_rn(v);
      static_cast<__half*>(out0)[(size_t)orow * dp + c] = h;
      const float vr = __half2float(h);
      acc += (double)vr * (double)vr;
    } else {
      const __nv_bfloat16 h = __float2bfloat16_rn(v);
      const float vr = __bfloat162float(h);
      if (!(fold && c >= d && c < d + 3))
        static_cast<__nv_bfloat16*>(out0)[(size_t)orow * dp + c] = (fold == 1) ? __float2bfloat16_rn(-2.f * vr) : h;
      acc += (double)vr * (double)vr;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, off);
  const float xn = static_cast<float>(acc);
  if (lane == 0 && norms != nullptr) norms[orow] = xn;
  if (MODE == 2 && fold && lane < 3) {
    // xn = h0 + h1 + h2 exactly: each bf16 takes the next 8 significant bits
    // (a non-finite norm goes whole into h0: inf - inf would make h1 NaN)
    float part = xn, hv = 0.f;
    for (int i = 0; i <= lane; ++i) {
      hv = __bfloat162float(__float2bfloat16_rn(part));
      part = isfinite(part) ? part - hv : 0.f;  // exact (Sterbenz / representable remainder)
    }
    static_cast<__nv_bfloat16*>(out0)[(size_t)orow * dp + d + lane] = __float2bfloat16_rn(fold == 1 ? hv : 1.f);
  }
}

// Stored rows (by position) back to float32 n x d.
template <int MODE>
__global__ void reconstruct_kernel(const void* __restrict__ s0, const void* __restrict__ s1, int dp, int d,
                                   const int64_t* __restrict__ positions, int64_t n, float* __restrict__ out,
                                   float scale) {
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const int64_t r = positions[i];
  for (int c = lane; c < d; c += 32) {
    float v;
    if (MODE == 0)
      v = static_cast<const float*>(s0)[(size_t)r * dp + c] + static_cast<const float*>(s1)[(size_t)r * dp + c];
    else if (MODE == 4)
      v = static_cast<const float*>(s0)[(size_t)r * dp + c];
    else if (MODE == 1)
      v = __half2float(static_cast<const __half*>(s0)[(size_t)r * dp + c]);
    else
      v = __bfloat162float(static_cast<const __nv_bfloat16*>(s0)[(size_t)r * dp + c]);
    out[(size_t)i * d + c] = v * scale;  // scale -0.5 undoes the folded -2x (exact)
  }
}

// Gather rows (by position) of a row-major [*, row_bytes] buffer.
__global__ void gather_rows_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, size_t row_bytes,
                                   const int64_t* __restrict__ keep, int64_t n) {
  const int64_t i = blockIdx.x;
  if (i >= n) return;
  const uint8_t* s = src + (size_t)keep[i] * row_bytes;
  uint8_t* o = dst + (size_t)i * row_bytes;
  for (size_t b = threadIdx.x * 4; b < row_bytes; b += blockDim.x * 4)
    *reinterpret_cast<uint32_t*>(o + b) = *reinterpret_cast<const uint32_t*>(s + b);
}

// Running max of non-negative float norms (uint compare == float compare for
// x >= 0; a NaN norm wins, which disables the fast filter -- still exact).
__global__ void norm_max_kernel(const float* __restrict__ norms, int64_t n, unsigned int* out) {
  unsigned int m = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, __float_as_uint(fabsf(norms[i])) | (isnan(norms[i]) ? 0x7FC00000u : 0u));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, off));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

__global__ void iota_ids_kernel(int64_t* ids, int64_t start, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) ids[i] = start + i;
}

__global__ void fill_sentinel_kernel(float* D, int64_t* I, int64_t* P, size_t n, float v) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    D[i] = v;
    I[i] = -1;
    if (P) P[i] = -1;
  }
}

// ------------------------------------------------------------ range search
// Exact direct distance of every candidate (reference range search goes
// through pairwise_distances -> the direct per-pair loops, flat.py:121-144,
// _ckernels.pyx dist_one): L2 sum (q - x)^2, IP sum q x, accumulated in fp64
// and rounded once to fp32, from the STORED operands (fp32: hi + lo == x
// exactly; fold: -2x scaled back).  Survivors (<= radius, >= for IP) get
// sort keys: key_id = user id, key_rd = (row << 32) | monotone(best-first value).
template <int MODE>
__global__ void range_exact_kernel(const unsigned long long* __restrict__ cand, unsigned long long n,
                                   const void* __restrict__ q0, const void* __restrict__ q1, const void* __restrict__ s0,
                                   const void* __restrict__ s1, int d, int dp, int is_ip, int fold, float radius,
                                   const int64_t* __restrict__ ids, float* __restrict__ dist,
                                   unsigned long long* __restrict__ key_id, unsigned long long* __restrict__ key_rd,
                                   unsigned int* __restrict__ keep, unsigned int* __restrict__ row_count) {
  const unsigned long long i = (unsigned long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const unsigned long long e = cand[i];
  const uint32_t row = static_cast<uint32_t>(e >> 32), pos = static_cast<uint32_t>(e);
  auto val = [&](const void* a, const void* b, size_t off) -> double {
    if (MODE == 0) return (double)(static_cast<const float*>(a)[off] + static_cast<const float*>(b)[off]);
    if (MODE == 4) return (double)static_cast<const float*>(a)[off];
    if (MODE == 1) return (double)__half2float(static_cast<const __half*>(a)[off]);
    return (double)__bfloat162float(static_cast<const __nv_bfloat16*>(a)[off]);
  };
  double acc = 0.0;
  for (int c = lane; c < d; c += 32) {
    const double qv = val(q0, q1, (size_t)row * dp + c);
    double xv = val(s0, s1, (size_t)pos * dp + c);
    if (fold) xv *= -0.5;  // stored -2x (exact)
    if (is_ip) acc = fma(qv, xv, acc);
    else {
      const double t = qv - xv;
      acc = fma(t, t, acc);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(FULLMASK, acc, off);
  if (lane == 0) {
    const float v = static_cast<float>(acc);
    const bool in = is_ip ? (v >= radius) : (v <= radius);  // flat.py:134 (NaN never matches)
    keep[i] = in ? 1u : 0u;
    dist[i] = v;
    key_id[i] = static_cast<unsigned long long>(ids[pos]);
    key_rd[i] = (static_cast<unsigned long long>(row) << 32) | dist_key(v, is_ip != 0);
    if (in) atomicAdd(row_count + row, 1u);
  }
}

// ------------------------------------------------------------ k-means assignment (fp64)
// Reference quantize.py:38-62 (_assign): nearest centroid in fp64,
// L2: argmin(cnorm - 2 ip), IP: argmax(ip), first index wins ties; the error
// is max(xnorm + cnorm[a] - 2 ip[a], 0).  One warp per row evaluates `kc`
// candidate centroids (the fp32 GPU shortlist, or every centroid) in fp64.
// With `approx` (the shortlist's fp32 distances, best first) a row is flagged
// uncertain when the shortlist's first and last values are closer than the
// fp32 error bound `margin * (xnorm + cmax)`: the true best might then lie
// outside the shortlist, and the caller rescores that row over all centroids.
__global__ void kmeans_rescore_kernel(const float* __restrict__ x, int64_t n, int d, const double* __restrict__ c,
                                      const double* __restrict__ cnorm, int64_t nc, const int64_t* __restrict__ cand,
                                      int kc, int by_ip, const float* __restrict__ approx, double margin, double cmax,
                                      int64_t* __restrict__ assign, double* __restrict__ err,
                                      int* __restrict__ uncertain) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const float* xr = x + (size_t)row * d;
  double xn = 0.0;
  for (int i = lane; i < d; i += 32) xn += (double)xr[i] * (double)xr[i];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) xn += __shfl_xor_sync(FULLMASK, xn, off);
  int64_t best = -1;
  double bval = 0.0, bip = 0.0;
  for (int j = 0; j < kc; ++j) {
    const int64_t cj = cand ? cand[(size_t)row * kc + j] : j;
    if (cj < 0 || cj >= nc) continue;
    const double* cr = c + (size_t)cj * d;
    double ip = 0.0;
    for (int i = lane; i < d; i += 32) ip = fma((double)xr[i], cr[i], ip);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ip += __shfl_xor_sync(FULLMASK, ip, off);
    const double v = by_ip ? ip : cnorm[cj] - 2.0 * ip;
    const bool better = best < 0 || (by_ip ? (v > bval || (v == bval && cj < best))
                                           : (v < bval || (v == bval && cj < best)));
    if (better) {
      best = cj;
      bval = v;
      bip = ip;
    }
  }
  if (lane == 0) {
    assign[row] = best;
    const double e = best >= 0 ? xn + cnorm[best] - 2.0 * bip : 0.0;
    err[row] = e > 0.0 ? e : 0.0;  // np.maximum(err, 0.0)
    if (uncertain) {
      int u = 0;
      if (approx && kc > 1) {
        const float a0 = approx[(size_t)row * kc], a1 = approx[(size_t)row * kc + kc - 1];
        const double gap = by_ip ? (double)a0 - (double)a1 : (double)a1 - (double)a0;
        u = !(gap > margin * (xn + cmax));  // NaN-safe: NaN gap -> uncertain
      } else if (approx) {
        u = 1;  // a one-entry shortlist cannot be certified
      }
      uncertain[row] = u;
    }
  }
}

}  // namespace fk
