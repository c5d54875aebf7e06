// The hot kernel of the B200-native exact flat k-NN engine (and the key /
// queue / selection helpers it shares with the merge kernels).
//
//   prep_rows_kernel   : f32/f16/bf16 rows -> stored operand layout
//                        (3xTF32 hi/lo split or RNE fp16/bf16) + fp32 norms.
//                        Base side = FlatIndex._add + norms einsum
//                        (reference flat.py:28-32); query side = the qn einsum
//                        of flat_search_blas (flat.py:110).
//   fused_knn_kernel   : persistent, warp-specialised tcgen05 GEMM
//                        (TMA -> smem -> tcgen05.mma -> TMEM) with the L2/IP
//                        epilogue (flat.py:108-114) and the per-row top-k
//                        selection (core.py:205-236) fused behind it, so the
//                        nq x nb distance matrix never reaches HBM.
//   merge_kernel       : split-N partial lists -> final top-k, position -> id
//                        (flat.py:68-73).
//   shard_merge_kernel : per-shard top-k lists -> single-index order (8(e)).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "sm100.cuh"

// FK_DEV=1 (libflatknn_dev.so, scripts only) compiles in the clock64 timeline
// trace and the bottleneck-experiment flags; the product build has neither.
#ifndef FK_DEV
#define FK_DEV 0
#endif
// experiment switch (variant builds): 1 = unrolled 4-MMA issue for full
// K-chunks (A/B on cfg2: MMA-only 2.09 vs 2.19 ms but the full kernel 3.68 vs
// 3.44 ms -- off)
#ifndef FK_LD_X64  // 64-column TMEM loads in the two-group epilogue (0: two 32-column loads)
#define FK_LD_X64 1
#endif
#ifndef FK_LD_X128  // one 128-column TMEM load in the one-group epilogue (experiment)
#define FK_LD_X128 0
#endif
#ifndef FK_ISSUER_FAST
#define FK_ISSUER_FAST 0
#endif

namespace fk {

constexpr int BM = 128;                        // queries per tile (TMEM lanes)
constexpr int BN = 128;                        // base rows per tile (TMEM columns)
constexpr uint32_t CHUNK_BYTES = 128u * 128u;  // one 128-row x 128-byte K-chunk
constexpr int EPI_WARP0 = 4;                   // warps 0-3: producer, MMA, TMEM alloc, spare

// ------------------------------------------------------------ key helpers
// Order-preserving float32 -> uint32 (core.py:193-197): NaN above +inf,
// -0.0 below +0.0.  Comparing (key, position) reproduces the reference's
// 64-bit composite sort key (core.py:219).
__device__ __forceinline__ uint32_t monotone(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
// Sort key of a reference distance value (IP ranks -value, core.py:217).
// A NaN is ranked as the positive quiet NaN a NaN input carries (np.nan):
// worst for L2 (above +inf), best for IP (its negation has the sign bit set).
// Canonical, so it also stays below the all-ones "empty slot" key.
__device__ __forceinline__ uint32_t dist_key(float v, bool ip) {
  uint32_t b = (v != v) ? 0x7FC00000u : __float_as_uint(v);
  if (ip) b ^= 0x80000000u;  // -v as a bit operation (neg.f32 of a NaN is unspecified)
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
// Reported distance of a key (IP: the inner product again).
__device__ __forceinline__ float key_dist(uint32_t k, bool ip) {
  uint32_t b = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
  if (ip) b ^= 0x80000000u;
  return __uint_as_float(b);
}
__device__ __forceinline__ float unmonotone(uint32_t k) {
  const uint32_t b = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
  return __uint_as_float(b);
}

struct SearchParams {
  const float* qnorm;  // [nq]
  const float* xnorm;  // [cap], cap padded to BN
  const float* xn_max; // device scalar: max stored norm (bounds the filter's rounding margin)
  uint32_t* part_key;  // [nq][S][k]
  uint32_t* part_pos;  // [nq][S][k]
  uint32_t* thr_key;   // [nq] shared per-query bound: min over units of their k-th key
  int* part_cnt;       // [nq][S_tot] valid entries per partial list (large-k mode)
  uint64_t* cbuf;      // large-k candidate buffers [grid][EPI][32][cap] of (key<<32 | pos)
  int cap;             // large-k buffer capacity per row
  float* dbg_ip;       // optional raw inner products [nq][nb] (debug)
  const void* qa0;     // query operand rows [nq][dp] (hi / f16 / bf16) -- A_TMEM mode
  const void* qa1;     // lo part (fp32 mode)
  int nq, nb, k;
  int num_m, n_tiles, chunk_tiles, S, num_units;
  int probe_tiles;  // > 0: chunk 0 is a short probe chunk [0, probe_tiles), the others follow it
  int num_kb;      // padded d / elements-per-128B-chunk
  int a_mode;      // 0: queries in TMEM, 1: resident in smem, 2: streamed per stage, 3: split (below)
  int a_kt;        // a_mode 3: K-chunks [0, a_kt) of the queries in TMEM, the rest resident in smem
  int stages;      // B (and streamed A) pipeline depth
  int xn_slots;    // base-norm tile ring depth (prefetched by the producer)
  unsigned long long* trace;  // debug timeline (CTA 0): [tile][16] clock64 stamps
  int n_issuers;   // MMA-issuing threads (warps 1 and 3)
  int n_producers; // TMA producer threads: 1 (warp 0 serves every ring) or one per issuer ring (warps 0, 2)
  int acc_stages;  // TMEM accumulator buffers (2..4); the query operand (a_mode 0) follows them
  int kk_last;     // MMA K-steps in the last 128-byte K-chunk (trims the zero padding of d)
  int b_policy;    // L2 eviction policy of the streamed base tiles (0 first, 1 normal, 2 last)
  int cluster;     // 1, or 2: CTA pairs share each base tile (each loads half, TMA multicast to both)
  int num_mu;      // query-tile units per chunk: num_m, or ceil(num_m / 2) pairs in cluster mode
  int bn;          // base rows per tile (template TBN of the launched kernel)
  const void* xbase;  // stored base rows (MODE 4: raw fp32, read for exact rescoring)
  // MODE 4 band filter: lists keep k (= p.k) slots, the filter/publish bound
  // is (own kfinal-th tf32 value + band); a row whose queue dropped an entry
  // inside that band is flagged in rflag (the merge then uses the fallback)
  int kfinal;
  // {base, queries}: nonzero when some value needs its lo part; when both
  // are zero the 1-pass tf32 products are exact and the band collapses
  const unsigned int* inexact;
  // MODE 5: 2^-s of each query row's fp16 scale [nq] and of the base's
  // (device scalar); NaN marks an unusable scale (row -> exact fallback)
  const float* qinv;
  const float* xinv;
  float band_l2;  // F1P rounding-band coefficient of |q| max|x| (L2; IP half)
  int pub_mask;  // publish the own bound / fetch the shared one every pub_mask+1 own tiles
  // MODE 4: per-query running union of the finished units' best k' tf32 keys
  // (lock-protected), so the shared bound tightens towards the global k-th
  unsigned int* glock;  // [nq]
  uint32_t* gkeys;      // [nq][32]
  unsigned int* rflag;
  // F1P: entries inside the band that a full register queue had to drop go
  // to a per-query overflow list [nq][ovf_cap] (count may exceed the cap:
  // the row is then flagged for the exact fallback)
  uint32_t* ovf_key;
  uint32_t* ovf_pos;
  unsigned int* ovf_cnt;
  int ovf_cap;
  // range search (KQ == -1): every (row, position) whose fast-filter value
  // passes the conservative radius bound is appended to rcand (the exact
  // direct distance and the radius test follow in range_exact_kernel)
  float radius;
  unsigned long long* rcand;  // [rcap] (row << 32 | position)
  unsigned long long* rcount; // device counter (may exceed rcap: caller grows and reruns)
  unsigned long long rcap;
  int dbg_flags;   // bottleneck experiments (FK_DEBUG_FLAGS): 1 = epilogue skips TMEM loads + compute,
                   // 2 = producer skips TMA, 4 = no slow path, 8 = TMEM loads without the filter
};

// Base tiles [t0, t1) of N-chunk `chunk`.  With a probe chunk, chunk 0 is
// short so the first units of every query finish early and publish a bound
// (the running union) before the long chunks have inserted much.
__device__ __forceinline__ void chunk_range(const SearchParams& p, int chunk, int& t0, int& t1) {
  if (p.probe_tiles > 0) {
    t0 = chunk == 0 ? 0 : p.probe_tiles + (chunk - 1) * p.chunk_tiles;
    t1 = chunk == 0 ? p.probe_tiles : t0 + p.chunk_tiles;
  } else {
    t0 = chunk * p.chunk_tiles;
    t1 = t0 + p.chunk_tiles;
  }
  t1 = min(t1, p.n_tiles);
}

// ------------------------------------------------------------ register queue
// Sorted ascending (worst at KQ-1).  Slots [0, KQ-k) hold phantom key 0 which
// nothing displaces, so a runtime k <= KQ needs only static register indices.
// Ties: a new candidate always has a larger position than every queued one
// (columns are streamed in order), so strict `<` keeps the smaller position
// first -- the reference's (value, column) order.
template <int KQ>
__device__ __forceinline__ void queue_insert(uint32_t (&keys)[KQ], uint32_t (&pos)[KQ], uint32_t key,
                                             uint32_t p) {
  if (key < keys[KQ - 1]) {
#pragma unroll
    for (int i = KQ - 1; i > 0; --i) {
      const bool shift = key < keys[i - 1];
      const uint32_t nk = shift ? keys[i - 1] : key;
      const uint32_t np = shift ? pos[i - 1] : p;
      if (key < keys[i]) {
        keys[i] = nk;
        pos[i] = np;
      }
    }
    if (key < keys[0]) {
      keys[0] = key;
      pos[0] = p;
    }
  }
}

// a[idx] for a runtime idx without dynamic register indexing (which would
// move the whole array to local memory): a log2(N)-deep tree of selects
// (N a power of two), short latency on the insertion path
template <int N>
__device__ __forceinline__ uint32_t select_static(const uint32_t (&a)[N], int idx) {
  if constexpr (N == 1) {
    return a[0];
  } else {
    uint32_t t[N / 2];
#pragma unroll
    for (int i = 0; i < N / 2; ++i) t[i] = (idx & 1) ? a[2 * i + 1] : a[2 * i];
    return select_static<N / 2>(t, idx >> 1);
  }
}

// Sort a bitonic sequence of 32 keys ascending (half-cleaner network, static
// indices only: the array stays in registers).
__device__ __forceinline__ void bitonic_merge32(uint32_t (&x)[32]) {
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if ((i & s) == 0) {
        const uint32_t a = x[i], b = x[i + s];
        x[i] = min(a, b);
        x[i + s] = max(a, b);
      }
    }
  }
}

// ------------------------------------------------------------ exact selection (large k)
constexpr unsigned FULLMASK = 0xFFFFFFFFu;

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const uint64_t o = __shfl_xor_sync(FULLMASK, v, off);
    v = o < v ? o : v;
  }
  return v;
}

// Exact k-th smallest (1-based) of cnt 64-bit composites (key<<32 | position)
// read through load(e): warp-cooperative MSB-first 8-bit radix select with a
// 256-bin smem histogram; stops as soon as the k-th is alone in its bucket.
template <class Load>
__device__ uint64_t warp_kth(Load load, int cnt, uint32_t k, uint32_t* hist) {
  const int lane = threadIdx.x & 31;
  uint64_t prefix = 0;
  uint32_t need = k;
#pragma unroll 1
  for (int shift = 56; shift >= 0; shift -= 8) {
    const uint64_t hmask = (shift == 56) ? 0ull : (~0ull << (shift + 8));
    for (int b = lane; b < 256; b += 32) hist[b] = 0;
    __syncwarp();
    for (int e = lane; e < cnt; e += 32) {
      const uint64_t v = load(e);
      if ((v & hmask) == prefix) atomicAdd(&hist[static_cast<uint32_t>(v >> shift) & 255u], 1u);
    }
    __syncwarp();
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
    const unsigned own = __ballot_sync(FULLMASK, excl < need && need <= incl);
    const int src = own ? __ffs(own) - 1 : 31;
    uint32_t bin = 0, before = 0, bcnt = 0;
    if (lane == src) {
      uint32_t run = excl;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (bcnt == 0 && run < need && need <= run + c[i]) {
          bin = lane * 8 + i;
          before = run;
          bcnt = c[i];
        }
        run += c[i];
      }
    }
    bin = __shfl_sync(FULLMASK, bin, src);
    before = __shfl_sync(FULLMASK, before, src);
    bcnt = __shfl_sync(FULLMASK, bcnt, src);
    need -= before;
    prefix |= static_cast<uint64_t>(bin) << shift;
    __syncwarp();
    if (bcnt == 1) {  // the k-th is the only value in its bucket
      const uint64_t m2 = ~0ull << shift;
      uint64_t found = ~0ull;
      for (int e = lane; e < cnt; e += 32) {
        const uint64_t v = load(e);
        if ((v & m2) == prefix) found = v;
      }
      return warp_min_u64(found);
    }
  }
  return prefix;
}

// In-place, order-preserving compaction of buf[0..cnt) to the values <= kth.
__device__ __forceinline__ int warp_compact_le(uint64_t* buf, int cnt, uint64_t kth) {
  const int lane = threadIdx.x & 31;
  int out = 0;
  for (int base = 0; base < cnt; base += 32) {
    const int e = base + lane;
    const uint64_t v = e < cnt ? buf[e] : ~0ull;
    const bool keep = e < cnt && v <= kth;
    const unsigned b = __ballot_sync(FULLMASK, keep);
    __syncwarp();
    if (keep) buf[out + __popc(b & ((1u << lane) - 1u))] = v;
    out += __popc(b);
    __syncwarp();
  }
  return out;
}

// ------------------------------------------------------------ fused kernel
// Work unit = (128-query tile m, N-chunk): the CTA keeps the queries of tile m
// resident (TMEM or smem) and streams the chunk's base tiles through a TMA ring.
//
// Warp roles (1 CTA per SM, persistent):
//   warp 0      TMA producer (one lane): B tiles (and A when not resident)
//   warp 1      MMA issuer (one lane): tcgen05.mma into a double-buffered
//               TMEM accumulator; also bulk-copies the tile's base norms
//   warp 2      TMEM allocator
//   warps 4..   EPI epilogue warps: write the query tile into TMEM (A_TMEM
//               mode), then per accumulator tile: tcgen05.ld -> distance
//               -> NaN-propagating min-tree filter -> rare exact insertion
//               into a per-row register queue.
//
// a_mode 0: queries in TMEM (TS MMA; frees smem, halves smem operand reads)
// a_mode 1: queries resident in smem for the unit
// a_mode 2: queries streamed with every B stage (large d)
// a_mode 3: split -- the first a_kt K-chunks in TMEM (TS MMAs), the rest in
//           smem (SS MMAs): a query operand too large for TMEM beside two
//           accumulators (d = 768 16-bit) keeps two accumulators (no drain of
//           the MMA pipe at every tile)
constexpr int MAX_ACC = 4;      // TMEM accumulator buffers
constexpr int MAX_STAGES = 32;  // smem operand ring  // TMEM accumulator buffers (runtime p.acc_stages); A operand columns follow them

// NaN-propagating min / max over 32 values with 3-input FMNMX (16 instructions).
template <bool MAX>
__device__ __forceinline__ float reduce32(const float (&v)[32]) {
  auto op3 = [](float a, float b, float c) { return MAX ? fmax3_nan(a, b, c) : fmin3_nan(a, b, c); };
  auto op2 = [](float a, float b) { return MAX ? fmax_nan(a, b) : fmin_nan(a, b); };
  float l1[11];
#pragma unroll
  for (int i = 0; i < 10; ++i) l1[i] = op3(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
  l1[10] = op2(v[30], v[31]);
  const float a = op3(l1[0], l1[1], l1[2]);
  const float b = op3(l1[3], l1[4], l1[5]);
  const float c = op3(l1[6], l1[7], l1[8]);
  const float d = op2(l1[9], l1[10]);
  return op2(op3(a, b, c), d);
}

__device__ __forceinline__ float select32(const float (&s)[32], int j) {
  float t16[16], t8[8], t4[4], t2[2];
#pragma unroll
  for (int i = 0; i < 16; ++i) t16[i] = (j & 1) ? s[2 * i + 1] : s[2 * i];
#pragma unroll
  for (int i = 0; i < 8; ++i) t8[i] = (j & 2) ? t16[2 * i + 1] : t16[2 * i];
#pragma unroll
  for (int i = 0; i < 4; ++i) t4[i] = (j & 4) ? t8[2 * i + 1] : t8[2 * i];
#pragma unroll
  for (int i = 0; i < 2; ++i) t2[i] = (j & 8) ? t4[2 * i + 1] : t4[2 * i];
  return (j & 16) ? t2[1] : t2[0];
}

template <int MODE, int KQ, bool IS_IP, int EPI, int TBN>
__global__ void __launch_bounds__(128 + 32 * EPI, 1)
    fused_knn_kernel(const __grid_constant__ CUtensorMap tm_a0, const __grid_constant__ CUtensorMap tm_a1,
                     const __grid_constant__ CUtensorMap tm_b0, const __grid_constant__ CUtensorMap tm_b1,
                     const SearchParams p) {
  // MODE 0: fp32 3xTF32 hi/lo; 4: fp32, ONE tf32 pass as a filter with a
  // proven margin and exact fp32 rescoring of the survivors; 5: the same
  // filter on power-of-two-scaled fp16 copies of the fp32 rows (same 11-bit
  // precision as tf32, twice the MMA rate, half the bytes; filter16_kernels.cuh);
  // 1/2: fp16/bf16 storage
  constexpr bool TF32 = (MODE == 0 || MODE == 4);
  constexpr bool F1P = (MODE == 4 || MODE == 5);  // 1-pass filter + certified exact rescoring
  constexpr int SPLIT = (MODE == 0) ? 2 : 1;
  constexpr int BK = TF32 ? 32 : 64;  // elements per 128-byte K-chunk
  constexpr uint32_t AB_FMT = TF32 ? 2u : ((MODE == 1 || MODE == 5) ? 0u : 1u);
  // MODE 3 (bf16, L2): base rows are stored as [-2x | xn split in 3 bf16] and
  // query rows as [q | 1 1 1], so the accumulator already holds xn - 2 q.x and
  // the epilogue needs no base-norm tile (FOLD).
  constexpr bool FOLD = (MODE == 3);
  constexpr bool XN_TILE = !IS_IP && !FOLD;
  // TBN: base rows per tile = accumulator columns (128, or 64 when a large
  // query operand leaves TMEM room for only 2 x 64 accumulator columns)
  constexpr int BN = TBN;
  constexpr uint32_t B_CHUNK = (uint32_t)TBN * 128u;  // one TBN-row x 128-byte K-chunk of the base
  constexpr uint32_t IDESC = make_idesc(AB_FMT, BM, BN);
  constexpr int NH = EPI / 4;       // epilogue warp groups (one warp per TMEM lane quarter each)
  constexpr int NG = NH;            // group g owns the tiles with tcount % NG == g
  constexpr int PIECE = (NG == 1) ? BN : 64;  // accumulator columns per TMEM load batch

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // debug timeline window (FK_DEV): tiles [TOFF, TOFF + 256) of CTA 0, epilogue lane quarter TQ
  const uint32_t TOFF = FK_DEV ? (uint32_t)(p.dbg_flags >> 20) * 256u : 0u;
  const int TQ = FK_DEV ? (p.dbg_flags >> 16) & 3 : 0;
  const int num_kb = p.num_kb;
  const int stages = p.stages;
  const int a_mode = p.a_mode;
  const int a_kt = (a_mode == 3) ? p.a_kt : (a_mode == 0 ? num_kb : 0);  // K-chunks of A in TMEM
  const uint32_t a_bytes = (a_mode == 1 || a_mode == 3) ? SPLIT * (num_kb - a_kt) * CHUNK_BYTES : 0u;
  // stage = [B hi (| B lo)] (a_mode 2: + [A hi (| A lo)], 128-row chunks)
  const uint32_t stage_bytes = SPLIT * B_CHUNK + (a_mode == 2 ? SPLIT * CHUNK_BYTES : 0u);
  constexpr uint32_t tmem_cols = 512u;  // 1 CTA per SM: take the whole TMEM

  uint8_t* a_region = smem;
  uint8_t* st_region = smem + a_bytes;
  const int xn_slots = p.xn_slots;
  float* xn_s = reinterpret_cast<float*>(st_region + stages * stage_bytes);  // [xn_slots][BN]
  uint32_t* hist_base = reinterpret_cast<uint32_t*>(xn_s + xn_slots * BN);  // large-k: [EPI][256]
  // barriers live in static shared memory: constant addresses, nothing to
  // rematerialise inside the hot loops
  __shared__ __align__(8) uint64_t bars[92];
  uint64_t* full = bars;         // [MAX_STAGES]
  uint64_t* empty = bars + 32;   // [MAX_STAGES]
  uint64_t* tfull = bars + 64;   // [MAX_ACC]
  uint64_t* tempty = bars + 68;  // [MAX_ACC]
  uint64_t* xfull = bars + 72;   // [8]
  uint64_t* xempty = bars + 80;  // [8]
  uint64_t* afull = bars + 88;
  uint64_t* aempty = bars + 89;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 90);
  const uint32_t acc_stages = p.acc_stages;
  const uint32_t tmem_a_col = acc_stages * BN;
  // cluster mode: the CTA pair walks the same (chunk, tile) sequence with
  // query tiles m = 2*mu + crank; each CTA loads half of every base tile and
  // multicasts it, so a stage is reusable only after BOTH CTAs' MMAs read it
  const int CL = p.cluster;
  const uint32_t crank = CL == 2 ? cluster_ctarank() : 0u;
  const int ublock = blockIdx.x / CL, ugrid = gridDim.x / CL;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_b0);
    if (SPLIT == 2) tma_prefetch_desc(&tm_b1);
    if (a_mode != 0) {
      tma_prefetch_desc(&tm_a0);
      if (SPLIT == 2) tma_prefetch_desc(&tm_a1);
    }
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL);  // one commit from each CTA's MMA issuer
    }
    for (int b = 0; b < (int)acc_stages; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);  // the 4 warps of the tile's epilogue group
    }
    for (int x = 0; x < xn_slots; ++x) {
      mbar_init(&xfull[x], 1);
      mbar_init(&xempty[x], 4);
    }
    mbar_init(afull, a_mode == 0 ? EPI : (a_mode == 3 ? EPI + 1 : 1));
    mbar_init(aempty, p.n_issuers);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  if (CL == 2) cluster_sync();  // peers' barriers are initialised before any multicast targets them
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0 || (warp == 2 && p.n_issuers == 2 && p.n_producers == 2)) {
    // ===================== TMA producers =====================
    // One producer per MMA issuer (warp 0 -> ring 0, warp 2 -> ring 1): a
    // producer blocked on one ring's free slots never stalls the other ring.
    if (lane == 0) {
      const uint32_t myring = (warp == 0) ? 0u : 1u;
      const uint64_t pol_a = policy_evict_last();
      // streamed base: evict_last by default (FK_B_POLICY=0 first, 1 normal)
      const uint64_t pol_b = p.b_policy == 2 ? policy_evict_last()
                             : p.b_policy == 1 ? policy_evict_normal() : policy_evict_first();
      // one FIFO sub-ring of `sh` slots per MMA issuer (tile t -> ring t % nis)
      const uint32_t nis = p.n_issuers;
      const uint32_t sh = (uint32_t)stages / nis;
      // per-ring positions (a single producer serves both rings when
      // n_producers == 1); norm-tile sub-ring of ring r: slots [r*xh, +xh)
      uint32_t rs0 = 0, rph0 = 0, rs1 = 0, rph1 = 0, xt0 = 0, xp0 = 0, xt1 = 0, xp1 = 0;
      const uint32_t xh = (uint32_t)xn_slots / nis;
      uint32_t tc = 0;
      int j = 0;
      for (int u = ublock; u < p.num_units; u += ugrid, ++j) {
        const int chunk = u / p.num_mu;
        const int m = (u - chunk * p.num_mu) * CL + (int)crank;
        int t0, t1;
        chunk_range(p, chunk, t0, t1);
        if ((a_mode == 1 || a_mode == 3) && myring == 0) {  // smem-resident K-chunks [a_kt, num_kb)
          if (j > 0) mbar_wait(aempty, (j - 1) & 1);
          mbar_arrive_expect_tx(afull, a_bytes);
          const int nka = num_kb - a_kt;
          for (int part = 0; part < SPLIT; ++part)
            for (int kb = a_kt; kb < num_kb; ++kb)
              tma_load_2d(a_region + (part * nka + kb - a_kt) * CHUNK_BYTES, part ? &tm_a1 : &tm_a0, afull,
                          kb * BK, m * BM, pol_a);
        }
        for (int t = t0; t < t1; ++t, ++tc) {
          const uint32_t ring = (nis == 2) ? (tc & 1) : 0;
          if (p.n_producers == 2 && ring != myring) continue;  // the other producer's tile
          uint32_t& rs = ring ? rs1 : rs0;
          uint32_t& rph = ring ? rph1 : rph0;
          if (XN_TILE) {  // base norms of this tile -> the ring's norm sub-ring (consumed by the epilogue)
            uint32_t& xt = ring ? xt1 : xt0;
            uint32_t& xphase = ring ? xp1 : xp0;
            const uint32_t xs = ring * xh + xt, xph = xphase;
            if (++xt == xh) {
              xt = 0;
              xphase ^= 1;
            }
            mbar_wait(&xempty[xs], xph ^ 1);
            mbar_arrive_expect_tx(&xfull[xs], BN * sizeof(float));
            bulk_load(xn_s + xs * BN, p.xnorm + (size_t)t * BN, BN * sizeof(float), &xfull[xs]);
          }
          for (int kb = 0; kb < num_kb; ++kb) {
            const uint32_t stage = ring * sh + rs, phase = rph;
            if (++rs == sh) {
              rs = 0;
              rph ^= 1;
            }
            mbar_wait(&empty[stage], phase ^ 1);
            if (p.dbg_flags & 2) {  // experiment: no data movement
              mbar_arrive(&full[stage]);
              continue;
            }
            mbar_arrive_expect_tx(&full[stage], stage_bytes);
            uint8_t* sb = st_region + stage * stage_bytes;
            if (CL == 2) {  // my half of the tile's rows (swizzle-atom aligned) to both CTAs
              const uint32_t hoff = crank * (B_CHUNK / 2);
              tma_load_2d_mc(sb + hoff, &tm_b0, &full[stage], kb * BK, t * BN + (int)crank * (BN / 2), 0x3, pol_b);
              if (SPLIT == 2)
                tma_load_2d_mc(sb + B_CHUNK + hoff, &tm_b1, &full[stage], kb * BK, t * BN + (int)crank * (BN / 2),
                               0x3, pol_b);
            } else {
              tma_load_2d(sb, &tm_b0, &full[stage], kb * BK, t * BN, pol_b);
              if (SPLIT == 2) tma_load_2d(sb + B_CHUNK, &tm_b1, &full[stage], kb * BK, t * BN, pol_b);
            }
            if (a_mode == 2) {
              tma_load_2d(sb + SPLIT * B_CHUNK, &tm_a0, &full[stage], kb * BK, m * BM, pol_a);
              if (SPLIT == 2)
                tma_load_2d(sb + SPLIT * B_CHUNK + CHUNK_BYTES, &tm_a1, &full[stage], kb * BK, m * BM, pol_a);
            }
          }
        }
      }
    }
  } else if (warp == 1 || (warp == 3 && p.n_issuers == 2)) {
    // ===================== MMA issuers (whole warp, one elected lane issues) =====================
    // With two issuers (warps 1 and 3), issuer w owns the tiles with
    // tcount % 2 == w: while one waits on its barriers the other keeps the
    // tensor pipe fed.  The loop runs on all 32 lanes so every descriptor is
    // warp-uniform; elect_one() picks the lane that issues.
    {
      const uint32_t nis = p.n_issuers;
      const uint32_t mw = (warp == 1) ? 0u : 1u;
      const uint32_t sh = (uint32_t)stages / nis;
      uint32_t rslot = 0, rphase = 0;  // position in this issuer's sub-ring
      uint32_t tcount = 0, buf = 0, tph = 0;  // accumulator ring position of tile tcount
      int j = 0;
      const uint32_t a_tm = tmem_base + tmem_a_col;
      const uint32_t a_lo_off = (MODE == 0) ? (uint32_t)(num_kb * 32) : 0u;  // lo half after hi (columns)
      const uint64_t st_desc0 = smem_desc_sw128(smem_u32(st_region));
      const uint64_t a_desc0 = smem_desc_sw128(smem_u32(a_region));
      const int kk_last = p.kk_last;
      for (int u = ublock; u < p.num_units; u += ugrid, ++j) {
        const int chunk = u / p.num_mu;
        int t0, t1;
        chunk_range(p, chunk, t0, t1);
        if (a_mode != 2) {
          mbar_wait(afull, j & 1);
          tc_fence_after();
        }
        for (int t = t0; t < t1; ++t, ++tcount) {
          const uint32_t cbuf = buf, cph = tph;
          if (++buf == acc_stages) {
            buf = 0;
            tph ^= 1;
          }
          if (nis == 2 && (tcount & 1) != mw) continue;
          const bool tr = FK_DEV && p.trace != nullptr && blockIdx.x == 0 && tcount - TOFF < 256u && lane == 0;
          if (tr) p.trace[(tcount - TOFF) * 16 + 0] = clock64();
          mbar_wait(&tempty[cbuf], cph ^ 1);
          tc_fence_after();
          if (tr) p.trace[(tcount - TOFF) * 16 + 1] = clock64();
          const uint32_t d_tmem = tmem_base + cbuf * BN;
          for (int kb = 0; kb < num_kb; ++kb) {
            const int nkk = (kb == num_kb - 1) ? kk_last : 4;  // skip all-zero K padding steps
            const uint32_t stage = mw * sh + rslot, phase = rphase;
            if (++rslot == sh) {
              rslot = 0;
              rphase ^= 1;
            }
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            if (tr && kb < 4) p.trace[(tcount - TOFF) * 16 + 13 + (kb < 3 ? kb : 2)] = clock64();
            // descriptor start address is in 16-byte units (bits 0-13)
            const uint64_t bd0 = st_desc0 + ((stage * stage_bytes) >> 4);
            const uint64_t bd1 = bd0 + (B_CHUNK >> 4);
            if (elect_one()) {
              if (a_mode == 0 || (a_mode == 3 && kb < a_kt)) {
                const uint32_t ah = a_tm + kb * 32;
                if (MODE == 0) {
#pragma unroll
                  for (int kk = 0; kk < 4; ++kk) {
                    if (kk >= nkk) break;
                    const uint64_t off = 2 * kk;  // 32 B = K 8 (tf32) per step, 16-byte units
                    mma_tf32_ts(d_tmem, ah + a_lo_off + 8 * kk, bd0 + off, IDESC, (kb | kk) != 0);  // lo*hi
                    mma_tf32_ts(d_tmem, ah + 8 * kk, bd1 + off, IDESC, 1u);                        // hi*lo
                    mma_tf32_ts(d_tmem, ah + 8 * kk, bd0 + off, IDESC, 1u);                        // hi*hi
                  }
                } else if (FK_ISSUER_FAST && nkk == 4) {  // full 128-byte K-chunk: 4 MMAs, no padding checks
                  const uint32_t acc0 = kb != 0;
                  if (MODE == 4) {
                    mma_tf32_ts(d_tmem, ah, bd0, IDESC, acc0);
                    mma_tf32_ts(d_tmem, ah + 8, bd0 + 2, IDESC, 1u);
                    mma_tf32_ts(d_tmem, ah + 16, bd0 + 4, IDESC, 1u);
                    mma_tf32_ts(d_tmem, ah + 24, bd0 + 6, IDESC, 1u);
                  } else {
                    mma_f16_ts(d_tmem, ah, bd0, IDESC, acc0);
                    mma_f16_ts(d_tmem, ah + 8, bd0 + 2, IDESC, 1u);
                    mma_f16_ts(d_tmem, ah + 16, bd0 + 4, IDESC, 1u);
                    mma_f16_ts(d_tmem, ah + 24, bd0 + 6, IDESC, 1u);
                  }
                } else {
#pragma unroll
                  for (int kk = 0; kk < 4; ++kk) {
                    if (kk >= nkk) break;  // one K-step = 32 B of K = 8 TMEM columns (tf32 or 16-bit pairs)
                    if (MODE == 4) mma_tf32_ts(d_tmem, ah + 8 * kk, bd0 + 2 * kk, IDESC, (kb | kk) != 0);
                    else mma_f16_ts(d_tmem, ah + 8 * kk, bd0 + 2 * kk, IDESC, (kb | kk) != 0);
                  }
                }
              } else {
                const uint64_t ad0 = (a_mode == 1 || a_mode == 3) ? a_desc0 + (((kb - a_kt) * CHUNK_BYTES) >> 4)
                                                                  : bd0 + ((SPLIT * B_CHUNK) >> 4);
                if (MODE == 0) {
                  const uint64_t ad1 = (a_mode == 1) ? a_desc0 + (((num_kb + kb) * CHUNK_BYTES) >> 4)
                                                     : bd0 + ((2 * B_CHUNK + CHUNK_BYTES) >> 4);
#pragma unroll
                  for (int kk = 0; kk < 4; ++kk) {
                    if (kk >= nkk) break;
                    const uint64_t off = 2 * kk;
                    mma_tf32(d_tmem, ad1 + off, bd0 + off, IDESC, (kb | kk) != 0);
                    mma_tf32(d_tmem, ad0 + off, bd1 + off, IDESC, 1u);
                    mma_tf32(d_tmem, ad0 + off, bd0 + off, IDESC, 1u);
                  }
                } else if (FK_ISSUER_FAST && nkk == 4) {  // full 128-byte K-chunk: 4 MMAs, no padding checks
                  const uint32_t acc0 = kb != 0;
                  if (MODE == 4) {
                    mma_tf32(d_tmem, ad0, bd0, IDESC, acc0);
                    mma_tf32(d_tmem, ad0 + 2, bd0 + 2, IDESC, 1u);
                    mma_tf32(d_tmem, ad0 + 4, bd0 + 4, IDESC, 1u);
                    mma_tf32(d_tmem, ad0 + 6, bd0 + 6, IDESC, 1u);
                  } else {
                    mma_f16(d_tmem, ad0, bd0, IDESC, acc0);
                    mma_f16(d_tmem, ad0 + 2, bd0 + 2, IDESC, 1u);
                    mma_f16(d_tmem, ad0 + 4, bd0 + 4, IDESC, 1u);
                    mma_f16(d_tmem, ad0 + 6, bd0 + 6, IDESC, 1u);
                  }
                } else {
#pragma unroll
                  for (int kk = 0; kk < 4; ++kk) {
                    if (kk >= nkk) break;
                    if (MODE == 4) mma_tf32(d_tmem, ad0 + 2 * kk, bd0 + 2 * kk, IDESC, (kb | kk) != 0);
                    else mma_f16(d_tmem, ad0 + 2 * kk, bd0 + 2 * kk, IDESC, (kb | kk) != 0);
                  }
                }
              }
              if (CL == 2) mma_commit_mc(&empty[stage], 0x3);  // frees the stage in both CTAs
              else mma_commit(&empty[stage]);
            }
            __syncwarp();
            if (tr && kb < 4) p.trace[(tcount - TOFF) * 16 + 9 + kb] = clock64();
          }
          if (elect_one()) mma_commit(&tfull[cbuf]);
          __syncwarp();
          if (tr) p.trace[(tcount - TOFF) * 16 + 3] = clock64();
        }
        if (a_mode != 2) {  // the unit's MMAs retired: A may be replaced (smem: producer, TMEM: epilogue)
          if (elect_one()) mma_commit(aempty);
          __syncwarp();
        }
      }
    }
  } else if (warp >= EPI_WARP0) {
    // ===================== epilogue =====================
    const int ew = warp - EPI_WARP0;
    const int eq = warp & 3;  // TMEM lane quarter this warp may access
    const int g = ew >> 2;    // warp group: owns every NG-th tile (and partial list g of each unit)
    const int h = g;
    const uint32_t lane_addr = static_cast<uint32_t>(eq * 32) << 16;
    const int k = p.k;
    const int dp = num_kb * BK;
    const int a_cols = (MODE == 0) ? 2 * dp : (MODE == 4 ? dp : dp / 2);  // TMEM columns of the query operand
    uint32_t tcount = 0, a_buf = 0, a_ph = 0;
    uint32_t xs0 = 0, xp0 = 0, xs1 = 0, xp1 = 0;  // norm sub-ring positions (ring = tile % n_issuers)
    const uint32_t xn_s_a = smem_u32(xn_s);
    const uint32_t xh = (uint32_t)xn_slots / (uint32_t)p.n_issuers;
    int uj = 0;  // units processed by this CTA
    for (int u = ublock; u < p.num_units; u += ugrid, ++uj) {
      const int chunk = u / p.num_mu;
      const int m = (u - chunk * p.num_mu) * CL + (int)crank;
      int t0, t1;
      chunk_range(p, chunk, t0, t1);
      const int row = m * BM + eq * 32 + lane;
      const bool row_ok = row < p.nq;

      if (a_mode == 0 || a_mode == 3) {
        // Query tile -> TMEM (lane = query row, columns = K; fp32: [hi | lo]).
        // Only after EVERY MMA of the previous unit retired (both issuers
        // commit aempty at unit end): with two epilogue groups, this group's
        // last tile is not necessarily the unit's last MMA.
        if (uj > 0) mbar_wait(aempty, (uj - 1) & 1);
        const int a_ccn = (a_mode == 3) ? a_kt : a_cols / 32;  // 32-column groups written (a_mode 3: TMEM part)
        for (int cc = h; cc < a_ccn; cc += NH) {
          uint32_t v[32];
          const uint32_t* src;
          if (MODE == 0)
            src = (cc * 32 < dp) ? reinterpret_cast<const uint32_t*>(p.qa0) + (size_t)row * dp + cc * 32
                                 : reinterpret_cast<const uint32_t*>(p.qa1) + (size_t)row * dp + (cc * 32 - dp);
          else if (MODE == 4)
            src = reinterpret_cast<const uint32_t*>(p.qa0) + (size_t)row * dp + cc * 32;
          else
            src = reinterpret_cast<const uint32_t*>(p.qa0) + (size_t)row * (dp / 2) + cc * 32;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            uint4 w = make_uint4(0u, 0u, 0u, 0u);
            if (row_ok) w = __ldg(reinterpret_cast<const uint4*>(src) + i);
            v[4 * i] = w.x;
            v[4 * i + 1] = w.y;
            v[4 * i + 2] = w.z;
            v[4 * i + 3] = w.w;
          }
          tmem_st_32x32b_x32(tmem_base + lane_addr + tmem_a_col + cc * 32, v);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(afull);
      }

      constexpr bool RANGE = KQ < 0;
      const float qn = ((!IS_IP || RANGE || F1P) && row_ok) ? p.qnorm[row] : 0.f;
      // MODE 5: accumulator -> inner product scale 2^-(s_q + s_x) (exact)
      const float sc = (MODE == 5 && row_ok) ? __ldg(p.qinv + row) * __ldg(p.xinv) : 1.f;
      const float c2 = -2.f * sc;
      constexpr int KQS = KQ > 0 ? KQ : 1;
      uint32_t keys[KQS], pos[KQS];
      if constexpr (KQ > 0) {
#pragma unroll
        for (int i = 0; i < KQ; ++i) {
          keys[i] = (i < KQ - k) ? 0u : 0xFFFFFFFFu;
          pos[i] = 0xFFFFFFFFu;
        }
      }
      // large k: unsorted per-row candidate buffer + exact compaction
      uint64_t* mybuf = nullptr;
      int cnt = 0;
      uint32_t lkey = 0xFFFFFFFFu;  // key of the k-th after the last compaction
      uint32_t* hist = hist_base + ew * 256;
      if constexpr (KQ == 0) mybuf = p.cbuf + (((size_t)blockIdx.x * EPI + ew) * 32 + lane) * (size_t)p.cap;
      // MODE 4: |t - v| <= e for every pair, band = 2e with 2x safety (see
      // merge_rescore_kernel); the bound we filter and publish with is
      // (own kfinal-th t) + band >= (global kfinal-th t) + band
      const bool tf32_exact = p.inexact != nullptr && (p.inexact[0] | p.inexact[1]) == 0u;
      // rounding term (host-chosen p.band_l2, IP half): one filter pass errs
      // by |t - ip| <= (2^-10 + 2^-20) |q||x| (tf32 truncation) or
      // (2^-10 + 2^-27) |q||x| (RNE scaled fp16, incl. subnormals), so the
      // filter value xn - 2t by twice that, and a true top-k member lies within
      // 2x of it above the k-th filter value: band = 2^-7 / 2^-8 |q| max|x|
      // (+ 2^-10 margin)
      const float band4 = (F1P && KQ > 0 && !RANGE && row_ok)
                              ? (tf32_exact ? 0.f : (IS_IP ? 0.5f * p.band_l2 : p.band_l2)) *
                                        sqrtf(band_norm(p.qnorm[row]) * band_norm(*p.xn_max)) +
                                    // fp32 accumulation: the tensor core (possibly truncating,
                                    // <= dp 2^-23) and the sequential-FMA rescoring (<= dp 2^-24)
                                    // each err by <= dp u (qn + max xn); band = 2e, 2x safety,
                                    // + the final (qn + xn) - 2ip roundings
                                    (4.f * (float)dp + 8.f) * 1.1920928955078125e-07f *
                                        (band_norm(p.qnorm[row]) + band_norm(*p.xn_max))
                              : 0.f;
      uint32_t min_lost = 0xFFFFFFFFu;  // F1P: smallest band key lost (overflow list full)
      // queue slot of the caller's k-th (MODE 4 keeps k' >= kfinal entries);
      // read through a static select so the queue stays in registers
      const int kf_slot = (KQS - k) + p.kfinal - 1;
      // F1P: (kfinal-th filter key + band), cached -- it only changes when an
      // insertion lands at or before the kfinal-th slot
      auto band_bound = [&](uint32_t kk) -> uint32_t {
        if (kk == 0xFFFFFFFFu) return kk;
        const float b = unmonotone(kk) + band4;
        return (b != b) ? 0xFFFFFFFFu : monotone(b);
      };
      uint32_t kth_f1p = 0xFFFFFFFFu, own_f1p = 0xFFFFFFFFu;
      auto own_key = [&]() -> uint32_t {
        if constexpr (KQ > 0) {
          if (F1P) return own_f1p;
          return keys[KQS - 1];
        }
        return lkey;
      };
      // Effective threshold = min(own k-th, best k-th published by any unit of
      // this query): every true top-k member has key <= the global k-th <= it.
      uint32_t gkey = (row_ok && !RANGE) ? __ldcg(p.thr_key + row) : 0xFFFFFFFFu;
      float thr = unmonotone(gkey);  // NaN while nothing is known: everything passes
      if constexpr (RANGE) thr = IS_IP ? -p.radius : p.radius;  // IP ranks -ip (core.py:217)
      // Conservative fast-filter bound on f = fl(xn - 2ip): the reference value
      // fl(fl(qn + xn) - 2ip) differs from qn + f by < 3u(qn + xn + |v|); the
      // 2^-20 margin (u = 2^-24) over max-norm covers it with room to spare.
      const float xmax = (IS_IP && !F1P) ? 0.f : *p.xn_max;
      // MODE 4 range search: the single tf32 pass rounds each operand to 11
      // significant bits, |ip_tf32 - ip| <= 2^-9 sum|q_i||x_i| <= 2^-9 |q||x|,
      // so f = xn - 2 ip moves by <= 2^-8 |q| max|x|: widen by 2^-7 (2x) before
      // the exact direct-distance pass.  (Top-k queues stay in tf32 space.)
      const float tf32_margin =
          (MODE == 4 && RANGE) ? 0.0078125f * sqrtf(fmaxf(qn, 0.f) * fmaxf(xmax, 0.f)) : 0.f;
      auto filter_bound = [&](float th) -> float {
        if (MODE == 4 && RANGE) {
          if (IS_IP) return th + 0.5f * tf32_margin;  // IP filters on -ip: half the L2 widening
          return (th - qn) + (qn + xmax + fabsf(th)) * 9.5367431640625e-07f + tf32_margin;
        }
        if (IS_IP) {
          // range search compares the GEMM inner product with the exact
          // direct one: widen by 2^-18 |q| max|x| (>> the 3xTF32 / fp32 error)
          if (RANGE) return th + 3.814697265625e-06f * sqrtf(qn * *p.xn_max);
          return th;
        }
        return (th - qn) + (qn + xmax + fabsf(th)) * 9.5367431640625e-07f;
      };
      float T = filter_bound(thr);
      // warp-uniform: compact every lane whose buffer holds more than `limit`
      auto compact_lanes = [&](int limit) {
        unsigned todo = __ballot_sync(FULLMASK, cnt > limit);
        while (todo) {
          const int L = __ffs(todo) - 1;
          todo &= todo - 1;
          const int cL = __shfl_sync(FULLMASK, cnt, L);
          uint64_t* bL = reinterpret_cast<uint64_t*>(
              __shfl_sync(FULLMASK, reinterpret_cast<unsigned long long>(mybuf), L));
          const uint64_t kth = warp_kth([&](int e) { return bL[e]; }, cL, (uint32_t)k, hist);
          const int nc = warp_compact_le(bL, cL, kth);
          if (lane == L) {
            cnt = nc;
            lkey = static_cast<uint32_t>(kth >> 32);
            thr = unmonotone(min(lkey, gkey));
            T = filter_bound(thr);
          }
        }
      };

      uint32_t own_tiles = 0;  // tiles of this unit processed by this warp group (publish cadence)
      for (int t = t0; t < t1; ++t, ++tcount) {
        const uint32_t buf = a_buf, tph = a_ph;
        if (++a_buf == acc_stages) {
          a_buf = 0;
          a_ph ^= 1;
        }
        uint32_t xslot = 0, xph = 0;
        if (XN_TILE) {
          const uint32_t ring = (p.n_issuers == 2) ? (tcount & 1) : 0;
          uint32_t& xs = ring ? xs1 : xs0;
          uint32_t& xp = ring ? xp1 : xp0;
          xslot = ring * xh + xs;
          xph = xp;
          if (++xs == xh) {
            xs = 0;
            xp ^= 1;
          }
        }
        if (NG > 1 && (tcount & (NG - 1)) != (uint32_t)g) continue;  // another group's tile
        const bool tr = FK_DEV && p.trace != nullptr && blockIdx.x == 0 && tcount - TOFF < 256u && eq == TQ && lane == 0;
        if (tr) p.trace[(tcount - TOFF) * 16 + 4] = clock64();
        mbar_wait(&tfull[buf], tph);
        if (tr) p.trace[(tcount - TOFF) * 16 + 5] = clock64();
        if (XN_TILE) mbar_wait(&xfull[xslot], xph);
        tc_fence_after();
        if (tr) p.trace[(tcount - TOFF) * 16 + 6] = clock64();
        const int n0 = t * BN;
        const int nvalid = p.nb - n0;
        const uint32_t xs_a = xn_s_a + xslot * (BN * 4u);  // this tile's base norms (shared address)
        // Filter on f = xn - 2 ip (L2; one FMA) or -ip (IP) against T; the
        // exact reference value (qn + xn) - 2 ip is computed for survivors only.
        auto chunk_f = [&](const uint32_t (&r)[32], int c0, float (&f)[32]) {
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            if (IS_IP && MODE == 5) {
              f[4 * j4 + 0] = __uint_as_float(r[4 * j4 + 0]) * sc;
              f[4 * j4 + 1] = __uint_as_float(r[4 * j4 + 1]) * sc;
              f[4 * j4 + 2] = __uint_as_float(r[4 * j4 + 2]) * sc;
              f[4 * j4 + 3] = __uint_as_float(r[4 * j4 + 3]) * sc;
            } else if (IS_IP || FOLD) {
              f[4 * j4 + 0] = __uint_as_float(r[4 * j4 + 0]);
              f[4 * j4 + 1] = __uint_as_float(r[4 * j4 + 1]);
              f[4 * j4 + 2] = __uint_as_float(r[4 * j4 + 2]);
              f[4 * j4 + 3] = __uint_as_float(r[4 * j4 + 3]);
            } else {
              // c2 = -2 (MODE 5: -2 * 2^-(s_q + s_x), so c2 * acc is exactly -2 t)
              const float4 x = lds_f4_at(xs_a + (uint32_t)(c0 + 4 * j4) * 4u);
              f[4 * j4 + 0] = fmaf(c2, __uint_as_float(r[4 * j4 + 0]), x.x);
              f[4 * j4 + 1] = fmaf(c2, __uint_as_float(r[4 * j4 + 1]), x.y);
              f[4 * j4 + 2] = fmaf(c2, __uint_as_float(r[4 * j4 + 2]), x.z);
              f[4 * j4 + 3] = fmaf(c2, __uint_as_float(r[4 * j4 + 3]), x.w);
            }
          }
        };
        // rare path for one 32-column chunk: exact value + insertion per survivor
        auto slow_chunk = [&](const uint32_t (&r)[32], int c0) {
          float f[32];
          chunk_f(r, c0, f);
          const int lim = nvalid - c0;
          const uint32_t valid = lim >= 32 ? 0xFFFFFFFFu : (lim <= 0 ? 0u : ((1u << lim) - 1u));
          uint32_t cand = 0;
#pragma unroll
          for (int j = 0; j < 32; ++j) cand |= ((IS_IP ? !(-f[j] > T) : !(f[j] > T)) ? 1u : 0u) << j;
          cand &= valid;
          if constexpr (RANGE) {  // append every candidate; the exact test happens later
            const unsigned nc = __popc(cand);
            if (nc) {
              unsigned long long slot = atomicAdd(p.rcount, (unsigned long long)nc);
              while (cand) {
                const int j = __ffs(cand) - 1;
                cand &= cand - 1;
                if (slot < p.rcap)
                  p.rcand[slot] = (static_cast<unsigned long long>(row) << 32) | static_cast<uint32_t>(n0 + c0 + j);
                ++slot;
              }
            }
            return;
          }
          while (cand) {
            const int j = __ffs(cand) - 1;
            cand &= cand - 1;
            // (MODE 4: a 1-pass tf32 value; the queue works in that space and
            // merge_rescore_kernel recomputes the survivors exactly)
            const float ip = select32(reinterpret_cast<const float(&)[32]>(r), j) * sc;
            // flat.py:111: dmat = (qn + norms) - 2.0*ip  (2*ip exact -> one FMA;
            // FOLD: the accumulator already is xn - 2 ip)
            float v;
            if (IS_IP) v = -ip;
            else if (FOLD) v = qn + ip;
            else v = fmaf(-2.f, ip, qn + lds_f32_at(xs_a + (uint32_t)(c0 + j) * 4u));
            if (!(v > thr)) {
              if (!IS_IP) v = (v <= 0.f) ? 0.f : v;  // np.maximum(dmat, 0) (flat.py:112)
              const uint32_t kv = IS_IP ? dist_key(ip, true) : dist_key(v, false);
              if constexpr (KQ > 0) {
                uint32_t lk = 0xFFFFFFFFu, lp = 0u;  // F1P: the entry a full queue drops
                if (F1P) {
                  if (kv >= keys[KQS - 1]) {
                    lk = kv;
                    lp = static_cast<uint32_t>(n0 + c0 + j);
                  } else if (pos[KQS - 1] != 0xFFFFFFFFu) {
                    lk = keys[KQS - 1];
                    lp = pos[KQS - 1];
                  }
                }
                queue_insert<KQS>(keys, pos, kv, static_cast<uint32_t>(n0 + c0 + j));
                if (F1P) {
                  if (kv < kth_f1p) {  // the kfinal-th slot moved
                    kth_f1p = select_static<KQS>(keys, kf_slot);
                    own_f1p = band_bound(kth_f1p);
                  }
                }
                const uint32_t bk = min(own_key(), gkey);
                thr = unmonotone(bk);
                T = filter_bound(thr);
                if (F1P && lk != 0xFFFFFFFFu && lk <= bk) {
                  // a band member: keep it in the query's overflow list
                  if (p.ovf_cnt != nullptr) {
                    const unsigned slot = atomicAdd(p.ovf_cnt + row, 1u);
                    if (slot < (unsigned)p.ovf_cap) {
                      p.ovf_key[(size_t)row * p.ovf_cap + slot] = lk;
                      p.ovf_pos[(size_t)row * p.ovf_cap + slot] = lp;
                    } else {
                      min_lost = min(min_lost, lk);
                    }
                  } else {
                    min_lost = min(min_lost, lk);
                  }
                }
              } else {
                mybuf[cnt++] = (static_cast<uint64_t>(kv) << 32) | static_cast<uint32_t>(n0 + c0 + j);
              }
            }
          }
        };
        // Per PIECE of columns: (1) accumulators -> registers; after the last
        // piece (2) hand the TMEM buffer back to the MMA issuer; (3) filter +
        // select from registers.  Tiles alternate between warp groups, so a
        // group has NG tile periods to finish one tile.
        const bool do_epi = !(p.dbg_flags & 1);
        const bool do_cmp = do_epi && !(p.dbg_flags & 8);  // 8: TMEM loads without the filter
#pragma unroll
        for (int pc = 0; pc < BN / PIECE; ++pc) {
          uint32_t racc[PIECE];
          if (tr && pc == 0) p.trace[(tcount - TOFF) * 16 + 2] = clock64();
          if (do_epi) {
            if constexpr (FK_LD_X64 && PIECE == 64) {  // one 64-column load
              tmem_ld_32x32b_x64(tmem_base + lane_addr + buf * BN + pc * PIECE, racc);
            } else if constexpr (FK_LD_X128 && PIECE == 128) {  // the whole tile row in one load
              tmem_ld_32x32b_x128(tmem_base + lane_addr + buf * BN, racc);
            } else {
#pragma unroll
              for (int c = 0; c < PIECE / 32; ++c)
                tmem_ld_32x32b_x32(tmem_base + lane_addr + buf * BN + pc * PIECE + c * 32,
                                   *reinterpret_cast<uint32_t(*)[32]>(&racc[32 * c]));
            }
            tmem_ld_wait();
          }
          if (tr && pc < 2) p.trace[(tcount - TOFF) * 16 + 11 + pc] = clock64();
          if (pc == BN / PIECE - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
          }
          if (do_cmp) {
            if (p.dbg_ip != nullptr && row_ok) {
              for (int j = 0; j < PIECE; ++j)
                if (pc * PIECE + j < nvalid) p.dbg_ip[(size_t)row * p.nb + n0 + pc * PIECE + j] = __uint_as_float(racc[j]);
            }
            // fast path: straight-line min tree, a single branch per piece;
            // the 32-column minima are kept so the slow path visits only the
            // chunks that hold a candidate
            float m = 0.f;
            float mcs[PIECE / 32];
#pragma unroll
            for (int c = 0; c < PIECE / 32; ++c) {
              float f[32];
              chunk_f(*reinterpret_cast<const uint32_t(*)[32]>(&racc[32 * c]), pc * PIECE + c * 32, f);
              const float mc = IS_IP ? -reduce32<true>(f) : reduce32<false>(f);
              mcs[c] = mc;
              m = (c == 0) ? mc : fmin_nan(m, mc);
            }
            const bool slow = !(m > T) && row_ok && !(p.dbg_flags & 4);
            if (FK_DEV && p.trace != nullptr) {
              const unsigned sb = __ballot_sync(FULLMASK, slow);
              if (tr) p.trace[(tcount - TOFF) * 16 + 8] += __popc(sb);
            }
            if (FK_DEV && p.trace != nullptr && !(p.dbg_flags & 0x8000)) {  // slow-path statistics over all CTAs (trace row 256; 0x8000: off)
              const unsigned sbl = __ballot_sync(FULLMASK, slow);
              if (lane == 0) {
                atomicAdd(reinterpret_cast<unsigned long long*>(p.trace + 256 * 16 + 0), 1ull);  // warp-pieces
                if (sbl) atomicAdd(reinterpret_cast<unsigned long long*>(p.trace + 256 * 16 + 1), 1ull);
                atomicAdd(reinterpret_cast<unsigned long long*>(p.trace + 256 * 16 + 2), (unsigned long long)__popc(sbl));
                // slow warp-pieces by chunk (slots 3..14: chunks 0..11; and by wave: units < grid)
                if (sbl) atomicAdd(reinterpret_cast<unsigned long long*>(p.trace + 256 * 16 + 3 + min(chunk, 11)), 1ull);
              }
            }
            if (slow) {  // divergent, rare
#pragma unroll
              for (int c = 0; c < PIECE / 32; ++c)
                if (!(mcs[c] > T))  // (T only tightens while inserting: re-checked per chunk)
                  slow_chunk(*reinterpret_cast<const uint32_t(*)[32]>(&racc[32 * c]), pc * PIECE + c * 32);
            }
            __syncwarp();
            // warp-uniform: make room for the next piece's candidates per row
            if constexpr (KQ == 0) compact_lanes(p.cap - PIECE);
          }
        }
        __syncwarp();
        if (tr) p.trace[(tcount - TOFF) * 16 + 7] = clock64();
        if (lane == 0 && XN_TILE) mbar_arrive(&xempty[xslot]);
        if (!RANGE && (++own_tiles & p.pub_mask) == 0 && row_ok) {  // publish own k-th, fetch the shared bound
          const uint32_t mine = own_key();
          gkey = min(atomicMin(p.thr_key + row, mine), mine);
          thr = unmonotone(min(mine, gkey));
          T = filter_bound(thr);
        }
      }
      const int S_tot = p.S * NH;
      const size_t base = ((size_t)row * S_tot + chunk * NH + h) * (size_t)k;
      if constexpr (RANGE) {
        // nothing per unit: candidates went straight to rcand
      } else if constexpr (KQ > 0) {
        if (row_ok) {
          atomicMin(p.thr_key + row, own_key());
          if (p.gkeys != nullptr && k <= 32) {
            // merge this unit's list into the query's running union (sorted,
            // 32 deep) and publish (union k-th + band): a valid bound that,
            // unlike one unit's own k-th, improves as units finish.
            // Register-only: [phantoms -> max | queue ascending | max pad] is
            // bitonic, half-cleaners sort it; min(x[i], g[31-i]) of two sorted
            // lists is a bitonic sequence of the 32 smallest of the union.
            uint32_t x[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) x[i] = (i < KQS && i >= KQS - k) ? keys[i < KQS ? i : 0] : 0xFFFFFFFFu;
            bitonic_merge32(x);
            unsigned int* lk = p.glock + row;
            uint32_t* G = p.gkeys + (size_t)row * 32;
            while (atomicCAS(lk, 0u, 1u) != 0u) __nanosleep(64);
            __threadfence();
#pragma unroll
            for (int i = 0; i < 32; ++i) x[i] = min(x[i], __ldcg(G + 31 - i));
            bitonic_merge32(x);
#pragma unroll
            for (int o = 0; o < 32; ++o) __stcg(G + o, x[o]);
            __threadfence();
            atomicExch(lk, 0u);
            const uint32_t uk = select_static<32>(x, p.kfinal - 1);
            if (uk != 0xFFFFFFFFu) {
              const float bnd = unmonotone(uk) + band4;
              if (bnd == bnd) atomicMin(p.thr_key + row, monotone(bnd));
            }
          }
          if (F1P && ((min_lost != 0xFFFFFFFFu && min_lost <= own_key()) || !(sc == sc))) {
            atomicOr(p.rflag + row, 1u);  // band member dropped
            if (FK_DEV && row < 3)
              printf("row %d chunk %d: min_lost %f own(kth+band) %f keys0 %f keys9 %f keys31 %f band %f gkey %f\n", row,
                     chunk, unmonotone(min_lost), unmonotone(own_key()), unmonotone(keys[0]),
                     unmonotone(keys[KQS - k + p.kfinal - 1]), unmonotone(keys[KQS - 1]), band4, unmonotone(gkey));
          }
#pragma unroll
          for (int i = 0; i < KQ; ++i) {
            if (i >= KQ - k) {
              p.part_key[base + i - (KQ - k)] = keys[i];
              p.part_pos[base + i - (KQ - k)] = pos[i];
            }
          }
        }
      } else {
        compact_lanes(k);  // exact top-k of this unit's survivors
        if (row_ok) {
          if (lkey != 0xFFFFFFFFu) atomicMin(p.thr_key + row, lkey);
          for (int i = 0; i < cnt; ++i) {
            const uint64_t v = mybuf[i];
            p.part_key[base + i] = static_cast<uint32_t>(v >> 32);
            p.part_pos[base + i] = static_cast<uint32_t>(v);
          }
          p.part_cnt[(size_t)row * S_tot + chunk * NH + h] = cnt;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (CL == 2) cluster_sync();  // no CTA leaves while its peer may still multicast into it
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, tmem_cols);
  }
}

}  // namespace fk
