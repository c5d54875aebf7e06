// tcgen05.mma dependency test (sm_100a): kind::f16 M128 N128 K16, A in TMEM,
// B from smem.  NACC independent accumulators are used round-robin (NACC = 1:
// every MMA accumulates into the previous one's result -- a dependent chain,
// like the K loop of one tile).  Also: B descriptor stepping through K like
// the fused kernel (4 K-steps of 32 B per 128-byte chunk, 2 chunks).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2401_08281_b200/csrc
//        -o scripts/microbench_mma3 scripts/microbench_mma3.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace fk;

template <int NACC, bool STEP, int COMMIT = 0>
__global__ void chain(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar, dummy[4];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (warp == 0) tmem_alloc(&slot, 512);
  if (threadIdx.x == 32) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&dummy[i], 1 << 20);  // never completes: commits only count
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 1) {
    constexpr uint32_t idesc = make_idesc(0u, 128, 128);
    const uint64_t b0 = smem_desc_sw128(smem_u32(smem));
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; i += 8 * NACC) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {        // 8 K-steps of a d=128 fp16 tile
#pragma unroll
        for (int a = 0; a < NACC; ++a) {     // NACC tiles interleaved
          const uint64_t bd = STEP ? b0 + (uint64_t)((kk >> 2) * (16384 >> 4)) + 2 * (kk & 3) : b0;
          if (elect_one()) {
            mma_f16_ts(tmem + a * 96, tmem + 448 + 8 * (kk & 3), bd, idesc, kk != 0);
            if (COMMIT && ((kk + 1) % COMMIT) == 0) mma_commit(&dummy[(kk >> 2) & 3]);
          }
          __syncwarp();
        }
      }
    }
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// Pipeline replica of the fused kernel's MMA issuer without TMA: producer
// warp waits empty[s] -> arrives full[s]; issuer waits full[s] -> fence ->
// 4 MMAs (one 128-byte K-chunk) -> commit empty[s]; FENCE toggles the
// tcgen05.fence::after_thread_sync after each wait.
template <bool FENCE, int NS>
__global__ void pipe(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar, full[NS], empty[NS];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (warp == 0) tmem_alloc(&slot, 512);
  if (threadIdx.x == 32) {
    mbar_init(&bar, 1);
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const int nstage = iters / 4;
  if (warp == 2 && (threadIdx.x & 31) == 0) {
    for (int j = 0; j < nstage; ++j) {
      const int s = j % NS;
      mbar_wait(&empty[s], ((j / NS) & 1) ^ 1);
      mbar_arrive(&full[s]);
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = make_idesc(0u, 128, 128);
    const uint64_t b0 = smem_desc_sw128(smem_u32(smem));
    const unsigned long long t0 = clock64();
    for (int j = 0; j < nstage; ++j) {
      const int s = j % NS;
      mbar_wait(&full[s], (j / NS) & 1);
      if (FENCE) tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_f16_ts(tmem + ((j >> 1) & 1) * 128, tmem + 448 + 8 * kk, b0 + 2 * kk, idesc, (j & 1) | kk);
        mma_commit(&empty[s]);
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <bool FENCE, int NS>
void runp(unsigned long long* d) {
  auto k = pipe<FENCE, NS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  const int iters = 8 * 4 * 256;
  k<<<148, 128, 65536 + 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("pipe: %s\n", cudaGetErrorString(e));
    return;
  }
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; ++i) c += h[i];
  c /= 148;
  printf("pipe fence %d stages %d: %6.1f cyc/MMA\n", (int)FENCE, NS, c / iters);
}

// Closer replica: NIS issuer warps alternate tiles (2 stages of 4 MMAs
// each, own sub-rings), accumulator ring of NACC buffers (tfull commit per
// tile), NG epilogue groups of 4 warps alternate tiles: wait tfull ->
// (optionally LDTM the tile) -> arrive tempty.  SS: A from smem.
template <int NIS, bool SS, int NACC, int NG, bool LD, int BSTRIDE = 4096, bool RANDOM = false>
__global__ void pipe2(int tiles, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int NS = 8;
  __shared__ uint32_t slot;
  __shared__ uint64_t full[NS], empty[NS], tfull[NACC], tempty[NACC];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (BSTRIDE * 8 + 32768) / 4; i += blockDim.x) {
    uint32_t v = 0;
    if (RANDOM) {  // two fp16 values in [-2, 2): sign, exponent 14..15, random mantissa
      uint32_t h = (uint32_t)i * 2654435761u ^ (blockIdx.x * 40503u);
      h ^= h >> 13;
      h *= 0x5bd1e995u;
      h ^= h >> 15;
      const uint32_t lo = (h & 0x83FFu) | 0x3800u, hi = ((h >> 16) & 0x83FFu) | 0x3C00u;
      v = lo | (hi << 16);
    }
    reinterpret_cast<uint32_t*>(smem)[i] = v;
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  if (threadIdx.x == 32) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < NACC; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t sh = NS / NIS;
  unsigned long long t0 = clock64();
  if (warp == 0 || (warp == 2 && NIS == 2)) {  // producers, one per ring
    if (lane == 0) {
      const uint32_t ring = warp == 0 ? 0 : 1;
      uint32_t rs = 0, ph = 0;
      for (int t = 0; t < tiles; ++t) {
        if (NIS == 2 && (t & 1) != (int)ring) continue;
        for (int kb = 0; kb < 2; ++kb) {
          const uint32_t s = ring * sh + rs, p = ph;
          if (++rs == sh) { rs = 0; ph ^= 1; }
          mbar_wait(&empty[s], p ^ 1);
          mbar_arrive(&full[s]);
        }
      }
    }
  } else if (warp == 1 || (warp == 3 && NIS == 2)) {
    constexpr uint32_t idesc = make_idesc(0u, 128, 128);
    const uint64_t b0 = smem_desc_sw128(smem_u32(smem));
    const uint64_t a0 = smem_desc_sw128(smem_u32(smem + BSTRIDE * 8));
    const uint32_t mw = warp == 1 ? 0 : 1;
    uint32_t rs = 0, rph = 0, buf = 0, tph = 0;
    for (int t = 0; t < tiles; ++t) {
      const uint32_t cb = buf, cph = tph;
      if (++buf == NACC) { buf = 0; tph ^= 1; }
      if (NIS == 2 && (t & 1) != (int)mw) continue;
      mbar_wait(&tempty[cb], cph ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < 2; ++kb) {
        const uint32_t s = mw * sh + rs, p = rph;
        if (++rs == sh) { rs = 0; rph ^= 1; }
        mbar_wait(&full[s], p);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            if (SS) mma_f16(tmem + cb * 128, a0 + (kb * 16384 >> 4) + 2 * kk, b0 + (s * BSTRIDE >> 4) + 2 * kk, idesc, kb | kk);
            else mma_f16_ts(tmem + cb * 128, tmem + 448 + 8 * kk, b0 + (s * BSTRIDE >> 4) + 2 * kk, idesc, kb | kk);
          }
          mma_commit(&empty[s]);
        }
        __syncwarp();
      }
      if (elect_one()) mma_commit(&tfull[cb]);
      __syncwarp();
    }
  } else if (warp >= 4) {  // epilogue groups
    const int g = (warp - 4) >> 2, eq = warp & 3;
    uint32_t buf = 0, tph = 0;
    uint32_t acc = 0;
    for (int t = 0; t < tiles; ++t) {
      const uint32_t cb = buf, cph = tph;
      if (++buf == NACC) { buf = 0; tph ^= 1; }
      if (NG == 2 && (t & 1) != g) continue;
      mbar_wait(&tfull[cb], cph);
      tc_fence_after();
      if (LD) {
        uint32_t r[32];
        for (int c = 0; c < 4; ++c) {
          tmem_ld_32x32b_x32(tmem + ((uint32_t)(eq * 32) << 16) + cb * 128 + c * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) acc += r[i];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[cb]);
    }
    if (acc == 0xdeadbeef) out[0] = acc;
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int NIS, bool SS, int NACC, int NG, bool LD, int BSTRIDE = 4096, bool RANDOM = false>
void runp2(unsigned long long* d, int tiles = 1024) {
  auto k = pipe2<NIS, SS, NACC, NG, LD, BSTRIDE, RANDOM>;
  const int smem = BSTRIDE * 8 + 32768 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<148, 128 + 32 * 4 * NG, smem>>>(tiles, d);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  if (e != cudaSuccess) {
    printf("pipe2: %s\n", cudaGetErrorString(e));
    return;
  }
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; ++i) c += h[i];
  c /= 148;
  printf("pipe2 random %d bstride %d issuers %d %s acc %d groups %d ldtm %d tiles %d: %6.1f cyc/MMA  %.3f ms  %.0f MHz  %.0f TF/s\n", (int)RANDOM, BSTRIDE, NIS,
         SS ? "SS" : "TS", NACC, NG, (int)LD, tiles, c / (tiles * 8), ms, c / (ms * 1e3),
         2.0 * 128 * 128 * 16 * 8.0 * tiles * 148 / (ms * 1e9));
}

template <int NACC, bool STEP, int COMMIT = 0>
void run(unsigned long long* d) {
  auto k = chain<NACC, STEP, COMMIT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  const int iters = 8 * 4 * 256;
  k<<<148, 128, 65536 + 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("NACC %d: %s\n", NACC, cudaGetErrorString(e));
    return;
  }
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; ++i) c += h[i];
  c /= 148;
  const int n = (iters / (8 * NACC)) * 8 * NACC;
  printf("NACC %d step %d commit/%d: %6.1f cyc/MMA  (%.0f flop/cyc/SM)\n", NACC, (int)STEP, COMMIT, c / n, 2.0 * 128 * 128 * 16 * n / c);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  run<1, false>(d);
  run<1, true>(d);
  run<2, true>(d);
  run<3, true>(d);
  run<4, true>(d);
  run<1, true, 4>(d);
  run<1, true, 8>(d);
  run<2, true, 4>(d);
  run<1, true, 1>(d);
  runp<true, 8>(d);
  runp<false, 8>(d);
  runp<true, 4>(d);
  runp<true, 2>(d);
  runp2<1, false, 2, 1, false>(d);
  runp2<2, false, 2, 1, false>(d);
  runp2<2, true, 4, 2, false>(d);
  runp2<2, false, 2, 2, false>(d);
  runp2<1, true, 4, 2, false>(d);
  runp2<2, true, 4, 2, true>(d);
  runp2<1, false, 2, 1, true>(d);
  runp2<2, false, 2, 2, true>(d);
  runp2<2, true, 4, 2, true, 16384>(d, 8192);
  runp2<2, true, 4, 2, true, 16384, true>(d, 8192);
  runp2<1, false, 2, 1, false, 16384>(d, 8192);
  runp2<1, false, 2, 1, false, 16384, true>(d, 8192);
  runp2<2, true, 4, 2, true, 16384, true>(d, 65536);
  return 0;
}
