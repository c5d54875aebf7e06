// tcgen05.mma issue-rate microbenchmark (sm_100a): cycles per instruction for
// M=128, N in {64,128,256}, kind::f16 (K=16) and kind::tf32 (K=8), A from TMEM
// (TS) or shared memory (SS).  Operands are zero-filled smem / TMEM: only the
// pipe rate is measured.  One CTA per SM, one elected issuing thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2401_08281_b200/csrc
//        -o scripts/microbench_mma scripts/microbench_mma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace fk;

template <bool TF32, bool TS, int N>
__global__ void mma_rate(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (warp == 0) tmem_alloc(&slot, 512);
  if (threadIdx.x == 32) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 32) {
    constexpr uint32_t idesc = make_idesc(TF32 ? 2u : 1u, 128, N);
    const uint64_t bdesc = smem_desc_sw128(smem_u32(smem));
    const uint64_t adesc = smem_desc_sw128(smem_u32(smem + 32768));
    const uint32_t a_tm = tmem + 256 + (N == 256 ? 0 : 0);  // A columns (TS); overlaps D for N=256 (values irrelevant)
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = tmem + ((i & 1) && N <= 128 ? 128 : 0);
      if (TF32) {
        if (TS) mma_tf32_ts(d, a_tm, bdesc, idesc, 1u);
        else mma_tf32(d, adesc, bdesc, idesc, 1u);
      } else {
        if (TS) mma_f16_ts(d, a_tm, bdesc, idesc, 1u);
        else mma_f16(d, adesc, bdesc, idesc, 1u);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <bool TF32, bool TS, int N>
void run(const char* name, unsigned long long* dout) {
  auto k = mma_rate<TF32, TS, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  const int iters = 4096;
  k<<<148, 128, 65536 + 1024>>>(iters, dout);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(e));
    return;
  }
  unsigned long long h[148];
  cudaMemcpy(h, dout, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; ++i) c += h[i];
  c /= 148;
  const double kdim = TF32 ? 8 : 16;
  const double flop = 2.0 * 128 * N * kdim;
  printf("%-22s %.1f cyc/instr  %.0f flop/cyc/SM\n", name, c / iters, flop * iters / c);
}

int main2();
int main() {
  if (main2()) return 1;
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  run<false, true, 128>("f16  TS  M128 N128", d);
  run<false, false, 128>("f16  SS  M128 N128", d);
  run<false, true, 256>("f16  TS  M128 N256", d);
  run<false, false, 256>("f16  SS  M128 N256", d);
  run<false, true, 64>("f16  TS  M128 N64", d);
  run<true, true, 128>("tf32 TS  M128 N128", d);
  run<true, false, 128>("tf32 SS  M128 N128", d);
  run<true, true, 256>("tf32 TS  M128 N256", d);
  return 0;
}

// ---------------------------------------------------------------------------
// Contention: one warp streams kind::f16 M128 N128 K16 MMAs into TMEM columns
// [0,128) while `nld` warps read columns [256,384) with tcgen05.ld 32x32b.x32
// (2 per wait, results consumed).  Reports MMA cycles/instr and per-warp LDTM
// round-trip latency with and without the MMA stream.
__global__ void contention(int iters, int mma_on, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  __shared__ int done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (warp == 0) tmem_alloc(&slot, 512);
  if (threadIdx.x == 32) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    done = 0;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 1) {
    if (mma_on) {
      constexpr uint32_t idesc = make_idesc(1u, 128, 128);
      const uint64_t bdesc = smem_desc_sw128(smem_u32(smem));
      const unsigned long long t0 = clock64();
      int n = 0;
      const int nld = (blockDim.x >> 5) - 4;
      while (*(volatile int*)&done < nld) {
        if (elect_one()) mma_f16_ts(tmem + ((n & 1) ? 128 : 0), tmem + 448, bdesc, idesc, 1u);
        __syncwarp();
        ++n;
      }
      if (elect_one()) mma_commit(&bar);
      __syncwarp();
      mbar_wait(&bar, 0);
      const unsigned long long t1 = clock64();
      if (lane == 0) out[blockIdx.x * 4 + 0] = (t1 - t0) * 1000 / (unsigned long long)max(n, 1);
    }
  } else if (warp >= 4) {
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 256 + ((warp >> 2) & 1) * 64;
    uint32_t r[64];
    uint32_t acc = 0;
    unsigned long long lat = 0;
    for (int it = 0; it < iters; ++it) {
      const unsigned long long a = clock64();
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
            "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
            "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
            "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(base));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += r[i];
      asm volatile("" ::"r"(acc));
      lat += clock64() - a;
    }
    if (lane == 0 && warp == 4) out[blockIdx.x * 4 + 1] = lat / iters;
    if (acc == 0xdeadbeef) out[blockIdx.x * 4 + 2] = acc;
    __syncwarp();
    if (lane == 0) atomicAdd(&done, 1);
  }
  __syncthreads();
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int main2() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 4 * 8);
  cudaFuncSetAttribute(contention, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  for (int nw : {4, 8}) {
    for (int on : {0, 1}) {
      cudaMemset(d, 0, 148 * 4 * 8);
      contention<<<148, 128 + 32 * nw, 65536 + 1024>>>(4000, on, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("err %s\n", cudaGetErrorString(e));
        return 1;
      }
      unsigned long long h[148 * 4];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("ld warps=%d mma=%d: LDTM x32 round trip %llu cyc, MMA %.1f cyc/instr\n", nw, on, h[1],
             h[0] / 1000.0);
    }
  }
  return 0;
}
