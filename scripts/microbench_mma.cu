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

int main() {
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
