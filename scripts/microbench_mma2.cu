// tcgen05.mma rate with STREAMING operands (sm_100a): the B descriptor walks
// `npos` distinct K-slices of a 128 KB smem ring (as the fused kernel's
// stages do), for
//   * cta_group::1, M=128 N=128 K=16 (kind::f16), A from TMEM (TS) or smem (SS)
//   * cta_group::2, M=256 N=128 K=16: CTA pair, each CTA holds 128 rows of A
//     and 64 rows of B; only the leader issues.
// Reports cycles per instruction and flop/cycle per SM.  Operands are zero.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2401_08281_b200/csrc
//        -o scripts/microbench_mma2 scripts/microbench_mma2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace fk;

__device__ __forceinline__ void mma2_f16_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma2_f16_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

constexpr int SMEM = 192 * 1024;

// cta_group::1: A region at +128 KB (SS), B ring [0, 128 KB)
template <bool TS>
__global__ void mma1(int iters, int npos, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < SMEM / 4 - 256; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
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
  if (warp == 1) {
    constexpr uint32_t idesc = make_idesc(0u, 128, 128);
    const uint64_t b0 = smem_desc_sw128(smem_u32(smem));
    const uint64_t a0 = smem_desc_sw128(smem_u32(smem + 128 * 1024));
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int p = i % npos;  // chunk p/4 (16 KB apart), K-step p%4 (32 B)
      const uint64_t bd = b0 + (uint64_t)(((p >> 2) * 16384) >> 4) + 2 * (p & 3);
      const uint64_t ad = a0 + 2 * (p & 3);
      const uint32_t d = tmem + ((i >> 3) & 1) * 128;
      if (elect_one()) {
        if (TS) mma_f16_ts(d, tmem + 256 + 8 * (p & 3), bd, idesc, 1u);
        else mma_f16(d, ad, bd, idesc, 1u);
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

// cta_group::2: cluster of 2; each CTA: A half (128 rows) at +128 KB, B half
// (64 rows per 8 KB chunk) ring in [0, 128 KB)
template <bool TS>
__global__ void mma2(int iters, int npos, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_ctarank();
  for (int i = threadIdx.x; i < SMEM / 4 - 256; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 32) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 1) {
    constexpr uint32_t idesc = make_idesc(0u, 256, 128);
    const uint64_t b0 = smem_desc_sw128(smem_u32(smem));
    const uint64_t a0 = smem_desc_sw128(smem_u32(smem + 128 * 1024));
    const unsigned long long t0 = clock64();
    if (rank == 0) {
      for (int i = 0; i < iters; ++i) {
        const int p = i % npos;
        const uint64_t bd = b0 + (uint64_t)(((p >> 2) * 8192) >> 4) + 2 * (p & 3);
        const uint64_t ad = a0 + 2 * (p & 3);
        const uint32_t d = tmem + ((i >> 3) & 1) * 128;
        if (elect_one()) {
          if (TS) mma2_f16_ts(d, tmem + 256 + 8 * (p & 3), bd, idesc, 1u);
          else mma2_f16_ss(d, ad, bd, idesc, 1u);
        }
        __syncwarp();
      }
      if (elect_one())
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&bar)),
            "h"((uint16_t)3)
            : "memory");
      __syncwarp();
    }
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

template <class K>
void launch(K k, int cluster, int iters, int npos, unsigned long long* d, const char* name, double flop_per_instr_per_sm) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM + 1024);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = SMEM + 1024;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, iters, npos, d);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%-34s npos %2d: %s\n", name, npos, cudaGetErrorString(e));
    return;
  }
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; ++i) c += h[i];
  c /= 148;
  printf("%-34s npos %2d: %7.1f cyc/instr  %6.0f flop/cyc/SM\n", name, npos, c / iters,
         flop_per_instr_per_sm * iters / c);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int iters = 8192;
  const double f1 = 2.0 * 128 * 128 * 16;  // per SM per instruction (cta_group::1 and ::2 alike)
  for (int npos : {1, 4, 32}) {
    launch(mma1<true>, 1, iters, npos, d, "cta_group::1 TS M128 N128 K16", f1);
    launch(mma1<false>, 1, iters, npos, d, "cta_group::1 SS M128 N128 K16", f1);
    launch(mma2<true>, 2, iters, npos, d, "cta_group::2 TS M256 N128 K16", f1);
    launch(mma2<false>, 2, iters, npos, d, "cta_group::2 SS M256 N128 K16", f1);
  }
  return 0;
}
