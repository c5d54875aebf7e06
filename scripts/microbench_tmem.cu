// TMEM read-throughput microbenchmark (sm_100a): how many bytes/cycle/SM can
// tcgen05.ld move, by shape, repetition and number of warps?  Decides whether
// the 16-bit small-d search is TMEM-read bound (64 KB of fp32 accumulators per
// 128x128 tile).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o
// scripts/microbench_tmem scripts/microbench_tmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int X>
__device__ __forceinline__ void ld32x32b(uint32_t taddr, uint32_t* r);

#define R8(o) "=r"(r[o]), "=r"(r[o + 1]), "=r"(r[o + 2]), "=r"(r[o + 3]), "=r"(r[o + 4]), "=r"(r[o + 5]), "=r"(r[o + 6]), "=r"(r[o + 7])
template <>
__device__ __forceinline__ void ld32x32b<32>(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : R8(0), R8(8), R8(16), R8(24)
      : "r"(taddr));
}
template <>
__device__ __forceinline__ void ld32x32b<16>(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : R8(0), R8(8)
               : "r"(taddr));
}
// 16x256b.x8: 16 lanes x 256 bits, 8 repetitions -> 32 regs per thread
__device__ __forceinline__ void ld16x256b_x8(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : R8(0), R8(8), R8(16), R8(24)
      : "r"(taddr));
}
// 16x128b.x16 -> 32 regs
__device__ __forceinline__ void ld16x128b_x16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x128b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : R8(0), R8(8), R8(16), R8(24)
      : "r"(taddr));
}
__device__ __forceinline__ void ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// mode 0: 32x32b.x32 (4 KB/warp/instr), mode 1: 32x32b.x16, mode 2: 16x256b.x8, mode 3: 16x128b.x16
// per_wait: instructions issued between waits
__global__ void bench(int mode, int iters, int per_wait, unsigned long long* out, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16);
  const int nw = blockDim.x >> 5;
  uint32_t acc = 0;
  uint32_t r[32];
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int j = 0; j < per_wait; ++j) {
      const uint32_t col = ((it * per_wait + j) * 64 + (warp >> 2) * 128) & 448;
      if (mode == 0) ld32x32b<32>(base + col, r);
      else if (mode == 1) ld32x32b<16>(base + col, r);
      else if (mode == 2) ld16x256b_x8(base + col, r);
      else ld16x128b_x16(base + col, r);
      ld_wait();  // registers are reused: wait per instruction (per_wait>1 -> back-to-back after wait)
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += r[i];
    }
  }
  const unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
  (void)nw;
}

// Same but with two independent register sets in flight per wait (ILP in TMEM loads).
__global__ void bench2(int iters, unsigned long long* out, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16);
  uint32_t acc = 0;
  uint32_t r[128];
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t col = (it * 128) & 511;
    ld32x32b<32>(base + col, r);
    ld32x32b<32>(base + col + 32, r + 32);
    ld32x32b<32>(base + col + 64, r + 64);
    ld32x32b<32>(base + col + 96, r + 96);
    ld_wait();
#pragma unroll
    for (int i = 0; i < 128; ++i) acc += r[i];
  }
  const unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

int main() {
  unsigned long long* out;
  uint32_t* sink;
  cudaMalloc(&out, 148 * 8);
  cudaMalloc(&sink, 148 * 1024 * 4);
  const char* names[4] = {"32x32b.x32", "32x32b.x16", "16x256b.x8", "16x128b.x16"};
  const int bytes_per_instr[4] = {4096, 2048, 4096, 4096};  // per warp
  const int iters = 2000;
  for (int mode = 0; mode < 4; ++mode)
    for (int nw : {4, 8, 16}) {
      bench<<<148, nw * 32>>>(mode, iters, 1, out, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("%s nw=%d error %s\n", names[mode], nw, cudaGetErrorString(e));
        return 1;
      }
      unsigned long long h[148];
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      double cyc = 0;
      for (int i = 0; i < 148; ++i) cyc += h[i];
      cyc /= 148;
      const double bytes = (double)bytes_per_instr[mode] * nw * iters;
      printf("%-12s warps=%2d  %.1f B/cyc/SM  (%.0f cyc per 64KB tile)\n", names[mode], nw, bytes / cyc,
             65536.0 / (bytes / cyc));
    }
  for (int nw : {4, 8, 16}) {
    bench2<<<148, nw * 32>>>(iters, out, sink);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    double cyc = 0;
    for (int i = 0; i < 148; ++i) cyc += h[i];
    cyc /= 148;
    const double bytes = 4096.0 * 4 * nw * iters;
    printf("4x x32 per wait warps=%2d  %.1f B/cyc/SM  (%.0f cyc per 64KB tile)\n", nw, bytes / cyc,
           65536.0 / (bytes / cyc));
  }
  return 0;
}
