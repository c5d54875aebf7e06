// Peer-memory exchange for the row-sharded index (the fused
// alternative to NCCL all-gather + merge): every rank exports ONE device
// block (CUDA IPC) holding its per-search top-k lists and two counters; each
// rank's merge kernel reads every peer's lists directly over NVLink P2P (or
// the same device) and writes the single-index answer -- no collective, no
// host round trip.
//
// Block layout: [ready u32 | done u32 | blocks-finished u32 | error u32 | pad
// to 256 B][D f32 cap][P i64 cap][I i64 cap], cap = nq_cap * k_cap.
//
// One search (sequence number s = 1, 2, ...), all on the rank's stream:
//   1. fk_xchg_acquire: wait until every peer's `done` >= s-1 (peers have
//      finished reading this rank's previous lists) -- then the lists may be
//      overwritten;
//   2. the local search writes D / global positions / ids (fk_xchg_put);
//   3. fk_xchg_merge: `ready` = s (release, system scope); one kernel waits
//      for every peer's `ready` >= s (acquire), merges by (distance, global
//      position) exactly like fk_merge_shards, and its last block sets
//      `done` = s.
// Spin waits are bounded (FK_XCHG_TIMEOUT_MS, default 20 s): on timeout the
// kernel records an error (fk_xchg_status) instead of hanging the GPU.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "fk_host.cuh"

using namespace fk;
using fkh::set_err;

namespace {

constexpr int XMAX = 64;          // ranks
constexpr size_t HDR = 256;       // header bytes of an exported block
constexpr int XHANDLE = sizeof(cudaIpcMemHandle_t);

struct Peer {
  const float* D;
  const int64_t* P;
  const int64_t* I;
  const unsigned int* ctr;  // [ready, done, ...]
};
struct Peers {
  Peer p[XMAX];
};

__device__ __forceinline__ unsigned int ld_acquire_sys(const unsigned int* a) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned int* a, unsigned int v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Wait until ctr[which] >= want on every peer (one thread); false on timeout.
__device__ bool wait_peers(const Peers& ps, int n, int which, unsigned int want, unsigned long long timeout_ns) {
  const unsigned long long t0 = gtimer();
  for (int g = 0; g < n; ++g) {
    while (ld_acquire_sys(ps.p[g].ctr + which) < want) {
      if (gtimer() - t0 > timeout_ns) return false;
      __nanosleep(256);
    }
  }
  return true;
}

__global__ void xchg_acquire_kernel(Peers ps, int n, unsigned int want, unsigned long long timeout_ns,
                                    unsigned int* my_ctr) {
  if (threadIdx.x == 0 && !wait_peers(ps, n, 1, want, timeout_ns)) atomicOr(my_ctr + 3, 1u);
}

__global__ void xchg_signal_kernel(unsigned int* ctr, unsigned int v) {
  if (threadIdx.x == 0) {
    __threadfence_system();
    st_release_sys(ctr, v);
  }
}

template <bool IS_IP>
__global__ void xchg_merge_kernel(Peers ps, int nshard, int nq, int k, int stride_k, unsigned int seq,
                                  unsigned long long timeout_ns, unsigned int* my_ctr, float* __restrict__ D,
                                  int64_t* __restrict__ I) {
  __shared__ int ok;
  if (threadIdx.x == 0) {
    ok = wait_peers(ps, nshard, 0, seq, timeout_ns) ? 1 : 0;
    if (!ok) atomicOr(my_ctr + 3, 2u);
  }
  __syncthreads();
  const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (ok && q < nq) {
    // lane l owns shards l, l+32: head-of-list merge by (key, global position)
    auto head = [&](int s, int h, int64_t& id) -> uint64_t {
      if (s >= nshard || h >= k) return ~0ull;
      const size_t o = (size_t)q * stride_k + h;
      const int64_t pos = ps.p[s].P[o];
      if (pos < 0) return ~0ull;
      id = ps.p[s].I[o];
      return (static_cast<uint64_t>(dist_key(ps.p[s].D[o], IS_IP)) << 32) | static_cast<uint32_t>(pos);
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
        D[o] = w == ~0ull ? (IS_IP ? -INFINITY : INFINITY) : key_dist(static_cast<uint32_t>(w >> 32), IS_IP);
        I[o] = w == ~0ull ? -1 : wid;
      }
    }
  }
  // the last block to finish publishes done = seq (peers may reuse their lists)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned int fin = atomicAdd(my_ctr + 2, 1u);
    if (fin == gridDim.x - 1) {
      my_ctr[2] = 0u;
      st_release_sys(my_ctr + 1, seq);
    }
  }
}

}  // namespace

struct fk_xchg {
  int device = 0, rank = 0, world = 1;
  int64_t nq_cap = 0;
  int k_cap = 0;
  void* block = nullptr;  // this rank's exported block
  size_t bytes = 0;
  void* peer_base[XMAX] = {nullptr};
  Peers peers{};
  bool connected = false;
  unsigned int seq = 0;
  unsigned long long timeout_ns = 20000000000ull;
};

extern "C" {

int fk_xchg_create(int device, int rank, int world, int64_t nq_cap, int k_cap, fk_xchg** out, void* handle_out) {
  if (!out || !handle_out) return set_err(FK_E_INVALID, "NULL argument");
  if (world < 1 || world > XMAX || rank < 0 || rank >= world) return set_err(FK_E_INVALID, "bad rank/world");
  if (nq_cap < 1 || k_cap < 1) return set_err(FK_E_INVALID, "bad capacity");
  CK(cudaSetDevice(device));
  auto* x = new fk_xchg;
  x->device = device;
  x->rank = rank;
  x->world = world;
  x->nq_cap = nq_cap;
  x->k_cap = k_cap;
  const size_t cap = (size_t)nq_cap * k_cap;
  x->bytes = HDR + cap * (4 + 8 + 8);
  if (const char* e = getenv("FK_XCHG_TIMEOUT_MS")) x->timeout_ns = (unsigned long long)atoll(e) * 1000000ull;
  cudaError_t e = cudaMalloc(&x->block, x->bytes);
  if (e == cudaSuccess) e = cudaMemset(x->block, 0, HDR);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t*>(handle_out), x->block);
  if (e != cudaSuccess) {
    if (x->block) cudaFree(x->block);
    delete x;
    return set_err(FK_E_CUDA, "exchange block: %s", cudaGetErrorString(e));
  }
  *out = x;
  return FK_OK;
}

int fk_xchg_handle_bytes(void) { return XHANDLE; }

// all_handles: world x fk_xchg_handle_bytes(), rank order (this rank's own
// entry is ignored: its block is used directly)
int fk_xchg_connect(fk_xchg* x, const void* all_handles) {
  if (!x || !all_handles) return set_err(FK_E_INVALID, "NULL argument");
  CK(cudaSetDevice(x->device));
  const size_t cap = (size_t)x->nq_cap * x->k_cap;
  for (int g = 0; g < x->world; ++g) {
    void* base = x->block;
    if (g != x->rank) {
      cudaIpcMemHandle_t hd;
      std::memcpy(&hd, static_cast<const uint8_t*>(all_handles) + (size_t)g * XHANDLE, XHANDLE);
      CK(cudaIpcOpenMemHandle(&base, hd, cudaIpcMemLazyEnablePeerAccess));
      x->peer_base[g] = base;
    }
    auto* b = static_cast<uint8_t*>(base);
    x->peers.p[g].ctr = reinterpret_cast<const unsigned int*>(b);
    x->peers.p[g].D = reinterpret_cast<const float*>(b + HDR);
    x->peers.p[g].P = reinterpret_cast<const int64_t*>(b + HDR + cap * 4);
    x->peers.p[g].I = reinterpret_cast<const int64_t*>(b + HDR + cap * 12);
  }
  x->connected = true;
  return FK_OK;
}

// Step 1: before the local search overwrites this rank's lists.
int fk_xchg_acquire(fk_xchg* x, void* stream) {
  if (!x || !x->connected) return set_err(FK_E_INVALID, "exchange not connected");
  CK(cudaSetDevice(x->device));
  xchg_acquire_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      x->peers, x->world, x->seq, x->timeout_ns, static_cast<unsigned int*>(x->block));
  CKL();
  return FK_OK;
}

// Step 2: copy this rank's results (device, nq x k: distances, GLOBAL
// positions, ids) into the exported block.
int fk_xchg_put(fk_xchg* x, int64_t nq, int k, const float* D, const int64_t* P, const int64_t* I, void* stream) {
  if (!x) return set_err(FK_E_INVALID, "NULL exchange");
  if (nq > x->nq_cap || k > x->k_cap) return set_err(FK_E_INVALID, "results exceed the exchange capacity");
  CK(cudaSetDevice(x->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t cap = (size_t)x->nq_cap * x->k_cap;
  auto* b = static_cast<uint8_t*>(x->block);
  // rows are stored with stride k_cap (the peers' merge reads that layout)
  CK(cudaMemcpy2DAsync(b + HDR, (size_t)x->k_cap * 4, D, (size_t)k * 4, (size_t)k * 4, nq, cudaMemcpyDeviceToDevice,
                       st));
  CK(cudaMemcpy2DAsync(b + HDR + cap * 4, (size_t)x->k_cap * 8, P, (size_t)k * 8, (size_t)k * 8, nq,
                       cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpy2DAsync(b + HDR + cap * 12, (size_t)x->k_cap * 8, I, (size_t)k * 8, (size_t)k * 8, nq,
                       cudaMemcpyDeviceToDevice, st));
  return FK_OK;
}

// Step 3: publish, wait for every peer's lists, merge into D_out / I_out.
int fk_xchg_merge(fk_xchg* x, int metric, int64_t nq, int k, float* D_out, int64_t* I_out, void* stream) {
  if (!x || !x->connected) return set_err(FK_E_INVALID, "exchange not connected");
  if (nq > x->nq_cap || k > x->k_cap) return set_err(FK_E_INVALID, "results exceed the exchange capacity");
  CK(cudaSetDevice(x->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const unsigned int seq = ++x->seq;
  auto* ctr = static_cast<unsigned int*>(x->block);
  xchg_signal_kernel<<<1, 32, 0, st>>>(ctr, seq);
  CKL();
  const int wpb = 8;
  const unsigned grid = (unsigned)std::max<int64_t>(1, (nq + wpb - 1) / wpb);
  if (metric == FK_METRIC_IP)
    xchg_merge_kernel<true><<<grid, wpb * 32, 0, st>>>(x->peers, x->world, (int)nq, k, x->k_cap, seq, x->timeout_ns,
                                                       ctr, D_out, I_out);
  else
    xchg_merge_kernel<false><<<grid, wpb * 32, 0, st>>>(x->peers, x->world, (int)nq, k, x->k_cap, seq, x->timeout_ns,
                                                        ctr, D_out, I_out);
  CKL();
  return FK_OK;
}

// Synchronises the device and reports a timed-out wait (FK_E_CUDA) if any.
int fk_xchg_status(fk_xchg* x) {
  if (!x) return set_err(FK_E_INVALID, "NULL exchange");
  CK(cudaSetDevice(x->device));
  CK(cudaDeviceSynchronize());
  unsigned int err = 0;
  CK(cudaMemcpy(&err, static_cast<unsigned int*>(x->block) + 3, 4, cudaMemcpyDeviceToHost));
  if (err) return set_err(FK_E_CUDA, "peer exchange wait timed out (code %u)", err);
  return FK_OK;
}

void fk_xchg_destroy(fk_xchg* x) {
  if (!x) return;
  cudaSetDevice(x->device);
  cudaDeviceSynchronize();
  for (int g = 0; g < XMAX; ++g)
    if (x->peer_base[g]) cudaIpcCloseMemHandle(x->peer_base[g]);
  if (x->block) cudaFree(x->block);
  delete x;
}

}  // extern "C"
