// Definition of fkh::launch_fused_mode<MODE>: template dispatch from the
// runtime plan (epilogue width, queue bucket, metric, tile width, cluster
// mode) to the fused_knn_kernel instantiations of one operand MODE.
// Included only by fused_m<MODE>.cu, which instantiates it once.
#pragma once
#include "fk_host.cuh"

namespace fkh {

template <int MODE, int KQ, bool IP, int EPI, int TBN>
int launch_fused_tb(const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b0, const CUtensorMap& b1,
                    const fk::SearchParams& sp, int grid, int smem, cudaStream_t st) {
  auto kern = fk::fused_knn_kernel<MODE, KQ, IP, EPI, TBN>;
  static std::atomic<uint64_t> configured{0};  // per instantiation, per device
  int rc = once_per_device(configured, [&]() -> int {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
    return FK_OK;
  });
  if (rc) return rc;
  if (sp.cluster == 2) {  // CTA pairs sharing base tiles (TMA multicast)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(128 + 32 * EPI);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, kern, a0, a1, b0, b1, sp));
  } else {
    kern<<<grid, 128 + 32 * EPI, smem, st>>>(a0, a1, b0, b1, sp);
  }
  CKL();
  return FK_OK;
}

// 64-column tiles are instantiated only for each storage's default epilogue
// width (fp32: 4 warps, 16-bit: 8)
template <int MODE, int KQ, bool IP, int EPI>
int launch_fused_t(const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b0, const CUtensorMap& b1,
                   const fk::SearchParams& sp, int grid, int smem, cudaStream_t st) {
  if (sp.bn == 64) {
    if constexpr ((MODE == 0 || MODE == 4) == (EPI == 4))
      return launch_fused_tb<MODE, KQ, IP, EPI, 64>(a0, a1, b0, b1, sp, grid, smem, st);
    return set_err(FK_E_UNSUPPORTED, "64-column tiles need the default epilogue width");
  }
  return launch_fused_tb<MODE, KQ, IP, EPI, 128>(a0, a1, b0, b1, sp, grid, smem, st);
}

template <int MODE, bool IP, int EPI>
int launch_fused_k(int kq, const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b0,
                   const CUtensorMap& b1, const fk::SearchParams& sp, int grid, int smem, cudaStream_t st) {
  switch (kq) {
    case 8: return launch_fused_t<MODE, 8, IP, EPI>(a0, a1, b0, b1, sp, grid, smem, st);
    case 16: return launch_fused_t<MODE, 16, IP, EPI>(a0, a1, b0, b1, sp, grid, smem, st);
    case 32: return launch_fused_t<MODE, 32, IP, EPI>(a0, a1, b0, b1, sp, grid, smem, st);
    case 0: return launch_fused_t<MODE, 0, IP, EPI>(a0, a1, b0, b1, sp, grid, smem, st);
    case -1:  // range search: default epilogue width only (not on the MODE 5 filter)
      if constexpr (MODE != 5 && (MODE == 0 || MODE == 4) == (EPI == 4))
        return launch_fused_t<MODE, -1, IP, EPI>(a0, a1, b0, b1, sp, grid, smem, st);
      return set_err(FK_E_UNSUPPORTED, "range search runs with the default epilogue width");
  }
  return set_err(FK_E_UNSUPPORTED, "queue bucket %d", kq);
}

template <int MODE>
int launch_fused_mode(int epi, bool ip, int kq, const CUtensorMap& a0, const CUtensorMap& a1,
                      const CUtensorMap& b0, const CUtensorMap& b1, const fk::SearchParams& sp, int grid, int smem,
                      cudaStream_t st) {
  if constexpr (MODE == 3) {  // folded bf16 norms: L2 only
    if (ip) return set_err(FK_E_INVALID, "folded norms are an L2 layout");
    return epi == 8 ? launch_fused_k<3, false, 8>(kq, a0, a1, b0, b1, sp, grid, smem, st)
                    : launch_fused_k<3, false, 4>(kq, a0, a1, b0, b1, sp, grid, smem, st);
  } else {
    if (epi == 8)
      return ip ? launch_fused_k<MODE, true, 8>(kq, a0, a1, b0, b1, sp, grid, smem, st)
                : launch_fused_k<MODE, false, 8>(kq, a0, a1, b0, b1, sp, grid, smem, st);
    return ip ? launch_fused_k<MODE, true, 4>(kq, a0, a1, b0, b1, sp, grid, smem, st)
              : launch_fused_k<MODE, false, 4>(kq, a0, a1, b0, b1, sp, grid, smem, st);
  }
}

}  // namespace fkh

#define FK_INSTANTIATE_FUSED(M)                                                                              \
  template int fkh::launch_fused_mode<M>(int, bool, int, const CUtensorMap&, const CUtensorMap&,             \
                                         const CUtensorMap&, const CUtensorMap&, const fk::SearchParams&, int, \
                                         int, cudaStream_t);
