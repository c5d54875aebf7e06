// fused_knn_kernel instantiations for operand MODE 5 (see fused_launch.cuh).
#include "fused_launch.cuh"
FK_INSTANTIATE_FUSED(5)
