#!/bin/bash
# Bottleneck decomposition of the fused kernel (dev build flags):
# 1 = epilogue skips TMEM loads + compute, 2 = producer skips TMA, 4 = no slow path
mkdir -p gpurun_out
TAG=${TAG:-dc}
for ov in ${OVERRIDES:-"storage=fp16"}; do
FK_DEV_LIB=1 CFG=${CFG:-2} OVERRIDE=$ov timeout 600 python scripts/sweep.py "" "FK_DEBUG_FLAGS=1" "FK_DEBUG_FLAGS=2" "FK_DEBUG_FLAGS=3" "FK_DEBUG_FLAGS=4" ${VARIANTS} 2>&1 | grep -E "variant|rror" | cut -c1-200 | sed "s/^/$ov /"
done
