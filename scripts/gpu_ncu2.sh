#!/bin/bash
# one ncu --set full capture of the cfg2 fused kernel (TAG names the report)
TAG=${TAG:-x}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_knn -s 2 -c 1 \
   -o gpurun_out/full2_${TAG} -f python scripts/prof_search.py --config 2 --iters 3 > gpurun_out/ncu_full2_${TAG}.log 2>&1; echo "ncu cfg2 rc=$?"
