#!/bin/bash
# cfg3 main pass (the 4th fused launch: bound, main per search) and the cfg5
# kernel at 4M rows, where the one-epilogue-group plan of the full 100M-row
# search applies (nq * rows * dp >= 4e12); then the cfg1 1-pass sweeps
mkdir -p gpurun_out
TAG=${TAG:-r02n}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_knn -s 3 -c 1 \
   -o gpurun_out/full3_${TAG} -f python scripts/prof_search.py --config 3 --iters 3 > gpurun_out/ncu_full3_${TAG}.log 2>&1; echo "ncu cfg3 main rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_knn -s 1 -c 1 \
   -o gpurun_out/full5b_${TAG} -f python scripts/prof_search.py --config 5 --nb 4000000 --iters 2 > gpurun_out/ncu_full5b_${TAG}.log 2>&1; echo "ncu cfg5 4M rc=$?"
grep plan gpurun_out/ncu_full3_${TAG}.log gpurun_out/ncu_full5b_${TAG}.log | cut -c1-300
bash scripts/gpu_r02m_sweeps.sh
