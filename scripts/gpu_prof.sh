#!/bin/bash
# ncu capture of the fused kernel + launch list of the bench command.
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_knn -s 1 -c 1 \
   -o gpurun_out/prof_${TAG} -f python scripts/prof_search.py --config ${CFG:-2} --iters 2 ${PROF_ARGS} > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_${TAG}.log
if [ -n "$LAUNCHES" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches_bench_${TAG}.log 2>&1
echo "launches rc=$?"
fi
