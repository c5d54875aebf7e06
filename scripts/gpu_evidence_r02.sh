#!/bin/bash
# Round-2 evidence pass: GPU suite, bench lines for every config (N=1), the
# ncu launch list of the cfg2 bench command, ncu --set full captures of the
# fused kernel for cfg2/cfg3/cfg4/cfg5 shapes (reports kept in gpurun_out/).
mkdir -p gpurun_out
TAG=${TAG:-r02e}
if [ -z "$NO_TESTS" ]; then
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 --durations=20 > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|ERROR" gpurun_out/pytest_${TAG}.log | tail -20
fi
for c in 2 2 1 3 4 5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_cfg$c.json 2> gpurun_out/bench_${TAG}_cfg$c.err; echo "bench cfg$c rc=$?"
  tail -1 gpurun_out/bench_${TAG}_cfg$c.json | cut -c1-300
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-gate > gpurun_out/launches_bench_${TAG}.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_knn -s 2 -c 1 \
   -o gpurun_out/full2_${TAG} -f python scripts/prof_search.py --config 2 --iters 3 > gpurun_out/ncu_full2_${TAG}.log 2>&1; echo "ncu cfg2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_knn -s 2 -c 1 \
   -o gpurun_out/full3_${TAG} -f python scripts/prof_search.py --config 3 --iters 3 > gpurun_out/ncu_full3_${TAG}.log 2>&1; echo "ncu cfg3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_knn -s 1 -c 1 \
   -o gpurun_out/full4_${TAG} -f python scripts/prof_search.py --config 4 --nb 2000000 --iters 2 > gpurun_out/ncu_full4_${TAG}.log 2>&1; echo "ncu cfg4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_knn -s 1 -c 1 \
   -o gpurun_out/full5_${TAG} -f python scripts/prof_search.py --config 5 --nb 2000000 --iters 2 > gpurun_out/ncu_full5_${TAG}.log 2>&1; echo "ncu cfg5 rc=$?"
ls -la gpurun_out/*.ncu-rep
