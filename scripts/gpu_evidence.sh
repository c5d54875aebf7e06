#!/bin/bash
# Evidence pass: bench line (N=1, cfg2), the ncu launch list of the same bench
# command, one ncu --set full capture of the fused kernel (cfg2 and the cfg5
# shape; reports stay in /tmp, their summaries land in gpurun_out/), plus
# per-config timings.
mkdir -p gpurun_out /tmp/reps
TAG=${TAG:-r01}
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
tail -1 gpurun_out/bench_${TAG}.json | cut -c1-400
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches_bench_${TAG}.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_knn -s 2 -c 1 \
   -o /tmp/reps/full_${TAG} -f python scripts/prof_search.py --config 2 --iters 3 > gpurun_out/ncu_full_${TAG}.log 2>&1; echo "ncu full rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_knn -s 1 -c 1 \
   -o /tmp/reps/full5_${TAG} -f python scripts/prof_search.py --config 5 --nb 2000000 --iters 2 > gpurun_out/ncu_full5_${TAG}.log 2>&1; echo "ncu full cfg5 rc=$?"
python scripts/make_profiles.py ${TAG} --reps /tmp/reps --out gpurun_out/profiles_${TAG}
for c in 1 3 4 5; do CFG=$c timeout 900 python scripts/sweep.py 2>&1 | grep -E "variant|rror" | sed "s/^/cfg$c /"; done > gpurun_out/sweep_${TAG}.jsonl
cat gpurun_out/sweep_${TAG}.jsonl | cut -c1-200
