#!/bin/bash
# bench (cfg2) + decomposition (MODE 5 fp32 and MODE 1 fp16) + ncu full of the MODE 5 fused kernel
mkdir -p gpurun_out
TAG=${TAG:-r02c}
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
tail -1 gpurun_out/bench_${TAG}.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d.get(k) for k in ('value','ms_per_step','kernel_sum_ms','gpu_launches')}, d['roofline']['kernel_ms'], d['roofline']['merge_ms'], d['roofline']['frac'], d['e2e']['value'])"
OVERRIDES="storage=fp32 storage=fp16" bash scripts/gpu_decomp.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_knn -s 2 -c 1 \
   -o gpurun_out/full_${TAG} -f python scripts/prof_search.py --config 2 --iters 3 > gpurun_out/ncu_full_${TAG}.log 2>&1; echo "ncu full rc=$?"
