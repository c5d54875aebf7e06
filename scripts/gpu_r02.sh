#!/bin/bash
# Round-2 GPU pass: GPU tests, two bench lines (cfg2), per-config timings.
mkdir -p gpurun_out
TAG=${TAG:-r02a}
python -c "import torch; print(torch.cuda.get_device_name(0))"
if [ -z "$NO_TESTS" ]; then
timeout 2400 python -m pytest tests -m gpu -q ${PYTEST_X} --timeout 900 --durations=15 ${PYTEST_ARGS} > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|ERROR" gpurun_out/pytest_${TAG}.log | tail -30
fi
if [ -z "$NO_BENCH" ]; then
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench_${TAG}_$i.json 2> gpurun_out/bench_${TAG}_$i.err; echo "bench rc=$?"
tail -1 gpurun_out/bench_${TAG}_$i.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d.get(k) for k in ('value','ms_per_step','ms_per_step_median','kernel_sum_ms','gpu_launches','clocks')}, d['roofline']['kernel_ms'], d['roofline']['frac'], d['e2e'])"
done
fi
if [ -n "$SWEEP" ]; then
for c in $SWEEP; do CFG=$c timeout 900 python scripts/sweep.py 2>&1 | grep -E "variant|rror" | sed "s/^/cfg$c /"; done > gpurun_out/sweep_${TAG}.jsonl
cut -c1-250 gpurun_out/sweep_${TAG}.jsonl
fi
