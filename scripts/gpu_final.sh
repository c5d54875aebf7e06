#!/bin/bash
# end-of-round validation: GPU suite, every config's bench line, range search timing
TAG=${TAG:-r02i}
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 --durations=15 > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|ERROR" gpurun_out/pytest_${TAG}.log | tail -5
for c in 2 1 3 4 5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_cfg$c.json 2> gpurun_out/bench_${TAG}_cfg$c.err; echo "bench cfg$c rc=$?"
  tail -1 gpurun_out/bench_${TAG}_cfg$c.json | cut -c1-200
done
for s in 1e-5 1e-4; do SEL=$s CFG=2 timeout 600 python scripts/range_bench.py 2>&1 | tail -1; done
