#!/bin/bash
TAG=${TAG:-r02h}
for c in 3 2; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_cfg$c.json 2> gpurun_out/bench_${TAG}_cfg$c.err; echo "bench cfg$c rc=$?"
  tail -1 gpurun_out/bench_${TAG}_cfg$c.json | cut -c1-300
done
