#!/bin/bash
# Round re-entry check: smoke, GPU tests, bench line, per-config sweep.
mkdir -p gpurun_out
bash scripts/gpu_check.sh
for c in 1 3 4 5; do
  echo "== cfg$c"
  CFG=$c timeout 600 python scripts/sweep.py 2>&1 | grep -E "variant|Error|error" | cut -c1-300
done
