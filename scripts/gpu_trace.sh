#!/bin/bash
# clock64 timelines (dev build) of the fused kernel for a few variants
mkdir -p gpurun_out
for v in "${@:-}"; do
  echo "=== variant: $v"
  env $v timeout 300 python scripts/trace.py 2>&1 | tail -12
done
