#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for c in "CFG=5 OVERRIDE=nb=4000000" "CFG=2 OVERRIDE=storage=bf16" "CFG=2"; do
  echo "== $c"
  env $c timeout 300 python scripts/sweep.py ${SWEEP:-"FK_ACC=2" "FK_ACC=3" "FK_ACC=2;FK_EPI=8" "FK_ACC=3;FK_EPI=8"} 2>&1 | grep -E "variant|Error|error" | cut -c1-150
done
