#!/bin/bash
# sweep EPI variants on cfg2 fp32 and the bf16 / fp16 storage of the same shape
for c in "CFG=2" "CFG=2 OVERRIDE=storage=bf16" ${EXTRA_CFGS}; do
  echo "== $c"
  env $c timeout 300 python scripts/sweep.py ${SWEEP:-"FK_EPI=4" "FK_EPI=8"} 2>&1 | grep -E "variant|Error|error" | cut -c1-240
done
