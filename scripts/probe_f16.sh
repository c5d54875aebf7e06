#!/bin/bash
# cfg2 shape with 16-bit storage: the speed a 16-bit filter pass could reach
mkdir -p gpurun_out
for ov in "storage=fp16" "storage=fp16,k=32" "storage=bf16,k=32"; do
  CFG=2 OVERRIDE=$ov timeout 300 python scripts/sweep.py "" "FK_EPI=4" 2>&1 | grep -E "variant|rror" | sed "s/^/$ov /"
done
CFG=2 timeout 300 python scripts/sweep.py "" 2>&1 | grep -E "variant|rror" | sed "s/^/fp32 /"
