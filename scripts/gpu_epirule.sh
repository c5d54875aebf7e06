#!/bin/bash
# when does one epilogue group beat two on 16-bit data? (fold L2 / IP / plain L2; small and large bases)
for ov in "nb=1000000" "nb=16000000"; do
  CFG=5 OVERRIDE=$ov timeout 900 python scripts/sweep.py "" "FK_EPI=4" "" "FK_EPI=4" 2>&1 | grep -E "variant|rror" | cut -c1-75 | sed "s/^/fold-bf16-d96 $ov /"
done
CFG=2 OVERRIDE=storage=fp16,metric=ip timeout 900 python scripts/sweep.py "" "FK_EPI=4" "" "FK_EPI=4" 2>&1 | grep -E "variant|rror" | cut -c1-75 | sed "s/^/ip-fp16-d128 /"
CFG=2 OVERRIDE=storage=bf16,d=96 timeout 900 python scripts/sweep.py "" "FK_EPI=4" 2>&1 | grep -E "variant|rror" | cut -c1-75 | sed "s/^/fold-bf16-d96-1M-cfg2q /"
CFG=2 OVERRIDE=storage=fp16 timeout 900 python scripts/sweep.py "" "FK_EPI=4" 2>&1 | grep -E "variant|rror" | cut -c1-75 | sed "s/^/l2-fp16-d128 /"
