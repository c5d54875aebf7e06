#!/bin/bash
# SS (A in smem) vs TS (A in TMEM) MMA on the 16-bit filter path, cfg2 shape
for ov in "storage=fp32" "storage=fp16"; do
CFG=2 OVERRIDE=$ov timeout 600 python scripts/sweep.py "" "FK_FORCE_AMODE=0" "FK_EPI5=4;FK_EPI=4" "FK_EPI5=4;FK_EPI=4;FK_FORCE_AMODE=1" "FK_EPI5=4;FK_EPI=4;FK_FORCE_AMODE=1;FK_ACC=2" "FK_FORCE_AMODE=1;FK_ACC=2" 2>&1 | grep -E "variant|rror" | cut -c1-330 | sed "s/^/$ov /"
done
