#!/bin/bash
# MMA-only rate (dev flags 3) with A in smem (SS) vs TMEM (TS)
for c in "2 storage=fp16" "2 storage=fp32" "5 nb=4000000"; do set -- $c
FK_DEV_LIB=1 CFG=$1 OVERRIDE=$2 timeout 600 python scripts/sweep.py "FK_DEBUG_FLAGS=3" "FK_DEBUG_FLAGS=3;FK_FORCE_AMODE=0" "FK_DEBUG_FLAGS=3;FK_FORCE_AMODE=1;FK_ACC=2" "FK_DEBUG_FLAGS=1;FK_FORCE_AMODE=0" "FK_FORCE_AMODE=0" 2>&1 | grep -E "variant|rror" | cut -c1-250 | sed "s/^/cfg$1 $2 /"
done
