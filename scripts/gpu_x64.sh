#!/bin/bash
for v in "" x64 "" x64; do
  FK_LIB_VARIANT=$v CFG=2 timeout 300 python scripts/sweep.py "" 2>&1 | grep -E "variant|rror" | cut -c1-90 | sed "s/^/[$v] /"
  FK_LIB_VARIANT=$v CFG=5 OVERRIDE=nb=4000000 timeout 300 python scripts/sweep.py "" 2>&1 | grep -E "variant|rror" | cut -c1-90 | sed "s/^/[$v cfg5-4M] /"
done
