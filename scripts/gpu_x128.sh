#!/bin/bash
# one 128-column TMEM load (one-group epilogues: cfg1/cfg3 3xTF32, cfg4 split, cfg5 long fold)
for v in "" x128 "" x128; do
  FK_LIB_VARIANT=$v CFG=1 timeout 300 python scripts/sweep.py "" 2>&1 | grep -E "variant|rror" | cut -c1-80 | sed "s/^/[$v cfg1] /"
  FK_LIB_VARIANT=$v CFG=3 timeout 300 python scripts/sweep.py "" 2>&1 | grep -E "variant|rror" | cut -c1-80 | sed "s/^/[$v cfg3] /"
  FK_LIB_VARIANT=$v CFG=4 OVERRIDE=nb=2000000 timeout 300 python scripts/sweep.py "" 2>&1 | grep -E "variant|rror" | cut -c1-80 | sed "s/^/[$v cfg4-2M] /"
  FK_LIB_VARIANT=$v CFG=5 OVERRIDE=nb=16000000 timeout 600 python scripts/sweep.py "" 2>&1 | grep -E "variant|rror" | cut -c1-80 | sed "s/^/[$v cfg5-16M] /"
done
