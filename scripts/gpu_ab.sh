#!/bin/bash
for v in "" nofast "" nofast; do
  FK_LIB_VARIANT=$v CFG=2 timeout 300 python scripts/sweep.py "" "FK_DEBUG_FLAGS=3" 2>&1 | grep -E "variant|rror" | cut -c1-100 | sed "s/^/[$v] /"
done
CFG=5 OVERRIDE=nb=4000000 timeout 300 python scripts/sweep.py "" 2>&1 | grep -E "variant|rror" | cut -c1-100
FK_LIB_VARIANT=nofast CFG=5 OVERRIDE=nb=4000000 timeout 300 python scripts/sweep.py "" 2>&1 | grep -E "variant|rror" | cut -c1-100 | sed "s/^/[nofast] /"
FK_DIAG=1 CFG=1 timeout 300 python scripts/sweep.py "FK_FP32_1PASS_MINROWS=0" 2>&1 | grep -E "variant|rror|uncert" | sort | uniq -c | cut -c1-140
for k in 32 64 100 128; do FK_DIAG=1 CFG=2 OVERRIDE=k=$k timeout 300 python scripts/sweep.py "" "FK_FP32_1PASS_MAXK=2048" 2>&1 | grep -E "variant|rror|uncert" | sort | uniq -c | cut -c1-140 | sed "s/^/k=$k /"; done
