#!/bin/bash
# cfg1 (100k rows, below the 1-pass row floor) through the 1-pass scaled-fp16
# filter vs 3xTF32, and the floor itself at 200k rows
mkdir -p gpurun_out
for nb in 100000 200000; do
CFG=1 OVERRIDE=nb=$nb timeout 600 python scripts/sweep.py "" "FK_FP32_1PASS_MINROWS=50000" "FK_FP32_1PASS_MINROWS=50000;FK_EPI5=4" "" 2>&1 | grep -E "variant|rror" | cut -c1-330 | sed "s/^/nb=$nb /"
done
for nq in 100 10000; do
CFG=1 OVERRIDE=nq=$nq timeout 600 python scripts/sweep.py "" "FK_FP32_1PASS_MINROWS=50000" 2>&1 | grep -E "variant|rror" | cut -c1-330 | sed "s/^/nq=$nq /"
done
