#!/bin/bash
# Bottleneck decomposition for the 16-bit small-d path (cfg5 shape, 4M rows) and cfg4.
for c in "CFG=5 OVERRIDE=nb=4000000" "CFG=2 OVERRIDE=storage=bf16"; do
  echo "== $c"
  env $c timeout 300 python scripts/sweep.py "FK_EPI=4" "FK_EPI=8" "FK_EPI=4;FK_DEBUG_FLAGS=1" "FK_EPI=8;FK_DEBUG_FLAGS=1" "FK_EPI=4;FK_DEBUG_FLAGS=3" "FK_EPI=8;FK_DEBUG_FLAGS=3" 2>&1 | grep -E "variant|Error|error" | cut -c1-200
done
for e in 4 8; do CFG=5 OVERRIDE=nb=2000000 FK_EPI=$e timeout 120 python scripts/trace.py 2>&1 | tail -4; done
