#!/bin/bash
for c in "CFG=2" "CFG=2 OVERRIDE=storage=bf16"; do
  env $c python scripts/sweep.py "FK_DEBUG_FLAGS=0" "FK_DEBUG_FLAGS=1" "FK_DEBUG_FLAGS=2" "FK_DEBUG_FLAGS=3" "FK_DEBUG_FLAGS=1;FK_EPI=8" "FK_DEBUG_FLAGS=0;FK_EPI=8" 2>&1 | grep variant
done
