#!/bin/bash
for v in "FK_ACC=3 FK_EPI=8" "FK_ACC=3 FK_EPI=8 FK_DEBUG_FLAGS=4" "FK_ACC=3 FK_EPI=4"; do
  echo "== $v"; env $v CFG=5 OVERRIDE=nb=2000000 timeout 120 python scripts/trace.py 2>&1 | tail -5
done
CFG=5 OVERRIDE=nb=4000000 timeout 300 python scripts/sweep.py "FK_ACC=3;FK_EPI=8" "FK_ACC=3;FK_EPI=8;FK_DEBUG_FLAGS=4" "FK_ACC=3;FK_EPI=4;FK_DEBUG_FLAGS=4" 2>&1 | grep variant | cut -c1-120
