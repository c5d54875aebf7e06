#!/bin/bash
# upper bound on a folded MODE 5 epilogue: no-insertion timing with / without the per-column norm term
for v in "" noxn; do
  FK_LIB_VARIANT=$v CFG=2 timeout 300 python scripts/sweep.py "FK_DEBUG_FLAGS=4" "FK_DEBUG_FLAGS=4" "FK_DEBUG_FLAGS=3" 2>&1 | grep -E "variant|rror" | cut -c1-100 | sed "s/^/[$v] /"
done
