#!/bin/bash
# same sweep across experiment library variants (FK_LIB_VARIANT)
for v in "" spin hint1k; do
  FK_LIB_VARIANT=$v CFG=${CFG:-2} OVERRIDE=${OVERRIDE:-} timeout 300 python scripts/sweep.py "" "FK_DEBUG_FLAGS=3" ${VARIANTS} 2>&1 | grep -E "variant|rror" | cut -c1-110 | sed "s/^/[$v] /"
done
