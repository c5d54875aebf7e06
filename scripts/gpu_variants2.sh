#!/bin/bash
for v in "" nofull notempty fixedb; do
  FK_LIB_VARIANT=$v CFG=2 timeout 300 python scripts/sweep.py "FK_DEBUG_FLAGS=3" "FK_DEBUG_FLAGS=3;FK_EPI5=4" 2>&1 | grep -E "variant|rror" | cut -c1-100 | sed "s/^/[$v] /"
done
