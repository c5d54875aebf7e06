#!/bin/bash
# default-plan fp32 searches around nq = 4 x SMs (where the rescoring merge
# stops holding every list entry): look for whole-base fallbacks
for nb in 300000 500000 1000000; do for nq in 600 1000 1500; do for k in 1 10 16; do
CFG=2 OVERRIDE=nb=$nb,nq=$nq,k=$k FK_DIAG=1 timeout 300 python scripts/sweep.py "" 2>&1 | grep -E "variant|rror|uncert|fallback" | head -3 | cut -c1-200 | sed "s/^/nb=$nb nq=$nq k=$k /"
done; done; done
