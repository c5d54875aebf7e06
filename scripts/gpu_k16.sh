#!/bin/bash
# fp32 1-pass searches with 10 < k <= 16: 16-deep queues (k' = 16, little or
# no slack for the rounding band) vs 32-deep queues (k' = 32) with one or two
# epilogue groups; diag lines count uncertified queries
for nq in 10000 1000; do for k in 11 12 13 14 16; do
CFG=2 OVERRIDE=nq=$nq,k=$k FK_DIAG=1 timeout 600 python scripts/sweep.py "" "FK_KP=32;FK_EPI5=4" "FK_KP=32" 2>&1 | grep -E "variant|uncertified" | awk '/uncertified/{u=$0; next} {print substr($0,1,120), "|", substr(u, index(u,"uncertified"), 60)}' | sed "s/^/nq=$nq k=$k /"
done; done
