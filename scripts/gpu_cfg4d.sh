#!/bin/bash
# cfg4 shape under the split plan: decomposition + multicast
CFG=4 OVERRIDE=nb=2000000 timeout 900 python scripts/sweep.py "" "FK_DEBUG_FLAGS=1" "FK_DEBUG_FLAGS=3" "FK_CLUSTER=2" "FK_STAGES=6" "" "FK_CLUSTER=2" 2>&1 | grep -E "variant|rror" | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    p=d['plan']; print(d['variant'] or '-', d['ms'], d['prep_fused_merge_ms'], 'amode', p['a_mode'], 'acc', p['acc_stages'], 'epi', p['epi'], 'stages', p['stages'], 'same', d['same_as_first'])
"
