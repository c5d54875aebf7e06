#!/bin/bash
# cfg5 16M-row shape under the one-group plan: CTA-pair multicast, stage depth
CFG=5 OVERRIDE=nb=16000000 timeout 900 python scripts/sweep.py "" "FK_CLUSTER=2" "FK_STAGES=8" "" "FK_CLUSTER=2" 2>&1 | grep -E "variant|rror" | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    p=d['plan']; print(d['variant'] or '-', d['ms'], d['prep_fused_merge_ms'], 'amode', p['a_mode'], 'acc', p['acc_stages'], 'epi', p['epi'], 'stages', p['stages'], 'same', d['same_as_first'])
"
