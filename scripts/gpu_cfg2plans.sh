#!/bin/bash
# cfg2 MODE 5 plan variants: A placement x epilogue groups x accumulators
CFG=2 timeout 900 python scripts/sweep.py "" "FK_FORCE_AMODE=0" "FK_EPI5=4" "FK_EPI5=4;FK_FORCE_AMODE=1" "FK_ACC=2" "" 2>&1 | grep -E "variant|rror" | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    p=d['plan']; print(d['variant'] or '-', d['ms'], d['prep_fused_merge_ms'], 'amode', p['a_mode'], 'acc', p['acc_stages'], 'epi', p['epi'], 'stages', p['stages'], 'same', d['same_as_first'])
"
