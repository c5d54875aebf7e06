#!/bin/bash
CFG=4 OVERRIDE=nb=2000000 timeout 900 python scripts/sweep.py "" "FK_ACC=1;FK_BN=128" "FK_ACC=1;FK_BN=128;FK_EPI=8" 2>&1 | grep -E "variant|rror" | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    p=d['plan']; print(d['variant'] or '-', d['ms'], d['prep_fused_merge_ms'], 'amode',p['a_mode'],'acc',p['acc_stages'],'epi',p['epi'],'bn',p['bn'],'stages',p['stages'], 'same', d['same_as_first'])
"
