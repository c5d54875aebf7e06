#!/bin/bash
for ov in "metric=ip" "storage=fp16,metric=ip" "storage=fp16"; do
CFG=2 OVERRIDE=$ov timeout 600 python scripts/sweep.py "FK_DEBUG_FLAGS=3" "FK_DEBUG_FLAGS=3;FK_EPI5=4;FK_EPI=4" "" 2>&1 | grep -E "variant|rror" | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    p=d['plan']; print('$ov', d['variant'] or '-', 'fused', d['prep_fused_merge_ms'][1], 'amode',p['a_mode'],'acc',p['acc_stages'],'epi',p['epi'],'stages',p['stages'])
"
done
