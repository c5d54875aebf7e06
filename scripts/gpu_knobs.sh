#!/bin/bash
CFG=2 timeout 600 python scripts/sweep.py "FK_DEBUG_FLAGS=3" "FK_DEBUG_FLAGS=3;FK_ISSUERS=1" "FK_DEBUG_FLAGS=3;FK_STAGES=8" "FK_DEBUG_FLAGS=3;FK_STAGES=4" "FK_DEBUG_FLAGS=3;FK_PRODUCERS=1" "FK_DEBUG_FLAGS=3;FK_EPI5=4" "FK_DEBUG_FLAGS=3;FK_FORCE_AMODE=0" "FK_DEBUG_FLAGS=3;FK_NO_UNION=1" "FK_DEBUG_FLAGS=3;FK_PUB=1023" 2>&1 | grep -E "variant|rror" | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    p=d['plan']; print(d['variant'] or '-', 'fused', d['prep_fused_merge_ms'][1], 'amode',p['a_mode'],'acc',p['acc_stages'],'epi',p['epi'],'stages',p['stages'])
"
