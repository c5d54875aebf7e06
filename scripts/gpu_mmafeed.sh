#!/bin/bash
# what paces the MMA-only kernel (FK_DEBUG_FLAGS=3: no epilogue math, no TMA)
CFG=2 timeout 900 python scripts/sweep.py "FK_DEBUG_FLAGS=3" "FK_DEBUG_FLAGS=3;FK_STAGES=8" "FK_DEBUG_FLAGS=3;FK_STAGES=4" "FK_DEBUG_FLAGS=3;FK_FORCE_S=7" "FK_DEBUG_FLAGS=3;FK_PRODUCERS=1" "FK_DEBUG_FLAGS=3;FK_FORCE_AMODE=0" "FK_DEBUG_FLAGS=3;FK_ACC=2" "FK_DEBUG_FLAGS=3;FK_EPI5=4" "FK_DEBUG_FLAGS=3;FK_EPI5=4;FK_FORCE_AMODE=0" 2>&1 | grep -E "variant|rror" | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    p=d['plan']; print(d['variant'] or '-', d['ms'], d['prep_fused_merge_ms'], 'amode',p['a_mode'],'acc',p['acc_stages'],'epi',p['epi'],'stages',p['stages'],'S',p.get('S'),'iss',p.get('n_issuers'))
"
