#!/bin/bash
# cfg4 shape decomposition: full / no epilogue / no TMA / neither; 1 vs 2 producers
CFG=4 OVERRIDE=nb=2000000 timeout 900 python scripts/sweep.py "" "FK_DEBUG_FLAGS=1" "FK_DEBUG_FLAGS=2" "FK_DEBUG_FLAGS=3" "FK_STAGES=8" 2>&1 | grep -E "variant|rror" | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    p=d['plan']; print(d['variant'] or '-', d['ms'], d['prep_fused_merge_ms'], 'stages', p['stages'], 'acc', p['acc_stages'])
"
