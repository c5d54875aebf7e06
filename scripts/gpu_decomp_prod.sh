#!/bin/bash
# Bottleneck decomposition on the PRODUCT build (FK_DEBUG_FLAGS: 1 no TMEM loads/filter,
# 2 no TMA, 4 no slow path, 8 TMEM loads but no filter)
for c in "2 storage=fp32" "2 storage=fp16" "5 nb=4000000"; do set -- $c
CFG=$1 OVERRIDE=$2 timeout 600 python scripts/sweep.py "" "FK_DEBUG_FLAGS=4" "FK_DEBUG_FLAGS=8" "FK_DEBUG_FLAGS=1" "FK_DEBUG_FLAGS=3" "FK_DEBUG_FLAGS=10" ${VARIANTS} 2>&1 | grep -E "variant|rror" | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    p=d['plan']; print('cfg$1 $2', d['variant'] or '-', 'fused', d['prep_fused_merge_ms'][1], 'merge', d['prep_fused_merge_ms'][2], 'amode',p['a_mode'],'acc',p['acc_stages'],'epi',p['epi'],'stages',p['stages'])
"
done
