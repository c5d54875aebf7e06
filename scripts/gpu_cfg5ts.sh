#!/bin/bash
# cfg5 shape (power-capped): query operand placement x epilogue groups
CFG=5 OVERRIDE=nb=8000000 timeout 900 python scripts/sweep.py "" "FK_FORCE_AMODE=0;FK_EPI=4" "FK_EPI=4" "FK_FORCE_AMODE=0;FK_EPI=4;FK_ISSUERS=1" "" "FK_FORCE_AMODE=0;FK_EPI=4" 2>&1 | grep -E "variant|rror" | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    p=d['plan']; print(d['variant'] or '-', d['ms'], d['prep_fused_merge_ms'], 'amode', p['a_mode'], 'acc', p['acc_stages'], 'epi', p['epi'], 'stages', p['stages'], 'same', d['same_as_first'])
"
for C in 2; do CFG=$C OVERRIDE=storage=bf16 timeout 900 python scripts/sweep.py "" "FK_FORCE_AMODE=0;FK_EPI=4" 2>&1 | grep -E "variant|rror" | cut -c1-100 | sed "s/^/cfg2-bf16 /"; done
