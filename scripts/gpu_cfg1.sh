#!/bin/bash
# cfg1 (100k rows, 1k queries): epilogue width, publish cadence, split count
CFG=1 timeout 900 python scripts/sweep.py "" "FK_EPI=8" "FK_PUB=3" "FK_PUB=1" "FK_FORCE_S=9" "FK_FORCE_S=36" "FK_EPI=8;FK_PUB=3" "" 2>&1 | grep -E "variant|rror" | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    p=d['plan']; print(d['variant'] or '-', d['ms'], d['prep_fused_merge_ms'], 'S', p['S'], 'grid', p['grid'], 'amode', p['a_mode'], 'acc', p['acc_stages'], 'epi', p['epi'], 'same', d['same_as_first'])
"
