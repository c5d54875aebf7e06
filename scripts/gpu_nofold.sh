#!/bin/bash
# cfg5 16M-row shape: folded norms (7 K-steps, light epilogue) vs unfolded (6 K-steps + norm term)
CFG=5 OVERRIDE=nb=16000000 timeout 1200 python scripts/sweep.py "" "FK_NO_FOLD=1" "FK_NO_FOLD=1;FK_EPI=4" 2>&1 | grep -E "variant|rror" | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    p=d['plan']; print(d['variant'] or '-', d['ms'], d['prep_fused_merge_ms'], 'amode', p['a_mode'], 'acc', p['acc_stages'], 'epi', p['epi'], 'kmode', p['kmode'], 'same', d['same_as_first'])
"
