#!/bin/bash
# stage-ring depth on the full kernels (cfg2 MODE 5, cfg5-shape MODE 3, cfg1, cfg3 shapes)
for C in 2 5; do
OV=""; [ $C = 5 ] && OV="nb=4000000"
CFG=$C OVERRIDE=$OV timeout 900 python scripts/sweep.py "" "FK_STAGES=8" "FK_STAGES=6" "FK_STAGES=4" "" "FK_STAGES=6" 2>&1 | grep -E "variant|rror" | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    p=d['plan']; print('cfg$C', d['variant'] or '-', d['ms'], d['prep_fused_merge_ms'], 'amode',p['a_mode'],'acc',p['acc_stages'],'epi',p['epi'],'stages',p['stages'],'same',d['same_as_first'])
"
done
