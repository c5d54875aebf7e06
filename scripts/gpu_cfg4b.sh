#!/bin/bash
# cfg4 shape (2M x 768 fp16 IP k=100): multicast pairs / streamed A / 64-col tiles
CFG=4 OVERRIDE=nb=2000000 timeout 900 python scripts/sweep.py "" "FK_CLUSTER=2" "FK_FORCE_AMODE=2" "FK_FORCE_AMODE=2;FK_CLUSTER=2" "FK_BN=64" "FK_BN=64;FK_CLUSTER=2" 2>&1 | grep -E "variant|rror" | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    p=d['plan']; print(d['variant'] or '-', d['ms'], d['prep_fused_merge_ms'], 'amode',p['a_mode'],'acc',p['acc_stages'],'epi',p['epi'],'bn',p['bn'],'stages',p['stages'],'cl',p.get('cluster'), 'same', d['same_as_first'])
"
