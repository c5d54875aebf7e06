#!/bin/bash
# large-k merge tuning (cfg3 k=1024, cfg4-shape k=100)
CFG=3 timeout 900 python scripts/sweep.py "FK_MERGE_SMC=8192;FK_MERGE_THREADS=512" "FK_MERGE_SMC=10240;FK_MERGE_THREADS=512" "FK_MERGE_SMC=12288;FK_MERGE_THREADS=512" "FK_MERGE_SMC=8192;FK_MERGE_THREADS=1024" "FK_MERGE_SMC=12288;FK_MERGE_THREADS=1024" "FK_MERGE_SMC=6144;FK_MERGE_THREADS=512" "FK_MERGE_SMC=8192;FK_MERGE_THREADS=256" 2>&1 | grep -E "variant|rror" | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print(d['variant'] or '-', d['ms'], d['prep_fused_merge_ms'], 'same', d['same_as_first'])
"
CFG=4 OVERRIDE=nb=2000000 timeout 900 python scripts/sweep.py "" "FK_MERGE_THREADS=512" "FK_MERGE_SMC=8192;FK_MERGE_THREADS=512" 2>&1 | grep -E "variant|rror" | cut -c1-120
