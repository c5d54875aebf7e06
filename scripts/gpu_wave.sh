#!/bin/bash
# first-wave bound knobs on cfg2: publish cadence, probe chunk, bound pre-pass
CFG=2 timeout 900 python scripts/sweep.py "" "FK_PUB=7" "FK_PUB=3" "FK_PUB=1" "FK_PROBE=16" "FK_PROBE=64" "FK_PREPASS=8192" "FK_PUB=3;FK_PROBE=32" "" 2>&1 | grep -E "variant|rror" | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print(d['variant'] or '-', d['ms'], d['prep_fused_merge_ms'], 'same', d['same_as_first'])
"
