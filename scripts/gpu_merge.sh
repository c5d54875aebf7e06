#!/bin/bash
# large-k merge (cfg3, k=1024): survivor buffer and threads per query CTA; + the cfg3 main-pass capture
CFG=3 timeout 900 python scripts/sweep.py "" "FK_MERGE_THREADS=512" "FK_MERGE_THREADS=1024" "FK_MERGE_SMC=16384" "FK_MERGE_SMC=16384;FK_MERGE_THREADS=1024" "FK_MERGE_SMC=8192;FK_MERGE_THREADS=512" 2>&1 | grep -E "variant|rror" | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print(d['variant'] or '-', d['ms'], d['prep_fused_merge_ms'], 'same', d['same_as_first'])
"
TAG=${TAG:-r02g}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fused_knn python scripts/prof_search.py --config 3 --iters 2 2>&1 | grep -E "fused_knn_kernel<|gpu__time_duration" | head -8
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_knn -s 3 -c 1 \
   -o gpurun_out/full3_${TAG} -f python scripts/prof_search.py --config 3 --iters 3 > gpurun_out/ncu_full3_${TAG}.log 2>&1; echo "ncu cfg3 rc=$?"
