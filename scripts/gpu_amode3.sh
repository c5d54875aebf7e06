#!/bin/bash
# split query operand (a_mode 3) for d = 768 16-bit: speed vs the single-accumulator plan + parity
CFG=4 OVERRIDE=nb=2000000 timeout 900 python scripts/sweep.py "" "FK_AMODE3=0" "" 2>&1 | grep -E "variant|rror" | python3 -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    p=d['plan']; print(d['variant'] or '-', d['ms'], d['prep_fused_merge_ms'], 'amode', p['a_mode'], 'acc', p['acc_stages'], 'epi', p['epi'], 'stages', p['stages'], 'same', d['same_as_first'])
"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_range.py -m gpu -q -x --timeout 900 -k "split_query or large_query or range_16bit" 2>&1 | tail -2
timeout 1500 python -m pytest "tests/test_fullsize_parity.py::test_fullsize_config_vs_sharded_oracle[4]" -m gpu -q -x --timeout 1200 2>&1 | tail -2
timeout 900 python bench.py --config 4 --steps 10 --warmup 3 > gpurun_out/bench_a3_cfg4.json 2> gpurun_out/bench_a3_cfg4.err; tail -1 gpurun_out/bench_a3_cfg4.json | cut -c1-250
