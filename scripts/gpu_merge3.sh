#!/bin/bash
# large-k merge with warp-aggregated atomics: cfg3 (k=1024) and cfg4 shape (k=100) + tests
CFG=3 timeout 900 python scripts/sweep.py "" "" 2>&1 | grep -E "variant|rror" | cut -c1-100 | sed "s/^/cfg3 /"
CFG=4 OVERRIDE=nb=2000000 timeout 900 python scripts/sweep.py "" 2>&1 | grep -E "variant|rror" | cut -c1-100 | sed "s/^/cfg4-2M /"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_fp32_filter16.py tests/test_fp32_tf32x1.py tests/test_range.py -m gpu -q -x --timeout 900 2>&1 | tail -2
