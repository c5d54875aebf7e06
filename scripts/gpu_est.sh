#!/bin/bash
timeout 900 python scripts/scan_300k.py 2>&1 | grep -E "^300000 - |^1000000 - " | cut -c1-40
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_fp32_filter16.py -m gpu -q -x --timeout 900 -k "large_k or estimate or est or plan_invariance" 2>&1 | tail -2
