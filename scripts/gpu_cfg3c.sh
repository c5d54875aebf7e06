#!/bin/bash
FK_DIAG=1 FK_FP32_1PASS_MAXK=2048 CFG=3 timeout 300 python scripts/prof_search.py --config 3 --iters 1 2>&1 | grep -E "uncert|rror" | head -3
FK_DIAG=1 CFG=3 timeout 600 python scripts/sweep.py "" "FK_FP32_1PASS_MAXK=2048" "FK_FP32_1PASS_MAXK=2048;FK_EPI5=4" 2>&1 | grep -E "variant|rror|uncert" | sort | uniq -c | cut -c1-250
timeout 900 python -m pytest tests/test_fp32_filter16.py -q -m gpu -k "large_k or coherent" > gpurun_out/pytest_lk.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_lk.log
