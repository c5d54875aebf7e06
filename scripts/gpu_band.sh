#!/bin/bash
timeout 900 python -m pytest tests/test_fp32_filter16.py tests/test_fp32_tf32x1.py -q -m gpu > gpurun_out/pytest_band.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_band.log; grep -E "FAILED|Error" gpurun_out/pytest_band.log | head
FK_DIAG=1 CFG=2 timeout 600 python scripts/sweep.py "FK_BAND=2" "" 2>&1 | grep -E "variant|rror|uncert" | sort | uniq -c | cut -c1-230
FK_DIAG=1 FK_FP32_1PASS_MAXK=2048 CFG=3 timeout 300 python scripts/prof_search.py --config 3 --iters 1 2>&1 | grep -E "uncert|plan|rror" | head -5
