#!/bin/bash
timeout 900 python -m pytest tests/test_fp32_filter16.py tests/test_fp32_tf32x1.py -q -m gpu -x > gpurun_out/pytest_pre.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_pre.log
FK_DIAG=1 CFG=2 timeout 600 python scripts/sweep.py "FK_PREPASS=0" "" "FK_PREPASS=8192" "FK_PREPASS=32768" "FK_PREPASS=65536" 2>&1 | grep -E "variant|rror" | cut -c1-130
FK_DIAG=1 CFG=2 timeout 600 python scripts/sweep.py "FK_PREPASS=32768" 2>&1 | grep uncert | sort | uniq -c | head -3
