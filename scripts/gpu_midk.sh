#!/bin/bash
CFG=2 timeout 300 python scripts/sweep.py "" 2>&1 | grep -E "variant|rror" | cut -c1-100
for k in 32 64 100 128; do FK_DIAG=1 CFG=2 OVERRIDE=k=$k timeout 300 python scripts/sweep.py "" "FK_FP32_1PASS_MAXK=2048" 2>&1 | grep -E "variant|rror|uncert" | sort | uniq -c | cut -c1-140 | sed "s/^/k=$k /"; done
timeout 900 python -m pytest tests/test_fp32_filter16.py -q -m gpu > gpurun_out/pytest_midk.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_midk.log
