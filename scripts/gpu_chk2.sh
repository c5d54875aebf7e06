#!/bin/bash
timeout 1500 python -m pytest tests/test_fp32_filter16.py tests/test_fp32_tf32x1.py tests/test_edge_values.py -q -m gpu > gpurun_out/pytest_chk2.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_chk2.log; grep -E "^FAILED|Error" gpurun_out/pytest_chk2.log | head
CFG=2 timeout 300 python scripts/sweep.py "" 2>&1 | grep -E "variant|rror" | cut -c1-120
FK_DIAG=1 CFG=2 OVERRIDE=k=1 timeout 300 python scripts/sweep.py "" 2>&1 | grep -E "variant|rror|uncert" | sort | uniq -c | cut -c1-160
