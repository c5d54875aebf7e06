#!/bin/bash
timeout 1500 python -m pytest tests/test_fp32_filter16.py tests/test_edge_values.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_chk3.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_chk3.log; grep -E "^FAILED|Error" gpurun_out/pytest_chk3.log | head
CFG=2 timeout 300 python scripts/sweep.py "" "" 2>&1 | grep -E "variant|rror" | cut -c1-120
CFG=5 OVERRIDE=nb=4000000 timeout 300 python scripts/sweep.py "" 2>&1 | grep -E "variant|rror" | cut -c1-120
