#!/bin/bash
# quick GPU check: selected tests + cfg2/cfg4 timings
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_fp32_filter16.py "tests/test_fullsize_parity.py::test_fullsize_config_vs_sharded_oracle[4]" -q -m gpu ${PYTEST_ARGS} > gpurun_out/pytest_chk.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_chk.log; grep -E "^FAILED|Error" gpurun_out/pytest_chk.log | head
CFG=2 timeout 300 python scripts/sweep.py "" 2>&1 | grep -E "variant|rror" | cut -c1-120
timeout 900 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-200
