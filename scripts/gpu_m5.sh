#!/bin/bash
# MODE 5 (scaled fp16 filter) checks: fp32 parity tests + cfg2 variants
mkdir -p gpurun_out
TAG=${TAG:-m5a}
timeout 900 python -m pytest tests/test_fp32_filter16.py tests/test_fp32_tf32x1.py tests/test_edge_values.py tests/test_gpu_parity.py -q -m gpu ${PYTEST_ARGS} > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_${TAG}.log | tail -15
FK_DIAG=1 CFG=2 timeout 600 python scripts/sweep.py "" "FK_EPI5=4" "FK_KP=16" "FK_KP=16;FK_EPI5=4" "FK_KP=8" "FK_KP=8;FK_EPI5=4" ${VARIANTS} > gpurun_out/sweep_${TAG}.txt 2>&1
grep -E "variant|rror" gpurun_out/sweep_${TAG}.txt | cut -c1-230
grep -E "uncert" gpurun_out/sweep_${TAG}.txt | sort | uniq -c | sort -rn | head -12
