#!/bin/bash
# fallback with the row-split composites: few uncertified queries (k = 14 with
# 16-deep queues), many (k = 16 with 16-deep queues), the fallback tests
mkdir -p gpurun_out
for k in 14 16; do
CFG=2 OVERRIDE=k=$k FK_DIAG=1 timeout 300 python scripts/sweep.py "" "FK_KP=16" 2>&1 | grep -E "variant|uncertified" | awk '/uncertified/{u=$0; next} {print substr($0,1,110), "|", substr(u, index(u,"uncertified"), 50)}' | sed "s/^/k=$k /"
done
timeout 900 python -m pytest tests/test_fp32_filter16.py tests/test_fp32_tf32x1.py tests/test_edge_values.py tests/test_concurrency_gpu.py tests/test_gpu_parity.py -q -m gpu > gpurun_out/pytest_fb.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_fb.log
