#!/bin/bash
timeout 900 python -m pytest tests/test_fp32_filter16.py -q -m gpu -k large_k > gpurun_out/pytest_lk.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_lk.log
FK_DIAG=1 CFG=3 timeout 600 python scripts/sweep.py "" "FK_FP32_1PASS_MAXK=2048" "FK_FP32_1PASS_MAXK=2048;FK_EPI5=4" 2>&1 | grep -E "variant|rror|uncert" | sort | uniq -c | cut -c1-250
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_knn -s 3 -c 1 \
   -o gpurun_out/full3b -f python scripts/prof_search.py --config 3 --iters 3 > gpurun_out/ncu_full3b.log 2>&1; echo "ncu cfg3 rc=$?"
