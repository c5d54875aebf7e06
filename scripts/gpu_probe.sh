#!/bin/bash
FK_DIAG=1 CFG=2 timeout 600 python scripts/sweep.py "" "FK_PROBE=16" "FK_PROBE=32" "FK_PROBE=64" "FK_PROBE=128" "FK_PROBE=32;FK_PUB=3" 2>&1 | grep -E "variant|rror" | cut -c1-160
CFG=5 OVERRIDE=nb=4000000 timeout 600 python scripts/sweep.py "" "FK_PROBE=32" "FK_PROBE=64" 2>&1 | grep -E "variant|rror" | cut -c1-160
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "plan_invariance or many_chunks" > gpurun_out/pytest_probe.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_probe.log
