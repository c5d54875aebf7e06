#!/bin/bash
# Fast iteration: GPU tests (subset via PYTEST_ARGS) + variant sweep on cfg2.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/pytest_gpu.log
timeout 600 python scripts/sweep.py ${SWEEP} > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?"
cat gpurun_out/sweep.log | tail -20
