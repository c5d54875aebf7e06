#!/bin/bash
# after the k' slack rule: the filter16 tests, then cfg2-shape k = 10/13/14/16 default plans
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fp32_filter16.py -q -m gpu > gpurun_out/pytest_k16.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_k16.log
for k in 10 13 14 16; do for nq in 10000 1000; do
CFG=2 OVERRIDE=nq=$nq,k=$k FK_DIAG=1 timeout 300 python scripts/sweep.py "" 2>&1 | grep -E "variant|uncertified" | awk '/uncertified/{u=$0; next} {print substr($0,1,110), "|", substr(u, index(u,"uncertified"), 50)}' | sed "s/^/nq=$nq k=$k /"
done; done
