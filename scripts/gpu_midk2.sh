#!/bin/bash
for k in 32 64 100; do FK_DIAG=1 CFG=2 OVERRIDE=k=$k timeout 300 python scripts/sweep.py "" "FK_FP32_1PASS_MAXK=2048" 2>&1 | grep -E "variant|rror|uncert" | sort | uniq -c | cut -c1-140 | sed "s/^/k=$k /"; done
