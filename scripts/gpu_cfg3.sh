#!/bin/bash
FK_DIAG=1 CFG=3 timeout 600 python scripts/sweep.py "" "FK_FP32_1PASS_MAXK=2048" "FK_FP32_1PASS_MAXK=2048;FK_EPI5=4" "FK_FP32_1PASS_MAXK=2048;FK_FP32_FILTER=tf32" 2>&1 | grep -E "variant|rror|uncert" | cut -c1-220
FK_DIAG=1 CFG=2 OVERRIDE=k=32 timeout 600 python scripts/sweep.py "" "FK_FP32_1PASS_MAXK=2048" 2>&1 | grep -E "variant|rror|uncert" | cut -c1-220
FK_DIAG=1 CFG=2 OVERRIDE=k=100 timeout 600 python scripts/sweep.py "" "FK_FP32_1PASS_MAXK=2048" 2>&1 | grep -E "variant|rror|uncert" | cut -c1-220
