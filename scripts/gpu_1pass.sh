#!/bin/bash
FK_DIAG=1 CFG=1 timeout 300 python scripts/sweep.py "" "FK_FP32_1PASS_MINROWS=0" 2>&1 | grep -E "variant|rror|uncert" | sort | uniq -c | cut -c1-140
FK_DIAG=1 CFG=3 timeout 600 python scripts/sweep.py "" "FK_FP32_1PASS_MAXK=2048" 2>&1 | grep -E "variant|rror|uncert" | sort | uniq -c | cut -c1-140
FK_DIAG=1 CFG=2 OVERRIDE=k=32 timeout 300 python scripts/sweep.py "" "FK_FP32_1PASS_MAXK=2048" 2>&1 | grep -E "variant|rror|uncert" | sort | uniq -c | cut -c1-140
FK_DIAG=1 CFG=2 OVERRIDE=k=100 timeout 300 python scripts/sweep.py "" "FK_FP32_1PASS_MAXK=2048" 2>&1 | grep -E "variant|rror|uncert" | sort | uniq -c | cut -c1-140
