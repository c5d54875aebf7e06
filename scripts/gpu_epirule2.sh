#!/bin/bash
# epilogue width on long L2 searches with the per-column norm term (MODE 5 fp32 filter, MODE 1 fp16)
CFG=2 OVERRIDE=nb=8000000 timeout 900 python scripts/sweep.py "" "FK_EPI5=4" "" "FK_EPI5=4" 2>&1 | grep -E "variant|rror" | cut -c1-75 | sed "s/^/m5-fp32-8M /"
CFG=2 OVERRIDE=nb=8000000,storage=fp16 timeout 900 python scripts/sweep.py "" "FK_EPI=4" "" "FK_EPI=4" 2>&1 | grep -E "variant|rror" | cut -c1-75 | sed "s/^/l2-fp16-8M /"
