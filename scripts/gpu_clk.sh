#!/bin/bash
for f in "" 3 10 8 4; do FK_DEBUG_FLAGS=$f CFG=2 timeout 120 python scripts/clock_probe.py 2>&1 | tail -1; done
for f in "" 3; do FK_DEBUG_FLAGS=$f CFG=2 OVERRIDE=storage=fp16 timeout 120 python scripts/clock_probe.py 2>&1 | tail -1; done
