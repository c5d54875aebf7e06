#!/bin/bash
# epilogue timelines (dev build, global slow-path counters off: 0x8000) at tile windows 0, 8, 14 (x256)
for off in 0 8 14; do for q in 0; do
  f=$(( (off << 20) | (q << 16) | 0x8000 ))
  echo "=== off $off quarter $q"
  FK_DEBUG_FLAGS=$f CFG=2 timeout 300 python scripts/trace.py 2>&1 | grep -E "period|MMA issuer|epilogue|slow-path"
done; done
