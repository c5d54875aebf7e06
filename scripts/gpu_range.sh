#!/bin/bash
timeout 900 python -m pytest tests/test_range.py tests/test_concurrency_gpu.py -m gpu -q -x --timeout 600 2>&1 | tail -2
for s in 1e-5 1e-4; do SEL=$s CFG=2 timeout 600 python scripts/range_bench.py 2>&1 | tail -1; done
