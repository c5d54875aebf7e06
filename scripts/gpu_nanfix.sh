#!/bin/bash
for e in "" 1; do EDGE=$e FK_DIAG=1 timeout 300 python scripts/dbg_edge2.py 2>&1 | tail -2; done
timeout 1500 python -m pytest tests/test_edge_values.py tests/test_fp32_filter16.py tests/test_direct_path.py tests/test_fp32_tf32x1.py -m gpu -q -x --timeout 900 2>&1 | tail -3
timeout 600 python scripts/small_batch.py 2>&1 | tail -6
