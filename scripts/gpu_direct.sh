#!/bin/bash
timeout 600 python scripts/small_batch.py 2>&1 | tail -6
FK_DIRECT_WARP1=1 timeout 600 python scripts/small_batch.py 2>&1 | head -3
timeout 1500 python -m pytest tests/test_direct_path.py tests/test_edge_values.py tests/test_gpu_parity.py -m gpu -q -x --timeout 900 2>&1 | tail -3
