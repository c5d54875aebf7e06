#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 900 -k "epilogue_width or plan_invariance or split_query or large_query" 2>&1 | tail -2
timeout 1500 python -m pytest "tests/test_fullsize_parity.py::test_fullsize_config_vs_sharded_oracle[5]" -m gpu -q -x --timeout 1200 2>&1 | tail -2
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-200
