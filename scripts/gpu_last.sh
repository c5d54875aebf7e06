#!/bin/bash
# last validation of the round: smoke, GPU suite, default bench
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_r02k.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_r02k.log
timeout 900 python bench.py > gpurun_out/bench_r02k_default.json 2> gpurun_out/bench_r02k_default.err; echo "bench rc=$?"; tail -1 gpurun_out/bench_r02k_default.json | cut -c1-300
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 2>/dev/null | tail -1 | cut -c1-300
