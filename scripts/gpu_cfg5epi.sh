#!/bin/bash
# full cfg5: default plan vs one epilogue group (A in TMEM), alternating
for v in "" "FK_EPI=4" "" "FK_EPI=4"; do
  env $v timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python3 -c "
import sys,json; d=json.loads(sys.stdin.read()); print('$v' or '-', round(d['ms_per_step'],2), round(d['value']), d['clocks']['sm_mhz'], d['config']['plan']['epi'], d['config']['plan']['a_mode'])"
done
