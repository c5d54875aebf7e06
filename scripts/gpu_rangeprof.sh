#!/bin/bash
# launch list (ncu durations) of range searches on the cfg2 shape
SEL=1e-5 CFG=2 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/range_launches.csv python scripts/range_bench.py > /dev/null 2>&1; echo "ncu rc=$?"
python3 - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/range_launches.csv")))
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value"); ui = hdr.index("Metric Unit")
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[1:]:
    if len(r) <= vi: continue
    v = float(r[vi].replace(",", "")) * (1e-3 if r[ui] == "usecond" else (1e-6 if r[ui] == "nsecond" else 1.0))
    name = r[ki].split("(")[0][:80]
    tot[name] += v; cnt[name] += 1
for n, v in sorted(tot.items(), key=lambda x: -x[1])[:15]:
    print(f"{v:9.3f} ms  x{cnt[n]:3d}  {n}")
PY
