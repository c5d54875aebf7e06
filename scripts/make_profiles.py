"""Summarise an evidence pass (scripts/gpu_evidence.sh TAG=...) into profiles/<TAG>/.

    python scripts/make_profiles.py r01b

Writes the ncu summaries (key metrics, stall reasons, hottest SASS), the
launch list of the bench command, the bench JSON line and the per-config
sweep, plus profiles/ncu_traffic.json (DRAM bytes per fused launch from the
--set full capture) that bench.py reports as roofline.traffic.
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
src = os.path.join(REPO, "gpurun_out")
reps = sys.argv[sys.argv.index("--reps") + 1] if "--reps" in sys.argv else src
dst = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else os.path.join(REPO, "profiles", tag)
os.makedirs(dst, exist_ok=True)


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def to_ms(v, unit):
    return float(v.replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1, "msecond": 1,
                                         "s": 1e3, "second": 1e3}.get(unit, 1)


def to_bytes(v, unit):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


traffic = {}
for rep, name in ((f"full_{tag}.ncu-rep", "cfg2"), (f"full2_{tag}.ncu-rep", "cfg2"), (f"full3_{tag}.ncu-rep", "cfg3"),
                  (f"full4_{tag}.ncu-rep", "cfg4_2M"), (f"full5_{tag}.ncu-rep", "cfg5_2M"),
                  (f"full3b_{tag}.ncu-rep", "cfg3_boundpass"), (f"full5b_{tag}.ncu-rep", "cfg5_4M")):
    p = os.path.join(reps, rep)
    if not os.path.exists(p):
        continue
    summ = subprocess.run([sys.executable, os.path.join(REPO, "scripts", "ncu_summary.py"), p, "--source", "40"],
                          capture_output=True, text=True).stdout
    with open(os.path.join(dst, f"ncu_full_fused_{name}.txt"), "w") as f:
        f.write(summ)
    r, u = raw(p)
    rd = to_bytes(r["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
    wr = to_bytes(r["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
    traffic[name] = {"kernel": r["Kernel Name"], "dram_read_bytes": rd, "dram_write_bytes": wr,
                     "traffic_bytes": rd + wr, "duration_ms": to_ms(r["gpu__time_duration.sum"], u["gpu__time_duration.sum"]),
                     "capture": os.path.relpath(os.path.join(dst, f"ncu_full_fused_{name}.txt"), REPO)}
print("summaries ->", dst)
for c in range(1, 6):  # per-config bench lines of the evidence pass (last JSON line of each)
    b = os.path.join(src, f"bench_{tag}_cfg{c}.json")
    if os.path.exists(b):
        lines = [l for l in open(b) if l.startswith("{")]
        if lines:
            with open(os.path.join(dst, f"bench_cfg{c}.json"), "w") as f:
                f.write(lines[-1])
for f in (f"launches_{tag}.csv", f"bench_{tag}.json", f"sweep_{tag}.jsonl", f"pytest_{tag}.log"):
    if os.path.exists(os.path.join(src, f)):
        shutil.copy(os.path.join(src, f), os.path.join(dst, f))
with open(os.path.join(dst, "ncu_traffic.json"), "w") as f:
    json.dump(traffic, f, indent=1)
if traffic and ("--out" not in sys.argv or "--global" in sys.argv):
    with open(os.path.join(REPO, "profiles", "ncu_traffic.json"), "w") as f:
        json.dump(dict(traffic, tag=tag), f, indent=1)
print(json.dumps(traffic, indent=1))
