"""Summarise an ncu report: key metrics, stall reasons, hottest source lines.

    python scripts/ncu_summary.py gpurun_out/prof_r01.ncu-rep [--source N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
KEYS = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
        "launch__registers_per_thread", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed"]
for r in rows[2:]:
    print("----")
    for k in KEYS:
        for i, h in enumerate(hdr):
            if h == k:
                print(f"  {k:84s} {r[i]} {units[i]}")
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                st.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    print("  stall samples:", ", ".join(f"{n} {100 * v / tot:.1f}%" for v, n in sorted(st, reverse=True)[:12]))

if "--source" in sys.argv:
    # hottest SASS instructions by warp-stall samples (with the stall breakdown column)
    n = int(sys.argv[sys.argv.index("--source") + 1])
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    hi = next(i for i, r in enumerate(srows) if r and r[0] == "Address")
    h = srows[hi]
    ci = h.index("Warp Stall Sampling (All Samples)")
    ei = h.index("Instructions Executed")
    body = []
    for idx, r in enumerate(srows[hi + 1:]):
        try:
            body.append((float(r[ci] or 0), idx, float(r[ei] or 0), r[1].strip()[:90]))
        except (ValueError, IndexError):
            pass
    tot = sum(b[0] for b in body) or 1
    print(f"  {len(body)} SASS instructions; samples%  #idx  warp-instr executed  sass")
    for v, idx, ex, s in sorted(body, reverse=True)[:n]:
        print(f"  {100 * v / tot:5.1f}%  #{idx:<6} {ex:14.0f}  {s}")
    if "--dump" in sys.argv:
        with open(sys.argv[sys.argv.index("--dump") + 1], "w") as f:
            for v, idx, ex, s in body:
                f.write(f"{idx:6d} {100 * v / tot:6.2f}% {ex:12.0f}  {s}\n")
