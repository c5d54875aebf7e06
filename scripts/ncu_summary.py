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
    n = int(sys.argv[sys.argv.index("--source") + 1])
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    h = srows[0]
    try:
        ci = h.index("Warp Stall Sampling (All Samples)")
    except ValueError:
        ci = next(i for i, x in enumerate(h) if "Sampling" in x)
    li = h.index("Line") if "Line" in h else 0
    si = h.index("Source") if "Source" in h else 1
    body = []
    for r in srows[1:]:
        try:
            body.append((float(r[ci] or 0), r[li], r[si][:110]))
        except (ValueError, IndexError):
            pass
    tot = sum(b[0] for b in body) or 1
    for v, line, s in sorted(body, reverse=True)[:n]:
        print(f"  {100 * v / tot:5.1f}%  L{line:>5}  {s}")
