"""Attribute ncu per-instruction samples (``--page source --print-source sass``
CSV) to CUDA source lines through ``nvdisasm -g`` line info of the cubin.

    python scripts/sass_lines.py <sass.csv> <object.o> [top]
"""
import collections
import csv
import re
import subprocess
import sys
import tempfile
import os


def main():
    csv_path, obj = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    rows = list(csv.reader(open(csv_path)))
    kname = rows[0][1]
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[2:] if len(r) > 5]
    base = int(data[0][idx["Address"]], 16)
    samp = {int(r[idx["Address"]], 16) - base: (int(r[idx["Warp Stall Sampling (All Samples)"]] or 0),
                                                 int(r[idx["Instructions Executed"]] or 0), r[idx["Source"]])
            for r in data}
    # template args of the kernel name -> mangled name
    m = re.search(r"<\(int\)(-?\d+), \(int\)(-?\d+), \(bool\)(\d), \(int\)(\d+), \(int\)(\d+)>", kname)
    mode, kq, ip, epi, tbn = m.groups()
    kq_m = f"Li{kq}E" if not kq.startswith("-") else f"Lin{kq[1:]}E"
    mangled = f"_ZN2fk16fused_knn_kernelILi{mode}E{kq_m}Lb{ip}ELi{epi}ELi{tbn}EEEv14CUtensorMap_stS1_S1_S1_NS_12SearchParamsE"
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, capture_output=True)
        cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
        out = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(td, cub)], capture_output=True, text=True).stdout
    sec = out.split(f".text.{mangled}:")[1].split("//--------------------- .text.")[0]
    line = "?"
    by_line = collections.defaultdict(lambda: [0, 0])
    for ln in sec.splitlines():
        mm = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if mm:
            line = f"{os.path.basename(mm.group(1))}:{mm.group(2)}"
            continue
        mo = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if mo:
            off = int(mo.group(1), 16)
            if off in samp:
                s, e, _ = samp[off]
                b = by_line[line]
                b[0] += s
                b[1] += e
    tot = sum(v[0] for v in by_line.values())
    print(f"{kname[:90]}  total samples {tot}")
    for ln, (s, e) in sorted(by_line.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{s:8d} {100.0 * s / max(tot, 1):5.1f}%  inst {e:11d}  {ln}")


if __name__ == "__main__":
    main()
