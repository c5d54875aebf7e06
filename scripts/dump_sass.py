"""Regenerate profiles/r02/sass/: SASS of the shipped fused-kernel
instantiations (one per config plan) and of the auxiliary kernels, plus a
summary of tcgen05/TMA instruction counts, registers and spills.

    python scripts/dump_sass.py [out_dir]
"""
import os
import re
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(REPO, "paper_2401_08281_b200", "libflatknn.so")
out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(REPO, "profiles", "r02", "sass")
os.makedirs(out, exist_ok=True)
KERNELS = {  # (MODE, KQ, IP, EPI, TBN) -> which config runs it
    (5, 16, 0, 8, 128): "cfg2",
    (0, 16, 0, 4, 128): "cfg1",
    (0, 0, 0, 4, 128): "cfg3",
    (1, 0, 1, 4, 128): "cfg4",
    (3, 16, 0, 8, 128): "cfg5",
    (4, 16, 0, 4, 128): "tf32filter",
}


def mangled(m, kq, ip, epi, tbn):
    kqm = f"Li{kq}E" if kq >= 0 else f"Lin{-kq}E"
    return f"_ZN2fk16fused_knn_kernelILi{m}E{kqm}Lb{ip}ELi{epi}ELi{tbn}EEEv14CUtensorMap_stS1_S1_S1_NS_12SearchParamsE"


usage = subprocess.run(["cuobjdump", "--dump-resource-usage", LIB], capture_output=True, text=True).stdout.splitlines()
res = {}
for i, l in enumerate(usage):
    m = re.search(r"Function (\S+):", l)
    if m and i + 1 < len(usage):
        r = re.search(r"REG:(\d+) STACK:(\d+)", usage[i + 1])
        if r:
            res[m.group(1)] = (int(r.group(1)), int(r.group(2)))
for f in os.listdir(out):
    if f.startswith("fused_knn_kernel_"):
        os.remove(os.path.join(out, f))
lines = ["kernel | config | REG | STACK | UTCHMMA/UTCQMMA | UTMALDG | LDTM | STTM | UTCBAR | STL | LDL",
         "---|---|---|---|---|---|---|---|---|---|---"]
for key, cfg in KERNELS.items():
    name = mangled(*key)
    sass = subprocess.run(["cuobjdump", "-sass", "-fun", name, LIB], capture_output=True, text=True).stdout
    sass = "\n".join(l for l in sass.splitlines() if not re.fullmatch(r"\s*/\* [0-9a-fx]+ \*/\s*", l))
    fn = "fused_knn_kernel_" + "_".join(str(v) for v in key) + f"_{cfg}.sass"
    with open(os.path.join(out, fn), "w") as f:
        f.write(sass)
    cnt = lambda pat: len(re.findall(pat, sass))
    reg, stack = res.get(name, (None, None))
    lines.append(f"<{','.join(str(v) for v in key)}> | {cfg} | {reg} | {stack} | {cnt(r'UTC[HQ]MMA')} | {cnt(r'UTMALDG')} | "
                 f"{cnt(r'LDTM')} | {cnt(r'STTM')} | {cnt(r'UTCBAR')} | {cnt(r'STL')} | {cnt(r'LDL')}")
with open(os.path.join(out, "SUMMARY.md"), "w") as f:
    f.write("SASS of the shipped fused-kernel instantiations (`python scripts/dump_sass.py`), from "
            "`paper_2401_08281_b200/libflatknn.so` (sm_100a). Counts are static instruction counts.\n\n")
    f.write("\n".join(lines) + "\n")
print("\n".join(lines))
