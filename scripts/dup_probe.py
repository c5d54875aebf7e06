"""fp32 1-pass filter on bases with duplicated rows (each unique row stored
R times): time and certification (FK_DIAG=1) for R = 1, 2, 4, 8.
python scripts/dup_probe.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_08281_b200 import FlatIndex  # noqa: E402

nb, d, nq, k = 1_000_000, 128, 10_000, 10
for rep in (1, 2, 4, 8):
    g = torch.Generator(device="cuda").manual_seed(0)
    u = torch.randn(nb // rep, d, device="cuda", generator=g)
    xb = u.repeat(rep, 1)
    q = torch.randn(nq, d, device="cuda", generator=g)
    idx = FlatIndex(d, "l2")
    idx.add(xb)
    idx.search(q, k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    idx.search(q, k)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"dup": rep, "ms": round(e0.elapsed_time(e1), 3), "kmode": idx.last_plan()["kmode"]}), flush=True)
    del idx, xb, u
    torch.cuda.empty_cache()
