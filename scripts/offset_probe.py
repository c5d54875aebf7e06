"""fp32 1-pass filter on data far from the origin (norms >> neighbour
distances: the fp16 rounding band, 2^-8 (|q|^2 + max|x|^2), covers many
rows near the k-th): time and certification vs centred data and vs 3xTF32.
python scripts/offset_probe.py  (FK_DIAG=1 for the uncertified counts)"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_08281_b200 import FlatIndex  # noqa: E402

nb, d, nq, k = int(os.environ.get("NB", 1_000_000)), 128, int(os.environ.get("NQ", 10_000)), 10
for off in [float(x) for x in os.environ.get("OFFS", "0,1,3,10").split(",")]:
    g = torch.Generator(device="cuda").manual_seed(0)
    xb = torch.randn(nb, d, device="cuda", generator=g) + off
    q = torch.randn(nq, d, device="cuda", generator=g) + off
    idx = FlatIndex(d, "l2")
    idx.add(xb)
    for variant in ("", "FK_FP32_3X"):
        if variant:
            os.environ[variant] = "1"
        idx.search(q, k)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = idx.search(q, k)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"offset": off, "variant": variant or "default", "ms": round(e0.elapsed_time(e1), 3),
                          "kmode": idx.last_plan()["kmode"]}), flush=True)
        if variant:
            del os.environ[variant]
    del idx, xb
    torch.cuda.empty_cache()
