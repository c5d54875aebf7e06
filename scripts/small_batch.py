"""Latency of small query batches on the cfg2 base (1M x 128 fp32): nq < 20 takes
the reference's direct path (flat.py:58-62), nq >= 20 the fused GEMM path."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import CONFIGS, gen_base, gen_queries
from paper_2401_08281_b200 import IndexFlatL2
cfg = dict(CONFIGS[2])
idx = IndexFlatL2(cfg["d"])
idx.add(torch.from_numpy(gen_base(cfg)).cuda())
q = torch.from_numpy(gen_queries(cfg)).cuda()
for nq in (1, 4, 19, 20, 64, 256):
    qs = q[:nq].contiguous()
    for _ in range(3):
        idx.search(qs, 10)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        idx.search(qs, 10)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(json.dumps({"nq": nq, "ms": round(ms, 4), "plan": idx.last_plan().get("kmode")}))
