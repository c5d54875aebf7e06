"""Scan search latency over batch sizes, database sizes, k, storage and metric
to catch performance cliffs (plan corner cases) -- prints ms per search and
ns per (query x row) so outliers stand out.

    python scripts/shape_scan.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2401_08281_b200 import METRIC_IP, METRIC_L2, FlatIndex

D = 128
NQS = [1, 20, 100, 500, 3000]
KS = [1, 10, 100, 1000]
g = torch.Generator(device="cuda")
g.manual_seed(0)
for storage in ("fp32", "fp16"):
    for metric in ("l2", "ip"):
        for nb in (10_000, 300_000, 1_000_000):
            idx = FlatIndex(D, METRIC_L2 if metric == "l2" else METRIC_IP, storage=storage)
            idx.add(torch.randn((nb, D), generator=g, device="cuda"))
            qall = torch.randn((max(NQS), D), generator=g, device="cuda")
            for nq in NQS:
                q = qall[:nq].contiguous()
                for k in KS:
                    if k > nb:
                        continue
                    idx.search(q, k)
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(3):
                        idx.search(q, k)
                    e1.record()
                    torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1) / 3
                    p = idx.last_plan()
                    print(json.dumps({"storage": storage, "metric": metric, "nb": nb, "nq": nq, "k": k, "ms": round(ms, 3),
                                      "ns_per_pair": round(ms * 1e6 / (nq * nb), 4), "kmode": p.get("kmode"),
                                      "S": p.get("S"), "epi": p.get("epi")}), flush=True)
            del idx
            torch.cuda.empty_cache()
