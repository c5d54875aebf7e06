"""Second cliff scan: dimensions, bf16, k around the queue/list thresholds."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_08281_b200 import METRIC_L2, FlatIndex
g = torch.Generator(device="cuda"); g.manual_seed(1)
for d in (32, 256, 768):
    for storage in ("fp32", "bf16"):
        nb = 200_000
        idx = FlatIndex(d, METRIC_L2, storage=storage)
        idx.add(torch.randn((nb, d), generator=g, device="cuda"))
        qall = torch.randn((2000, d), generator=g, device="cuda")
        for nq in (19, 20, 129, 2000):
            q = qall[:nq].contiguous()
            for k in (1, 16, 33, 128, 600, 2048):
                idx.search(q, k); torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(3): idx.search(q, k)
                e1.record(); torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 3
                p = idx.last_plan()
                print(json.dumps({"d": d, "storage": storage, "nq": nq, "k": k, "ms": round(ms, 3),
                                  "ns_per_pair_dim": round(ms * 1e6 / (nq * nb * d) * 128, 4), "kmode": p.get("kmode"),
                                  "a_mode": p.get("a_mode"), "S": p.get("S")}), flush=True)
        del idx; torch.cuda.empty_cache()
