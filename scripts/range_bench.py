"""Time GPU range search on a config's shape (CUDA events), radius chosen so
that about `sel` of all pairs qualify; reports entries and the fused-pass time."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from bench import CONFIGS, gen_base, gen_queries
from paper_2401_08281_b200 import METRIC_IP, METRIC_L2, FlatIndex

cfg = dict(CONFIGS[int(os.environ.get("CFG", "2"))])
sel = float(os.environ.get("SEL", "1e-5"))
idx = FlatIndex(cfg["d"], METRIC_L2 if cfg["metric"] == "l2" else METRIC_IP, storage=cfg["storage"])
nb = min(cfg["nb"], 2_000_000)
xb = gen_base(cfg, 0, nb)
idx.add(torch.from_numpy(xb).cuda())
q = torch.from_numpy(gen_queries(cfg)).cuda()
# radius from a sample of exact distances
qs, xs = q[:64].double(), torch.from_numpy(xb[:200000]).cuda().double()
dm = ((qs * qs).sum(1)[:, None] + (xs * xs).sum(1)[None, :] - 2 * qs @ xs.T) if cfg["metric"] == "l2" else qs @ xs.T
radius = float(torch.quantile(dm.flatten()[:16_000_000].float(), 1 - sel if cfg["metric"] == "ip" else sel))
for _ in range(2):
    r = idx.range_search(q, radius)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 5
e0.record()
for _ in range(n):
    r = idx.range_search(q, radius)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
print(json.dumps({"workload": f"range search {cfg['name']} nb={nb}", "radius": radius, "entries": int(r.lims[-1]),
                  "ms": round(ms, 3), "qps": round(cfg["nq"] / ms * 1e3)}))
