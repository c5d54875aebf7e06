"""Small driver for ncu: build one config's index, warm up, then run N searches."""
import argparse
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from bench import CONFIGS, gen_base, gen_queries
from paper_2401_08281_b200 import FlatIndex, METRIC_L2, METRIC_IP

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--nq", type=int, default=0)
ap.add_argument("--nb", type=int, default=0)
ap.add_argument("--k", type=int, default=0)
ap.add_argument("--storage", default="")
a = ap.parse_args()
cfg = dict(CONFIGS[a.config])
if a.nq: cfg["nq"] = a.nq
if a.nb: cfg["nb"] = a.nb
if a.k: cfg["k"] = a.k
if a.storage: cfg["storage"] = a.storage
idx = FlatIndex(cfg["d"], METRIC_L2 if cfg["metric"] == "l2" else METRIC_IP, storage=cfg["storage"])
step = 2_000_000
for lo in range(0, cfg["nb"], step):
    idx.add(torch.from_numpy(gen_base(cfg, lo, min(cfg["nb"], lo + step))).cuda())
q = torch.from_numpy(gen_queries(cfg)).cuda()
for _ in range(a.iters):
    r = idx.search(q, cfg["k"])
torch.cuda.synchronize()
print("plan", idx.last_plan())
