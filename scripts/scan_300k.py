import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_08281_b200 import METRIC_L2, FlatIndex
g = torch.Generator(device="cuda"); g.manual_seed(0)
for nb in (300_000, 1_000_000):
    idx = FlatIndex(128, METRIC_L2, storage="fp16")
    idx.add(torch.randn((nb, 128), generator=g, device="cuda"))
    q = torch.randn((100, 128), generator=g, device="cuda")
    for env in ("", "FK_NO_EST=1", "FK_FORCE_S=40", "FK_FORCE_S=16"):
        for kv in env.split(";"):
            if kv: a, b = kv.split("="); os.environ[a] = b
        for k in (100, 1000):
            idx.search(q, k); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3): idx.search(q, k)
            e1.record(); torch.cuda.synchronize()
            print(nb, env or "-", k, round(e0.elapsed_time(e1) / 3, 3), idx.last_plan(), flush=True)
        for kv in env.split(";"):
            if kv: del os.environ[kv.split("=")[0]]
