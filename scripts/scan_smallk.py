import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_08281_b200 import METRIC_L2, FlatIndex
g = torch.Generator(device="cuda"); g.manual_seed(1)
for d, storage, nb in ((256, "bf16", 200_000), (32, "fp32", 200_000), (128, "fp16", 1_000_000)):
    idx = FlatIndex(d, METRIC_L2, storage=storage)
    idx.add(torch.randn((nb, d), generator=g, device="cuda"))
    qall = torch.randn((2000, d), generator=g, device="cuda")
    for env in ("", "FK_EST_SMALLK0=1"):
        if env: os.environ["FK_EST_SMALLK0"] = "1"
        for nq in (129, 2000):
            for k in (33, 48, 64):
                q = qall[:nq].contiguous()
                idx.search(q, k); torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(3): idx.search(q, k)
                e1.record(); torch.cuda.synchronize()
                print(d, storage, nb, env or "-", nq, k, round(e0.elapsed_time(e1) / 3, 3), flush=True)
        if env: del os.environ["FK_EST_SMALLK0"]
    del idx; torch.cuda.empty_cache()
