import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_08281_b200 import METRIC_L2, FlatIndex
g = torch.Generator(device="cuda"); g.manual_seed(1)
idx = FlatIndex(768, METRIC_L2, storage="fp32")
idx.add(torch.randn((200_000, 768), generator=g, device="cuda"))
qall = torch.randn((2000, 768), generator=g, device="cuda")
for env in ("", "FK_NO_EST=1"):
    if env: os.environ["FK_NO_EST"] = "1"
    for nq in (20, 129):
        for k in (33, 64, 128, 256, 600):
            q = qall[:nq].contiguous()
            idx.search(q, k); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3): idx.search(q, k)
            e1.record(); torch.cuda.synchronize()
            print(env or "-", nq, k, round(e0.elapsed_time(e1) / 3, 3), idx.last_plan(), flush=True)
    if env: del os.environ["FK_NO_EST"]
