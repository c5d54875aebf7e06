import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import CONFIGS, gen_base, gen_queries
from paper_2401_08281_b200 import IndexFlatL2
cfg = dict(CONFIGS[2])
idx = IndexFlatL2(cfg["d"])
idx.add(torch.from_numpy(gen_base(cfg)).cuda())
q = torch.from_numpy(gen_queries(cfg)).cuda()[:int(os.environ.get("NQ", "19"))].contiguous()
for _ in range(3):
    idx.search(q, 10)
torch.cuda.synchronize()
