#!/bin/bash
cat > /tmp/sb.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from bench import CONFIGS, gen_base, gen_queries
from paper_2401_08281_b200 import IndexFlatL2
cfg = dict(CONFIGS[2])
idx = IndexFlatL2(cfg["d"])
idx.add(torch.from_numpy(gen_base(cfg)).cuda())
q = torch.from_numpy(gen_queries(cfg)).cuda()
for nq in (20, 64, 128, 129, 256):
    r = idx.search(q[:nq].contiguous(), 10); torch.cuda.synchronize()
    print(nq, idx.last_plan(), flush=True)
PY
FK_DIAG=1 timeout 600 python /tmp/sb.py 2>&1 | tail -20
