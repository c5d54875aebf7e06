"""Full-size parity spot check (GPU vs oracle) for a storage / epilogue variant."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_2401_08281_b200 import FlatIndex, METRIC_L2, METRIC_IP
from oracle import flat_oracle as O
from parity import compare
nb, nq, d = int(os.environ.get("NB", "1000000")), int(os.environ.get("NQ", "3000")), int(os.environ.get("D", "128"))
storage, metric, k = os.environ.get("STORAGE", "fp32"), os.environ.get("METRIC", "l2"), int(os.environ.get("K", "10"))
rng = np.random.default_rng(1)
xb = rng.standard_normal((nb, d), dtype=np.float32); q = rng.standard_normal((nq, d), dtype=np.float32)
idx = FlatIndex(d, METRIC_L2 if metric == "l2" else METRIC_IP, storage=storage); idx.add(torch.from_numpy(xb).cuda())
xr, qr = O.round_to(xb, storage), O.round_to(q, storage)
wi, wd = O.flat_search_blas(xr, qr, k, metric)
for v in os.environ.get("VARIANTS", "FK_EPI=4,FK_EPI=8").split(","):
    a, b = v.split("=")
    os.environ[a] = b
    r = idx.search(torch.from_numpy(q).cuda(), k)
    print(v, idx.last_plan(), compare(r.ids.cpu().numpy(), r.distances.cpu().numpy(), wi, wd), flush=True)
    del os.environ[a]
