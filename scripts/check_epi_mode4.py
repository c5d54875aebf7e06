import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from paper_2401_08281_b200 import FlatIndex, METRIC_L2
from oracle import flat_oracle as O
from parity import compare
rng = np.random.default_rng(1)
xb = rng.standard_normal((int(os.environ.get("NB", "300000")), 128), dtype=np.float32); q = rng.standard_normal((int(os.environ.get("NQ", "2000")), 128), dtype=np.float32)
idx = FlatIndex(128, METRIC_L2); idx.add(torch.from_numpy(xb).cuda())
res = {}
for epi in ("4", "8"):
    os.environ["FK_EPI"] = epi
    r = idx.search(torch.from_numpy(q).cuda(), 10); res[epi] = (r.ids.cpu().numpy(), r.distances.cpu().numpy())
    print(epi, idx.last_plan())
del os.environ["FK_EPI"]
wi, wd = O.flat_search_blas(xb, q, 10, "l2")
for e, (i, d) in res.items():
    print(e, compare(i, d, wi, wd))
diff = np.nonzero((res["4"][0] != res["8"][0]).any(1))[0]
print("differing rows", len(diff), diff[:5])
for r in diff[:3]:
    print(res["4"][0][r], res["4"][1][r]); print(res["8"][0][r], res["8"][1][r]); print(wi[r], wd[r])
