import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
from paper_2401_08281_b200 import FlatIndex, METRIC_L2, config
from oracle import flat_oracle as O
config.blas_threshold = 0
rng = np.random.default_rng(33)
nb, d = 300_000, 32
xb = rng.standard_normal((nb, d), dtype=np.float32)
if os.environ.get("EDGE"):
    xb[np.array([3, 11, 12, nb - 1]), 2] = np.nan
    xb[np.array([5, 7, nb - 2])] = 1e20
q = rng.standard_normal((6, d), dtype=np.float32)
idx = FlatIndex(d, METRIC_L2); idx.add(xb)
res = idx.search(q, 10)
with np.errstate(invalid="ignore", over="ignore"):
    wi, wd = O.flat_search_blas(xb, q, 10, "l2")
print(os.environ.get("EDGE"), os.environ.get("FK_MERGE_SMC"), idx.last_plan()["S"], [bool(np.array_equal(res.ids[r], wi[r])) for r in range(6)])
