"""Where the end-to-end (host buffers) time of a cfg2 search goes, 1 GPU.

Times, per search of 10k queries over 1M x 128 fp32 (k = 10):
  dev   -- index.search(device tensor), synchronized per step
  e2e   -- index.search(pinned host tensor) -> numpy results (the bench's e2e leg)
  h2d   -- the 5.12 MB pinned query copy alone
  d2h_pageable / d2h_pinned -- the 1.2 MB result copy into fresh numpy / pinned memory
Usage: python scripts/e2e_probe.py [--iters N]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_08281_b200 import FlatIndex  # noqa: E402


def wall(fn, iters):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(iters):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=30)
    a = ap.parse_args()
    rng = np.random.default_rng(0)
    xb = rng.standard_normal((1_000_000, 128), dtype=np.float32)
    xq = np.random.default_rng(1).standard_normal((10_000, 128), dtype=np.float32)
    index = FlatIndex(128, "l2")
    index.add(torch.from_numpy(xb).cuda())
    q_dev = torch.from_numpy(xq).cuda()
    q_pin = torch.from_numpy(xq).pin_memory()
    k = 10
    out = {}
    out["dev"] = wall(lambda: (index.search(q_dev, k), torch.cuda.synchronize()), a.iters)
    out["e2e"] = wall(lambda: index.search(q_pin, k), a.iters)
    out["e2e_numpy_pageable_q"] = wall(lambda: index.search(xq, k), a.iters)
    buf = torch.empty_like(q_dev)
    out["h2d"] = wall(lambda: buf.copy_(q_pin, non_blocking=True), a.iters)
    rd = torch.empty((10_000, k), dtype=torch.float32, device="cuda")
    ri = torch.empty((10_000, k), dtype=torch.int64, device="cuda")

    def d2h_pageable():
        D = np.empty((10_000, k), np.float32)
        I = np.empty((10_000, k), np.int64)
        torch.from_numpy(D).copy_(rd)
        torch.from_numpy(I).copy_(ri)

    pd = torch.empty((10_000, k), dtype=torch.float32).pin_memory()
    pi = torch.empty((10_000, k), dtype=torch.int64).pin_memory()

    def d2h_pinned():
        pd.copy_(rd, non_blocking=True)
        pi.copy_(ri, non_blocking=True)
        torch.cuda.synchronize()

    def d2h_pinned_memcpy():
        d2h_pinned()
        D = np.empty((10_000, k), np.float32)
        I = np.empty((10_000, k), np.int64)
        D[...] = pd.numpy()
        I[...] = pi.numpy()

    out["d2h_pageable"] = wall(d2h_pageable, a.iters)
    out["d2h_pinned"] = wall(d2h_pinned, a.iters)
    out["d2h_pinned_memcpy"] = wall(d2h_pinned_memcpy, a.iters)
    print(json.dumps({k2: round(v, 4) for k2, v in out.items()}))


if __name__ == "__main__":
    main()
