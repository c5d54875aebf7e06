"""Time the §8(f) paths beside the flat search on one GPU (CUDA events, inputs
resident on the device), each with the numpy restatement of the reference
timed on a bounded sample of the same work (host cores):

  * kmeans_assign (quantize.py:38-62): 1M x 128 fp32 points, 4096 fp64 centroids
  * probe_lists (ivf.py:324-326): 10k queries, 4096-cell coarse quantizer, nprobe 32
  * refine_search (core.py:368-394): fp16 fast index -> exact fp32 re-rank, 1M x 128,
    10k queries, shortlist 100, k 10
  * remove_ids (flat.py:46-56): 10 % of 1M ids

    python scripts/aux_bench.py [out.jsonl]
One JSON line per path: GPU ms, rate, CPU-restatement rate and sample.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import flat_oracle as O  # CPU baseline leg only (test infrastructure)
from paper_2401_08281_b200 import FlatIndex, IndexFlatL2, kmeans_assign, coarse_quantizer, probe_lists, refine_search

out = open(sys.argv[1], "w") if len(sys.argv) > 1 else None
rng = np.random.default_rng(0)
NB, D, NQ = 1_000_000, 128, 10_000
xb = rng.standard_normal((NB, D), dtype=np.float32)
q = np.random.default_rng(1).standard_normal((NQ, D), dtype=np.float32)
xb_d, q_d = torch.from_numpy(xb).cuda(), torch.from_numpy(q).cuda()


def gpu_ms(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def emit(rec):
    line = json.dumps(rec)
    print(line, flush=True)
    if out:
        out.write(line + "\n")


# ---- k-means assignment (fp64 exact) ----
cent = rng.standard_normal((4096, D)).astype(np.float64)
cent_d = torch.from_numpy(cent).cuda()
ms = gpu_ms(lambda: kmeans_assign(xb_d, cent_d))
ns = 20_000
t0 = time.perf_counter()
x64 = xb[:ns].astype(np.float64)
dm = (x64 * x64).sum(1)[:, None] + (cent * cent).sum(1)[None, :] - 2.0 * x64 @ cent.T  # quantize.py:47-52
a_cpu = dm.argmin(1)
cpu_s = time.perf_counter() - t0
a_gpu, _ = kmeans_assign(xb_d[:ns], cent_d)
emit({"path": "kmeans_assign", "shape": "1M x 128 fp32, 4096 fp64 centroids", "gpu_ms": round(ms, 3),
      "rows_per_s": round(NB / ms * 1e3), "cpu_rows_per_s": round(ns / cpu_s), "cpu_sample": f"{ns} rows",
      "sample_agree": float((a_gpu.cpu().numpy() == a_cpu).mean())})

# ---- IVF probing ----
cq = coarse_quantizer(D)
cq.add(torch.from_numpy(cent.astype(np.float32)).cuda())
ms = gpu_ms(lambda: probe_lists(cq, q_d, 32))
nqs = 2000
t0 = time.perf_counter()
want, _ = O.flat_search_blas(cent.astype(np.float32), q[:nqs], 32, "l2")
cpu_s = time.perf_counter() - t0
got = probe_lists(cq, q[:nqs], 32)
gaps = [0.0]
c64 = cent.astype(np.float32).astype(np.float64)
for i in range(nqs):
    a, b = set(got[i].tolist()), set(want[i].tolist())
    if a != b:  # relative distance gap between the swapped cells (fp64 exact)
        qd = q[i].astype(np.float64)
        dist = lambda j: float(((qd - c64[j]) ** 2).sum())
        gaps.append(max(abs(dist(j) - dist(l)) / max(dist(l), 1e-30) for j in a - b for l in b - a))
emit({"path": "probe_lists", "shape": "10k queries, 4096 cells, nprobe 32", "gpu_ms": round(ms, 3),
      "qps": round(NQ / ms * 1e3), "cpu_qps": round(nqs / cpu_s), "cpu_sample": f"{nqs} queries",
      # (3xTF32 vs OpenBLAS sgemm rounding can swap exact near-ties at the 32nd place)
      "sample_rows_identical": float(np.mean([np.array_equal(a, b) for a, b in zip(got, want)])),
      "sample_recall": float(np.mean([len(set(a) & set(b)) / 32 for a, b in zip(got, want)])),
      "max_rel_gap_of_swaps": max(gaps)})

# ---- refine_search ----
fast = FlatIndex(D, storage="fp16")
fast.add(xb_d)
exact = IndexFlatL2(D)
exact.add(xb_d)
ms = gpu_ms(lambda: refine_search(fast, exact, q_d, 10, 100), reps=3)
ms_fast = gpu_ms(lambda: fast.search(q_d, 100), reps=3)
nqs = 200
cand = fast.search(q[:nqs], 100).ids
t0 = time.perf_counter()
want_ids, _ = O.refine_rerank(xb, np.arange(NB, dtype=np.int64), q[:nqs], cand, 10)
cpu_s = time.perf_counter() - t0
got = refine_search(fast, exact, q[:nqs], 10, 100)
emit({"path": "refine_search", "shape": "1M x 128, fp16 fast -> fp32 exact, 10k queries, shortlist 100, k 10",
      "gpu_ms": round(ms, 3), "gpu_ms_fast_search": round(ms_fast, 3), "gpu_ms_rerank": round(ms - ms_fast, 3),
      "qps": round(NQ / ms * 1e3), "cpu_rerank_qps": round(nqs / cpu_s), "cpu_sample": f"{nqs} queries (re-rank only)",
      "sample_equal": bool(np.array_equal(np.asarray(got.ids), want_ids))})

# ---- remove_ids ----
kill = np.random.default_rng(5).choice(NB, NB // 10, replace=False).astype(np.int64)


def remove_once():
    idx = IndexFlatL2(D)
    idx.add(xb_d)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = idx.remove_ids(kill)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), n, idx


remove_once()
ms, n, idx = remove_once()
t0 = time.perf_counter()
_, keep_ids, nrm = O.remove_ids(xb, np.arange(NB, dtype=np.int64), kill)
cpu_s = time.perf_counter() - t0
emit({"path": "remove_ids", "shape": "remove 100k of 1M x 128 fp32", "gpu_ms": round(ms, 3), "removed": int(n),
      "cpu_ms": round(cpu_s * 1e3, 3), "cpu_sample": "full", "ids_equal": bool(np.array_equal(np.asarray(idx.ids), keep_ids))})
