"""Time cfg searches under several plan/env variants in one process (GPU)."""
import os
import sys
import time
import json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import CONFIGS, gen_base, gen_base_device, gen_queries
from paper_2401_08281_b200 import FlatIndex, METRIC_L2, METRIC_IP

cfgn = int(os.environ.get("CFG", "2"))
cfg = dict(CONFIGS[cfgn])
for kv in os.environ.get("OVERRIDE", "").split(","):
    if kv:
        a, b = kv.split("=")
        cfg[a] = int(b) if b.isdigit() else b
if os.environ.get("FK_DEV_LIB") == "1":  # FK_DEBUG_FLAGS variants need the FK_DEV build
    from paper_2401_08281_b200 import build as B
    B.build(verbose=False, dev=True)


def make_index():
    idx = FlatIndex(cfg["d"], METRIC_L2 if cfg["metric"] == "l2" else METRIC_IP, storage=cfg["storage"])
    for lo in range(0, cfg["nb"], 2_000_000):
        hi = min(cfg["nb"], lo + 2_000_000)
        idx.add(torch.from_numpy(gen_base(cfg, lo, hi)).cuda() if cfg["nb"] <= 2_000_000 else gen_base_device(cfg, lo, hi))
        torch.cuda.empty_cache()
    return idx


CREATE_TIME = ("FK_NO_FOLD", "FK_NUM_SMS")  # read by fk_create: rebuild the index for these variants
idx = make_index()
q = torch.from_numpy(gen_queries(cfg)).cuda()
variants = [v for v in sys.argv[1:]] or [""]
ref = None
for v in variants:
    env = dict(kv.split("=") for kv in v.split(";") if kv)
    for a, b in env.items():
        os.environ[a] = b
    if any(a in CREATE_TIME for a in env):
        del idx
        torch.cuda.empty_cache()
        idx = make_index()
    for _ in range(3):
        r = idx.search(q, cfg["k"])
    torch.cuda.synchronize()
    n = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        r = idx.search(q, cfg["k"])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    idx.set_profiling(True)
    idx.kernel_times()
    for _ in range(3):
        idx.search(q, cfg["k"])
    (tp, tf, tm), nl = idx.kernel_times()
    idx.set_profiling(False)
    same = None
    if ref is None:
        ref = (r.ids.clone(), r.distances.clone())
    else:
        same = bool(torch.equal(ref[0], r.ids) and torch.equal(ref[1], r.distances))
    print(json.dumps({"variant": v, "ms": round(ms, 3), "prep_fused_merge_ms": [round(tp, 3), round(tf, 3), round(tm, 3)], "qps": round(cfg["nq"] / ms * 1e3), "plan": idx.last_plan(),
                      "same_as_first": same}), flush=True)
    for a in env:
        del os.environ[a]
    if any(a in CREATE_TIME for a in env):
        del idx
        torch.cuda.empty_cache()
        idx = make_index()
