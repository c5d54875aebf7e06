"""Experiment: is the fused kernel L2-bandwidth bound?  Time cfg2-shaped
searches with fewer SMs and with 16-bit storage (more B bytes per MMA cycle)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import CONFIGS, gen_base, gen_queries
from paper_2401_08281_b200 import FlatIndex, METRIC_L2

cfg = CONFIGS[2]
xb = torch.from_numpy(gen_base(cfg)).cuda()
q = torch.from_numpy(gen_queries(cfg)).cuda()
for storage in ("fp32", "bf16"):
    for nsm in (148, 74, 37):
        os.environ["FK_NUM_SMS"] = str(nsm)
        idx = FlatIndex(128, METRIC_L2, storage=storage)
        idx.add(xb)
        for _ in range(2):
            idx.search(q, 10)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            idx.search(q, 10)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        mult = 2 if storage == "fp32" else 1
        eb = 4 if storage == "fp32" else 2
        # L2->SM bytes: every unit streams its chunk of B (hi+lo)
        plan = idx.last_plan()
        bytes_l2 = 79 * 1_000_000 * 128 * eb * mult
        print(json.dumps({"storage": storage, "sms": nsm, "ms": round(ms, 3), "plan": plan,
                          "l2_to_sm_TBps": round(bytes_l2 / ms / 1e9, 2)}), flush=True)
        del idx
