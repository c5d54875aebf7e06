"""Per-tile clock64 timeline of CTA 0 (producer/MMA/epilogue handoffs)."""
import ctypes, os, sys, json
os.environ["FK_DEV_LIB"] = "1"  # timeline trace lives in the FK_DEV build only
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import CONFIGS, gen_base, gen_queries
from paper_2401_08281_b200 import FlatIndex, METRIC_L2, METRIC_IP
from paper_2401_08281_b200 import _native as N
from paper_2401_08281_b200 import build as B
B.build(verbose=False, dev=True)
cfg = dict(CONFIGS[int(os.environ.get("CFG", "2"))])
for kv in os.environ.get("OVERRIDE", "").split(","):
    if kv:
        a, b = kv.split("="); cfg[a] = int(b) if b.isdigit() else b
nb = min(cfg["nb"], 2_000_000)
idx = FlatIndex(cfg["d"], METRIC_L2 if cfg["metric"] == "l2" else METRIC_IP, storage=cfg["storage"])
idx.add(torch.from_numpy(gen_base(dict(cfg, nb=nb))).cuda())
q = torch.from_numpy(gen_queries(cfg)).cuda()
idx.search(q, cfg["k"]); torch.cuda.synchronize()
buf = torch.zeros(257 * 16, dtype=torch.int64, device="cuda")
N.check(N.lib().fk_debug_set_trace(idx._h, ctypes.c_void_p(buf.data_ptr())))
idx.search(q, cfg["k"]); torch.cuda.synchronize()
N.check(N.lib().fk_debug_set_trace(idx._h, None))
t_all = buf.cpu().numpy().reshape(257, 16).astype(np.int64)
t = t_all[:256]
t0 = t[0, 0]
print("plan", idx.last_plan(), os.environ.get("FK_DEBUG_FLAGS"))
for i in list(range(100, 106)):
    r = t[i] - t0
    print(i, f"wait_tempty {r[0]} got {r[1]} | kb0 full {r[13]} kb0 issued {r[9]} | kb1 full {r[14]} kb1 issued {r[10]} | commit {r[3]} || epi wait {r[4]} got {r[5]} done {r[7]}")
sl = slice(40, 240)
m = lambda a: float(np.median(a))
c = t[:, 3]
print("period/tile (commit[t+2]-commit[t])/2:", m((c[42:242] - c[40:240]) / 2))
print("MMA issuer: tempty wait", m(t[sl, 1] - t[sl, 0]), "| kb0 full wait", m(t[sl, 13] - t[sl, 1]),
      "| kb0 issue", m(t[sl, 9] - t[sl, 13]), "| kb1 full wait", m(t[sl, 14] - t[sl, 9]),
      "| kb1 issue", m(t[sl, 10] - t[sl, 14]), "| commit", m(t[sl, 3] - t[sl, 10]),
      "| idle before next own tile", m(t[42:242, 0] - t[40:240, 3]))
print("epilogue (warp 4): tfull wait", m(t[sl, 5] - t[sl, 4]), "| commit->got", m(t[sl, 5] - t[sl, 3]),
      "| busy", m(t[sl, 7] - t[sl, 6]), "| done->next wait", m(t[41:241, 4] - t[40:240, 7]))
ev = slice(40, 240, 2)
print("epilogue group 0: LDTM piece0 latency", m(t[ev, 11] - t[ev, 2]), "| piece0 compute + piece1 LDTM", m(t[ev, 12] - t[ev, 11]),
      "| piece1 compute + tail", m(t[ev, 7] - t[ev, 12]), "| got tfull -> ld issue", m(t[ev, 2] - t[ev, 6]))
slow = t[:, 8]
print("slow-path lanes per tile (warp 4): mean", slow[sl].mean(), "tiles with any", (slow[sl] > 0).mean())
print("slow warp-pieces by chunk 0..11:", list(t_all[256, 3:15]))
print("ALL CTAs: warp-pieces", t_all[256, 0], "with slow path", t_all[256, 1],
      f"({t_all[256, 1] / max(t_all[256, 0], 1):.4f})", "slow lanes", t_all[256, 2])
