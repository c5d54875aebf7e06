"""Run one config's search in a loop for ~3 s while nvidia-smi samples SM clock,
power and throttle reasons (is the kernel power-capped?)."""
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import CONFIGS, gen_base, gen_queries
from paper_2401_08281_b200 import FlatIndex, METRIC_L2, METRIC_IP
cfg = dict(CONFIGS[int(os.environ.get("CFG", "2"))])
for kv in os.environ.get("OVERRIDE", "").split(","):
    if kv:
        a, b = kv.split("="); cfg[a] = int(b) if b.isdigit() else b
idx = FlatIndex(cfg["d"], METRIC_L2 if cfg["metric"] == "l2" else METRIC_IP, storage=cfg["storage"])
idx.add(torch.from_numpy(gen_base(cfg)).cuda())
q = torch.from_numpy(gen_queries(cfg)).cuda()
for _ in range(3):
    idx.search(q, cfg["k"])
torch.cuda.synchronize()
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                        "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
time.sleep(0.3)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 0
t0 = time.time()
e0.record()
while time.time() - t0 < 3.0:
    for _ in range(20):
        idx.search(q, cfg["k"])
    n += 20
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
smi.terminate()
rows = [r.split(",") for r in smi.stdout.read().strip().splitlines()]
clk = sorted(float(r[0]) for r in rows if len(r) >= 3)
pw = sorted(float(r[1]) for r in rows if len(r) >= 3)
reasons = sorted(set(r[2].strip() for r in rows if len(r) >= 3))
print(f"{os.environ.get('FK_DEBUG_FLAGS', '-')} {cfg['storage']} ms/search {e0.elapsed_time(e1) / n:.3f}  sm_mhz median {clk[len(clk) // 2]:.0f} min {clk[0]:.0f}  power median {pw[len(pw) // 2]:.0f} W  reasons {reasons}")
