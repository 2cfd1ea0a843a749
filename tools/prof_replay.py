"""Run one replay (and optionally the data-parallel calls) of a C2/C3-shaped trace,
for ncu / timing experiments on the GPU box.  Usage:
    python tools/prof_replay.py [c2|c3] [n_calls] [mode] [n_users]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2411_15997_b200 import build as B  # noqa: E402
from paper_2411_15997_b200 import fairserve as F  # noqa: E402
from paper_2411_15997_b200 import tracegen as G  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
mode = int(sys.argv[3]) if len(sys.argv) > 3 else 1
nu = int(sys.argv[4]) if len(sys.argv) > 4 else 0
B.build()
cfg = dict(G.CONFIGS[name])
if n:
    cfg["n_users"] = max(50, int(cfg["n_users"] * n / cfg["n_calls"]))
    cfg["n_calls"] = n
if nu:
    cfg["n_users"] = nu
tr = G.generate(cfg)
ctx = F.Context(0)
T = F.Trace(tr)
prof = F.build_app_profiles(ctx, T, dict(tier_max=cfg["profile"]["tier_max"]))
eng = dict(cfg["engine"], mode=mode, tier_max=255, act=dict(window_ms=60000, limits_from_profile=1))
torch.cuda.synchronize()
t0 = time.time()
o, s = F.wsc_replay(ctx, T, prof, eng)
torch.cuda.synchronize()
dt = time.time() - t0
print(f"{name} n={tr['n_calls']} users={tr['n_users']} replay {dt*1e3:.1f} ms; "
      f"{dt*1e9/tr['n_calls']:.0f} ns/call; iterations {s['n_iterations']} admitted {s['n_admitted']} "
      f"blocked {sum(s['n_block'])} ovl_arrivals {s['n_ovl_arrivals']}", flush=True)
