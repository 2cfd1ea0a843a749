"""Time one fs_sweep of S scenarios over the C5 trace (C2-shaped, 1M calls).
Usage: python tools/prof_sweep.py [S] [n_calls] [n_users]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_15997_b200 import build as B  # noqa: E402
from paper_2411_15997_b200 import fairserve as F  # noqa: E402
from paper_2411_15997_b200 import tracegen as G  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 256
n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
nu = int(sys.argv[3]) if len(sys.argv) > 3 else 0
B.build()
cfg = dict(G.CONFIGS["c5"])
if n:
    cfg["n_users"] = max(50, int(cfg["n_users"] * n / cfg["n_calls"]))
    cfg["n_calls"] = n
if nu:
    cfg["n_users"] = nu
tr = G.generate(cfg)
ctx = F.Context(0)
T = F.Trace(tr)
prof = F.build_app_profiles(ctx, T, dict(tier_max=0))
c, eng, pcfg = bench.workload_cfg("c2")
scen = bench.sweep_scenarios(eng, S)
torch.cuda.synchronize()
t0 = time.time()
sums, codes = F.sweep(ctx, T, prof, scen)
torch.cuda.synchronize()
dt = time.time() - t0
ok = int((codes == 0).sum())
print(f"sweep S={S} n={tr['n_calls']}: {dt:.2f} s, {S * tr['n_calls'] / dt / 1e6:.1f} M calls/s, ok={ok}/{S}, "
      f"codes={sorted(set(codes.tolist()))}", flush=True)
