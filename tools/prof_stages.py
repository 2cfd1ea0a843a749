"""One profile + one ACT (overload = always) on a C3-shaped trace: the HBM-bound stages,
for ncu on the GPU box.  Usage: python tools/prof_stages.py [c3|c2] [n_calls]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2411_15997_b200 import build as B  # noqa: E402
from paper_2411_15997_b200 import fairserve as F  # noqa: E402
from paper_2411_15997_b200 import tracegen as G  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
B.build()
cfg = dict(G.CONFIGS[name])
if n:
    cfg["n_users"] = max(50, int(cfg["n_users"] * n / cfg["n_calls"]))
    cfg["n_calls"] = n
tr = G.generate(cfg)
ctx = F.Context(0)
T = F.Trace(tr)
ctx.set_timing(True)
torch.cuda.synchronize()
t0 = time.time()
prof = F.build_app_profiles(ctx, T, dict(tier_max=cfg["profile"]["tier_max"]))
t1 = time.time()
st, s = F.act_throttle(ctx, T, prof, dict(window_ms=60000, limits_from_profile=1))
torch.cuda.synchronize()
t2 = time.time()
print(f"{name} n={tr['n_calls']} profile {1e3*(t1-t0):.1f} ms act {1e3*(t2-t1):.1f} ms jacobi {s['jacobi_passes']}")
for k, v in sorted(ctx.timings().items(), key=lambda kv: -kv[1][1])[:20]:
    print(f"  {k:24s} {v[0]:5d} launches {v[1]:9.3f} ms")
