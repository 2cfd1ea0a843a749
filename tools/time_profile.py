"""Device time of fs_build_app_profiles on a device-generated trace (C4 by default), per kernel,
mean of `reps` L2-flushed calls after one warm-up.  Usage: python tools/time_profile.py [c4|c3] [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2411_15997_b200 import build as B  # noqa: E402
from paper_2411_15997_b200 import fairserve as F  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
B.build()
ctx = F.Context(0)
T = F.generate_trace(ctx, name)
pcfg = dict(tier_max=0, window_ms=60000, max_stage=64)
flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")
r = F.build_app_profiles(ctx, T, pcfg).read()
torch.cuda.synchronize()
ctx.timing_reset()
ctx.set_timing(True)
tot = 0.0
s = torch.cuda.current_stream()
for _ in range(reps):
    flush.zero_()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(s)
    F.build_app_profiles(ctx, T, pcfg)
    b.record(s)
    torch.cuda.synchronize()
    tot += a.elapsed_time(b)
print(f"{name} n={T.n} counted={int(r["n_app"].sum())} profile {tot / reps:.3f} ms per call")
for k, v in sorted(ctx.timings().items(), key=lambda kv: -kv[1][1])[:24]:
    print(f"  {k:24s} {v[0] / reps:5.1f} launches {v[1] / reps:9.3f} ms")
