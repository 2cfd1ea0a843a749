"""Device time of fs_act_throttle per kernel on a device-generated trace (C3 by default): with
replay-like arrival times (heads at their recorded time, continuations delayed 0-50 ms) and a
20 % overload mask, and with overload always.  Mean of `reps` L2-flushed calls after a warm-up.
Usage: python tools/time_act.py [c3|c2|c4] [reps] [both|replay|always]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2411_15997_b200 import build as B  # noqa: E402
from paper_2411_15997_b200 import fairserve as F  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
which = sys.argv[3] if len(sys.argv) > 3 else "both"
B.build()
ctx = F.Context(0)
T = F.generate_trace(ctx, name)
prof = F.build_app_profiles(ctx, T, dict(tier_max=0))
n = T.n
g = torch.Generator(device="cuda").manual_seed(7)
meta = T.t["meta"].to(torch.int64) & 0xFFFFFFFF
stage = (meta >> 8) & 255
tov = T.t["t_ms"].to(torch.int64) * 1_000_000
tov = tov + (stage > 1).to(torch.int64) * torch.randint(0, 50_000_000, (n,), device="cuda", generator=g)
ovl = (torch.rand(n, device="cuda", generator=g) < 0.2).to(torch.uint8)
act = dict(window_ms=60000, limits_from_profile=1)
flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")
s = torch.cuda.current_stream()
cases = [("replay-like arrivals, 20% overloaded", dict(overloaded=ovl, t_ns_override=tov)),
         ("recorded times, overload always", {})]
cases = cases[:1] if which == "replay" else cases[1:] if which == "always" else cases
for label, kw in cases:
    st, summ = F.act_throttle(ctx, T, prof, act, **kw)
    torch.cuda.synchronize()
    ctx.timing_reset()
    ctx.set_timing(True)
    tot = 0.0
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        F.act_throttle(ctx, T, prof, act, status=st, **kw)
        b.record(s)
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    ctx.set_timing(False)
    print(f"{name} n={n} ACT ({label}): {tot / reps:.3f} ms per call; blocked {sum(summ['n_block'])} "
          f"passes {summ['jacobi_passes']} fixup users {summ['n_fixup_users']}", flush=True)
    for k, v in sorted(ctx.timings().items(), key=lambda kv: -kv[1][1])[:16]:
        print(f"  {k:24s} {v[0] / reps:5.1f} launches {v[1] / reps:9.3f} ms", flush=True)
