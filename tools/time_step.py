"""Latency of the online form (fs_wsc_step) on the C2 trace: an online loop that
delivers the calls in trace order (64 per iteration boundary, recorded times), finishes admitted
calls L_O boundaries after admission and keeps a KV / batch budget; reports the k_step device time
and the host wall time per step.  Usage: python tools/time_step.py [steps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2411_15997_b200 import build as B  # noqa: E402
from paper_2411_15997_b200 import fairserve as F  # noqa: E402
from paper_2411_15997_b200 import tracegen as G  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
B.build()
tr = G.generate("c2")
ctx = F.Context(0)
T = F.Trace(tr)
prof = F.build_app_profiles(ctx, T, dict(tier_max=0))
eng = dict(G.CONFIGS["c2"]["engine"], mode=1, tier_max=255, act=dict(window_ms=60000, limits_from_profile=1))
st = F.WscState(ctx, T, prof, eng)
lo = tr["len_out"].astype(np.int64)
pi = tr["len_in"].astype(np.int64) + tr["len_sys"].astype(np.int64)
pos, occ, nb, running = 0, 0, 0, []
ctx.timing_reset()
ctx.set_timing(True)
t0 = time.time()
for it in range(steps):
    fin = [r for (f, r) in running if f <= it]
    running = [(f, r) for (f, r) in running if f > it]
    for r in fin:
        occ -= int(pi[r] + lo[r]); nb -= 1
    arr = list(range(pos, min(tr["n_calls"], pos + 64)))
    pos += len(arr)
    now = int(tr["t_ms"][arr[-1]]) * 1_000_000 if arr else it
    s, adm = st.step(now, occ, nb, fin, arr, [int(tr["t_ms"][r]) * 1_000_000 for r in arr])
    for r in adm:
        running.append((it + int(lo[r]), int(r)))
        occ += int(pi[r]); nb += 1
torch.cuda.synchronize()
wall = time.time() - t0
kt = ctx.timings()
ks = kt.get("wsc_step", (0, 0.0))
print(f"fs_wsc_step: {steps} steps, {pos} calls delivered; k_step {ks[1] / max(ks[0], 1) * 1e3:.1f} us per step "
      f"(device), {wall / steps * 1e6:.1f} us per step (host wall, incl. launch + sync + Python)", flush=True)
