"""A/B of the sweep's per-user ACT ring capacity (FS_SWEEP_RING_CAP): the 4096-scenario C5 sweep,
first launch and capacity-retry launch device times.  Usage: FS_SWEEP_RING_CAP=k python tools/exp_ring.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_15997_b200 import build as B  # noqa: E402
from paper_2411_15997_b200 import fairserve as F  # noqa: E402
from paper_2411_15997_b200 import tracegen as G  # noqa: E402

B.build()
tr = G.generate(G.CONFIGS["c5"])
ctx = F.Context(0)
T = F.Trace(tr)
prof = F.build_app_profiles(ctx, T, dict(tier_max=0))
c, eng, pcfg = bench.workload_cfg("c5")
scen = bench.sweep_scenarios(eng, 4096)
ref = None
for rep in range(2):
    torch.cuda.synchronize()
    ctx.timing_reset()
    ctx.set_timing(True)
    sums, codes = F.sweep(ctx, T, prof, scen)
    torch.cuda.synchronize()
    ctx.set_timing(False)
    tm = ctx.timings()
    dig = hash(tuple(int(s["digest"]) for s in sums))
    print(f"ring cap {os.environ.get('FS_SWEEP_RING_CAP', 'default')}: sweep {tm.get('wsc_sweep', (0, 0))[1]:.1f} ms, "
          f"retry {tm.get('wsc_sweep_retry', (0, 0))[1]:.1f} ms, codes {sorted(set(np.asarray(codes).tolist()))} digests {dig:x}", flush=True)
