"""Sweep-cost experiment: the bench's 4096 C5 scenarios as they are, then the same scenarios with every
(alpha, beta, gamma, E) replaced by one combination (one Eq. 3 increment table instead of 16: the
L2 working set of the sweep shrinks by ~120 MB).  Usage: python tools/exp_combo.py"""
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

B.build()
tr = G.generate("c5")
ctx = F.Context(0)
T = F.Trace(tr)
prof = F.build_app_profiles(ctx, T, dict(tier_max=0))
c, eng, pcfg = bench.workload_cfg("c2")
scen = bench.sweep_scenarios(eng, 4096)
one = [dict(s, alpha=1, beta=2, gamma=1, prio_abusive_q16=65536) for s in scen]
for name, sc in (("grid", scen), ("one-combo", one), ("grid", scen), ("one-combo", one)):
    torch.cuda.synchronize()
    t0 = time.time()
    sums, codes = F.sweep(ctx, T, prof, sc)
    torch.cuda.synchronize()
    print(f"{name}: {time.time() - t0:.2f} s", flush=True)
