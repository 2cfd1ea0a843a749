"""Projected strong scaling of the C5 sweep from one GPU: the grid split by fairserve.lpt_split over
N ranks; every rank's slice timed on this GPU (device time, CUDA events) -- T_N = the slowest slice.
Usage: python tools/scale_slices.py [N ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_15997_b200 import build as B  # noqa: E402
from paper_2411_15997_b200 import fairserve as F  # noqa: E402
from paper_2411_15997_b200 import tracegen as G  # noqa: E402

Ns = [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]
B.build()
tr = G.generate(G.CONFIGS["c5"])
ctx = F.Context(0)
T = F.Trace(tr)
prof = F.build_app_profiles(ctx, T, dict(tier_max=0))
c, eng, pcfg = bench.workload_cfg("c5")
scen = bench.sweep_scenarios(eng, 4096)
costs = F.scenario_costs(tr["meta"], scen)
s = torch.cuda.current_stream()


def timed(sc):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s)
    _, codes = F.sweep(ctx, T, prof, sc)
    b.record(s)
    torch.cuda.synchronize()
    assert (codes == 0).all()
    return a.elapsed_time(b) / 1e3


t1 = None
for N in Ns:
    parts = F.lpt_split(costs, N)
    ts = [timed([scen[i] for i in p]) for p in (parts if N > 1 else [list(range(len(scen)))])]
    tn = max(ts)
    if N == 1:
        t1 = tn
    eff = f"{t1 / (N * tn):.2f}" if t1 else "-"
    print(f"N={N}: slices {len(parts[0])} scenarios, slowest {tn:.2f} s (all: {' '.join(f'{x:.2f}' for x in ts)}), "
          f"T1/(N*TN) = {eff}", flush=True)
