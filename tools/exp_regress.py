"""Interleaved A/B of the C5 sweep between two builds of the library (this tree's and
ab_old/libfairserve.so built from an earlier tree), same box, same process order.
Usage: python tools/exp_regress.py [rounds]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import subprocess  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
code = r'''
import sys, time, torch
sys.path.insert(0, %r)
import bench
from paper_2411_15997_b200 import fairserve as F, tracegen as G
F.LIB_PATH = %r
tr = G.generate("c5"); ctx = F.Context(0); T = F.Trace(tr)
prof = F.build_app_profiles(ctx, T, dict(tier_max=0))
c, eng, pcfg = bench.workload_cfg("c2")
scen = bench.sweep_scenarios(eng, 4096)
torch.cuda.synchronize(); t0 = time.time()
F.sweep(ctx, T, prof, scen); torch.cuda.synchronize()
print(f"%s sweep {time.time() - t0:.3f} s", flush=True)
'''
new = os.path.join(ROOT, "paper_2411_15997_b200", "lib", "libfairserve.so")
old = os.path.join(ROOT, "ab_old", "libfairserve.so")
for r in range(rounds):
    for tag, path in (("new", new), ("old", old)):
        subprocess.run([sys.executable, "-c", code % (ROOT, path, tag)], check=False)
