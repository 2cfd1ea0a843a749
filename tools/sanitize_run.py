"""Every C-ABI call once on C1 and on a 100k-call C2-shaped trace (profile, FS(W+I) replay, ACT
on the replay's arrivals and with overload always, a 6-scenario sweep, online steps, the §5
metrics, the multi-GPU profile protocol with 2 virtual ranks), for compute-sanitizer runs:
    compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_run.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2411_15997_b200 import build as B  # noqa: E402
from paper_2411_15997_b200 import fairserve as F  # noqa: E402
from paper_2411_15997_b200 import tracegen as G  # noqa: E402

B.build()
ctx = F.Context(0)
small = len(sys.argv) > 1 and sys.argv[1] == "small"
cases = [("c1", G.generate("c1"))]
if not small:
    cases.append(("c2-100k", G.generate(dict(G.CONFIGS["c2"], n_users=200, n_calls=100_000, seed=5))))
for name, tr in cases:
    T = F.Trace(tr)
    prof = F.build_app_profiles(ctx, T, dict(tier_max=255 if name == "c1" else 0))
    eng = dict(G.CONFIGS["c1" if name == "c1" else "c2"]["engine"], mode=1, tier_max=255,
               act=dict(window_ms=60000, limits_from_profile=1))
    o, s = F.wsc_replay(ctx, T, prof, eng)
    st, _ = F.act_throttle(ctx, T, prof, eng["act"], overloaded=o["ovl"], t_ns_override=o["arrive_ns"])
    st2, _ = F.act_throttle(ctx, T, prof, eng["act"])
    scen = [dict(eng, tier_max=tm, alpha=a) for tm, a in ((255, 1), (0, 1), (255, 2), (3, 1))]
    scen += [dict(eng, mode=0), dict(eng, mode=2)]
    F.sweep(ctx, T, prof, scen)
    F.replay_metrics(ctx, T, o, 5_000_000)
    ws = F.WscState(ctx, T, prof, eng)
    heads = [i for i in range(min(tr["n_calls"], 400)) if (int(tr["meta"][i]) >> 8) & 255 == 1][:8]
    st_, adm = ws.step(0, 0, 0, [], heads, [int(tr["t_ms"][i]) * 1_000_000 for i in heads])
    ws.step(10_000_000, 0, len(adm), list(adm), [], [])
    ws.read()
    shards = [F.Trace(G.shard_by_user(tr, r, 2)) for r in range(2)]
    if name != "c1":
        import ctypes as C
        c = F._profile_cfg(dict(tier_max=0), [])
        parts, bufs = [], []
        for sh in shards:
            p, w = C.c_void_p(), C.c_size_t(0)
            ctx._check(F.lib().fs_profile_local(ctx.h, F._a(sh.c), F._a(c), C.byref(p), C.byref(w)))
            parts.append(p)
            bufs.append(torch.zeros(w.value, dtype=torch.int64, device="cuda"))
        for _ in range(24):
            ds, ws_ = [], []
            for p, b in zip(parts, bufs):
                w, d = C.c_size_t(0), C.c_int(0)
                ctx._check(F.lib().fs_profile_round(p, C.c_void_p(b.data_ptr()), C.byref(w), C.byref(d)))
                ds.append(d.value); ws_.append(w.value)
            if ds[0]:
                break
            tot = sum(b[: ws_[0]] for b in bufs)
            for b in bufs:
                b[: ws_[0]] = tot
        for p in parts:
            h = C.c_void_p()
            ctx._check(F.lib().fs_profile_finalize(p, C.byref(h)))
            F.Profile(ctx, h)
            F.lib().fs_profile_partial_free(p)
    print(name, "replay", s["n_admitted"], "blocked", sum(s["n_block"]), flush=True)
torch.cuda.synchronize()
print("sanitize run done", flush=True)
