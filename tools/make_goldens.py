"""Write full-size oracle goldens (tests/golden/full_<cfg>.json) for the GPU parity
tests at BASELINE sizes.  Calls only oracle/ and the seeded input generator.

    python tools/make_goldens.py c2 [c3 ...]

Each golden stores, for the bench's launch configuration (profile tier_max=0,
FS(W+I) replay with profile-derived limits over every user, ACT on the replay's
arrival times and overload flags) and for FS(W): the replay summary (incl. the
digest over every delivery, admission, final counter and the makespan), sha256
digests of the per-call output arrays, and the profile's small tables.
"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from paper_2411_15997_b200 import tracegen as G  # noqa: E402


def h(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run(name):
    c = G.CONFIGS[name]
    t0 = time.time()
    tr = G.generate(name)
    pcfg = dict(tier_max=c["profile"]["tier_max"], window_ms=60000, max_stage=64)
    p = O.profile(tr, pcfg)
    t1 = time.time()
    act = dict(window_ms=60000, limits_from_profile=1, limit_mult_q8=0, count_mode=0)
    eng = dict(c["engine"], mode=1, tier_max=255, alpha=1, beta=2, gamma=1, act=act)
    o, s = O.replay(tr, p, eng)
    t2 = time.time()
    st, sa = O.act(tr, p, act, overloaded=o["ovl"], t_ns_override=o["arrive_ns"])
    t3 = time.time()
    sta, saa = O.act(tr, p, act)                 # standalone screening: recorded times, overload always
    ow, sw = O.replay(tr, p, dict(eng, mode=0), outputs=False)
    out = {
        "citation": "written by tools/make_goldens.py from oracle/ only (SURVEY.md §8(c) O2-O5); "
                    "inputs: paper_2411_15997_b200/tracegen.py config " + name,
        "config": name, "n_calls": tr["n_calls"], "profile_cfg": pcfg, "engine": eng,
        "profile": {k: p[k].tolist() for k in ("T_req_a", "T_tok_a", "T_req_g", "T_tok_g", "nr_peak_r_a",
                                                "nr_peak_t_a", "maxstage")},
        "profile_sha": {k: h(p[k]) for k in ("cnt", "sum_in", "sum_sys", "sum_out", "hist", "nr_q", "peak_r_u",
                                             "peak_t_u", "peak_r_ua", "peak_t_ua")},
        "interp_q": p["interp_q"].tolist(),
        "replay_wi": s, "replay_w": sw,
        "replay_sha": {k: h(o[k]) for k in ("status", "ovl", "arrive_ns", "admit_ns", "first_ns", "finish_ns",
                                            "order", "counters", "admitted_per_app")},
        "act": {k: sa[k] for k in ("n_in", "n_admit", "n_block", "n_dropped", "n_filtered")},
        "act_sha": h(st),
        "act_equals_replay_status": bool((st == o["status"]).all()),
        "act_always": {k: saa[k] for k in ("n_in", "n_admit", "n_block", "n_dropped", "n_filtered")},
        "act_always_sha": h(sta),
        "oracle_seconds": {"profile": t1 - t0, "replay_wi": t2 - t1, "act": t3 - t2},
    }
    path = os.path.join(ROOT, "tests", "golden", f"full_{name}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(name, "written", path, out["oracle_seconds"], flush=True)




def run_c5(n_sample=12):
    """C5: oracle summaries of a seeded sample of the bench's 4096-scenario grid (bench.sweep_scenarios,
    the same list bench.py times), for the full-size sweep parity test."""
    import bench
    c = G.CONFIGS["c5"]
    tr = G.generate("c5")
    cfg, eng, pcfg = bench.workload_cfg("c2")
    p = O.profile(tr, pcfg)
    scen = bench.sweep_scenarios(eng, 4096)
    idx = sorted(int(i) for i in np.random.default_rng(55).choice(len(scen), n_sample, replace=False))
    t0 = time.time()
    sums, codes = O.sweep(tr, p, [scen[i] for i in idx])
    out = {"citation": "written by tools/make_goldens.py from oracle/ only (SURVEY.md §8(c) O4, A9); "
                       "inputs: tracegen config c5 and bench.sweep_scenarios(4096)",
           "config": "c5", "n_calls": tr["n_calls"], "seed": c["seed"], "profile_cfg": pcfg,
           "index": idx, "codes": [int(x) for x in codes], "summaries": sums,
           "oracle_seconds": time.time() - t0}
    path = os.path.join(ROOT, "tests", "golden", "full_c5_sample.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("c5 sample written", path, out["oracle_seconds"], flush=True)


def run_c5_full():
    """C5: oracle summaries of EVERY scenario of the bench's 4096-scenario grid
    (bench.sweep_scenarios, the list bench.py times), computed by P oracle replays in
    parallel threads (ctypes releases the GIL; the oracle keeps no global state), for the
    full-grid sweep parity test (tests/test_gpu_fullsize.py::test_sweep_c5_full)."""
    from concurrent.futures import ThreadPoolExecutor
    import bench
    c = G.CONFIGS["c5"]
    tr = G.generate("c5")
    cfg, eng, pcfg = bench.workload_cfg("c2")
    p = O.profile(tr, pcfg)
    scen = bench.sweep_scenarios(eng, 4096)
    P = len(os.sched_getaffinity(0))
    t0 = time.time()
    res = [None] * len(scen)
    done = [0]

    def one(i):
        s, cd = O.sweep(tr, p, [scen[i]])
        res[i] = (s[0], int(cd[0]))
        done[0] += 1
        if done[0] % 256 == 0:
            print(f"  {done[0]}/{len(scen)} scenarios, {time.time() - t0:.0f} s", flush=True)

    # longest first (participating calls grow with tier_max) for a balanced pool
    order = sorted(range(len(scen)), key=lambda i: -scen[i]["tier_max"])
    with ThreadPoolExecutor(P) as ex:
        list(ex.map(one, order))
    keys = list(res[0][0].keys())
    out = {"citation": "written by tools/make_goldens.py run_c5_full from oracle/ only (SURVEY.md §8(c) O4, "
                       "§8(d) run matrix 'C5: every scenario's summary + digest'); inputs: tracegen config c5 and "
                       "bench.sweep_scenarios(4096)",
           "config": "c5", "n_calls": tr["n_calls"], "seed": c["seed"], "profile_cfg": pcfg,
           "keys": keys, "codes": [r[1] for r in res],
           "summaries": [[r[0][k] for k in keys] for r in res],
           "oracle_threads": P, "oracle_seconds": time.time() - t0}
    path = os.path.join(ROOT, "tests", "golden", "full_c5.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("c5 full grid written", path, out["oracle_seconds"], flush=True)


def run_c2_metrics():
    """§5 metrics (oracle/metrics.py) of the full C2 FS(W+I) replay of the bench's configuration,
    global and per app, at three delay thresholds."""
    from oracle import metrics as M
    c = G.CONFIGS["c2"]
    tr = G.generate("c2")
    pcfg = dict(tier_max=c["profile"]["tier_max"], window_ms=60000, max_stage=64)
    p = O.profile(tr, pcfg)
    act = dict(window_ms=60000, limits_from_profile=1, limit_mult_q8=0, count_mode=0)
    eng = dict(c["engine"], mode=1, tier_max=255, alpha=1, beta=2, gamma=1, act=act)
    o, _ = O.replay(tr, p, eng)
    res = {}
    for thr in (0, 5_000_000, 1_000_000_000):
        g, per = M.replay_metrics(tr, o, thr)
        res[str(thr)] = {"global": g, "per_app": per}
    out = {"citation": "written by tools/make_goldens.py from oracle/ only (oracle/metrics.py, DESIGN.md R9); "
                       "inputs: tracegen config c2, the bench's FS(W+I) replay",
           "config": "c2", "n_calls": tr["n_calls"], "profile_cfg": pcfg, "engine": eng, "metrics": res}
    path = os.path.join(ROOT, "tests", "golden", "full_c2_metrics.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("c2 metrics written", path, flush=True)


def run_c4():
    """C4: the 100M-call profile (bench.py --workload c4 at one GPU builds exactly this trace)."""
    t0 = time.time()
    tr = G.generate("c4")
    t1 = time.time()
    pcfg = dict(tier_max=0, window_ms=60000, max_stage=64)
    p = O.profile(tr, pcfg)
    out = {
        "citation": "written by tools/make_goldens.py from oracle/ only (SURVEY.md §8(c) O2); inputs: tracegen config c4",
        "config": "c4", "n_calls": tr["n_calls"], "profile_cfg": pcfg,
        "profile": {k: p[k].tolist() for k in ("T_req_a", "T_tok_a", "T_req_g", "T_tok_g", "nr_peak_r_a",
                                                "nr_peak_t_a", "maxstage")},
        "profile_sha": {k: h(p[k]) for k in ("cnt", "sum_in", "sum_sys", "sum_out", "hist", "nr_q", "peak_r_u",
                                             "peak_t_u", "peak_r_ua", "peak_t_ua")},
        "interp_q": p["interp_q"].tolist(),
        "oracle_seconds": {"generate": t1 - t0, "profile": time.time() - t1},
    }
    path = os.path.join(ROOT, "tests", "golden", "full_c4.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("c4 written", path, out["oracle_seconds"], flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["c2"]:
        {"c5": run_c5, "c5full": run_c5_full, "c4": run_c4, "c2m": run_c2_metrics}.get(nm, lambda: run(nm))()
