"""GPU parity at BASELINE.json's full sizes, in bench.py's launch configuration,
against oracle goldens written by tools/make_goldens.py (oracle/ only):
profile tables, every per-call replay output (sha256), the replay digest/summary,
and the ACT statuses on the replay's arrivals (P8 cross-check)."""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2411_15997_b200 import tracegen as G

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def h(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_full_size(name):
    path = os.path.join(GOLD, f"full_{name}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    g = json.load(open(path))
    import torch
    from paper_2411_15997_b200 import build, fairserve as F
    build.build()
    ctx = F.Context(0)
    tr = G.generate(name)
    assert tr["n_calls"] == g["n_calls"]
    T = F.Trace(tr)
    prof = F.build_app_profiles(ctx, T, g["profile_cfg"])
    p = prof.read()
    for k, v in g["profile"].items():
        assert p[k].tolist() == v, k
    for k, v in g["profile_sha"].items():
        assert h(p[k]) == v, k
    np.testing.assert_allclose(p["interp_q"], np.array(g["interp_q"]), rtol=1e-6)
    o, s = F.wsc_replay(ctx, T, prof, g["engine"])
    for k in ("n_arrived", "n_block", "n_dropped", "n_admitted", "n_finished", "n_iterations", "n_ovl_arrivals",
              "makespan_ns", "sum_wait_ns", "max_wait_ns", "sum_ttft_ns", "u_min", "u_max", "digest"):
        assert s[k] == g["replay_wi"][k], (k, s[k], g["replay_wi"][k])
    conv = {"status": np.uint8, "ovl": np.uint8, "arrive_ns": np.int64, "admit_ns": np.int64, "first_ns": np.int64,
            "finish_ns": np.int64, "order": np.uint32, "counters": np.uint64, "admitted_per_app": np.uint64}
    for k, v in g["replay_sha"].items():
        a = o[k].cpu().numpy().view(conv[k]) if o[k].dtype != torch.uint8 else o[k].cpu().numpy()
        assert h(a) == v, k
    st, sa = F.act_throttle(ctx, T, prof, g["engine"]["act"], overloaded=o["ovl"], t_ns_override=o["arrive_ns"])
    assert h(st.cpu().numpy()) == g["act_sha"]
    for k, v in g["act"].items():
        assert sa[k] == v, k
    _, sw = F.wsc_replay(ctx, T, prof, dict(g["engine"], mode=0), outputs=False)
    assert sw["digest"] == g["replay_w"]["digest"]
    if "act_always_sha" in g:                   # ACT as standalone screening: overload always
        st2, sa2 = F.act_throttle(ctx, T, prof, g["engine"]["act"])
        assert h(st2.cpu().numpy()) == g["act_always_sha"]
        for k, v in g["act_always"].items():
            assert sa2[k] == v, k


def test_sweep_c5_full():
    """fs_sweep of the bench's whole 4096-scenario C5 grid (the launch bench.py times): EVERY
    scenario's summary (counts, times, counters, digest over every delivery / admission / final
    counter) and code equals the oracle's (tests/golden/full_c5.json, all 4096 oracle replays,
    tools/make_goldens.py run_c5_full); every scenario also satisfies the engine's conservation
    properties."""
    path = os.path.join(GOLD, "full_c5.json")
    assert os.path.exists(path), f"{path} missing (tools/make_goldens.py c5full)"
    g = json.load(open(path))
    import bench
    from paper_2411_15997_b200 import build, fairserve as F
    build.build()
    ctx = F.Context(0)
    tr = G.generate("c5")
    assert tr["n_calls"] == g["n_calls"]
    T = F.Trace(tr)
    _, eng, pcfg = bench.workload_cfg("c2")
    assert pcfg == g["profile_cfg"]
    prof = F.build_app_profiles(ctx, T, pcfg)
    scen = bench.sweep_scenarios(eng, 4096)
    sums, codes = F.sweep(ctx, T, prof, scen)
    assert len(g["summaries"]) == len(scen) == 4096
    keys = g["keys"]
    bad = [i for i in range(len(scen))
           if int(codes[i]) != g["codes"][i] or [sums[i][k] for k in keys] != g["summaries"][i]]
    assert not bad, (len(bad), bad[:5], sums[bad[0]], g["summaries"][bad[0]])
    tiers = tr["meta"] >> 24
    heads = ((tr["meta"] >> 8) & 255) == 1
    for s, c, sc in zip(sums, codes, scen):
        assert c == 0
        part = tiers <= sc["tier_max"]
        assert s["n_filtered"] == int((~part).sum())
        assert s["n_admitted"] == s["n_finished"]
        assert s["n_arrived"] == s["n_admitted"] + sum(s["n_block"])
        assert s["n_arrived"] + s["n_dropped"] + s["n_filtered"] == tr["n_calls"]
        assert sum(s["n_block"]) <= int((heads & part).sum())
        assert s["u_min"] <= s["u_max"]


@pytest.mark.parametrize("world", [2, 8])
def test_sweep_c5_slices(world):
    """The strong-scaling slices: the C5 grid split by fairserve.lpt_split over `world` ranks, each
    rank's slice (2048 / 512 scenarios: the solo-slot kernel) swept on this GPU -- every summary equals
    the oracle's golden for that scenario."""
    path = os.path.join(GOLD, "full_c5.json")
    assert os.path.exists(path), f"{path} missing (tools/make_goldens.py c5full)"
    g = json.load(open(path))
    import bench
    from paper_2411_15997_b200 import build, fairserve as F
    build.build()
    ctx = F.Context(0)
    tr = G.generate("c5")
    T = F.Trace(tr)
    _, eng, pcfg = bench.workload_cfg("c2")
    prof = F.build_app_profiles(ctx, T, pcfg)
    scen = bench.sweep_scenarios(eng, 4096)
    parts = F.lpt_split(F.scenario_costs(tr["meta"], scen), world)
    keys = g["keys"]
    for r in (0, world - 1):
        idx = parts[r]
        sums, codes = F.sweep(ctx, T, prof, [scen[i] for i in idx])
        bad = [j for j, i in enumerate(idx)
               if int(codes[j]) != g["codes"][i] or [sums[j][k] for k in keys] != g["summaries"][i]]
        assert not bad, (r, len(bad), bad[:5])


def test_profile_c4_full():
    """The 100M-call C4 profile (bench.py --workload c4 at one GPU) against the oracle's golden:
    every table bit-exact (sha256), interpolated quantiles within 1e-6."""
    path = os.path.join(GOLD, "full_c4.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    g = json.load(open(path))
    from paper_2411_15997_b200 import build, fairserve as F
    build.build()
    ctx = F.Context(0)
    tr = G.generate("c4")
    assert tr["n_calls"] == g["n_calls"]
    p = F.build_app_profiles(ctx, F.Trace(tr), g["profile_cfg"]).read()
    for k, v in g["profile"].items():
        assert p[k].tolist() == v, k
    for k, v in g["profile_sha"].items():
        assert h(p[k]) == v, k
    np.testing.assert_allclose(p["interp_q"], np.array(g["interp_q"]), rtol=1e-6)


def test_metrics_c2_full():
    """fs_replay_metrics over the full C2 FS(W+I) replay (the bench's configuration) against the
    oracle's §5 metrics (tests/golden/full_c2_metrics.json): every count exact, Jain within 1e-12."""
    path = os.path.join(GOLD, "full_c2_metrics.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    g = json.load(open(path))
    from paper_2411_15997_b200 import build, fairserve as F
    build.build()
    ctx = F.Context(0)
    tr = G.generate("c2")
    assert tr["n_calls"] == g["n_calls"]
    T = F.Trace(tr)
    prof = F.build_app_profiles(ctx, T, g["profile_cfg"])
    o, _ = F.wsc_replay(ctx, T, prof, g["engine"])
    for thr, want in g["metrics"].items():
        got, per = F.replay_metrics(ctx, T, o, int(thr))
        for a, b in [(got, want["global"])] + list(zip(per, want["per_app"])):
            for k, v in b.items():
                if k == "jain":
                    assert a[k] == pytest.approx(v, rel=1e-12), (thr, k)
                else:
                    assert a[k] == v, (thr, k, a[k], v)
