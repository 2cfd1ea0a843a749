"""GPU edge cases vs the oracle: empty and single-call traces, everything filtered,
and every error code (same code, same first offending index)."""
import numpy as np
import pytest

import oracle as O
from paper_2411_15997_b200 import tracegen as G

pytestmark = pytest.mark.gpu
MS = 10**6


@pytest.fixture(scope="module")
def F():
    import torch
    assert torch.cuda.is_available()
    from paper_2411_15997_b200 import build, fairserve
    build.build()
    return fairserve


@pytest.fixture(scope="module")
def ctx(F):
    return F.Context(0)


def _row(**k):
    r = dict(user=0, t_ms=0, app=0, inter=0, stage=1, ncalls=1, len_in=10, len_out=3)
    r.update(k)
    return r


ENG = dict(mode=1, kv_capacity=10**6, max_batch=4, overload_permille=0, iter_base_ns=MS, decode_ns_per_req=0,
           prefill_ns_per_tok=0, act=dict(window_ms=10, limits_from_profile=0, T_req_g=1, T_req_a=[1, 1]))


def _both(F, ctx, tr, op_host, cfg):
    """Run the replay on both sides; returns (oracle result or error, gpu result or error)."""
    A, J = op_host[0], op_host[1]
    op = O.profile_from_host(*op_host)
    gp = F.profile_from_host(ctx, *op_host)
    try:
        e = O.replay(tr, op, cfg)
    except O.OracleError as x:
        e = ("err", x.code, x.bad_index)
    try:
        g = F.wsc_replay(ctx, F.Trace(tr), gp, cfg)
    except F.FsError as x:
        g = ("err", x.code, x.bad_index)
    return e, g


PROF1 = (2, 1, [[0, 1], [0, 1]], [[0, 10], [0, 10]], [[0, 0], [0, 0]], [[0, 3], [0, 3]])


def test_empty_trace(F, ctx):
    tr = G.from_columns(3, 2, [])
    tr["n_inters"] = 0
    e, g = _both(F, ctx, tr, PROF1, ENG)
    assert g[1]["n_arrived"] == 0 and g[1]["digest"] == e[1]["digest"]
    p = F.build_app_profiles(ctx, F.Trace(tr), {}).read()
    assert p["cnt"].sum() == 0 and int(p["T_req_g"][0]) == 0
    st, s = F.act_throttle(ctx, F.Trace(tr), None, dict(limits_from_profile=0))
    assert s["n_in"] == 0


def test_single_call(F, ctx):
    tr = G.from_columns(1, 2, [_row()])
    e, g = _both(F, ctx, tr, PROF1, ENG)
    assert g[1] == e[1]
    assert int(g[0]["finish_ns"][0]) == int(e[0]["finish_ns"][0]) == 3 * MS


def test_all_filtered(F, ctx):
    rows = [_row(user=0, tier=3, inter=0), _row(user=1, tier=2, t_ms=1, inter=1)]
    tr = G.from_columns(2, 2, rows)
    cfg = dict(ENG, tier_max=1)
    e, g = _both(F, ctx, tr, PROF1, cfg)
    assert g[1] == e[1] and g[1]["n_filtered"] == 2 and g[1]["n_arrived"] == 0
    assert list(g[0]["status"].cpu().numpy()) == [6, 6]


@pytest.mark.parametrize("case", ["range_user", "range_lenout", "order_time", "order_chain", "order_dup",
                                  "profile", "oversize", "overflow"])
def test_error_codes(F, ctx, case):
    rows = [_row(inter=0, ncalls=2), _row(inter=0, stage=2, ncalls=2, t_ms=1), _row(user=1, inter=1, t_ms=2)]
    prof = PROF1
    cfg = dict(ENG)
    if case == "range_user":
        rows[2]["user"] = 7
    elif case == "range_lenout":
        rows[1]["len_out"] = 0
    elif case == "order_time":
        rows[2]["t_ms"] = 0
    elif case == "order_chain":
        rows[1]["stage"] = 3
        rows[1]["ncalls"] = 3
    elif case == "order_dup":
        rows.append(_row(inter=0, stage=2, ncalls=2, t_ms=3))
    elif case == "profile":
        prof = (2, 1, [[0, 1], [0, 0]], [[0, 10], [0, 0]], [[0, 0], [0, 0]], [[0, 3], [0, 0]])
        rows[2]["app"] = 1
    elif case == "oversize":
        cfg["kv_capacity"] = 12
    elif case == "overflow":
        prof = (2, 1, [[0, 65536], [0, 65536]], [[0, 1], [0, 1]], [[0, 0], [0, 0]], [[0, 0], [0, 0]])
        cfg.update(prio_benign_q16=(1 << 24) - 1, alpha=255, beta=255, gamma=255)
        for r in rows:
            r["len_in"] = (1 << 24) - 1
        cfg["kv_capacity"] = 1 << 26
    tr = G.from_columns(2, 2, rows)
    e, g = _both(F, ctx, tr, prof, cfg)
    assert e[0] == "err" and g[0] == "err", (e, g)
    assert g[1:] == e[1:], (case, e, g)


# ------------------------------------------------------------------ edge cases of the NEXT rows
@pytest.mark.parametrize("mode", [2, 3, 4])
def test_baseline_modes_empty_and_single(F, ctx, mode):
    cfg = dict(ENG, mode=mode)
    tr = G.from_columns(3, 2, [])
    tr["n_inters"] = 0
    e, g = _both(F, ctx, tr, PROF1, cfg)
    assert g[1] == e[1] and g[1]["n_arrived"] == 0
    tr = G.from_columns(1, 2, [_row()])
    e, g = _both(F, ctx, tr, PROF1, cfg)
    assert g[1] == e[1] and g[1]["n_admitted"] == 1


def test_rpm_blocks_the_second_call_of_a_user(F, ctx):
    """RPM with T_req_g = 1: a user's second call inside the window is blocked whatever its
    stage (here a continuation: the interaction is aborted midway)."""
    rows = [_row(inter=0, ncalls=3), _row(inter=0, stage=2, ncalls=3, t_ms=1), _row(inter=0, stage=3, ncalls=3, t_ms=2)]
    tr = G.from_columns(1, 2, rows)
    cfg = dict(ENG, mode=3, act=dict(window_ms=60000, limits_from_profile=0, T_req_g=1, T_req_a=[0, 0]))
    prof = (2, 3, [[0, 1, 1, 1], [0, 1, 1, 1]], [[0, 10, 10, 10]] * 2, [[0, 0, 0, 0]] * 2, [[0, 3, 3, 3]] * 2)
    e, g = _both(F, ctx, tr, prof, cfg)
    assert g[1] == e[1]
    assert list(g[0]["status"].cpu().numpy()) == list(e[0]["status"]) == [0, 1, 5]


def test_metrics_empty_and_single(F, ctx):
    from oracle import metrics as M
    tr = G.from_columns(3, 2, [])
    tr["n_inters"] = 0
    T = F.Trace(tr)
    out = F.replay_outputs(ctx, T)
    g, per = F.replay_metrics(ctx, T, out, 0)
    assert g["requests_total"] == 0 and g["ttft_n"] == 0 and g["jain"] == 0.0 and len(per) == 2
    tr = G.from_columns(1, 2, [_row()])
    e, _ = O.replay(tr, O.profile_from_host(*PROF1), ENG)
    go, _ = F.wsc_replay(ctx, F.Trace(tr), F.profile_from_host(ctx, *PROF1), ENG)
    g, _ = F.replay_metrics(ctx, F.Trace(tr), go, 0)
    eg, _ = M.replay_metrics(tr, e, 0)
    assert g == eg and g["users_served"] == 1 and g["jain"] == 1.0


def test_generate_tiny(F, ctx):
    T = F.generate_trace(ctx, "c1", n_calls=1, seed=3)
    assert T.n == 1 and T.X == 1
    assert int((T.t["meta"][0].item() >> 8) & 255) == 1          # the one call is a head


def test_sweep_empty_grid_and_bad_config(F, ctx):
    tr = G.from_columns(1, 2, [_row()])
    gp = F.profile_from_host(ctx, *PROF1)
    sums, codes = F.sweep(ctx, F.Trace(tr), gp, [])
    assert sums == [] and len(codes) == 0
    with pytest.raises(F.FsError) as e:                        # RPM takes explicit limits only (R8)
        F.sweep(ctx, F.Trace(tr), gp, [dict(ENG, mode=3, act=dict(window_ms=10, limits_from_profile=1))])
    assert e.value.code == -1


def _step_pair(F, ctx, tr, cfg):
    op = O.profile(tr, dict(tier_max=255))
    gp = F.build_app_profiles(ctx, F.Trace(tr), dict(tier_max=255))
    T = F.Trace(tr)
    return O.Step(tr, op, cfg), F.WscState(ctx, T, gp, cfg), T


def _step_err(fn):
    try:
        fn()
    except (O.OracleError, F_ERR) as x:
        return x.code, x.bad_index
    return None


F_ERR = RuntimeError


@pytest.mark.parametrize("case", ["finished_range", "arrived_range", "finished_filtered"])
def test_step_bad_ids_match_oracle(F, ctx, case):
    """fs_wsc_step with a call id >= n_calls (finished or arrived) returns FS_E_RANGE with the
    list position, and a finished call of a filtered user (tier > tier_max) FS_E_INVAL, as the
    oracle's or_step; the state is then poisoned (FS_E_PROTOCOL) instead of running on
    half-updated heaps."""
    tr = G.generate("c1")
    n = tr["n_calls"]
    eng = dict(G.CONFIGS["c1"]["engine"], mode=1, tier_max=0,
               act=dict(window_ms=60000, limits_from_profile=0, T_req_g=8, T_req_a=[5, 5]))
    so, sg, T = _step_pair(F, ctx, tr, eng)
    ab = int(np.nonzero((tr["meta"] >> 24) > 0)[0][0])         # a call of the abusive user
    args = {"finished_range": dict(finished=[0, n + 7]),
            "arrived_range": dict(arrived=[0, n], arrived_ns=[0, 0]),
            "finished_filtered": dict(finished=[ab])}[case]
    a = dict(finished=[], arrived=[], arrived_ns=[])
    a.update(args)
    eo = _step_err(lambda: so.step(0, 0, 0, **a))
    try:
        sg.step(0, 0, 0, **a)
        eg = None
    except F.FsError as x:
        eg = (x.code, x.bad_index)
    assert eo is not None and eg == eo, (eo, eg)
    with pytest.raises(F.FsError) as ex:
        sg.step(0, 0, 0, [], [0], [0])
    assert ex.value.code == -9                                   # FS_E_PROTOCOL


def test_replay_with_torch_allocator(F):
    """fs_ctx_set_allocator: with torch's caching allocator installed, every scratch / object
    allocation of a profile + FS(W+I) replay + ACT + sweep comes from torch's pool (its
    allocated-bytes counter moves) and the results equal the oracle's."""
    import torch
    c = F.Context(0)
    c.use_torch_allocator(True)
    tr = G.generate("c1")
    T = F.Trace(tr)
    before = torch.cuda.memory_stats()["allocation.all.allocated"]
    gp = F.build_app_profiles(c, T, dict(tier_max=255))
    eng = dict(G.CONFIGS["c1"]["engine"], mode=1, tier_max=255,
               act=dict(window_ms=60000, limits_from_profile=0, T_req_g=8, T_req_a=[5, 5]))
    o, s = F.wsc_replay(c, T, gp, eng)
    st, _ = F.act_throttle(c, T, gp, eng["act"], overloaded=o["ovl"], t_ns_override=o["arrive_ns"])
    gs, gc = F.sweep(c, T, gp, [eng, dict(eng, tier_max=0)])
    torch.cuda.synchronize()
    after = torch.cuda.memory_stats()["allocation.all.allocated"]
    assert after - before > 20                                   # the library's allocations went through torch
    op = O.profile(tr, dict(tier_max=255))
    eo, es = O.replay(tr, op, eng)
    assert s["digest"] == es["digest"]
    assert (st.cpu().numpy() == eo["status"]).all()
    e2, ec = O.sweep(tr, op, [eng, dict(eng, tier_max=0)])
    assert [x["digest"] for x in gs] == [x["digest"] for x in e2] and list(gc) == list(ec)
    del gp
    c.use_torch_allocator(False)
    _, s2 = F.wsc_replay(c, T, F.build_app_profiles(c, T, dict(tier_max=255)), eng, outputs=False)
    assert s2["digest"] == es["digest"]
