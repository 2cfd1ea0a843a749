"""Oracle pins for the NEXT-1 baseline policies (SPEC module
sched-baselines; PAPER.md P:59-66 (RPM, VTC), P:327-335 (RPM throttling)):
the SPEC's worked examples and stated invariants, and relations to the FairServe
modes that hold exactly (readings R7-R8)."""
import numpy as np

import oracle as O
from paper_2411_15997_b200.tracegen import from_columns
from tiny import tiny_profile, tiny_trace

UMAX = 0xFFFFFFFF
VTC, RPM, FCFS = 2, 3, 4


def eng(mode, **kw):
    c = dict(mode=mode, alpha=1, beta=1, gamma=2, kv_capacity=1000, max_batch=4, overload_permille=900,
             iter_base_ns=1_000_000, decode_ns_per_req=0, prefill_ns_per_tok=0,
             act=dict(window_ms=60000, limits_from_profile=0))
    c.update(kw)
    return c


def flat_profile(A, J=3, w=1):
    """Every (app, stage) has mean weighted tokens w (cnt 1, sum_in w): W_aj = w * 2^16 for (1, *, *)."""
    return O.profile_from_host(A, J, [[0] + [1] * J] * A, [[0] + [w] * J] * A, [[0] * (J + 1)] * A,
                               [[0] + [1] * J] * A)


def test_vtc_counter_example():
    """a finished request L_I = 100, L_O = 10 with weights (1, 2) adds 120 to the counter."""
    tr = from_columns(1, 1, [dict(user=0, t_ms=0, app=0, inter=0, stage=1, ncalls=1, len_in=100, len_out=10)])
    o, s = O.replay(tr, flat_profile(1), eng(VTC))
    assert int(o["counters"][0]) == 120 << 32


def test_vtc_ignores_app_normalisation():
    """S:342 / P:243: a heavy-app user and a light-app user with equal token consumption get equal
    VTC counters -- the inequity FairServe's app normalisation (Eq. 2-3) corrects."""
    rows = [dict(user=0, t_ms=0, app=0, inter=0, stage=1, ncalls=1, len_in=90, len_out=5),
            dict(user=1, t_ms=0, app=1, inter=1, stage=1, ncalls=1, len_in=90, len_out=5)]
    tr = from_columns(2, 2, rows)
    prof = O.profile_from_host(2, 1, [[0, 1], [0, 1]], [[0, 1000], [0, 10]], [[0, 0], [0, 0]], [[0, 1], [0, 1]])
    o, _ = O.replay(tr, prof, eng(VTC))
    assert int(o["counters"][0]) == int(o["counters"][1]) == 100 << 32
    o, _ = O.replay(tr, prof, eng(0))            # FS(W): the light app's user is charged more
    assert int(o["counters"][1]) > int(o["counters"][0])


def test_fcfs_examples():
    """t=1 before t=2; equal timestamps -> lower request id first."""
    rows = [dict(user=2, t_ms=1, app=0, inter=0, stage=1, ncalls=1, len_in=5, len_out=3),
            dict(user=1, t_ms=2, app=0, inter=1, stage=1, ncalls=1, len_in=5, len_out=3),
            dict(user=0, t_ms=2, app=0, inter=2, stage=1, ncalls=1, len_in=5, len_out=3)]
    tr = from_columns(3, 1, rows)
    o, _ = O.replay(tr, flat_profile(1), eng(FCFS, max_batch=1))
    assert list(o["order"]) == [0, 1, 2]


def _admission_sorted_by_arrival(o):
    adm = [i for i in range(len(o["order"])) if o["order"][i] != UMAX]
    by_order = sorted(adm, key=lambda i: o["order"][i])
    by_arrival = sorted(adm, key=lambda i: (o["arrive_ns"][i], i))
    return by_order == by_arrival


def test_fcfs_and_rpm_serve_in_arrival_order():
    """FCFS picks the globally earliest queued call, so admissions follow (arrival, id)
    exactly, whatever the KV budget and batch limit; RPM schedules FCFS among admitted calls."""
    for seed in range(150):
        rng = np.random.default_rng(700 + seed)
        A = int(rng.integers(1, 3))
        tr = tiny_trace(rng, n_users=3, n_apps=A)
        J, cnt, si, ss, so = tiny_profile(rng, A)
        prof = O.profile_from_host(A, J, cnt, si, ss, so)
        for mode in (FCFS, RPM):
            cfg = eng(mode, kv_capacity=int(rng.choice((30, 100))), max_batch=int(rng.choice((1, 2))))
            cfg["act"].update(T_req_g=int(rng.choice((0, 2))), T_req_a=[int(rng.choice((0, 3))) for _ in range(A)])
            try:
                o, _ = O.replay(tr, prof, cfg)
            except O.OracleError as e:
                assert e.code == -4          # oversize
                continue
            assert _admission_sorted_by_arrival(o), (seed, mode)


def _rpm_trace():
    """user 0: one 5-call interaction (stages 1 ms apart); user 1: a single call of app 1."""
    rows = [dict(user=0, t_ms=s - 1, app=0, inter=0, stage=s, ncalls=5, len_in=2, len_out=1, think_ms=0)
            for s in range(1, 6)]
    rows.insert(1, dict(user=1, t_ms=0, app=1, inter=1, stage=1, ncalls=1, len_in=2, len_out=1))
    return from_columns(2, 2, rows)


def test_rpm_blocks_mid_interaction():
    """stage 3 of 5 over the user limit -> blocked, the interaction is aborted midway: stages
    1-2 were served (their tokens wasted), stages 4-5 never arrive (DROPPED)."""
    tr = _rpm_trace()
    cfg = eng(RPM, iter_base_ns=100_000)
    cfg["act"].update(T_req_g=2, T_req_a=[0, 0])
    o, s = O.replay(tr, flat_profile(2, J=5), cfg)
    st = list(o["status"])
    ids = [i for i in range(tr["n_calls"]) if tr["user"][i] == 0]          # stages 1..5 of user 0
    assert [st[i] for i in ids] == [0, 0, 1, 5, 5]                        # ADMIT ADMIT USER_REQ DROPPED DROPPED
    assert o["finish_ns"][ids[0]] >= 0 and o["finish_ns"][ids[1]] >= 0
    assert s["n_block"] == [1, 0, 0, 0] and s["n_dropped"] == 2


def test_rpm_app_limit_and_under_limits():
    """app over its limit (counted over all users) with the user under -> blocked
    (APP_REQ); under both limits -> enqueued."""
    tr = _rpm_trace()
    prof = flat_profile(2, J=5)
    cfg = eng(RPM, iter_base_ns=100_000)
    cfg["act"].update(T_req_g=0, T_req_a=[3, 0])
    o, s = O.replay(tr, prof, cfg)
    ids = [i for i in range(tr["n_calls"]) if tr["user"][i] == 0]
    assert [int(o["status"][i]) for i in ids] == [0, 0, 0, 3, 5]
    cfg["act"].update(T_req_g=5, T_req_a=[5, 5])
    o, s = O.replay(tr, prof, cfg)
    assert all(int(x) == 0 for x in o["status"]) and sum(s["n_block"]) == 0


def test_rpm_is_overload_oblivious_and_vtc_never_blocks():
    """RPM decisions depend only on arrival history and limits (same under any theta);
    VTC never blocks."""
    for seed in range(80):
        rng = np.random.default_rng(1300 + seed)
        A = int(rng.integers(1, 3))
        tr = tiny_trace(rng, n_users=3, n_apps=A)
        J, cnt, si, ss, so = tiny_profile(rng, A)
        prof = O.profile_from_host(A, J, cnt, si, ss, so)
        lim = dict(T_req_g=int(rng.choice((1, 2))), T_req_a=[int(rng.choice((0, 1, 2))) for _ in range(A)])
        res = []
        for th in (0, 500, UMAX):
            cfg = eng(RPM, overload_permille=th, kv_capacity=100)
            cfg["act"].update(lim)
            try:
                o, s = O.replay(tr, prof, cfg)
            except O.OracleError:
                break
            res.append(list(o["status"]))
        assert all(r == res[0] for r in res)
        cfg = eng(VTC, overload_permille=0, kv_capacity=100)
        cfg["act"].update(lim)
        try:
            _, s = O.replay(tr, prof, cfg)
        except O.OracleError:
            continue
        assert sum(s["n_block"]) == 0 and s["n_dropped"] == 0


def test_rpm_without_limits_is_fcfs():
    for seed in range(60):
        rng = np.random.default_rng(1700 + seed)
        A = int(rng.integers(1, 3))
        tr = tiny_trace(rng, n_users=3, n_apps=A)
        J, cnt, si, ss, so = tiny_profile(rng, A)
        prof = O.profile_from_host(A, J, cnt, si, ss, so)
        try:
            _, a = O.replay(tr, prof, eng(FCFS, kv_capacity=100))
        except O.OracleError:
            continue
        cfg = eng(RPM, kv_capacity=100)
        cfg["act"].update(T_req_g=0, T_req_a=[0] * A)
        _, b = O.replay(tr, prof, cfg)
        assert a == b


def test_fs_w_equals_vtc_on_uniform_single_call_traces():
    """with every app's stage expectation equal (here W_aj = 2^16: one weighted token per
    call), single-call interactions and VTC weights equal to FS's, FS(W) and VTC make the same
    selections and reach the same counters."""
    for seed in range(80):
        rng = np.random.default_rng(2100 + seed)
        A = int(rng.integers(1, 3))
        tr = tiny_trace(rng, n_users=3, n_apps=A, m_choices=(1,), abusive_user=False)
        prof = flat_profile(A, J=1)
        w = dict(alpha=1, beta=0, gamma=0)
        a_out, a = O.replay(tr, prof, eng(0, **w, kv_capacity=30))
        b_out, b = O.replay(tr, prof, eng(VTC, **w, kv_capacity=30))
        assert list(a_out["order"]) == list(b_out["order"])
        assert list(a_out["counters"]) == list(b_out["counters"])
