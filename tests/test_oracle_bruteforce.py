"""Oracle pinned by brute force: the C++ oracle vs the
literal Python stepper (oracle/stepper.py: lists, full rescans, per-iteration
`done += 1` stepping) on seeded tiny traces, the O(n^2) ACT recount, and the
online step vs a literal step model."""
import numpy as np
import pytest

import oracle as O
from oracle import stepper as S
from tiny import tiny_profile, tiny_replay_cfg, tiny_trace

N_CASES = 400


def _oversize(tr, prof, cfg):
    calls = S._calls(tr)
    for c in calls:
        if c["tier"] > cfg.get("tier_max", 255):
            continue
        j = S._slot(prof, c["app"], c["stage"])
        R = int(prof["sum_out"][c["app"]][j]) // int(prof["cnt"][c["app"]][j])
        if c["L_I"] + c["L_S"] + R > cfg["kv_capacity"]:
            return True
    return False


@pytest.mark.parametrize("seed", range(N_CASES))
def test_replay_vs_stepper(seed):
    rng = np.random.default_rng(1000 + seed)
    A = int(rng.integers(1, 3))
    tr = tiny_trace(rng, n_users=int(rng.integers(1, 4)), n_apps=A)
    J, cnt, si, ss, so = tiny_profile(rng, A)
    prof = O.profile_from_host(A, J, cnt, si, ss, so)
    cfg = tiny_replay_cfg(rng, A)
    if _oversize(tr, prof, cfg):
        with pytest.raises(O.OracleError) as ei:
            O.replay(tr, prof, cfg)
        assert ei.value.code == -4
        return
    o, s = O.replay(tr, prof, cfg)
    eo, es = S.replay(tr, prof, cfg)
    for k in ("status", "ovl", "arrive_ns", "admit_ns", "first_ns", "finish_ns", "order", "counters"):
        assert list(o[k]) == list(eo[k]), (k, seed)
    for k in ("n_arrived", "n_block", "n_dropped", "n_admitted", "n_finished", "n_iterations",
              "n_ovl_arrivals", "makespan_ns", "digest"):
        assert s[k] == es[k], (k, seed)


@pytest.mark.parametrize("seed", range(300))
def test_replay_vs_stepper_baselines(seed):
    """NEXT-1 baseline policies (VTC, RPM, FCFS) against the literal stepper."""
    rng = np.random.default_rng(9000 + seed)
    A = int(rng.integers(1, 3))
    tr = tiny_trace(rng, n_users=int(rng.integers(1, 4)), n_apps=A)
    J, cnt, si, ss, so = tiny_profile(rng, A)
    prof = O.profile_from_host(A, J, cnt, si, ss, so)
    cfg = tiny_replay_cfg(rng, A, modes=(2, 3, 4))
    if _oversize(tr, prof, cfg):
        return
    o, s = O.replay(tr, prof, cfg)
    eo, es = S.replay(tr, prof, cfg)
    for k in ("status", "ovl", "arrive_ns", "admit_ns", "first_ns", "finish_ns", "order", "counters"):
        assert list(o[k]) == list(eo[k]), (k, seed)
    for k in ("n_arrived", "n_block", "n_dropped", "n_admitted", "n_finished", "n_iterations",
              "n_ovl_arrivals", "makespan_ns", "digest"):
        assert s[k] == es[k], (k, seed)


def test_replay_exhaustive_pairs():
    """Exhaustive grid: two single-call users x arrival times x lengths x Bmax."""
    n = 0
    for t1 in (0, 1, 2, 5):
        for L in ((1, 1), (1, 5), (5, 2), (2, 5)):
            for Lo in ((1, 2), (5, 1), (2, 2)):
                for Bmax in (1, 2):
                    for C in (8, 12):
                        rows = [dict(user=0, t_ms=0, app=0, inter=0, stage=1, ncalls=1, len_in=L[0], len_out=Lo[0]),
                                dict(user=1, t_ms=t1, app=1, inter=1, stage=1, ncalls=1, len_in=L[1], len_out=Lo[1]),
                                dict(user=0, t_ms=t1, app=0, inter=2, stage=1, ncalls=2, len_in=1, len_out=1, think_ms=1),
                                dict(user=0, t_ms=t1 + 1, app=0, inter=2, stage=2, ncalls=2, len_in=2, len_out=1)]
                        from paper_2411_15997_b200.tracegen import from_columns
                        tr = from_columns(2, 2, rows)
                        prof = O.profile_from_host(2, 2, [[0, 2, 1], [0, 1, 0]], [[0, 4, 2], [0, 3, 0]],
                                                   [[0, 0, 0], [0, 0, 0]], [[0, 3, 1], [0, 2, 0]])
                        for mode in (0, 1, 2, 3, 4):
                            cfg = dict(mode=mode, kv_capacity=C, max_batch=Bmax, overload_permille=500,
                                       iter_base_ns=1_000_000, decode_ns_per_req=0, prefill_ns_per_tok=0,
                                       act=dict(window_ms=3, limits_from_profile=0, T_req_g=1, T_req_a=[1, 1]))
                            o, s = O.replay(tr, prof, cfg)
                            eo, es = S.replay(tr, prof, cfg)
                            for k in ("status", "admit_ns", "finish_ns", "counters"):
                                assert list(o[k]) == list(eo[k])
                            assert s["digest"] == es["digest"]
                            n += 1
    assert n == 4 * 4 * 3 * 2 * 2 * 5


@pytest.mark.parametrize("seed", range(200))
def test_act_vs_recount(seed):
    rng = np.random.default_rng(5000 + seed)
    A = int(rng.integers(1, 3))
    tr = tiny_trace(rng, n_users=2, n_apps=A, max_inters=5, max_calls=9)
    J, cnt, si, ss, so = tiny_profile(rng, A)
    prof = O.profile_from_host(A, J, cnt, si, ss, so)
    n = tr["n_calls"]
    cfg = dict(window_ms=int(rng.choice((1, 2, 4))), limits_from_profile=0, T_req_g=int(rng.choice((0, 1, 2))),
               T_req_a=[int(rng.choice((0, 1, 2))) for _ in range(A)], T_tok_g=int(rng.choice((0, 8))),
               T_tok_a=[int(rng.choice((0, 6))) for _ in range(A)], count_mode=int(rng.integers(0, 2)),
               tier_max=int(rng.choice((0, 255))))
    ovl = (rng.random(n) < 0.7).astype(np.uint8) if rng.random() < 0.8 else None
    tov = None
    if rng.random() < 0.5:         # replay-like overrides: continuations later than their heads
        _, head_of, _ = O.validate(tr)[1:] if False else (None, *O.validate(tr)[2:])
        tov = tr["t_ms"].astype(np.int64) * 1_000_000
        tov = tov + rng.integers(0, 3, size=n) * 1_000_000
        for i in range(n):
            if int(head_of[i]) != i:
                tov[i] = max(tov[i], tov[int(head_of[i])] + 1)
        tov[rng.random(n) < 0.1] = -1
    st, _ = O.act(tr, prof, cfg, overloaded=ovl, t_ns_override=tov)

    def ohat(c):
        j = S._slot(prof, c["app"], c["stage"])
        return int(prof["sum_out"][c["app"]][j]) // int(prof["cnt"][c["app"]][j])

    ref = S.act(tr, ohat, cfg, overloaded=ovl, t_ns_override=tov,
                limits=(cfg["T_req_g"], cfg["T_tok_g"], cfg["T_req_a"], cfg["T_tok_a"]))
    assert list(st) == ref


@pytest.mark.parametrize("seed", range(200))
def test_act_vs_recount_app_global(seed):
    """NEXT-3 app-global counters (FS_SCOPE_APP_GLOBAL, R10) vs the O(n^2) recount."""
    rng = np.random.default_rng(15000 + seed)
    A = int(rng.integers(1, 3))
    tr = tiny_trace(rng, n_users=3, n_apps=A, max_inters=5, max_calls=9)
    J, cnt, si, ss, so = tiny_profile(rng, A)
    prof = O.profile_from_host(A, J, cnt, si, ss, so)
    n = tr["n_calls"]
    cfg = dict(window_ms=int(rng.choice((1, 2, 4))), limits_from_profile=0, T_req_g=int(rng.choice((0, 2, 3))),
               T_req_a=[int(rng.choice((0, 1, 2, 3))) for _ in range(A)], T_tok_g=int(rng.choice((0, 12))),
               T_tok_a=[int(rng.choice((0, 9))) for _ in range(A)], count_mode=int(rng.integers(0, 2)),
               tier_max=int(rng.choice((0, 255))), app_scope=1)
    ovl = (rng.random(n) < 0.7).astype(np.uint8) if rng.random() < 0.8 else None
    st, _ = O.act(tr, prof, cfg, overloaded=ovl)

    def ohat(c):
        j = S._slot(prof, c["app"], c["stage"])
        return int(prof["sum_out"][c["app"]][j]) // int(prof["cnt"][c["app"]][j])

    ref = S.act(tr, ohat, cfg, overloaded=ovl,
                limits=(cfg["T_req_g"], cfg["T_tok_g"], cfg["T_req_a"], cfg["T_tok_a"]))
    assert list(st) == ref


@pytest.mark.parametrize("seed", range(200))
def test_replay_vs_stepper_app_global(seed):
    rng = np.random.default_rng(16000 + seed)
    A = int(rng.integers(1, 3))
    tr = tiny_trace(rng, n_users=int(rng.integers(2, 4)), n_apps=A)
    J, cnt, si, ss, so = tiny_profile(rng, A)
    prof = O.profile_from_host(A, J, cnt, si, ss, so)
    cfg = tiny_replay_cfg(rng, A, modes=(1,))
    cfg["act"]["app_scope"] = 1
    if _oversize(tr, prof, cfg):
        return
    o, s = O.replay(tr, prof, cfg)
    eo, es = S.replay(tr, prof, cfg)
    for k in ("status", "ovl", "arrive_ns", "admit_ns", "first_ns", "finish_ns", "order", "counters"):
        assert list(o[k]) == list(eo[k]), (k, seed)
    assert s["digest"] == es["digest"] and s["n_block"] == es["n_block"]


@pytest.mark.parametrize("seed", range(150))
def test_act_vs_recount_tau_weighted(seed):
    """NEXT-3 weighted token load (R11): tau = w_in L_I + w_sys L_S + w_out O-hat, vs the recount."""
    rng = np.random.default_rng(17000 + seed)
    A = int(rng.integers(1, 3))
    tr = tiny_trace(rng, n_users=2, n_apps=A, max_inters=5, max_calls=9)
    J, cnt, si, ss, so = tiny_profile(rng, A)
    prof = O.profile_from_host(A, J, cnt, si, ss, so)
    n = tr["n_calls"]
    tw = tuple(int(x) for x in rng.integers(0, 4, size=3))
    cfg = dict(window_ms=int(rng.choice((1, 2, 4))), limits_from_profile=0, T_req_g=int(rng.choice((0, 2))),
               T_req_a=[int(rng.choice((0, 2))) for _ in range(A)], T_tok_g=int(rng.choice((0, 8, 20))),
               T_tok_a=[int(rng.choice((0, 6, 15))) for _ in range(A)], count_mode=int(rng.integers(0, 2)),
               tier_max=255, app_scope=int(rng.integers(0, 2)), tau_weights=tw)
    ovl = (rng.random(n) < 0.7).astype(np.uint8)
    st, _ = O.act(tr, prof, cfg, overloaded=ovl)

    def ohat(c):
        j = S._slot(prof, c["app"], c["stage"])
        return int(prof["sum_out"][c["app"]][j]) // int(prof["cnt"][c["app"]][j])

    ref = S.act(tr, ohat, cfg, overloaded=ovl,
                limits=(cfg["T_req_g"], cfg["T_tok_g"], cfg["T_req_a"], cfg["T_tok_a"]))
    assert list(st) == ref


@pytest.mark.parametrize("seed", range(150))
def test_replay_vs_stepper_tau_weighted(seed):
    rng = np.random.default_rng(18000 + seed)
    A = int(rng.integers(1, 3))
    tr = tiny_trace(rng, n_users=int(rng.integers(1, 4)), n_apps=A)
    J, cnt, si, ss, so = tiny_profile(rng, A)
    prof = O.profile_from_host(A, J, cnt, si, ss, so)
    cfg = tiny_replay_cfg(rng, A, modes=(1,))
    cfg["act"]["tau_weights"] = tuple(int(x) for x in rng.integers(0, 4, size=3))
    cfg["act"]["app_scope"] = int(rng.integers(0, 2))
    if _oversize(tr, prof, cfg):
        return
    o, s = O.replay(tr, prof, cfg)
    eo, es = S.replay(tr, prof, cfg)
    for k in ("status", "admit_ns", "order", "counters"):
        assert list(o[k]) == list(eo[k]), (k, seed)
    assert s["digest"] == es["digest"]


def test_tau_weighted_example():
    """R11 by hand: one call L_I = 10, L_S = 5, profiled output mean O-hat = 20; weights (2, 0, 1)
    give tau = 40: T_tok_g = 39 blocks it (USER_TOK), 40 admits it; the profile's token peak of
    the user is 40 too."""
    from paper_2411_15997_b200.tracegen import from_columns
    tr = from_columns(1, 1, [dict(user=0, t_ms=0, app=0, inter=0, stage=1, ncalls=1, len_in=10, len_sys=5,
                                  len_out=20)])
    prof = O.profile_from_host(1, 1, [[0, 1]], [[0, 10]], [[0, 5]], [[0, 20]])
    base = dict(window_ms=60000, limits_from_profile=0, tau_weights=(2, 0, 1))
    assert list(O.act(tr, prof, dict(base, T_tok_g=39))[0]) == [2]
    assert list(O.act(tr, prof, dict(base, T_tok_g=40))[0]) == [0]
    p = O.profile(tr, dict(tier_max=255, tau_weights=(2, 0, 1)))
    assert int(p["peak_t_u"][0]) == 40
    assert int(O.profile(tr, dict(tier_max=255))["peak_t_u"][0]) == 35
    with pytest.raises(O.OracleError):
        O.act(tr, prof, dict(base, tau_weights=(16, 0, 1)))


def test_app_global_example():
    """S:217 (c^r_a over the app's arrivals): user 0's head and then user 1's head of the same app
    inside one window, T^r_a = 1, always overloaded -> user 1 is blocked (APP_REQ) with app-global
    counters and admitted with per-(user, app) counters (Q2)."""
    from paper_2411_15997_b200.tracegen import from_columns
    rows = [dict(user=0, t_ms=0, app=0, inter=0, stage=1, ncalls=1, len_in=1, len_out=1),
            dict(user=1, t_ms=1, app=0, inter=1, stage=1, ncalls=1, len_in=1, len_out=1)]
    tr = from_columns(2, 1, rows)
    prof = O.profile_from_host(1, 1, [[0, 1]], [[0, 1]], [[0, 0]], [[0, 1]])
    cfg = dict(window_ms=60000, limits_from_profile=0, T_req_g=0, T_req_a=[1])
    st, _ = O.act(tr, prof, dict(cfg, app_scope=1))
    assert list(st) == [0, 3]
    st, _ = O.act(tr, prof, cfg)
    assert list(st) == [0, 0]
    with pytest.raises(O.OracleError) as e:                      # R10: explicit limits only
        O.act(tr, prof, dict(cfg, app_scope=1, limits_from_profile=1))
    assert e.value.code == -1


@pytest.mark.parametrize("seed", range(60))
def test_step_vs_literal(seed):
    """Random step sequences: oracle Step vs the literal Sched of the stepper."""
    rng = np.random.default_rng(9000 + seed)
    A = 2
    tr = tiny_trace(rng, n_users=3, n_apps=A, max_inters=6, max_calls=12, thinks=(0,))
    J, cnt, si, ss, so = tiny_profile(rng, A)
    prof = O.profile_from_host(A, J, cnt, si, ss, so)
    cfg = tiny_replay_cfg(rng, A)
    cfg["kv_capacity"] = 100
    cfg["tier_max"] = 255
    st = O.Step(tr, prof, cfg)
    lit = S.Sched(tr, prof, cfg)
    n = tr["n_calls"]
    order = list(range(n))
    pos = 0
    admitted = []
    for it in range(12):
        k = int(rng.integers(0, 4))
        arr = order[pos:pos + k]
        pos += len(arr)
        t = np.full(len(arr), it * 1_000_000, np.int64)
        fin = [admitted.pop(0) for _ in range(min(len(admitted), int(rng.integers(0, 3))))]
        occ = int(rng.integers(0, 100))
        nb = int(rng.integers(0, 3))
        s1, a1 = st.step(it * 1_000_000, occ, nb, fin, arr, t)
        for r in fin:
            lit.finish(r)
        s2 = [lit.deliver(r, it * 1_000_000, lit.overloaded(occ)) for r in arr]
        a2 = []
        o, b = occ, nb
        while True:
            r = lit.pick(o, b)
            if r is None:
                break
            a2.append(r)
            c = lit.calls[r]
            o += c["L_I"] + c["L_S"]
            b += 1
        assert list(s1) == s2
        assert list(a1) == a2
        admitted += a2
        u, e = st.read()
        assert list(u) == lit.u
        assert (e if e >= 0 else None) == lit.e
