"""Oracle invariants on seeded C1-shaped traces and
tiny traces: I1-I4, I11-I13; lift/monotonicity I5-I6 on the literal stepper
(which brute force ties to the oracle)."""
import numpy as np
import pytest

import oracle as O
from oracle import stepper as S
from paper_2411_15997_b200 import tracegen as G
from tiny import tiny_profile, tiny_trace

UMAX = 0xFFFFFFFF


def _c1(seed):
    tr = G.generate("c1", seed=seed)
    c = G.CONFIGS["c1"]
    prof = O.profile(tr, dict(tier_max=255))
    cfg = dict(c["engine"], mode=1, tier_max=255,
               act=dict(window_ms=60000, limits_from_profile=0, T_req_g=8, T_req_a=[5, 5]))
    return tr, prof, cfg


@pytest.mark.parametrize("seed", range(100, 200))
def test_replay_invariants(seed):
    tr, prof, cfg = _c1(seed)
    o, s = O.replay(tr, prof, cfg)
    st, adm = o["status"], o["admit_ns"]
    meta = tr["meta"].astype(np.int64)
    stage, nc = (meta >> 8) & 255, (meta >> 16) & 255
    # I1 nothing blocked/dropped/filtered is admitted
    assert (adm[st != 0] == -1).all() and (adm[st == 0] >= 0).all()
    # I2 blocks only at heads and only under overload
    blk = (st >= 1) & (st <= 4)
    assert (stage[blk] == 1).all() and (o["ovl"][blk] == 1).all()
    # I3 zero waste: every admitted head's interaction finishes completely
    for x in np.unique(tr["inter"][(stage == 1) & (st == 0)]):
        calls = np.nonzero(tr["inter"] == x)[0]
        assert (o["finish_ns"][calls] >= 0).all()
    # I13 accounting
    assert s["n_arrived"] == s["n_admitted"] + sum(s["n_block"])
    assert s["n_admitted"] == s["n_finished"]
    assert s["n_dropped"] == int(((st == 5)).sum())
    # clocks: admit <= first <= finish; first - admit >= one iteration
    a = st == 0
    assert (o["arrive_ns"][a] <= adm[a]).all() and (adm[a] < o["first_ns"][a]).all()
    assert (o["first_ns"][a] <= o["finish_ns"][a]).all()
    # I4 FS(W) never blocks; FS(W+I) never overloaded == FS(W)
    ow, sw = O.replay(tr, prof, dict(cfg, mode=0))
    assert (ow["status"] == 0).all()
    _, sn = O.replay(tr, prof, dict(cfg, overload_permille=UMAX))
    assert sn["digest"] == sw["digest"]


def test_c1_exercises_throttling():
    hits = 0
    for seed in range(100, 130):
        tr, prof, cfg = _c1(seed)
        _, s = O.replay(tr, prof, cfg)
        hits += sum(s["n_block"]) > 0
    assert hits > 0


@pytest.mark.parametrize("seed", range(40))
def test_spread_bound_bmax(seed):
    """I11: single-call trace, FS(W), equal E: while users i, j are both backlogged
    after each was picked once, u_i - u_j <= F_i * Dmax <= Bmax * Dmax."""
    rng = np.random.default_rng(seed)
    Bmax = int(rng.integers(1, 4))
    rows = []
    for k in range(30):
        rows.append(dict(user=k % 2, t_ms=0, app=k % 2, inter=len(rows), stage=1, ncalls=1,
                         len_in=int(rng.integers(1, 20)), len_out=int(rng.integers(1, 6))))
    tr = G.from_columns(2, 2, rows)
    prof = O.profile_from_host(2, 1, [[0, 1], [0, 1]], [[0, 7], [0, 3]], [[0, 0], [0, 0]], [[0, 3], [0, 2]])
    cfg = dict(mode=0, kv_capacity=10**6, max_batch=Bmax, iter_base_ns=1_000_000, decode_ns_per_req=0,
               prefill_ns_per_tok=0)
    Sd = S.Sched(tr, prof, cfg)
    dmax = max((Sd.prio(c) * (c["L_I"] + 2 * c["L_S"] + c["L_O"]) << 32) // Sd.weight(c) for c in Sd.calls)
    # drive the literal scheduler with the replay's own event order via the oracle replay times
    o, _ = O.replay(tr, prof, cfg)
    eo, _ = S.replay(tr, prof, cfg)
    assert list(o["admit_ns"]) == list(eo["admit_ns"])
    # reconstruct counters at each admission time from finish times
    inc = {c["id"]: (Sd.prio(c) * (c["L_I"] + 2 * c["L_S"] + c["L_O"]) << 32) // Sd.weight(c) for c in Sd.calls}
    user = tr["user"]
    picked = {0: False, 1: False}
    for r in np.argsort(o["order"]):
        T = o["admit_ns"][r]
        u = [sum(inc[x] for x in range(len(rows)) if user[x] == k and 0 <= o["finish_ns"][x] <= T) for k in (0, 1)]
        backlog = [any(user[x] == k and o["admit_ns"][x] > T for x in range(len(rows))) for k in (0, 1)]
        if all(picked.values()) and all(backlog):
            assert abs(u[0] - u[1]) <= Bmax * dmax
        picked[int(user[r])] = True


def test_unit_normalisation():
    """I12: calls equal to their (app, stage) means with E = 1 charge exactly 2^32 each."""
    rows = []
    x = 0
    for k in range(12):
        m = 1 + k % 3
        for s in range(1, m + 1):
            rows.append(dict(user=k % 4, t_ms=10 * k + s, app=k % 2, inter=x, stage=s, ncalls=m,
                             len_in=5 * s + (k % 2), len_sys=s, len_out=3 + s))
        x += 1
    tr = G.from_columns(4, 2, rows)
    prof = O.profile(tr, dict(max_stage=8))
    cfg = dict(mode=0, kv_capacity=10**6, max_batch=4, iter_base_ns=1_000_000, decode_ns_per_req=0,
               prefill_ns_per_tok=0)
    st = O.Step(tr, prof, cfg)
    for r in range(len(rows)):
        u0, _ = st.read()
        st.step(0, 0, 0, finished=[r])
        u1, _ = st.read()
        d = u1.astype(object) - u0.astype(object)
        assert d[rows[r]["user"]] == 1 << 32 and sum(d) == 1 << 32


@pytest.mark.parametrize("seed", range(60))
def test_lift_and_monotone_on_stepper(seed):
    """I5 counters nondecreasing; I6 after a lift with Q non-empty, u_u >= min_Q u."""
    rng = np.random.default_rng(300 + seed)
    tr = tiny_trace(rng, n_users=3, n_apps=2, max_inters=6, max_calls=10)
    J, cnt, si, ss, so = tiny_profile(rng, 2)
    prof = O.profile_from_host(2, J, cnt, si, ss, so)
    cfg = dict(mode=0, kv_capacity=100, max_batch=2, iter_base_ns=1_000_000, decode_ns_per_req=0,
               prefill_ns_per_tok=0, act={})
    Sd = S.Sched(tr, prof, cfg)
    orig_deliver, orig_finish = Sd.deliver, Sd.finish
    hist = []

    def deliver(r, t, ovl):
        k = Sd.calls[r]["user"]
        before = list(Sd.u)
        queued_users = {Sd.calls[q[0]]["user"] for q in Sd.Q}
        res = orig_deliver(r, t, ovl)
        assert all(a >= b for a, b in zip(Sd.u, before))
        if queued_users and k not in queued_users:
            assert Sd.u[k] >= min(before[v] for v in queued_users)
        hist.append(1)
        return res

    def finish(r):
        before = list(Sd.u)
        orig_finish(r)
        assert all(a >= b for a, b in zip(Sd.u, before))

    Sd.deliver, Sd.finish = deliver, finish
    # run the stepper's replay loop with the instrumented scheduler
    import oracle.stepper as st_mod
    real = st_mod.Sched
    st_mod.Sched = lambda *a, **k: Sd
    try:
        st_mod.replay(tr, prof, cfg)
    finally:
        st_mod.Sched = real
    assert hist
