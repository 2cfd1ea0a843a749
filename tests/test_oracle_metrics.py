"""Pins for the §5 metric-suite oracle (oracle/metrics.py; NEXT-2, SPEC S:366-413,
PAPER.md P:534-576): the SPEC's worked examples, the paper's stated properties, and the
accounting identities."""
import numpy as np
import pytest

import oracle as O
from oracle import metrics as M
from paper_2411_15997_b200 import tracegen as G
from paper_2411_15997_b200.tracegen import from_columns

ADDITIVE = [f for f in M.FIELDS if f not in ("users_feedback", "users_served", "users_delayed", "ttft_p50_ns",
                                            "ttft_p99_ns", "jain")]


def test_jain_examples():
    """S:391-393."""
    assert M.jain_index([5, 5, 5, 5]) == 1.0
    assert M.jain_index([1, 0, 0, 0]) == 0.25
    assert M.jain_index([1, 2, 3]) == pytest.approx(36 / 42, rel=1e-15)


def test_nearest_rank():
    assert M._nearest_rank([10, 20, 30, 40], 500_000) == 20
    assert M._nearest_rank([10, 20, 30, 40], 990_000) == 40
    assert M._nearest_rank([7], 990_000) == 7 and M._nearest_rank([], 500_000) == 0


def test_wasted_tokens_example():
    """one 3-call interaction aborted after call 2 finished (100+0 in / 10 out, 50+20 in /
    5 out) wastes (100+10)+(50+20+5) = 185 tokens; built here as an RPM replay whose third call
    exceeds the user limit."""
    rows = [dict(user=0, t_ms=0, app=0, inter=0, stage=1, ncalls=3, len_in=100, len_out=10),
            dict(user=0, t_ms=1, app=0, inter=0, stage=2, ncalls=3, len_in=50, len_sys=20, len_out=5),
            dict(user=0, t_ms=2, app=0, inter=0, stage=3, ncalls=3, len_in=5, len_out=5)]
    tr = from_columns(1, 1, rows)
    prof = O.profile_from_host(1, 3, [[0, 1, 1, 1]], [[0, 1, 1, 1]], [[0, 0, 0, 0]], [[0, 1, 1, 1]])
    cfg = dict(mode=3, kv_capacity=1000, max_batch=4, overload_permille=900, iter_base_ns=100_000,
               decode_ns_per_req=0, prefill_ns_per_tok=0,
               act=dict(window_ms=60000, limits_from_profile=0, T_req_g=2, T_req_a=[0]))
    o, s = O.replay(tr, prof, cfg)
    assert list(o["status"]) == [0, 0, 1]
    g, per_app = M.replay_metrics(tr, o, 10**9)
    assert g["wasted_tokens"] == 185
    assert g["interactions_aborted_midway"] == 1 and g["interactions_completed"] == 0
    assert g["users_feedback"] == 1 and g["users_served"] == 0


def _cases():
    tr = G.generate(dict(G.CONFIGS["c2"], n_users=60, n_calls=6000, seed=81))
    op = O.profile(tr, dict(tier_max=255))
    base = dict(G.CONFIGS["c2"]["engine"], tier_max=255, alpha=1, beta=2, gamma=1)
    out = {}
    out["wi"] = O.replay(tr, op, dict(base, mode=1, act=dict(window_ms=60000, limits_from_profile=1)))[0]
    out["w"] = O.replay(tr, op, dict(base, mode=0))[0]
    out["vtc"] = O.replay(tr, op, dict(base, mode=2, beta=1, gamma=2))[0]
    out["rpm"] = O.replay(tr, op, dict(base, mode=3, act=dict(window_ms=60000, limits_from_profile=0, T_req_g=3,
                                                              T_req_a=[20] * tr["n_apps"])))[0]
    return tr, out


@pytest.fixture(scope="module")
def cases():
    return _cases()


def test_properties(cases):
    """P:535-539 / S:384: FS(W+I) never aborts an interaction midway, FS(W) and VTC
    never throttle (every user with feedback is served, nothing wasted); RPM aborts midway."""
    tr, out = cases
    thr = 10**9
    for k in ("wi", "w", "vtc"):
        g, _ = M.replay_metrics(tr, out[k], thr)
        assert g["interactions_aborted_midway"] == 0 and g["wasted_tokens"] == 0
    for k in ("w", "vtc"):
        g, _ = M.replay_metrics(tr, out[k], thr)
        assert g["users_served"] == g["users_feedback"] and g["requests_blocked"] == 0
    g, _ = M.replay_metrics(tr, out["rpm"], thr)
    assert g["interactions_aborted_midway"] > 0 and g["wasted_tokens"] > 0


def test_accounting_identities(cases):
    """every participating request is served, blocked or dropped (a replay runs to
    completion); every interaction is completed, blocked at its head or aborted midway; the
    per-app breakdown sums to the global values; delayed users fall as the threshold grows."""
    tr, out = cases
    for k, o in out.items():
        g, per_app = M.replay_metrics(tr, o, 5 * 10**6)
        assert g["requests_total"] == g["requests_served"] + g["requests_blocked"] + g["requests_dropped"]
        assert g["interactions_total"] == (g["interactions_completed"] + g["interactions_blocked_at_head"] +
                                           g["interactions_aborted_midway"])
        assert g["requests_total"] == int(tr["n_calls"])
        for f in ADDITIVE:
            assert sum(p[f] for p in per_app) == g[f], (k, f)
        assert 0 < g["jain"] <= 1
        assert g["ttft_p50_ns"] <= g["ttft_p99_ns"]
        assert g["ttft_n"] == g["requests_served"]
        d = [M.replay_metrics(tr, o, th)[0]["users_delayed"] for th in (0, 10**7, 10**9, 10**13)]
        assert d == sorted(d, reverse=True)
