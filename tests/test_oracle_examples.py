"""Oracle pinned to the hand-worked examples and printed values (not to itself).

Examples W, WI, A, P: tests/golden/*.json (each cites its passage).  Closed
forms: Eq. 2 / Eq. 3 evaluations printed in PAPER.md §3.2 and the
graph-size table row "1", can_admit arithmetic.
"""
import numpy as np
import pytest

import oracle as O
from conftest import golden, golden_trace
from paper_2411_15997_b200.tracegen import from_columns

MS = 10**6


def _prof(g, A):
    p = g["profile"]
    return O.profile_from_host(A, p["max_stage"], p["cnt"], p["sum_in"], p["sum_sys"], p["sum_out"])


def _ms(a):
    return [int(x) // MS if x >= 0 else -1 for x in a]


def test_example_W():
    g = golden("example_W")
    tr = golden_trace(g)
    o, s = O.replay(tr, _prof(g, g["n_apps"]), g["cfg"])
    e = g["expect"]
    assert list(np.argsort(o["order"])) == e["order"]
    assert _ms(o["admit_ns"]) == e["admit_ms"]
    assert _ms(o["first_ns"]) == e["first_ms"]
    assert _ms(o["finish_ns"]) == e["finish_ms"]
    assert list(o["counters"]) == e["counters"]
    assert list(o["status"]) == e["status"]
    # FCFS by (t, id) would have been c0, c2, c3, c1, ... -- WSC differs
    assert s["n_admitted"] == 7 and s["n_finished"] == 7 and s["makespan_ns"] == 70 * MS


def test_example_WI():
    g = golden("example_WI")
    tr = golden_trace(g)
    prof = _prof(g, 1)
    o, s = O.replay(tr, prof, g["cfg"])
    e = g["expect"]
    assert list(o["status"]) == e["status"]
    assert list(o["ovl"]) == e["ovl"]
    assert _ms(o["admit_ns"]) == e["admit_ms"]
    assert _ms(o["first_ns"]) == e["first_ms"]
    assert _ms(o["finish_ns"]) == e["finish_ms"]
    assert list(o["counters"]) == e["counters"]
    assert s["n_block"] == [2, 0, 0, 0]
    # P8 cross-check: ACT on the replay's arrival times + overload flags reproduces statuses
    st, _ = O.act(tr, prof, g["cfg"]["act"], overloaded=o["ovl"], t_ns_override=o["arrive_ns"])
    assert list(st) == e["status"]
    # contrast: FS(W) -- d1 blocks the admission round (Q16), d2 admitted only at 5 ms
    cfg = dict(g["cfg"], mode=0)
    o2, _ = O.replay(tr, prof, cfg)
    assert o2["admit_ns"][2] == g["contrast_fs_w"]["d2_admit_ms"] * MS


def test_example_A():
    g = golden("example_A")
    tr = golden_trace(g)
    st, summ = O.act(tr, None, g["cfg"], overloaded=np.array(g["overloaded"], np.uint8))
    assert list(st) == g["expect_all"]
    st2, _ = O.act(tr, None, dict(g["cfg"], count_mode=1), overloaded=np.array(g["overloaded"], np.uint8))
    assert list(st2) == g["expect_heads_only"]
    assert summ["n_dropped"] == 2 and summ["n_block"] == [3, 0, 2, 0]


def test_example_P():
    g = golden("example_P")
    tr = golden_trace(g)
    p = O.profile(tr, g["cfg"])
    e = g["expect"]
    for j in (1, 2):
        assert int(p["cnt"][0, j]) == e[f"cnt_{j}"]
        assert int(p["sum_in"][0, j]) == e[f"sum_in_{j}"]
        assert int(p["sum_sys"][0, j]) == e[f"sum_sys_{j}"]
        assert int(p["sum_out"][0, j]) == e[f"sum_out_{j}"]
        assert int(p["ohat"][0, j]) == e[f"ohat_{j}"]
    W = O.weights(p, 1, 2, 1)
    assert int(W[0, 1]) == e["W_1"] and int(W[0, 2]) == e["W_2"]
    assert list(p["peak_r_u"]) == e["peak_r_u"]
    assert list(p["peak_t_u"]) == e["peak_t_u"]
    assert int(p["T_req_g"][0]) == e["T_req_g"] and list(p["T_req_a"]) == e["T_req_a"]
    assert int(p["T_tok_g"][0]) == e["T_tok_g"] and list(p["T_tok_a"]) == e["T_tok_a"]
    h = p["hist"][0, 0]
    assert {str(b): int(h[b]) for b in np.nonzero(h)[0]} == e["len_in_bins"]
    q = list(g["cfg"]["q_ppm"])
    for qq, v in e["nr_len_in"].items():
        assert int(p["nr_q"][0, 0, q.index(int(qq))]) == v
    for qq, v in e["interp_len_in"].items():
        assert float(p["interp_q"][0, 0, q.index(int(qq))]) == pytest.approx(v, rel=1e-12)
    hm = p["hist"][0, 4]
    assert {str(b): int(hm[b]) for b in np.nonzero(hm)[0]} == e["m_hist"]
    # Eq. 3 increment if q1 finished alone: replay a one-call trace against this profile
    one = from_columns(1, 1, [dict(user=0, t_ms=0, app=0, inter=0, stage=1, ncalls=1,
                                   len_in=300, len_sys=50, len_out=40)])
    o, _ = O.replay(one, p, dict(mode=0, kv_capacity=10**6, max_batch=1, iter_base_ns=MS,
                                  decode_ns_per_req=0, prefill_ns_per_tok=0))
    assert int(o["counters"][0]) == e["inc_q1"]


def _one_call_inc(L_I, L_S, L_O, cnt, s_in, s_sys, s_out, alpha=1, beta=2, gamma=1, E=65536):
    tr = from_columns(1, 1, [dict(user=0, t_ms=0, app=0, inter=0, stage=1, ncalls=1,
                                  len_in=L_I, len_sys=L_S, len_out=L_O)])
    p = O.profile_from_host(1, 1, [[0, cnt]], [[0, s_in]], [[0, s_sys]], [[0, s_out]])
    o, _ = O.replay(tr, p, dict(mode=0, alpha=alpha, beta=beta, gamma=gamma, prio_benign_q16=E,
                                kv_capacity=10**7, max_batch=1, iter_base_ns=MS,
                                decode_ns_per_req=0, prefill_ns_per_tok=0))
    return int(o["counters"][0])


def test_eq2_printed_values():
    # Eq. 2 with (alpha,beta,gamma)=(1,2,1): (10,5,20)->40, (10,0,0)->10
    p = O.profile_from_host(2, 1, [[0, 1], [0, 1]], [[0, 10], [0, 10]], [[0, 5], [0, 0]], [[0, 20], [0, 0]])
    W = O.weights(p, 1, 2, 1)
    assert int(W[0, 1]) == 40 << 16 and int(W[1, 1]) == 10 << 16
    # graph-size table row "1": avg input 4994.65, output 136.86 over 100 interactions
    p = O.profile_from_host(1, 1, [[0, 100]], [[0, 499465]], [[0, 0]], [[0, 13686]])
    assert int(O.weights(p, 1, 2, 1)[0, 1]) == 336298639      # 5131.51 in Q16, truncated


def test_eq3_section32_worked_case():
    # PAPER.md §3.2: apps with average length 10 and 50; 5 tokens processed
    # -> 5/10 = 50% and 5/50 = 10% (alpha,beta,gamma) = (1,0,0)
    assert _one_call_inc(5, 0, 1, 1, 10, 0, 0, 1, 0, 0) == 1 << 31
    assert _one_call_inc(5, 0, 1, 1, 50, 0, 0, 1, 0, 0) == 429496729    # floor(0.1 * 2^32)
    # a request matching its app's expectations -> exactly 1.0; E = 2 -> 2.0
    assert _one_call_inc(10, 5, 20, 1, 10, 5, 20) == 1 << 32
    assert _one_call_inc(10, 5, 20, 1, 10, 5, 20, E=2 * 65536) == 1 << 33


def test_can_admit_arithmetic():
    # capacity 1000, occupied 900, candidate 50 + reserve 60 -> 1010 > 1000 -> no admit.
    # Realise occ = 900 with an in-flight call of prompt 899 (+1 decoded token).
    rows = [dict(user=0, t_ms=0, app=0, inter=0, stage=1, ncalls=1, len_in=899, len_out=100),
            dict(user=1, t_ms=0, app=1, inter=1, stage=1, ncalls=1, len_in=50, len_out=1)]
    tr = from_columns(2, 2, rows)
    p = O.profile_from_host(2, 1, [[0, 1], [0, 1]], [[0, 1], [0, 1]], [[0, 0], [0, 0]], [[0, 1], [0, 60]])
    cfg = dict(mode=0, kv_capacity=1000, max_batch=8, iter_base_ns=MS, decode_ns_per_req=0,
               prefill_ns_per_tok=0)
    o, _ = O.replay(tr, p, cfg)
    assert o["admit_ns"][1] == 100 * MS          # waits for call 0 to finish at 100 ms
    p2 = O.profile_from_host(2, 1, [[0, 1], [0, 1]], [[0, 1], [0, 1]], [[0, 0], [0, 0]], [[0, 1], [0, 50]])
    o2, _ = O.replay(tr, p2, cfg)                 # 900 + 50 + 50 = 1000 <= 1000 fits at 1 ms
    assert o2["admit_ns"][1] == 0


def test_single_call_ttft():
    # TTFT = iter_base + 10 * prefill + 1 * decode; finish after 5 decode iterations
    tr = from_columns(1, 1, [dict(user=0, t_ms=0, app=0, inter=0, stage=1, ncalls=1, len_in=10, len_out=5)])
    p = O.profile_from_host(1, 1, [[0, 1]], [[0, 10]], [[0, 0]], [[0, 5]])
    cfg = dict(mode=0, kv_capacity=1000, max_batch=4, iter_base_ns=2 * MS, decode_ns_per_req=500_000,
               prefill_ns_per_tok=10_000)
    o, s = O.replay(tr, p, cfg)
    assert o["first_ns"][0] == 2 * MS + 10 * 10_000 + 500_000
    assert s["n_iterations"] == 5
    assert o["finish_ns"][0] == o["first_ns"][0] + 4 * (2 * MS + 500_000)
