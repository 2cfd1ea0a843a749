"""ORACLE -- TEST INFRASTRUCTURE ONLY.

Plain definitional implementation of the §5 evaluation quantities (NEXT-2; PAPER.md
§5; SPEC module `metrics` S:366-413) over one replay's per-call outputs.
Python loops over calls and interactions, exact integers; only tests/ may import it.
Readings (R9):
  * a participating call is one with status != FILTERED; served = ADMIT (the replay
    runs every admitted call to completion); blocked = USER_REQ..APP_TOK; dropped = DROPPED;
  * an interaction (its participating calls) is completed when every call is served,
    blocked at its head when the head is blocked, aborted midway when the head is served
    and a later call is blocked (RPM);
  * wasted tokens = L_I + L_S + L_O of the served calls of aborted-midway interactions
    (S:376, S:383 example: 185);
  * prompt / decode tokens = L_I + L_S / L_O of served calls; abuser tokens = both over
    calls of users with tier > 0;
  * TTFT = first_ns - arrive_ns of served calls; p50 / p99 by nearest rank (Q30);
  * users with feedback = users with a participating interaction; served users = with a
    completed interaction; delayed users = with a served call whose wait
    admit_ns - arrive_ns exceeds the threshold (S:404 leaves it open: a parameter);
  * Jain's index over the per-user served tokens of the users with feedback:
    (sum x)^2 / (n sum x^2); 0 when every x is 0 (S:391 makes that an error; we report 0).
Per-app values restrict every quantity to the calls / interactions / users of that app.
"""
from __future__ import annotations

import numpy as np

ADMIT, DROPPED, FILTERED = 0, 5, 6

FIELDS = ["requests_total", "requests_served", "requests_blocked", "requests_dropped",
          "interactions_total", "interactions_completed", "interactions_blocked_at_head",
          "interactions_aborted_midway", "wasted_tokens", "prompt_tokens", "decode_tokens", "abuser_tokens",
          "users_feedback", "users_served", "users_delayed", "ttft_n", "ttft_sum_ns", "ttft_p50_ns",
          "ttft_p99_ns", "jain"]


def _nearest_rank(sorted_vals, q_ppm):
    """x_(max(1, ceil(q n))) of a sorted list (nearest rank, Q30); 0 if empty."""
    n = len(sorted_vals)
    if n == 0:
        return 0
    r = max(1, -(-q_ppm * n // 1_000_000))
    return int(sorted_vals[r - 1])


def jain_index(xs):
    """(sum x)^2 / (n sum x^2); 0.0 for an empty or all-zero list."""
    xs = [int(x) for x in xs]
    s2 = sum(x * x for x in xs)
    if not xs or s2 == 0:
        return 0.0
    return float(sum(xs)) ** 2 / (len(xs) * float(s2))


def _block(st):
    return 1 <= st <= 4


def replay_metrics(tr, out, delay_threshold_ns):
    """Returns (global dict, list of per-app dicts) of FIELDS."""
    n = int(tr["n_calls"])
    A = int(tr["n_apps"])
    status = [int(x) for x in np.asarray(out["status"])]
    arrive = [int(x) for x in np.asarray(out["arrive_ns"])]
    admit = [int(x) for x in np.asarray(out["admit_ns"])]
    first = [int(x) for x in np.asarray(out["first_ns"])]
    meta = [int(x) for x in tr["meta"]]
    user = [int(x) for x in tr["user"]]
    inter = [int(x) for x in tr["inter"]]
    Li = [int(x) for x in tr["len_in"]]
    Ls = [int(x) for x in tr["len_sys"]]
    Lo = [int(x) for x in tr["len_out"]]
    app = [m & 255 for m in meta]
    stage = [(m >> 8) & 255 for m in meta]
    tier = [m >> 24 for m in meta]

    def empty():
        return {k: 0 for k in FIELDS}

    res = [empty() for _ in range(A + 1)]          # index A = global
    ttft = [[] for _ in range(A + 1)]
    calls_of = {}
    for i in range(n):
        if status[i] == FILTERED:
            continue
        calls_of.setdefault(inter[i], []).append(i)
        for g in (app[i], A):
            r = res[g]
            r["requests_total"] += 1
            if status[i] == ADMIT:
                r["requests_served"] += 1
                r["prompt_tokens"] += Li[i] + Ls[i]
                r["decode_tokens"] += Lo[i]
                if tier[i] > 0:
                    r["abuser_tokens"] += Li[i] + Ls[i] + Lo[i]
                ttft[g].append(first[i] - arrive[i])
            elif _block(status[i]):
                r["requests_blocked"] += 1
            elif status[i] == DROPPED:
                r["requests_dropped"] += 1
    users_fb = [set() for _ in range(A + 1)]
    users_served = [set() for _ in range(A + 1)]
    users_delayed = [set() for _ in range(A + 1)]
    tokens = [dict() for _ in range(A + 1)]
    for x, cs in calls_of.items():
        h = next(i for i in cs if stage[i] == 1)
        a, k = app[h], user[h]
        completed = all(status[i] == ADMIT for i in cs)
        at_head = _block(status[h])
        midway = status[h] == ADMIT and any(_block(status[i]) for i in cs)
        wasted = sum(Li[i] + Ls[i] + Lo[i] for i in cs if status[i] == ADMIT) if midway else 0
        for g in (a, A):
            r = res[g]
            r["interactions_total"] += 1
            r["interactions_completed"] += int(completed)
            r["interactions_blocked_at_head"] += int(at_head)
            r["interactions_aborted_midway"] += int(midway)
            r["wasted_tokens"] += wasted
            users_fb[g].add(k)
            tokens[g].setdefault(k, 0)
            if completed:
                users_served[g].add(k)
        for i in cs:
            if status[i] == ADMIT:
                for g in (a, A):
                    tokens[g][k] += Li[i] + Ls[i] + Lo[i]
                    if admit[i] - arrive[i] > delay_threshold_ns:
                        users_delayed[g].add(k)
    for g in range(A + 1):
        r = res[g]
        r["users_feedback"] = len(users_fb[g])
        r["users_served"] = len(users_served[g])
        r["users_delayed"] = len(users_delayed[g])
        v = sorted(ttft[g])
        r["ttft_n"] = len(v)
        r["ttft_sum_ns"] = sum(v)
        r["ttft_p50_ns"] = _nearest_rank(v, 500_000)
        r["ttft_p99_ns"] = _nearest_rank(v, 990_000)
        r["jain"] = jain_index(tokens[g].values())
    return res[A], res[:A]
