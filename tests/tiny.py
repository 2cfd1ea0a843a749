"""Seeded tiny-trace and tiny-config generators for brute-force tests (inputs only)."""
import numpy as np

from paper_2411_15997_b200.tracegen import from_columns

UMAX = 0xFFFFFFFF


def tiny_trace(rng, n_users=3, n_apps=2, max_inters=4, times=(0, 1, 2, 5), lens=(1, 2, 5),
               m_choices=(1, 1, 2, 3), thinks=(0, 1, 3), abusive_user=True, max_calls=6):
    rows = []
    n_int = int(rng.integers(1, max_inters + 1))
    tiers = [0] * n_users
    if abusive_user and rng.random() < 0.5:
        tiers[int(rng.integers(0, n_users))] = int(rng.integers(1, 3))
    ncalls_total = 0
    for x in range(n_int):
        m = int(rng.choice(m_choices))
        if ncalls_total + m > max_calls:
            m = max_calls - ncalls_total
        if m <= 0:
            break
        u = int(rng.integers(0, n_users))
        a = int(rng.integers(0, n_apps))
        t0 = int(rng.choice(times))
        for s in range(1, m + 1):
            if s > 1:
                t0 += int(rng.integers(0, 3))
            rows.append(dict(user=u, t_ms=t0, app=a, inter=x, stage=s,
                             ncalls=m, len_in=int(rng.choice(lens)), len_sys=int(rng.choice((0, 0, 1))),
                             len_out=int(rng.choice(lens)), think_ms=int(rng.choice(thinks)), tier=tiers[u]))
        ncalls_total += m
    rows.sort(key=lambda r: (r["t_ms"], r["inter"], r["stage"]))
    # inter ids dense in head order
    ren = {}
    for r in rows:
        if r["stage"] == 1:
            ren.setdefault(r["inter"], len(ren))
    for r in rows:
        r["inter"] = ren[r["inter"]]
    return from_columns(n_users, n_apps, rows)


def tiny_replay_cfg(rng, n_apps, modes=(0, 1)):
    cfg = dict(mode=int(modes[int(rng.integers(0, len(modes)))]), alpha=int(rng.choice((1, 2))), beta=int(rng.choice((1, 2))),
               gamma=int(rng.choice((1, 3))), prio_benign_q16=65536,
               prio_abusive_q16=int(rng.choice((65536, 131072, 32768))),
               kv_capacity=int(rng.choice((14, 20, 30, 100))), max_batch=int(rng.choice((1, 2, 3))),
               overload_permille=int(rng.choice((0, 300, 500, 900, UMAX))),
               iter_base_ns=1_000_000, decode_ns_per_req=int(rng.choice((0, 500_000))),
               prefill_ns_per_tok=int(rng.choice((0, 100_000))),
               tier_max=int(rng.choice((0, 255, 255))))
    cfg["act"] = dict(window_ms=int(rng.choice((1, 3, 10))), limits_from_profile=0,
                      T_req_g=int(rng.choice((0, 1, 2))),
                      T_req_a=[int(rng.choice((0, 1, 2))) for _ in range(n_apps)],
                      T_tok_g=int(rng.choice((0, 0, 12))),
                      T_tok_a=[int(rng.choice((0, 0, 9))) for _ in range(n_apps)],
                      count_mode=int(rng.integers(0, 2)))
    if cfg["mode"] == 3:         # RPM: explicit request limits only (R8)
        cfg["act"]["T_tok_g"] = 0
        cfg["act"]["T_tok_a"] = [0] * n_apps
    return cfg


def tiny_profile(rng, n_apps, J=3):
    cnt = rng.integers(1, 4, size=(n_apps, J + 1))
    cnt[:, 0] = 0
    s_in = cnt * rng.integers(1, 5, size=cnt.shape)
    s_sys = cnt * rng.integers(0, 2, size=cnt.shape)
    s_out = cnt * rng.integers(1, 5, size=cnt.shape) + rng.integers(0, 2, size=cnt.shape)
    s_out[:, 0] = 0
    if rng.random() < 0.3:         # shallower profile: exercises the stage clamp
        cnt[:, 2:] = 0
        s_in[:, 2:] = s_sys[:, 2:] = s_out[:, 2:] = 0
    return J, cnt, s_in, s_sys, s_out
