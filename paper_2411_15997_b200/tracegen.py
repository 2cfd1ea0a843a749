"""Seeded synthetic trace generator (input plumbing only).

This module is the ONE piece shared by the CUDA path and the CPU oracle: it
draws the synthetic, Copilot-shaped request traces both sides are run on.  It
holds none of the method's arithmetic (no profiles, windows, counters,
weights or scheduling) -- only random numbers turned into trace records.

Workload shape:
  * apps with distinct token-length ranges (§3.2, P:212-248;
    case-study apps 14/7/12, `tab:application_comparison` P:615-616);
  * heavy-tailed lognormal lengths;
  * calls per interaction from the graph-size table `tab:graph_table`
    (P:302-322): 73.22 / 26.09 / 0.50 / 0.11 / 0.0267 x3 %;
  * heterogeneous per-user rates, a minority of abusive users
     with 20x head rate and ON/OFF bursts;
  * diurnal head arrivals over one day ("a full day").

Record layout: eight little-endian u32 arrays, sorted by
(t_ms, index); index = call id.
    user, t_ms, len_in, len_sys, len_out, think_ms, inter, meta
    meta = app | stage << 8 | ncalls << 16 | tier << 24
"""
from __future__ import annotations

import numpy as np

FIELDS = ("user", "t_ms", "len_in", "len_sys", "len_out", "think_ms", "inter", "meta")

# (name, mean L_I, mean L_S, mean L_O)
APP_TEMPLATES = [
    ("QA", 600, 200, 180),
    ("SUM", 6000, 300, 110),
    ("CODE", 400, 600, 450),
    ("app14", 6370, 0, 102),
    ("app7", 14854, 0, 74),
    ("app12", 999, 0, 32),
]

# graph-size table buckets: (lo, hi, percent)
GRAPH_BUCKETS = [
    (1, 1, 73.22), (2, 10, 26.09), (11, 20, 0.50), (21, 30, 0.11),
    (31, 40, 0.0267), (41, 50, 0.0267), (51, 100, 0.0267),
]

DAY_MS = 86_400_000

# Engine / profile / ACT parameters travel with the workload.  Times in ns.
CONFIGS = {
    "c1": dict(name="c1", n_users=4, apps=["QA", "SUM"], app_scales=[1.0], n_calls=200,
               n_abusive=1, seed=1, duration_ms=600_000, m_dist="c1",
               in_cap=8000, sys_cap=2000, out_cap=2000,
               engine=dict(kv_capacity=20_000, max_batch=4, overload_permille=900,
                           iter_base_ns=2_000_000, decode_ns_per_req=500_000,
                           prefill_ns_per_tok=10_000),
               act=dict(window_ms=60_000, T_req_g=8, T_req_a=[5, 5]),
               profile=dict(tier_max=255)),
    "c2": dict(name="c2", n_users=1000, apps=[t[0] for t in APP_TEMPLATES], app_scales=[1.0],
               n_calls=1_000_000, abusive_frac=0.05, seed=2, duration_ms=DAY_MS, m_dist="graph",
               in_cap=16_000, sys_cap=4000, out_cap=4000,
               engine=dict(kv_capacity=49_152, max_batch=256, overload_permille=900,
                           iter_base_ns=2_000_000, decode_ns_per_req=20_000,
                           prefill_ns_per_tok=10_000),
               act=dict(window_ms=60_000),
               profile=dict(tier_max=0)),
    "c3": dict(name="c3", n_users=10_000, apps=[t[0] for t in APP_TEMPLATES], app_scales=[0.5, 2.0],
               n_calls=10_000_000, abusive_frac=0.05, seed=3, duration_ms=DAY_MS, m_dist="graph",
               in_cap=16_000, sys_cap=4000, out_cap=4000,
               engine=dict(kv_capacity=49_152, max_batch=256, overload_permille=900,
                           iter_base_ns=200_000, decode_ns_per_req=2_000,
                           prefill_ns_per_tok=1_500),   # calibrated (oracle, FS(W)): 22.5 % of arrivals
                                                        # overloaded with every tier, 3.0 % benign only
               act=dict(window_ms=60_000),
               profile=dict(tier_max=0)),
    "c4": dict(name="c4", n_users=100_000, apps=[t[0] for t in APP_TEMPLATES],
               app_scales=[0.5, 0.75, 1.0, 1.5, 2.0, 3.0], n_apps=34,
               n_calls=100_000_000, abusive_frac=0.05, seed=4, duration_ms=DAY_MS, m_dist="graph",
               in_cap=16_000, sys_cap=4000, out_cap=4000,
               engine=None, act=dict(window_ms=60_000), profile=dict(tier_max=0)),
}
CONFIGS["c5"] = dict(CONFIGS["c2"], name="c5", seed=2)


def _app_table(cfg):
    names, means = [], []
    for s in cfg["app_scales"]:
        for (nm, mi, ms, mo) in APP_TEMPLATES:
            if nm not in cfg["apps"]:
                continue
            names.append(nm if len(cfg["app_scales"]) == 1 else f"{nm}x{s}")
            means.append((mi * s, ms * s, mo * s))
    n_apps = cfg.get("n_apps", len(names))
    names, means = names[:n_apps], means[:n_apps]
    return names, np.array(means, dtype=np.float64)


def _lognormal_int(rng, mean, sigma, lo, hi):
    """Lognormal with the given mean, clipped to [lo, hi], rounded."""
    mean = np.maximum(mean, 1e-9)
    mu = np.log(mean) - 0.5 * sigma * sigma
    v = np.exp(mu + sigma * rng.standard_normal(mean.shape))
    v = np.rint(v)
    return np.clip(v, lo, hi)


def _sample_m(rng, n, m_dist):
    if m_dist == "c1":
        return np.where(rng.random(n) < 0.8, 1, 3).astype(np.int64)
    p = np.array([b[2] for b in GRAPH_BUCKETS])
    p = p / p.sum()
    b = rng.choice(len(GRAPH_BUCKETS), size=n, p=p)
    lo = np.array([x[0] for x in GRAPH_BUCKETS])[b]
    hi = np.array([x[1] for x in GRAPH_BUCKETS])[b]
    return lo + np.floor(rng.random(n) * (hi - lo + 1)).astype(np.int64)


def _diurnal_times(rng, n, duration_ms, diurnal):
    u = rng.random(n)
    if not diurnal:
        return u * duration_ms
    # inverse CDF of density ∝ 1 - 0.5 cos(2π t / T) on a fine grid
    g = np.linspace(0.0, 1.0, 20001)
    cdf = (g - 0.5 * np.sin(2 * np.pi * g) / (2 * np.pi))
    return np.interp(u, cdf, g) * duration_ms


def generate(cfg_or_name, n_calls=None, seed=None):
    """Return a dict: the eight u32 arrays + n_calls/n_users/n_apps/n_inters + app names."""
    cfg = dict(CONFIGS[cfg_or_name]) if isinstance(cfg_or_name, str) else dict(cfg_or_name)
    if n_calls is not None:
        cfg["n_calls"] = int(n_calls)
    if seed is not None:
        cfg["seed"] = int(seed)
    rng = np.random.Generator(np.random.PCG64(cfg["seed"]))
    N = int(cfg["n_calls"])
    U = int(cfg["n_users"])
    T = int(cfg["duration_ms"])
    app_names, app_means = _app_table(cfg)
    A = len(app_names)

    # ---- users: tier, home app, rate weight
    if "n_abusive" in cfg:
        n_ab = int(cfg["n_abusive"])
    else:
        n_ab = max(1, int(round(cfg["abusive_frac"] * U)))
    tier = np.zeros(U, dtype=np.int64)
    ab_users = rng.choice(U, size=n_ab, replace=False)
    tier[ab_users] = rng.integers(1, 16, size=n_ab)
    zipf = 1.0 / np.arange(1, A + 1) ** 1.1
    home = rng.choice(A, size=U, p=zipf / zipf.sum())
    has_sec = rng.random(U) < 0.3
    sec = rng.integers(0, A, size=U)
    w = np.exp(1.5 * rng.standard_normal(U))
    w[tier > 0] *= 20.0
    abusive = tier > 0

    # ---- interactions: sizes with exact total N
    m_all = []
    tot = 0
    while tot < N:
        m = _sample_m(rng, max(16, int((N - tot) / 2.0) + 16), cfg["m_dist"])
        m_all.append(m)
        tot += int(m.sum())
    m = np.concatenate(m_all)
    cs = np.cumsum(m)
    X = int(np.searchsorted(cs, N) + 1)
    m = m[:X].copy()
    m[-1] -= int(cs[X - 1] - N)
    assert m[-1] >= 1 and int(m.sum()) == N

    # ---- interaction -> user, app, head time
    iu = rng.choice(U, size=X, p=w / w.sum())
    use_sec = has_sec[iu] & (rng.random(X) < 0.2)
    iapp = np.where(use_sec, sec[iu], home[iu])
    th = _diurnal_times(rng, X, T, diurnal=cfg["name"] != "c1")
    ab = abusive[iu]
    if ab.any():
        # ON/OFF bursts: 25% duty, period = T/24, random phase per user
        period = T / 24.0
        phase = rng.random(U) * period
        k = rng.integers(0, 24, size=int(ab.sum()))
        within = rng.random(int(ab.sum())) * 0.25 * period
        tt = (k * period + phase[iu[ab]] + within) % T
        th[ab] = tt
    th = np.floor(th).astype(np.int64)

    # ---- calls
    inter_tmp = np.repeat(np.arange(X, dtype=np.int64), m)
    start = np.concatenate([[0], np.cumsum(m)[:-1]])
    stage = np.arange(N, dtype=np.int64) - np.repeat(start, m) + 1
    ncalls = np.repeat(m, m)
    capp = iapp[inter_tmp]
    mean_in = app_means[capp, 0] * (1.0 + 0.25 * np.minimum(stage - 1, 4))
    mean_sys = app_means[capp, 1]
    mean_out = app_means[capp, 2] * np.where((stage > 1) & (stage < ncalls), 0.6, 1.0)
    L_I = _lognormal_int(rng, mean_in, 1.0, 1, np.minimum(8 * mean_in, cfg["in_cap"]))
    L_S = np.where(mean_sys > 0,
                   _lognormal_int(rng, mean_sys, 0.5, 0, np.minimum(8 * mean_sys, cfg["sys_cap"])), 0)
    L_O = _lognormal_int(rng, mean_out, 0.9, 1, np.minimum(8 * mean_out, cfg["out_cap"]))
    think = np.floor(rng.exponential(500.0, size=N)).astype(np.int64)
    # recorded continuation time = previous time + nominal service + think
    step = 50 + L_O.astype(np.int64) + think            # ms after this call's arrival
    cstep = np.cumsum(step)
    excl = cstep - step                                   # global exclusive prefix
    t = th[inter_tmp] + (excl - np.repeat(excl[start], m))
    order = np.lexsort((stage, inter_tmp, t))
    # renumber interactions by head position
    pos = np.empty(N, dtype=np.int64)
    pos[order] = np.arange(N)
    head_pos = pos[start]
    inter_rank = np.empty(X, dtype=np.int64)
    inter_rank[np.argsort(head_pos, kind="stable")] = np.arange(X)

    user = iu[inter_tmp]
    meta = capp | (stage << 8) | (ncalls << 16) | (tier[user] << 24)
    out = {
        "user": user[order],
        "t_ms": t[order],
        "len_in": L_I[order],
        "len_sys": L_S[order],
        "len_out": L_O[order],
        "think_ms": think[order],
        "inter": inter_rank[inter_tmp][order],
        "meta": meta[order],
    }
    for k in FIELDS:
        assert out[k].min() >= 0 and out[k].max() < 2**32, k
        out[k] = np.ascontiguousarray(out[k].astype(np.uint32))
    out.update(n_calls=N, n_users=U, n_apps=A, n_inters=X, app_names=app_names,
               config=cfg["name"], seed=cfg["seed"])
    return out


def from_columns(n_users, n_apps, rows):
    """Hand-written tiny traces (tests): rows of dicts with user, t_ms, app,
    inter, stage, ncalls, len_in, len_sys, len_out, think_ms, tier.  Rows must
    already be in (t_ms, id) order; n_inters = max(inter)+1."""
    n = len(rows)
    out = {k: np.zeros(n, dtype=np.uint32) for k in FIELDS}
    for i, r in enumerate(rows):
        out["user"][i] = r["user"]
        out["t_ms"][i] = r["t_ms"]
        out["len_in"][i] = r["len_in"]
        out["len_sys"][i] = r.get("len_sys", 0)
        out["len_out"][i] = r["len_out"]
        out["think_ms"][i] = r.get("think_ms", 0)
        out["inter"][i] = r["inter"]
        out["meta"][i] = (r["app"] | (r["stage"] << 8) | (r["ncalls"] << 16)
                          | (r.get("tier", 0) << 24))
    out.update(n_calls=n, n_users=n_users, n_apps=n_apps,
               n_inters=(max(r["inter"] for r in rows) + 1) if rows else 0,
               app_names=[f"app{a}" for a in range(n_apps)], config="hand", seed=0)
    return out


def sm64(x):
    """splitmix64 finaliser on a u64 numpy array (used only to shard users)."""
    x = (np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15))
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def shard_by_user(tr, rank, world):
    """Rank's user-hash shard (calls of users with sm64(user) % world == rank),
    keeping (t_ms, id) order.  Interaction ids are renumbered densely."""
    with np.errstate(over="ignore"):
        h = sm64(tr["user"].astype(np.uint64)) % np.uint64(world)
    keep = np.nonzero(h == np.uint64(rank))[0]
    out = {k: np.ascontiguousarray(tr[k][keep]) for k in FIELDS}
    inter = out["inter"].astype(np.int64)
    uniq, inv = np.unique(inter, return_inverse=True)
    # keep interaction numbering in order of first (head) appearance
    first = np.full(len(uniq), len(inter), dtype=np.int64)
    np.minimum.at(first, inv, np.arange(len(inter)))
    rank_of = np.empty(len(uniq), dtype=np.int64)
    rank_of[np.argsort(first, kind="stable")] = np.arange(len(uniq))
    out["inter"] = rank_of[inv].astype(np.uint32)
    out.update(n_calls=len(keep), n_users=tr["n_users"], n_apps=tr["n_apps"],
               n_inters=len(uniq), app_names=tr["app_names"], config=tr["config"],
               seed=tr["seed"])
    return out
