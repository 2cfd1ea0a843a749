"""GPU parity: every fs_* call through the C ABI vs the CPU oracle, element by
element, on seeded inputs (tiny brute-force grids, C1, reduced C2 shapes).
Integer outputs bit-exact; interpolated percentiles within 1e-6 relative."""
import numpy as np
import pytest

import oracle as O
from conftest import golden, golden_trace
from paper_2411_15997_b200 import tracegen as G
from tiny import tiny_profile, tiny_replay_cfg, tiny_trace

pytestmark = pytest.mark.gpu
MS = 10**6
UMAX = 0xFFFFFFFF


@pytest.fixture(scope="module")
def F():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2411_15997_b200 import build, fairserve
    build.build()
    return fairserve


@pytest.fixture(scope="module")
def ctx(F):
    return F.Context(0)


def _np(t):
    import torch
    a = t.cpu().numpy()
    if t.dtype == torch.int32:
        return a.view(np.uint32)
    if t.dtype == torch.int64:
        return a
    return a


def gpu_prof_host(F, ctx, p):
    return F.profile_from_host(ctx, p["A"], p["J"], p["cnt"], p["sum_in"], p["sum_sys"], p["sum_out"],
                               p["T_req_a"], int(p["T_req_g"][0]), p["T_tok_a"], int(p["T_tok_g"][0]))


def cmp_replay(F, ctx, tr, gp, op, cfg, tag=""):
    T = F.Trace(tr)
    try:
        eo, es = O.replay(tr, op, cfg)
        ecode = 0
    except O.OracleError as e:
        ecode, eidx = e.code, e.bad_index
    if ecode:
        with pytest.raises(F.FsError) as ei:
            F.wsc_replay(ctx, T, gp, cfg)
        assert ei.value.code == ecode and ei.value.bad_index == eidx, tag
        return None
    o, s = F.wsc_replay(ctx, T, gp, cfg)
    for k, ek in (("status", "status"), ("ovl", "ovl"), ("arrive_ns", "arrive_ns"), ("admit_ns", "admit_ns"),
                  ("first_ns", "first_ns"), ("finish_ns", "finish_ns")):
        g = _np(o[k])
        bad = np.nonzero(g != eo[ek])[0]
        assert len(bad) == 0, (tag, k, bad[:5], g[bad[:5]], eo[ek][bad[:5]])
    assert (_np(o["order"]) == eo["order"]).all(), tag
    assert (_np(o["counters"]).view(np.uint64) == eo["counters"]).all(), tag
    assert (_np(o["admitted_per_app"]).view(np.uint64) == eo["admitted_per_app"]).all(), tag
    for k in O.SUMMARY_FIELDS:
        assert s[k] == es[k], (tag, k, s[k], es[k])
    return o, s


# ------------------------------------------------------------------ golden examples
def test_example_W_gpu(F, ctx):
    g = golden("example_W")
    tr = golden_trace(g)
    p = g["profile"]
    gp = F.profile_from_host(ctx, 2, p["max_stage"], p["cnt"], p["sum_in"], p["sum_sys"], p["sum_out"])
    op = O.profile_from_host(2, p["max_stage"], p["cnt"], p["sum_in"], p["sum_sys"], p["sum_out"])
    o, s = cmp_replay(F, ctx, tr, gp, op, g["cfg"], "W")
    assert list(_np(o["admit_ns"]) // MS) == g["expect"]["admit_ms"]
    assert list(_np(o["counters"])) == g["expect"]["counters"]


def test_example_WI_gpu(F, ctx):
    g = golden("example_WI")
    tr = golden_trace(g)
    p = g["profile"]
    gp = F.profile_from_host(ctx, 1, p["max_stage"], p["cnt"], p["sum_in"], p["sum_sys"], p["sum_out"])
    op = O.profile_from_host(1, p["max_stage"], p["cnt"], p["sum_in"], p["sum_sys"], p["sum_out"])
    o, s = cmp_replay(F, ctx, tr, gp, op, g["cfg"], "WI")
    assert list(_np(o["status"])) == g["expect"]["status"]
    assert list(_np(o["counters"])) == g["expect"]["counters"]
    # P8: ACT on the replay's arrivals + overload flags reproduces the statuses
    T = F.Trace(tr)
    st, _ = F.act_throttle(ctx, T, gp, g["cfg"]["act"], overloaded=o["ovl"], t_ns_override=o["arrive_ns"])
    assert list(_np(st)) == g["expect"]["status"]


def test_example_A_gpu(F, ctx):
    import torch
    g = golden("example_A")
    tr = golden_trace(g)
    T = F.Trace(tr)
    ovl = torch.tensor(g["overloaded"], dtype=torch.uint8, device="cuda")
    st, _ = F.act_throttle(ctx, T, None, g["cfg"], overloaded=ovl)
    assert list(_np(st)) == g["expect_all"]
    st, _ = F.act_throttle(ctx, T, None, dict(g["cfg"], count_mode=1), overloaded=ovl)
    assert list(_np(st)) == g["expect_heads_only"]


def _cmp_profile(gpr, op, nq):
    for k in ("cnt", "sum_in", "sum_sys", "sum_out", "ohat", "maxstage", "hist", "n_app", "nr_q", "peak_r_u",
              "peak_t_u", "peak_r_ua", "peak_t_ua", "nr_peak_r_a", "nr_peak_t_a", "nr_peak_r_g", "nr_peak_t_g",
              "T_req_a", "T_tok_a", "T_req_g", "T_tok_g"):
        a, b = np.asarray(gpr[k]), np.asarray(op[k])
        assert a.shape == b.shape and (a == b).all(), (k, np.nonzero(a != b))
    np.testing.assert_allclose(gpr["interp_q"], op["interp_q"], rtol=1e-6, atol=0)


def test_example_P_gpu(F, ctx):
    g = golden("example_P")
    tr = golden_trace(g)
    gpr = F.build_app_profiles(ctx, F.Trace(tr), g["cfg"]).read()
    _cmp_profile(gpr, O.profile(tr, g["cfg"]), 3)
    assert list(gpr["peak_r_u"]) == g["expect"]["peak_r_u"]


# ------------------------------------------------------------------ profiles
@pytest.mark.parametrize("case", ["c1", "mid", "c2small_t0", "heads"])
def test_profile_parity(F, ctx, case):
    if case == "c1":
        tr, cfg = G.generate("c1"), dict(tier_max=255)
    elif case == "mid":
        tr, cfg = G.generate(dict(G.CONFIGS["c3"], n_users=300, n_calls=150_000, seed=21)), dict(tier_max=255, max_stage=8)
    elif case == "c2small_t0":
        tr, cfg = G.generate(dict(G.CONFIGS["c2"], n_users=200, n_calls=60_000, seed=22)), dict(tier_max=0)
    else:
        tr, cfg = G.generate(dict(G.CONFIGS["c2"], n_users=100, n_calls=30_000, seed=23)), \
            dict(tier_max=3, count_mode=1, window_ms=30_000, limit_mult_q8=300)
    gpr = F.build_app_profiles(ctx, F.Trace(tr), cfg).read()
    _cmp_profile(gpr, O.profile(tr, cfg), 5)


@pytest.mark.parametrize("n", [1, 31, 4095, 4096, 4097, 12289])
def test_profile_tile_boundaries(F, ctx, n):
    """Sizes around the 4096-item tiles of the single-pass window scan and the device-wide scan
    (one tile, exact tiles, one item over, several tiles + a ragged tail)."""
    tr = G.generate(dict(G.CONFIGS["c2"], n_users=50, n_calls=n, seed=31 + n))
    assert tr["n_calls"] == n
    cfg = dict(tier_max=255, window_ms=20_000)
    gpr = F.build_app_profiles(ctx, F.Trace(tr), cfg).read()
    _cmp_profile(gpr, O.profile(tr, cfg), 5)


@pytest.mark.parametrize("case", ["dense", "dense_heads_tau", "users_2pass", "users_3pass"])
def test_profile_user_order(F, ctx, case):
    """The onesweep user order + segmented window kernel: dense users whose 60-s windows hold
    hundreds of calls (windows reaching back past a 32-position step, several apps per user),
    weighted token loads under heads-only counting, and user counts that need two (17 bits) and
    three (19 bits) radix passes."""
    if case.startswith("dense"):
        tr = G.generate(dict(G.CONFIGS["c3"], n_users=40, n_calls=100_000, duration_ms=3_600_000, seed=44))
        cfg = dict(tier_max=255) if case == "dense" else \
            dict(tier_max=7, count_mode=1, tau_w_in=2, tau_w_sys=0, tau_w_out=5, window_ms=90_000)
    elif case == "users_2pass":
        tr, cfg = G.generate(dict(G.CONFIGS["c2"], n_users=70_000, n_calls=200_000, seed=42)), dict(tier_max=255)
    else:
        tr, cfg = G.generate(dict(G.CONFIGS["c2"], n_users=300_000, n_calls=400_000, seed=43)), dict(tier_max=2)
    gpr = F.build_app_profiles(ctx, F.Trace(tr), cfg).read()
    op = O.profile(tr, cfg)
    _cmp_profile(gpr, op, 5)
    if case == "dense":
        assert int(np.max(op["peak_r_u"])) > 64                           # windows longer than two steps
        assert (op["peak_r_ua"] > 0).sum() > (op["peak_r_u"] > 0).sum()  # users with several apps


def test_profile_c2_full(F, ctx):
    tr = G.generate("c2")
    cfg = dict(tier_max=0)
    gpr = F.build_app_profiles(ctx, F.Trace(tr), cfg).read()
    _cmp_profile(gpr, O.profile(tr, cfg), 5)


def _cmp_profile_shard(gpr, op, nq, mine):
    """A rank's finalised profile: every global table equals the unsharded one; the per-user
    window peaks are the rank's own users' (zero elsewhere) -- they are never gathered."""
    for k in ("peak_r_u", "peak_t_u", "peak_r_ua", "peak_t_ua"):
        a, b = np.asarray(gpr[k]), np.asarray(op[k])
        m = mine if a.ndim == 1 else mine[:, None]
        assert a.shape == b.shape and (a == np.where(m, b, 0)).all(), k
    g = dict(gpr)
    for k in ("peak_r_u", "peak_t_u", "peak_r_ua", "peak_t_ua"):
        g[k] = op[k]
    _cmp_profile(g, op, nq)


def test_profile_window_load_over_2_32(F, ctx):
    """A user whose window token load passes 2^32 (400 calls of 16M input tokens inside 60 s): the
    window pieces keep ring prefixes mod 2^32 and must hand that user to the exact u64 kernel;
    peaks and limits equal the oracle's."""
    from paper_2411_15997_b200.tracegen import from_columns
    rows = []
    for k in range(400):
        rows.append(dict(user=0, t_ms=10 * k, app=0, inter=0, stage=1, ncalls=1, len_in=16_000_000, len_sys=0,
                         len_out=1, think_ms=0, tier=0))
    for k in range(300):
        rows.append(dict(user=1 + k % 3, t_ms=5 * k + 1, app=1, inter=0, stage=1, ncalls=1, len_in=100 + k,
                         len_sys=7, len_out=20, think_ms=0, tier=0))
    rows.sort(key=lambda r: r["t_ms"])
    for x, r in enumerate(rows):
        r["inter"] = x
    tr = from_columns(4, 2, rows)
    cfg = dict(tier_max=255)
    op = O.profile(tr, cfg)
    assert int(op["peak_t_u"][0]) >= 1 << 32
    _cmp_profile(F.build_app_profiles(ctx, F.Trace(tr), cfg).read(), op, 5)


def test_profile_many_apps(F, ctx):
    """A = 200 apps at J = 64: the Eq. 2 sums (200 x 65 x 4 u64) do not fit shared memory (global
    atomics), the histograms and the quantile tables run in app chunks; same profile as the oracle."""
    tr = G.generate(dict(G.CONFIGS["c2"], n_users=150, n_calls=30_000, seed=33))
    tr = dict(tr)
    A = 200
    app = (tr["inter"].astype(np.uint64) * np.uint64(2654435761) % np.uint64(A)).astype(np.uint32)
    tr["meta"] = (tr["meta"] & np.uint32(0xFFFFFF00)) | app
    tr["n_apps"] = A
    tr["app_names"] = [f"a{k}" for k in range(A)]
    cfg = dict(tier_max=255, max_stage=64)
    _cmp_profile(F.build_app_profiles(ctx, F.Trace(tr), cfg).read(), O.profile(tr, cfg), 5)


def test_profile_virtual_ranks(F, ctx):
    """The phased multi-GPU protocol with G virtual ranks on one GPU (SUM of the
    per-shard round payloads) finalises the unsharded profile bit for bit: sums, histograms,
    quantiles and the limits (radix-selected from digit histograms of the ranks' peaks)."""
    import ctypes as C
    import torch
    tr = G.generate(dict(G.CONFIGS["c2"], n_users=120, n_calls=40_000, seed=31))
    cfg = dict(tier_max=0)
    ref = O.profile(tr, cfg)
    for Gn in (2, 3):
        shards = [F.Trace(G.shard_by_user(tr, r, Gn)) for r in range(Gn)]
        keep = []
        c = F._profile_cfg(cfg, keep)
        parts, bufs = [], []
        for sh in shards:
            p = C.c_void_p()
            w = C.c_size_t(0)
            ctx._check(F.lib().fs_profile_local(ctx.h, F._a(sh.c), F._a(c), C.byref(p), C.byref(w)))
            parts.append(p)
            bufs.append(torch.zeros(w.value, dtype=torch.int64, device="cuda"))
        for _ in range(24):
            dones, ws = [], []
            for p, b in zip(parts, bufs):
                w = C.c_size_t(0)
                d = C.c_int(0)
                ctx._check(F.lib().fs_profile_round(p, C.c_void_p(b.data_ptr()), C.byref(w), C.byref(d)))
                dones.append(d.value)
                ws.append(w.value)
            assert len(set(dones)) == 1 and len(set(ws)) == 1
            if dones[0]:
                break
            tot = sum(b[: ws[0]] for b in bufs)
            for b in bufs:
                b[: ws[0]] = tot
        assert dones[0]
        with np.errstate(over="ignore"):
            owner = G.sm64(np.arange(tr["n_users"], dtype=np.uint64)) % np.uint64(Gn)
        for r, p in enumerate(parts):
            h = C.c_void_p()
            ctx._check(F.lib().fs_profile_finalize(p, C.byref(h)))
            _cmp_profile_shard(F.Profile(ctx, h).read(), ref, 5, owner == np.uint64(r))
            F.lib().fs_profile_partial_free(p)


def _shard_keep(tr, r, Gn):
    with np.errstate(over="ignore"):
        return np.nonzero(G.sm64(tr["user"].astype(np.uint64)) % np.uint64(Gn) == np.uint64(r))[0]


def test_act_user_sharded(F, ctx):
    """ACT shards by user with no exchange (windows are per user and per
    (user, app)) -- each user-hash shard throttled alone, with the replicated profile,
    gives exactly the unsharded statuses of its calls; overload always and replay-recorded."""
    tr = G.generate(dict(G.CONFIGS["c2"], n_users=150, n_calls=40_000, seed=41))
    gp = F.build_app_profiles(ctx, F.Trace(tr), dict(tier_max=0))
    act = dict(window_ms=60000, limits_from_profile=1)
    full, fs = F.act_throttle(ctx, F.Trace(tr), gp, act)
    full = full.cpu().numpy()
    assert fs["n_block"][0] + fs["n_block"][2] > 0
    eng = dict(G.CONFIGS["c2"]["engine"], mode=1, tier_max=255, act=act)
    o, _ = F.wsc_replay(ctx, F.Trace(tr), gp, eng)
    ovl, arr = o["ovl"].cpu().numpy(), o["arrive_ns"].cpu().numpy()
    full2, _ = F.act_throttle(ctx, F.Trace(tr), gp, act, overloaded=o["ovl"], t_ns_override=o["arrive_ns"])
    full2 = full2.cpu().numpy()
    import torch
    for Gn in (2, 4):
        tot = 0
        for r in range(Gn):
            keep = _shard_keep(tr, r, Gn)
            sh = F.Trace(G.shard_by_user(tr, r, Gn))
            st, ss = F.act_throttle(ctx, sh, gp, act)
            assert (st.cpu().numpy() == full[keep]).all()
            tot += ss["n_admit"]
            st2, _ = F.act_throttle(ctx, sh, gp, act, overloaded=torch.from_numpy(ovl[keep]).cuda(),
                                    t_ns_override=torch.from_numpy(arr[keep]).cuda())
            assert (st2.cpu().numpy() == full2[keep]).all()
        assert tot == fs["n_admit"]


# ------------------------------------------------------------------ ACT
@pytest.fixture(params=["1", "2", "1000"])
def jacobi(request, monkeypatch):
    """Jacobi passes before the sequential walk: walk-only, default, Jacobi-only."""
    monkeypatch.setenv("FS_ACT_JACOBI_MAX", request.param)
    return request.param


@pytest.mark.parametrize("seed", range(60))
def test_act_tiny(F, ctx, seed, jacobi):
    import torch
    rng = np.random.default_rng(5000 + seed)
    A = int(rng.integers(1, 3))
    tr = tiny_trace(rng, n_users=2, n_apps=A, max_inters=5, max_calls=9)
    J, cnt, si, ss, so = tiny_profile(rng, A)
    op = O.profile_from_host(A, J, cnt, si, ss, so)
    gp = F.profile_from_host(ctx, A, J, cnt, si, ss, so)
    n = tr["n_calls"]
    cfg = dict(window_ms=int(rng.choice((1, 2, 4))), limits_from_profile=0, T_req_g=int(rng.choice((0, 1, 2))),
               T_req_a=[int(rng.choice((0, 1, 2))) for _ in range(A)], T_tok_g=int(rng.choice((0, 8))),
               T_tok_a=[int(rng.choice((0, 6))) for _ in range(A)], count_mode=int(rng.integers(0, 2)),
               tier_max=int(rng.choice((0, 255))))
    ovl = (rng.random(n) < 0.7).astype(np.uint8) if rng.random() < 0.8 else None
    tov = None
    if rng.random() < 0.5:
        _, _, head_of, _ = O.validate(tr)
        tov = tr["t_ms"].astype(np.int64) * MS + rng.integers(0, 3, size=n) * MS
        for i in range(n):
            if int(head_of[i]) != i:
                tov[i] = max(tov[i], tov[int(head_of[i])] + 1)
        tov[rng.random(n) < 0.1] = -1
    est, esum = O.act(tr, op, cfg, overloaded=ovl, t_ns_override=tov)
    T = F.Trace(tr)
    st, s = F.act_throttle(ctx, T, gp, cfg,
                           overloaded=None if ovl is None else torch.tensor(ovl, device="cuda"),
                           t_ns_override=None if tov is None else torch.tensor(tov, device="cuda"))
    assert list(_np(st)) == list(est)
    for k in ("n_in", "n_admit", "n_block", "n_dropped", "n_filtered", "n_inter_blocked", "n_not_arrived"):
        assert s[k] == esum[k], k


@pytest.mark.parametrize("mode", ["always", "random", "heads_only", "replay"])
def test_act_c2_shape(F, ctx, mode, jacobi):
    import torch
    tr = G.generate(dict(G.CONFIGS["c2"], n_users=300, n_calls=200_000, seed=41))
    pcfg = dict(tier_max=0)
    op = O.profile(tr, pcfg)
    gp = F.build_app_profiles(ctx, F.Trace(tr), pcfg)
    cfg = dict(window_ms=60000, limits_from_profile=1, count_mode=1 if mode == "heads_only" else 0)
    n = tr["n_calls"]
    rng = np.random.default_rng(7)
    T = F.Trace(tr)
    ovl, tov = None, None
    if mode == "random":
        ovl = (rng.random(n) < 0.5).astype(np.uint8)
    if mode == "replay":
        eng = dict(G.CONFIGS["c2"]["engine"], mode=1, tier_max=255, act=cfg)
        eo, _ = O.replay(tr, op, eng)
        ovl, tov = eo["ovl"], eo["arrive_ns"]
    est, esum = O.act(tr, op, cfg, overloaded=ovl, t_ns_override=tov)
    st, s = F.act_throttle(ctx, T, gp, cfg, overloaded=None if ovl is None else torch.tensor(ovl, device="cuda"),
                           t_ns_override=None if tov is None else torch.tensor(tov, device="cuda"))
    g = _np(st)
    bad = np.nonzero(g != est)[0]
    assert len(bad) == 0, (bad[:10], g[bad[:10]], est[bad[:10]])
    assert s["n_block"] == esum["n_block"]


def dense_user_trace(rng, n_heads=1800, span_ms=20_000, n_apps=3):
    """One heavy user whose windows hold thousands of positions (the walk's global fallback beyond
    its 1024-position ring) plus a light user; 1-4 calls per interaction."""
    from paper_2411_15997_b200.tracegen import from_columns
    rows = []
    for x in range(n_heads):
        u = 0 if rng.random() < 0.9 else 1
        a = int(rng.integers(0, n_apps))
        m = int(rng.choice((1, 1, 2, 3, 4)))
        t0 = int(rng.integers(0, span_ms))
        for s in range(1, m + 1):
            if s > 1:
                t0 += int(rng.integers(0, 400))
            rows.append(dict(user=u, t_ms=t0, app=a, inter=x, stage=s, ncalls=m, len_in=int(rng.integers(1, 50)),
                             len_sys=int(rng.integers(0, 5)), len_out=int(rng.integers(1, 30)),
                             think_ms=int(rng.integers(0, 50)), tier=0))
    rows.sort(key=lambda r: (r["t_ms"], r["inter"], r["stage"]))
    ren = {}
    for r in rows:
        if r["stage"] == 1:
            ren.setdefault(r["inter"], len(ren))
    for r in rows:
        r["inter"] = ren[r["inter"]]
    return from_columns(2, n_apps, rows)


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("jmax", ["1", "2"])
def test_act_walk_long_windows(F, ctx, monkeypatch, seed, jmax):
    """ACT on a user whose windows span more positions than the walk's shared-memory ring (its global
    prefix copies), with limits near the windows' counts so decisions chain through continuations."""
    import torch
    monkeypatch.setenv("FS_ACT_JACOBI_MAX", jmax)
    rng = np.random.default_rng(9100 + seed)
    A = 3
    tr = dense_user_trace(rng, n_apps=A)
    J, cnt, si, ss, so = tiny_profile(rng, A)
    op = O.profile_from_host(A, J, cnt, si, ss, so)
    gp = F.profile_from_host(ctx, A, J, cnt, si, ss, so)
    n = tr["n_calls"]
    W = 15_000
    cfg = dict(window_ms=W, limits_from_profile=0, T_req_g=int(rng.integers(900, 1400)) if seed < 2 else 0,
               T_req_a=[int(rng.integers(300, 500)) for _ in range(A)], T_tok_g=int(rng.integers(40_000, 60_000)),
               T_tok_a=[int(rng.integers(12_000, 20_000)) for _ in range(A)], count_mode=0, tier_max=255)
    ovl = None if seed % 2 == 0 else (rng.random(n) < 0.8).astype(np.uint8)
    est, esum = O.act(tr, op, cfg, overloaded=ovl)
    st, s = F.act_throttle(ctx, F.Trace(tr), gp, cfg, overloaded=None if ovl is None else torch.tensor(ovl, device="cuda"))
    g = _np(st)
    bad = np.nonzero(g != est)[0]
    assert len(bad) == 0, (bad[:10], g[bad[:10]], est[bad[:10]])
    assert s["n_block"] == esum["n_block"] and sum(esum["n_block"]) > 0
    if jmax == "1":
        assert s["n_fixup_users"] >= 1


# ------------------------------------------------------------------ replay
@pytest.mark.parametrize("seed", range(150))
def test_replay_tiny(F, ctx, seed):
    rng = np.random.default_rng(1000 + seed)
    A = int(rng.integers(1, 3))
    tr = tiny_trace(rng, n_users=int(rng.integers(1, 4)), n_apps=A)
    J, cnt, si, ss, so = tiny_profile(rng, A)
    op = O.profile_from_host(A, J, cnt, si, ss, so)
    gp = F.profile_from_host(ctx, A, J, cnt, si, ss, so)
    cmp_replay(F, ctx, tr, gp, op, tiny_replay_cfg(rng, A), f"tiny{seed}")


@pytest.mark.parametrize("seed", range(1, 6))
@pytest.mark.parametrize("mode", [0, 1])
def test_replay_c1(F, ctx, seed, mode):
    tr = G.generate("c1", seed=seed)
    c = G.CONFIGS["c1"]
    op = O.profile(tr, dict(tier_max=255))
    gp = F.build_app_profiles(ctx, F.Trace(tr), dict(tier_max=255))
    cfg = dict(c["engine"], mode=mode, tier_max=255,
               act=dict(window_ms=60000, limits_from_profile=0, T_req_g=8, T_req_a=[5, 5]))
    cmp_replay(F, ctx, tr, gp, op, cfg, f"c1-{seed}-{mode}")


@pytest.mark.parametrize("variant", ["wi", "w", "t0", "heads", "tok"])
def test_replay_c2_shape(F, ctx, variant):
    tr = G.generate(dict(G.CONFIGS["c2"], n_users=200, n_calls=100_000, seed=51))
    pcfg = dict(tier_max=0)
    op = O.profile(tr, pcfg)
    gp = F.build_app_profiles(ctx, F.Trace(tr), pcfg)
    act = dict(window_ms=60000, limits_from_profile=1)
    cfg = dict(G.CONFIGS["c2"]["engine"], mode=1, tier_max=255, act=act)
    if variant == "w":
        cfg["mode"] = 0
    if variant == "t0":
        cfg["tier_max"] = 0
    if variant == "heads":
        act["count_mode"] = 1
    if variant == "tok":
        act["limit_mult_q8"] = 200
        cfg["prio_abusive_q16"] = 2 * 65536
        cfg["alpha"], cfg["beta"], cfg["gamma"] = 1, 1, 2
    cmp_replay(F, ctx, tr, gp, op, cfg, variant)


# ------------------------------------------------------------------ step
@pytest.mark.parametrize("seed", range(40))
def test_step_vs_oracle(F, ctx, seed):
    rng = np.random.default_rng(9000 + seed)
    A = 2
    tr = tiny_trace(rng, n_users=3, n_apps=A, max_inters=6, max_calls=12, thinks=(0,))
    J, cnt, si, ss, so = tiny_profile(rng, A)
    op = O.profile_from_host(A, J, cnt, si, ss, so)
    gp = F.profile_from_host(ctx, A, J, cnt, si, ss, so)
    cfg = tiny_replay_cfg(rng, A)
    cfg["kv_capacity"] = 100
    cfg["tier_max"] = 255
    so_ = O.Step(tr, op, cfg)
    sg = F.WscState(ctx, F.Trace(tr), gp, cfg)
    n = tr["n_calls"]
    pos = 0
    admitted = []
    for it in range(12):
        k = int(rng.integers(0, 4))
        arr = list(range(pos, min(n, pos + k)))
        pos += len(arr)
        t = [it * MS] * len(arr)
        fin = [admitted.pop(0) for _ in range(min(len(admitted), int(rng.integers(0, 3))))]
        occ = int(rng.integers(0, 100))
        nb = int(rng.integers(0, 3))
        s1, a1 = so_.step(it * MS, occ, nb, fin, arr, t)
        s2, a2 = sg.step(it * MS, occ, nb, fin, arr, t)
        assert list(s1) == list(s2)
        assert list(a1) == list(a2)
        admitted += list(a1)
        u1, e1 = so_.read()
        u2, e2 = sg.read()
        assert (u1 == u2).all() and e1 == e2


# ------------------------------------------------------------------ sweep
@pytest.mark.parametrize("kern", ["solo", "regular", "regular-generic"])
def test_sweep_small(F, ctx, monkeypatch, kern):
    """Small grids run on the solo-slot kernel (<= 16 scenarios per SM); the regular 16-per-SM kernel,
    with and without the FS(W+I)-only instantiation, is forced here."""
    if kern != "solo":
        monkeypatch.setenv("FS_SWEEP_SOLO", "0")
    if kern == "regular-generic":
        monkeypatch.setenv("FS_SWEEP_FWI", "0")
    tr = G.generate(dict(G.CONFIGS["c2"], n_users=100, n_calls=20_000, seed=61))
    op = O.profile(tr, dict(tier_max=0))
    gp = F.build_app_profiles(ctx, F.Trace(tr), dict(tier_max=0))
    base = dict(G.CONFIGS["c2"]["engine"], mode=1, act=dict(window_ms=60000, limits_from_profile=1))
    scen = []
    for k, w, tm in [(0, (1, 2, 1), 15), (128, (1, 1, 2), 15), (512, (2, 1, 1), 3), (UMAX, (1, 2, 1), 15),
                     (256, (1, 2, 1), 0), (384, (4, 1, 1), 7), (64, (1, 1, 4), 15), (1024, (1, 0, 1), 15)]:
        s = dict(base, alpha=w[0], beta=w[1], gamma=w[2], tier_max=tm, prio_abusive_q16=131072 if tm == 7 else 65536)
        s["act"] = dict(base["act"], limit_mult_q8=k)
        scen.append(s)
    scen.append(dict(scen[0], mode=0))
    es, ecodes = O.sweep(tr, op, scen)
    gs, gcodes = F.sweep(ctx, F.Trace(tr), gp, scen)
    assert list(gcodes) == list(ecodes)
    for a, b in zip(gs, es):
        assert a == b


def test_sweep_capacity_retry(F, ctx, monkeypatch):
    """Scenarios whose state outgrows the sweep's first capacities (a 512-entry ACT ring per user,
    a 65 536-entry RPM window log) run again with exact capacities: same summaries as the oracle,
    no FS_E_NOMEM.  Five users share 70 000 calls and the windows span the whole day."""
    tr = G.generate(dict(G.CONFIGS["c2"], n_users=5, n_calls=70_000, seed=62))
    op = O.profile(tr, dict(tier_max=255))
    gp = F.build_app_profiles(ctx, F.Trace(tr), dict(tier_max=255))
    A = tr["n_apps"]
    day = 86_400_000
    base = dict(G.CONFIGS["c2"]["engine"], tier_max=255)
    scen = [dict(base, mode=1, act=dict(window_ms=day, limits_from_profile=0, T_req_g=1 << 30, T_req_a=[1 << 30] * A)),
            dict(base, mode=1, overload_permille=0,
                 act=dict(window_ms=day, limits_from_profile=0, T_req_g=3000, T_req_a=[2000] * A)),
            dict(base, mode=0),
            dict(base, mode=3, act=dict(window_ms=day, limits_from_profile=0, T_req_g=1 << 30, T_req_a=[1 << 30] * A))]
    es, ecodes = O.sweep(tr, op, scen)
    assert list(ecodes) == [0] * len(scen)
    for solo in ("1", "0"):                  # the solo-slot and the regular kernel's retries
        monkeypatch.setenv("FS_SWEEP_SOLO", solo)
        for sub in (scen[:3], scen):        # FairServe modes only, then with RPM
            gs, gcodes = F.sweep(ctx, F.Trace(tr), gp, sub)
            assert list(gcodes) == [0] * len(sub)
            for a, b in zip(gs, es):
                assert a == b


# ------------------------------------------------------------------ errors
def test_error_parity(F, ctx):
    tr = G.generate("c1")
    T = lambda d: F.Trace(d)
    bad = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in tr.items()}
    bad["user"][17] = 99
    with pytest.raises(F.FsError) as ei:
        F.build_app_profiles(ctx, T(bad), {})
    assert ei.value.code == -2 and ei.value.bad_index == 17
    bad = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in tr.items()}
    bad["t_ms"][50] = 0
    code, idx = O.validate(bad)[:2]
    with pytest.raises(F.FsError) as ei:
        F.build_app_profiles(ctx, T(bad), {})
    assert ei.value.code == code and ei.value.bad_index == idx
    # oversize
    op = O.profile(tr, {})
    gp = F.build_app_profiles(ctx, T(tr), {})
    cfg = dict(G.CONFIGS["c1"]["engine"], mode=0, kv_capacity=3000)
    with pytest.raises(O.OracleError) as e1:
        O.replay(tr, op, cfg)
    with pytest.raises(F.FsError) as e2:
        F.wsc_replay(ctx, T(tr), gp, cfg)
    assert (e2.value.code, e2.value.bad_index) == (e1.value.code, e1.value.bad_index)


# ------------------------------------------------------------------ NEXT-1 baselines (VTC, RPM, FCFS)
@pytest.mark.parametrize("seed", range(120))
def test_replay_tiny_baselines(F, ctx, seed):
    rng = np.random.default_rng(9000 + seed)
    A = int(rng.integers(1, 3))
    tr = tiny_trace(rng, n_users=int(rng.integers(1, 4)), n_apps=A)
    J, cnt, si, ss, so = tiny_profile(rng, A)
    op = O.profile_from_host(A, J, cnt, si, ss, so)
    gp = F.profile_from_host(ctx, A, J, cnt, si, ss, so)
    cmp_replay(F, ctx, tr, gp, op, tiny_replay_cfg(rng, A, modes=(2, 3, 4)), f"base{seed}")


@pytest.mark.parametrize("mode", [2, 3, 4])
def test_replay_c2_shape_baselines(F, ctx, mode):
    """C2-shaped 100k-call trace: VTC (weights 1, 1, 2), RPM (user and app request limits), FCFS."""
    tr = G.generate(dict(G.CONFIGS["c2"], n_users=200, n_calls=100_000, seed=51))
    pcfg = dict(tier_max=0)
    op = O.profile(tr, pcfg)
    gp = F.build_app_profiles(ctx, F.Trace(tr), pcfg)
    cfg = dict(G.CONFIGS["c2"]["engine"], mode=mode, tier_max=255, alpha=1, beta=1, gamma=2,
               act=dict(window_ms=60000, limits_from_profile=0, T_req_g=6,
                        T_req_a=[40] * tr["n_apps"]))
    cmp_replay(F, ctx, tr, gp, op, cfg, f"c2base{mode}")


def test_sweep_baselines(F, ctx):
    """One sweep mixing FS(W+I), FS(W), VTC, RPM and FCFS scenarios over tier mixes."""
    tr = G.generate(dict(G.CONFIGS["c2"], n_users=100, n_calls=20_000, seed=61))
    op = O.profile(tr, dict(tier_max=0))
    gp = F.build_app_profiles(ctx, F.Trace(tr), dict(tier_max=0))
    base = dict(G.CONFIGS["c2"]["engine"], act=dict(window_ms=60000, limits_from_profile=0, T_req_g=4,
                                                   T_req_a=[30] * tr["n_apps"]))
    scen = []
    for mode, tm in [(2, 15), (3, 15), (4, 15), (2, 0), (3, 3), (4, 7), (0, 15)]:
        scen.append(dict(base, mode=mode, tier_max=tm, alpha=1, beta=1, gamma=2))
    scen.append(dict(base, mode=1, act=dict(window_ms=60000, limits_from_profile=1)))
    es, ecodes = O.sweep(tr, op, scen)
    gs, gcodes = F.sweep(ctx, F.Trace(tr), gp, scen)
    assert list(gcodes) == list(ecodes)
    for a, b in zip(gs, es):
        assert a == b


def test_rpm_profile_limits_rejected(F, ctx):
    """R8: RPM takes explicit limits; profile-derived ones are FS_E_INVAL on both sides, and the
    online step rejects RPM."""
    tr = G.generate("c1")
    op = O.profile(tr, dict(tier_max=255))
    gp = F.build_app_profiles(ctx, F.Trace(tr), dict(tier_max=255))
    cfg = dict(G.CONFIGS["c1"]["engine"], mode=3, act=dict(window_ms=60000, limits_from_profile=1))
    with pytest.raises(O.OracleError) as eo:
        O.replay(tr, op, cfg)
    with pytest.raises(F.FsError) as eg:
        F.wsc_replay(ctx, F.Trace(tr), gp, cfg)
    assert eo.value.code == eg.value.code == -1
    cfg["act"] = dict(window_ms=60000, limits_from_profile=0, T_req_g=3)
    with pytest.raises(F.FsError) as eg:
        F.WscState(ctx, F.Trace(tr), gp, cfg)
    assert eg.value.code == -1


# ------------------------------------------------------------------ NEXT-2 metric suite
def _cmp_metrics(F, ctx, tr, gout, eout, thr, name):
    from oracle import metrics as M
    g, per = F.replay_metrics(ctx, F.Trace(tr), gout, thr)
    eg, eper = M.replay_metrics(tr, eout, thr)
    for a, b in [(g, eg)] + list(zip(per, eper)):
        for k in M.FIELDS:
            if k == "jain":
                assert a[k] == pytest.approx(b[k], rel=1e-12, abs=0), (name, k)
            else:
                assert a[k] == b[k], (name, k, a[k], b[k])


@pytest.mark.parametrize("mode", [0, 1, 2, 3, 4])
def test_metrics_c2_shape(F, ctx, mode):
    """fs_replay_metrics vs oracle/metrics.py on the outputs of each policy's replay."""
    tr = G.generate(dict(G.CONFIGS["c2"], n_users=200, n_calls=30_000, seed=83))
    pcfg = dict(tier_max=255)
    op = O.profile(tr, pcfg)
    gp = F.build_app_profiles(ctx, F.Trace(tr), pcfg)
    act = dict(window_ms=60000, limits_from_profile=1) if mode == 1 else \
        dict(window_ms=60000, limits_from_profile=0, T_req_g=4, T_req_a=[30] * tr["n_apps"])
    cfg = dict(G.CONFIGS["c2"]["engine"], mode=mode, tier_max=255, act=act)
    go, _ = F.wsc_replay(ctx, F.Trace(tr), gp, cfg)
    eo, _ = O.replay(tr, op, cfg)
    for thr in (0, 5_000_000, 10**12):
        _cmp_metrics(F, ctx, tr, go, eo, thr, f"m{mode}-{thr}")


@pytest.mark.parametrize("seed", range(20))
def test_metrics_tiny(F, ctx, seed):
    rng = np.random.default_rng(4400 + seed)
    A = int(rng.integers(1, 3))
    tr = tiny_trace(rng, n_users=3, n_apps=A)
    J, cnt, si, ss, so = tiny_profile(rng, A)
    op = O.profile_from_host(A, J, cnt, si, ss, so)
    gp = F.profile_from_host(ctx, A, J, cnt, si, ss, so)
    cfg = tiny_replay_cfg(rng, A, modes=(0, 1, 2, 3, 4))
    try:
        eo, _ = O.replay(tr, op, cfg)
    except O.OracleError:
        return
    go, _ = F.wsc_replay(ctx, F.Trace(tr), gp, cfg)
    _cmp_metrics(F, ctx, tr, go, eo, int(rng.choice((0, 1_000_000, 10**9))), f"tiny{seed}")


# ------------------------------------------------------------------ NEXT-3 app-global counters
@pytest.mark.parametrize("seed", range(60))
def test_act_tiny_app_global(F, ctx, seed):
    import torch
    rng = np.random.default_rng(15000 + seed)
    A = int(rng.integers(1, 3))
    tr = tiny_trace(rng, n_users=3, n_apps=A, max_inters=5, max_calls=9)
    J, cnt, si, ss, so = tiny_profile(rng, A)
    op = O.profile_from_host(A, J, cnt, si, ss, so)
    gp = F.profile_from_host(ctx, A, J, cnt, si, ss, so)
    n = tr["n_calls"]
    cfg = dict(window_ms=int(rng.choice((1, 2, 4))), limits_from_profile=0, T_req_g=int(rng.choice((0, 2, 3))),
               T_req_a=[int(rng.choice((0, 1, 2, 3))) for _ in range(A)], T_tok_g=int(rng.choice((0, 12))),
               T_tok_a=[int(rng.choice((0, 9))) for _ in range(A)], count_mode=int(rng.integers(0, 2)),
               tier_max=int(rng.choice((0, 255))), app_scope=1)
    ovl = (rng.random(n) < 0.7).astype(np.uint8) if rng.random() < 0.8 else None
    est, esum = O.act(tr, op, cfg, overloaded=ovl)
    st, s = F.act_throttle(ctx, F.Trace(tr), gp, cfg,
                           overloaded=None if ovl is None else torch.tensor(ovl, device="cuda"))
    assert list(_np(st)) == list(est)
    assert s["n_block"] == esum["n_block"]


def test_act_c2_shape_app_global(F, ctx):
    tr = G.generate(dict(G.CONFIGS["c2"], n_users=300, n_calls=200_000, seed=41))
    op = O.profile(tr, dict(tier_max=0))
    gp = F.build_app_profiles(ctx, F.Trace(tr), dict(tier_max=0))
    cfg = dict(window_ms=60000, limits_from_profile=0, T_req_g=12, T_req_a=[60] * tr["n_apps"],
               T_tok_g=0, T_tok_a=[200000] * tr["n_apps"], app_scope=1)
    est, esum = O.act(tr, op, cfg)
    st, s = F.act_throttle(ctx, F.Trace(tr), gp, cfg)
    g = _np(st)
    bad = np.nonzero(g != est)[0]
    assert len(bad) == 0, (bad[:10], g[bad[:10]], est[bad[:10]])
    assert s["n_block"] == esum["n_block"] and sum(esum["n_block"]) > 0


@pytest.mark.parametrize("seed", range(60))
def test_replay_tiny_app_global(F, ctx, seed):
    rng = np.random.default_rng(16000 + seed)
    A = int(rng.integers(1, 3))
    tr = tiny_trace(rng, n_users=int(rng.integers(2, 4)), n_apps=A)
    J, cnt, si, ss, so = tiny_profile(rng, A)
    op = O.profile_from_host(A, J, cnt, si, ss, so)
    gp = F.profile_from_host(ctx, A, J, cnt, si, ss, so)
    cfg = tiny_replay_cfg(rng, A, modes=(1,))
    cfg["act"]["app_scope"] = 1
    cmp_replay(F, ctx, tr, gp, op, cfg, f"ag{seed}")


def test_sweep_app_global(F, ctx):
    tr = G.generate(dict(G.CONFIGS["c2"], n_users=100, n_calls=20_000, seed=61))
    op = O.profile(tr, dict(tier_max=0))
    gp = F.build_app_profiles(ctx, F.Trace(tr), dict(tier_max=0))
    base = dict(G.CONFIGS["c2"]["engine"], mode=1)
    scen = []
    for tm, lim, cm in [(15, 20, 0), (0, 10, 0), (7, 30, 1), (15, 5, 1)]:
        scen.append(dict(base, tier_max=tm, overload_permille=0, act=dict(window_ms=60000, limits_from_profile=0, T_req_g=8,
                                                     T_req_a=[lim] * tr["n_apps"], count_mode=cm, app_scope=1)))
    scen.append(dict(base, act=dict(window_ms=60000, limits_from_profile=1)))
    es, ecodes = O.sweep(tr, op, scen)
    gs, gcodes = F.sweep(ctx, F.Trace(tr), gp, scen)
    assert list(gcodes) == list(ecodes)
    for a, b in zip(gs, es):
        assert a == b
    assert sum(es[0]["n_block"]) > 0


# ------------------------------------------------------------------ NEXT-3 weighted token load (R11)
@pytest.mark.parametrize("seed", range(40))
def test_act_tiny_tau_weighted(F, ctx, seed):
    import torch
    rng = np.random.default_rng(17000 + seed)
    A = int(rng.integers(1, 3))
    tr = tiny_trace(rng, n_users=2, n_apps=A, max_inters=5, max_calls=9)
    J, cnt, si, ss, so = tiny_profile(rng, A)
    op = O.profile_from_host(A, J, cnt, si, ss, so)
    gp = F.profile_from_host(ctx, A, J, cnt, si, ss, so)
    n = tr["n_calls"]
    cfg = dict(window_ms=int(rng.choice((1, 2, 4))), limits_from_profile=0, T_req_g=int(rng.choice((0, 2))),
               T_req_a=[int(rng.choice((0, 2))) for _ in range(A)], T_tok_g=int(rng.choice((0, 8, 20))),
               T_tok_a=[int(rng.choice((0, 6, 15))) for _ in range(A)], count_mode=int(rng.integers(0, 2)),
               tier_max=255, app_scope=int(rng.integers(0, 2)),
               tau_weights=tuple(int(x) for x in rng.integers(0, 4, size=3)))
    ovl = (rng.random(n) < 0.7).astype(np.uint8)
    est, _ = O.act(tr, op, cfg, overloaded=ovl)
    st, _ = F.act_throttle(ctx, F.Trace(tr), gp, cfg, overloaded=torch.tensor(ovl, device="cuda"))
    assert list(_np(st)) == list(est)


@pytest.mark.parametrize("seed", range(40))
def test_replay_tiny_tau_weighted(F, ctx, seed):
    rng = np.random.default_rng(18000 + seed)
    A = int(rng.integers(1, 3))
    tr = tiny_trace(rng, n_users=int(rng.integers(1, 4)), n_apps=A)
    J, cnt, si, ss, so = tiny_profile(rng, A)
    op = O.profile_from_host(A, J, cnt, si, ss, so)
    gp = F.profile_from_host(ctx, A, J, cnt, si, ss, so)
    cfg = tiny_replay_cfg(rng, A, modes=(1,))
    cfg["act"]["tau_weights"] = tuple(int(x) for x in rng.integers(0, 4, size=3))
    cfg["act"]["app_scope"] = int(rng.integers(0, 2))
    cmp_replay(F, ctx, tr, gp, op, cfg, f"tw{seed}")


def test_profile_and_sweep_tau_weighted(F, ctx):
    """Weighted token peaks in the profile (and the limits derived from them), and a sweep whose
    FS(W+I) scenarios share one weight set."""
    tr = G.generate(dict(G.CONFIGS["c2"], n_users=100, n_calls=20_000, seed=61))
    pcfg = dict(tier_max=0, tau_weights=(2, 1, 3))
    op = O.profile(tr, pcfg)
    gpp = F.build_app_profiles(ctx, F.Trace(tr), pcfg)
    gpr = gpp.read()
    for k in ("peak_t_u", "peak_t_ua", "T_tok_a", "T_tok_g", "peak_r_u", "T_req_a"):
        assert (gpr[k] == op[k]).all(), k
    base = dict(G.CONFIGS["c2"]["engine"], mode=1, overload_permille=0)
    scen = [dict(base, tier_max=tm, act=dict(window_ms=60000, limits_from_profile=1, tau_weights=(2, 1, 3)))
            for tm in (15, 0, 7)]
    scen.append(dict(base, mode=0))
    es, ecodes = O.sweep(tr, op, scen)
    gs, gcodes = F.sweep(ctx, F.Trace(tr), gpp, scen)
    assert list(gcodes) == list(ecodes)
    for a, b in zip(gs, es):
        assert a == b
    assert sum(es[0]["n_block"]) > 0
