"""Oracle profile (O2) pinned to numpy library routines:
integer sums, np.percentile 'inverted_cdf' (nearest rank) and 'linear',
bin edges of the log-linear histogram, window counts via np.searchsorted."""
import numpy as np
import pytest

import oracle as O
from paper_2411_15997_b200 import tracegen as G

Q = [500000, 900000, 950000, 990000, 999000]


def _lower_edge(b):
    return b if b < 8 else (8 + b % 8) << (b // 8 - 1)


def _traces():
    yield G.generate("c1")
    cfg = dict(G.CONFIGS["c2"], n_users=60, n_calls=20000, seed=7)
    yield G.generate(cfg)
    cfg = dict(G.CONFIGS["c3"], n_users=40, n_calls=8000, seed=11)
    yield G.generate(cfg)


@pytest.mark.parametrize("k", range(3))
@pytest.mark.parametrize("tier_max", [0, 255])
@pytest.mark.parametrize("count_mode", [0, 1])
def test_profile_vs_numpy(k, tier_max, count_mode):
    tr = list(_traces())[k]
    J = 8
    W = 60000
    p = O.profile(tr, dict(max_stage=J, tier_max=tier_max, q_ppm=Q, window_ms=W, count_mode=count_mode,
                           limit_q_ppm=990000, limit_mult_q8=384))
    A, U = tr["n_apps"], tr["n_users"]
    meta = tr["meta"].astype(np.int64)
    app, stage, nc, tier = meta & 255, (meta >> 8) & 255, (meta >> 16) & 255, meta >> 24
    keep = tier <= tier_max
    j = np.minimum(stage, J)
    for name, col in (("cnt", np.ones(len(meta), np.int64)), ("sum_in", tr["len_in"]),
                      ("sum_sys", tr["len_sys"]), ("sum_out", tr["len_out"])):
        ref = np.zeros((A, J + 1), np.int64)
        np.add.at(ref, (app[keep], j[keep]), col.astype(np.int64)[keep])
        assert (p[name].astype(np.int64) == ref).all(), name
    vals = [tr["len_in"], tr["len_sys"], tr["len_out"],
            tr["len_in"].astype(np.int64) + tr["len_sys"] + tr["len_out"]]
    edges = np.array([_lower_edge(b) for b in range(240)] + [2**32], dtype=np.float64)
    for a in range(A):
        m = keep & (app == a)
        for f in range(4):
            v = np.sort(vals[f][m].astype(np.int64))
            h, _ = np.histogram(v, bins=edges)
            assert (p["hist"][a, f].astype(np.int64) == h).all()
            for qi, q in enumerate(Q):
                if len(v) == 0:
                    assert p["nr_q"][a, f, qi] == 0
                    continue
                assert int(p["nr_q"][a, f, qi]) == int(np.percentile(v, q / 1e6 * 100, method="inverted_cdf"))
                assert float(p["interp_q"][a, f, qi]) == pytest.approx(
                    float(np.percentile(v, q / 1e6 * 100, method="linear")), rel=1e-9)
        hm, _ = np.histogram(nc[m & (stage == 1)], bins=edges)
        assert (p["hist"][a, 4].astype(np.int64) == hm).all()
    # window peaks via searchsorted on per-user (t, id)-ordered times
    ohat = p["ohat"].astype(np.int64)
    tau = tr["len_in"].astype(np.int64) + tr["len_sys"] + ohat[app, j]
    cnt_ok = keep & ((stage == 1) if count_mode == 1 else True)
    t = tr["t_ms"].astype(np.int64)
    pr_u, pt_u = np.zeros(U, np.int64), np.zeros(U, np.int64)
    pr_ua, pt_ua = np.zeros((U, A), np.int64), np.zeros((U, A), np.int64)
    seen_u, seen_ua = np.zeros(U, bool), np.zeros((U, A), bool)
    for u in range(U):
        for a in [None] + list(range(A)):
            sel = np.nonzero(cnt_ok & (tr["user"] == u) & (True if a is None else app == a))[0]
            if len(sel) == 0:
                continue
            tt = t[sel]
            cs = np.concatenate([[0], np.cumsum(tau[sel])])
            lo = np.searchsorted(tt, tt - W, side="right")
            n = np.arange(len(sel)) - lo + 1
            tok = cs[1:] - cs[lo]
            if a is None:
                pr_u[u], pt_u[u], seen_u[u] = n.max(), tok.max(), True
            else:
                pr_ua[u, a], pt_ua[u, a], seen_ua[u, a] = n.max(), tok.max(), True
    assert (p["peak_r_u"] == pr_u).all() and (p["peak_t_u"] == pt_u).all()
    assert (p["peak_r_ua"] == pr_ua).all() and (p["peak_t_ua"] == pt_ua).all()

    def nr(x):
        return int(np.percentile(np.sort(x), 99.0, method="inverted_cdf")) if len(x) else 0

    def lim(v):
        return 0 if v == 0 else max(1, -(-384 * v // 256))

    assert int(p["nr_peak_r_g"][0]) == nr(pr_u[seen_u]) and int(p["T_req_g"][0]) == lim(nr(pr_u[seen_u]))
    assert int(p["nr_peak_t_g"][0]) == nr(pt_u[seen_u]) and int(p["T_tok_g"][0]) == lim(nr(pt_u[seen_u]))
    for a in range(A):
        assert int(p["T_req_a"][a]) == lim(nr(pr_ua[seen_ua[:, a], a]))
        assert int(p["T_tok_a"][a]) == lim(nr(pt_ua[seen_ua[:, a], a]))


def test_validation_errors():
    tr = G.generate("c1")
    assert O.validate(tr)[0] == 0
    bad = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in tr.items()}
    bad["user"][17] = 99
    assert O.validate(bad)[:2] == (-2, 17)
    bad = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in tr.items()}
    bad["t_ms"][50] = 0
    code, idx = O.validate(bad)[:2]
    assert code == -3 and idx <= 50
    bad = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in tr.items()}
    heads = np.nonzero(((bad["meta"] >> 8) & 255) == 1)[0]
    multi = [h for h in heads if ((bad["meta"][h] >> 16) & 255) > 1]
    h = multi[0]
    bad["meta"][h] = (bad["meta"][h] & ~np.uint32(255 << 8)) | np.uint32(2 << 8)   # head relabelled stage 2
    assert O.validate(bad)[0] == -3


def test_reachable_histogram_bins():
    """The CUDA stream pass keeps only the bins a validated field can reach (profile.cuh
    hb_off: 176 per length field, 192 for L_I + L_S + L_O, 48 for m): lengths < 2^24 (FS_E_RANGE
    beyond), their sum < 3 * 2^24, m <= 255 (8-bit field).  Pinned against the
    oracle's log-linear binning (monotone in the value, so the largest value gives the largest bin)."""
    assert O.bin_of(2**24 - 1) == 175
    assert O.bin_of(3 * (2**24 - 1)) <= 191
    assert O.bin_of(255) == 47
    vals = [0, 1, 7, 8, 9, 15, 16, 255, 256, 2**20, 2**24 - 1]
    assert [O.bin_of(v) for v in vals] == sorted(O.bin_of(v) for v in vals)
