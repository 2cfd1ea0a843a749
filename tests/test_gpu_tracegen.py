"""fs_generate_trace (NEXT-4 device trace generator): valid traces (the oracle's validator),
the same workload shape as tracegen.py (the CPU generator), and parity of the hot path on a
device-generated trace against the oracle on its host copy."""
import numpy as np
import pytest

import oracle as O
from paper_2411_15997_b200 import tracegen as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    from paper_2411_15997_b200 import build
    build.build()
    from paper_2411_15997_b200 import fairserve as F
    return F


@pytest.fixture(scope="module")
def ctx(F):
    return F.Context(0)


def _host(T):
    tr = {k: T.t[k].cpu().numpy().view(np.uint32) for k in G.FIELDS}
    tr.update(n_calls=T.n, n_users=T.U, n_apps=T.A, n_inters=T.X)
    return tr


def _stats(tr):
    meta = tr["meta"]
    app, stage, m, tier = meta & 255, (meta >> 8) & 255, (meta >> 16) & 255, meta >> 24
    heads = stage == 1
    A = int(tr["n_apps"])
    return dict(
        head_frac=heads.mean(), mean_m=m[heads].mean(), abusive_frac=(tier > 0).mean(),
        app_frac=np.bincount(app, minlength=A) / len(app),
        mean_in=np.array([tr["len_in"][app == a].mean() for a in range(A)]),
        mean_out=np.array([tr["len_out"][app == a].mean() for a in range(A)]),
        mean_think=tr["think_ms"].mean(), t_max=int(tr["t_ms"].max()))


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_generated_trace_is_valid_and_shaped(F, ctx, cfg):
    n = 200 if cfg == "c1" else 1_000_000
    T = F.generate_trace(ctx, cfg, n_calls=n, seed=7)
    tr = _host(T)
    assert tr["n_calls"] == n
    rc, bad, head_of, next_call = O.validate(tr)
    assert rc == 0, (rc, bad)
    assert (np.diff(tr["t_ms"].astype(np.int64)) >= 0).all()
    heads = ((tr["meta"] >> 8) & 255) == 1
    assert (tr["inter"][heads] == np.arange(int(heads.sum()))).all()       # dense ids in head order
    assert T.X == int(heads.sum())
    if cfg == "c1":
        return
    ref = _stats(G.generate(cfg))
    got = _stats(tr)
    assert abs(got["head_frac"] - ref["head_frac"]) < 0.01
    assert abs(got["mean_m"] - ref["mean_m"]) / ref["mean_m"] < 0.03
    # abusive users: 5 % of users with 20x rates carry about half of the calls (heavy-tailed weights)
    assert 0.25 < got["abusive_frac"] < 0.75 and 0.25 < ref["abusive_frac"] < 0.75
    assert np.allclose(got["mean_in"], ref["mean_in"], rtol=0.06)
    assert np.allclose(got["mean_out"], ref["mean_out"], rtol=0.06)
    assert abs(got["mean_think"] - ref["mean_think"]) / ref["mean_think"] < 0.03
    assert got["app_frac"].argmax() == ref["app_frac"].argmax()


def test_hot_path_on_generated_trace(F, ctx):
    """A device-generated trace through the profile and an FS(W+I) replay, against the oracle
    on its host copy (bit-exact tables and digest)."""
    T = F.generate_trace(ctx, "c2", n_calls=100_000, seed=11)
    tr = _host(T)
    pcfg = dict(tier_max=255)
    gp = F.build_app_profiles(ctx, T, pcfg)
    op = O.profile(tr, pcfg)
    g = gp.read()
    for k in ("cnt", "sum_in", "sum_out", "hist", "nr_q", "peak_r_u", "peak_t_ua", "T_req_a", "T_tok_g"):
        assert (g[k] == op[k]).all(), k
    eng = dict(G.CONFIGS["c2"]["engine"], mode=1, tier_max=255, act=dict(window_ms=60000, limits_from_profile=1))
    _, s = F.wsc_replay(ctx, T, gp, eng, outputs=False)
    _, es = O.replay(tr, op, eng, outputs=False)
    assert s["digest"] == es["digest"] and s["n_admitted"] == es["n_admitted"]


def test_generate_large(F, ctx):
    """10^8 calls (C4 size) on the device: the sort order and the chain structure hold."""
    import torch
    T = F.generate_trace(ctx, "c4", seed=4)
    t = T.t["t_ms"]
    assert T.n == 100_000_000
    assert bool((t[1:] >= t[:-1]).all())
    heads = ((T.t["meta"] >> 8) & 255) == 1
    assert int(heads.sum()) == T.X
