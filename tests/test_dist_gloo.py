"""Multi-process (gloo, world_size 2, CPU) tests of the multi-GPU host logic.

1. The user-hash-sharded profile protocol's decomposition: per-shard
   integer sums and histograms SUM-all-reduce to the unsharded ones; the per-user window
   peaks stay on their rank, and a radix select over SUM-all-reduced per-set counts and
   digit histograms gives the unsharded limits.  Computed with the oracle per shard.
2. The binding's round loop (build_app_profiles_dist) drives local -> rounds with
   all_reduce -> finalize in order, against a fake library speaking the protocol.
3. bench.py's max-over-ranks timing reduction.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(fn, world, *args):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_entry, args=(fn, r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        if isinstance(r, str):
            raise AssertionError(r)
    return res


def _entry(fn, rank, world, port, q, *args):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        out = globals()[fn](rank, world, *args)
        dist.destroy_process_group()
        q.put(out)
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")


def _profile_decomposition(rank, world):
    import oracle as O
    from paper_2411_15997_b200 import tracegen as G
    tr = G.generate(dict(G.CONFIGS["c2"], n_users=80, n_calls=30_000, seed=77))
    cfg = dict(tier_max=0, max_stage=16, q_ppm=[500000, 990000])
    ref = O.profile(tr, cfg)
    sh = G.shard_by_user(tr, rank, world)
    p = O.profile(sh, cfg)
    # R0: sums + histograms (u64 SUM)
    r0 = np.concatenate([p[k].ravel() for k in ("cnt", "sum_in", "sum_sys", "sum_out", "hist")]).astype(np.int64)
    t = torch.from_numpy(r0)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    want = np.concatenate([ref[k].ravel() for k in ("cnt", "sum_in", "sum_sys", "sum_out", "hist")]).astype(np.int64)
    assert (t.numpy() == want).all()
    # R1+: the window peaks stay on their rank (disjoint users).  The limits' nearest-rank
    # quantiles come from a radix select whose per-set counts and 8-bit digit histograms are
    # SUM-all-reduced: every rank picks the same digits and ends with the unsharded quantile.
    users = np.unique(sh["user"])
    mine = np.zeros(tr["n_users"], bool)
    mine[users] = True
    U, A = tr["n_users"], tr["n_apps"]
    sets = []                                         # (request values, token values) per set
    for a in range(A):
        pres = mine & (ref["peak_r_ua"][:, a] > 0)
        sets.append((ref["peak_r_ua"][pres, a].astype(np.uint64), ref["peak_t_ua"][pres, a].astype(np.uint64)))
    pres = mine & (ref["peak_r_u"] > 0)
    sets.append((ref["peak_r_u"][pres].astype(np.uint64), ref["peak_t_u"][pres].astype(np.uint64)))
    vals = [v[0] for v in sets] + [v[1] for v in sets]
    t = torch.tensor([len(v) for v in vals], dtype=torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    n = t.numpy()
    krank = [max(1, -(-990000 * int(x) // 1000000)) - 1 if x else 0 for x in n]
    prefix = [0] * len(vals)
    mx = torch.tensor([max([int(v.max()) if len(v) else 0 for v in vals])], dtype=torch.int64)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    top = max(0, (int(mx[0]).bit_length() + 7) // 8 - 1)
    for d in range(top, -1, -1):
        h = np.zeros((len(vals), 256), np.int64)
        for s_, v in enumerate(vals):
            sel = v if d == top else v[(v >> np.uint64(8 * d + 8)) == np.uint64(prefix[s_])]
            np.add.at(h[s_], ((sel >> np.uint64(8 * d)) & np.uint64(255)).astype(np.int64), 1)
        t = torch.from_numpy(h)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        for s_, row in enumerate(t.numpy()):
            if not n[s_]:
                continue
            c = np.cumsum(row)
            b = int(np.searchsorted(c, krank[s_], side="right"))
            krank[s_] -= int(c[b - 1]) if b else 0
            prefix[s_] = (prefix[s_] << 8) | b
    nr = [p_ if n[s_] else 0 for s_, p_ in enumerate(prefix)]
    assert nr[:A] == [int(x) for x in ref["nr_peak_r_a"]] and nr[A] == int(ref["nr_peak_r_g"][0])
    assert nr[A + 1:2 * A + 1] == [int(x) for x in ref["nr_peak_t_a"]] and nr[2 * A + 1] == int(ref["nr_peak_t_g"][0])
    assert max(1, -(-256 * nr[A] // 256)) == int(ref["T_req_g"][0])
    return int(mine.sum())


def _act_sharded(rank, world):
    """ACT shards by user with no exchange: the rank's shard throttled
    alone with the replicated profile gives the unsharded statuses of its calls, and the
    per-rank summaries SUM to the unsharded summary."""
    import oracle as O
    from paper_2411_15997_b200 import tracegen as G
    tr = G.generate(dict(G.CONFIGS["c2"], n_users=80, n_calls=20_000, seed=78))
    prof = O.profile(tr, dict(tier_max=0))
    act = dict(window_ms=60000, limits_from_profile=1)
    full, fsum = O.act(tr, prof, act)
    with np.errstate(over="ignore"):
        keep = np.nonzero(G.sm64(tr["user"].astype(np.uint64)) % np.uint64(world) == np.uint64(rank))[0]
    st, ssum = O.act(G.shard_by_user(tr, rank, world), prof, act)
    assert (np.asarray(st) == np.asarray(full)[keep]).all()
    keys = ("n_in", "n_admit", "n_dropped", "n_inter_blocked")
    t = torch.tensor([int(ssum[k]) for k in keys] + [int(x) for x in ssum["n_block"]], dtype=torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    assert t.tolist() == [int(fsum[k]) for k in keys] + [int(x) for x in fsum["n_block"]]
    return int(sum(fsum["n_block"]))


def test_act_user_sharded_gloo():
    res = _run("_act_sharded", 2)
    assert res[0] == res[1] and res[0] > 0


def test_profile_protocol_decomposition_gloo():
    res = _run("_profile_decomposition", 2)
    assert sum(res) > 0


class _FakeLib:
    """Speaks fs_profile_local/round/finalize: R0 payload = the rank's value, done after one reduce."""

    def __init__(self, value):
        self.value = value
        self.calls = []
        self.round = 0

    def fs_profile_local(self, ctx, trace, cfg, part, words):
        self.calls.append("local")
        words._obj.value = 4
        return 0

    def fs_profile_round(self, part, buf, words, done):
        import ctypes as C
        self.calls.append(f"round{self.round}")
        arr = (C.c_int64 * 4).from_address(buf.value)
        if self.round == 0:
            for i in range(4):
                arr[i] = self.value + i
            words._obj.value = 4
            done._obj.value = 0
        else:
            self.reduced = list(arr)
            words._obj.value = 0
            done._obj.value = 1
        self.round += 1
        return 0

    def fs_profile_finalize(self, part, out):
        self.calls.append("finalize")
        return 0

    def fs_profile_partial_free(self, part):
        self.calls.append("free")


def _binding_loop(rank, world):
    from paper_2411_15997_b200 import fairserve as F
    fake = _FakeLib(10 * (rank + 1))
    F._lib = fake

    class Ctx:
        device = torch.device("cpu")
        h = None

        def _check(self, code):
            assert code == 0

    class Tr:
        c = None

    orig = F.Profile
    F.Profile = lambda ctx, h: type("P", (), {})()
    orig_a = F._a
    F._a = lambda x: None
    try:
        F.build_app_profiles_dist(Ctx(), Tr(), {}, group=None)
    finally:
        F.Profile = orig
        F._a = orig_a
    assert fake.calls == ["local", "round0", "round1", "finalize", "free"], fake.calls
    return fake.reduced


def test_binding_dist_loop_gloo():
    res = _run("_binding_loop", 2)
    assert res[0] == res[1] == [30, 32, 34, 36]


def _max_reduce(rank, world):
    t = torch.tensor([100.0 + rank, 7.0 * (world - rank)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def test_bench_max_over_ranks_gloo():
    res = _run("_max_reduce", 2)
    assert res[0] == res[1] == [101.0, 14.0]


def _sweep_split(rank, world):
    """sweep_dist: LPT slices per rank, one all_gather of the summaries -> every rank holds the
    whole grid's results in grid order (the sweep itself is faked: summary = f(scenario))."""
    from paper_2411_15997_b200 import fairserve as F

    class Ctx:
        device = torch.device("cpu")

    rng = np.random.default_rng(3)
    meta = (rng.integers(0, 16, size=5000) << 24).astype(np.uint32)
    scen = [dict(tier_max=int(t), key=i) for i, t in enumerate(rng.integers(0, 16, size=37))]

    def fake(sc):
        out = []
        for s in sc:
            k = s["key"]
            out.append(dict(n_arrived=k, n_block=[k, 1, 2, 3], n_dropped=k + 1, n_filtered=s["tier_max"],
                            n_admitted=2 * k, n_finished=2 * k, n_iterations=3 * k, n_ovl_arrivals=4,
                            makespan_ns=10**12 + k, sum_wait_ns=5, max_wait_ns=6, sum_ttft_ns=7, u_min=8,
                            u_max=(1 << 64) - 1 - k, digest=(1 << 63) + k))
        return out, np.array([k % 3 for k in (s["key"] for s in sc)], np.int32)

    res, codes = F.sweep_dist(Ctx(), None, None, scen, meta, sweep_fn=fake)
    want, wcodes = fake(scen)
    assert res == want and list(codes) == list(wcodes)
    parts = F.lpt_split(F.scenario_costs(meta, scen), world)
    assert sorted(i for p in parts for i in p) == list(range(len(scen)))
    loads = [sum(F.scenario_costs(meta, scen)[i] for i in p) for p in parts]
    assert max(loads) - min(loads) <= max(F.scenario_costs(meta, scen))      # LPT balance bound
    return len(parts[rank])


def test_sweep_dist_gloo():
    res = _run("_sweep_split", 2)
    assert sum(res) == 37
