"""Benchmark of the FairServe trace-scale hot path on B200 (one JSON line on rank 0).

Default workload (BASELINE.json configs[4], the config the metric's "1/2/4/8 B200" is
quoted on): C5 -- a step is fs_build_app_profiles (A1-A5) on the 1M-call trace and an
fs_sweep of 4096 FS(W+I) replays over the grid throttle k x (alpha, beta, gamma) x
E_abusive x tier_max (A6-A9 inside every replay).  value = calls x scenarios / device
time of the step (requests throttled+scheduled/s).  One single C2 replay (configs[1])
is timed after the steps and reported as `single_replay`.

Other workloads: c2 / c3 (profile -> FS(W+I) replay -> ACT on the replay's arrival
times and overload flags), c4 (100M-call profile sharded by user, NCCL rounds).
N > 1: one process per GPU (torchrun).  c5 splits ONE 4096-scenario grid over the ranks
(longest-processing-time slices, NCCL all_gather of the summaries: strong scaling;
--sweep-split off gives every rank its own grid); c4 shards one trace by user (strong
scaling); c2/c3 run a replica per rank (the single replay does not shard -- DESIGN.md §8).
Time = max over ranks of CUDA-event time around the K steps.

--impl reference: the CPU oracle (oracle/, plain single-threaded C++) on this host,
timed on a bounded sample of the same workload, printed as the reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--calls", type=int, default=0, help="c4: total calls (default 100M)")
    ap.add_argument("--scenarios", type=int, default=4096, help="c5: scenarios per GPU (the whole grid with --sweep-split)")
    ap.add_argument("--sweep-split", default="auto", choices=["auto", "on", "off"],
                    help="c5 at N>1: one grid split over the ranks (LPT, all_gather of summaries; strong "
                         "scaling, the default) or an independent grid per rank (off: weak scaling)")
    ap.add_argument("--no-hbm", action="store_true", help="skip the full-size HBM lines (C4 profile, C3/C2 ACT)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--gen", default="gpu", choices=["cpu", "gpu"],
                    help="c4: trace from tracegen.py (cpu) or fs_generate_trace on the device (gpu)")
    ap.add_argument("--timings", action="store_true", help="print per-kernel timings to stderr")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (recipe's clocks line)."""

    def __init__(self, index):
        self.index = index
        self.p = None
        self.lines = []

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None
        return self

    def _read(self):
        for line in self.p.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.p:
            time.sleep(0.25)
            self.p.terminate()
            try:
                self.p.wait(timeout=2)
            except Exception:
                self.p.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def n_apps_of(wl):
    from paper_2411_15997_b200 import tracegen as G
    c = G.CONFIGS[wl]
    return c.get("n_apps", len(c["apps"]) * len(c["app_scales"]))


def workload_config(wl, n_calls, n_users, n_apps, scenarios, world, split=False):
    """The `config` object of the JSON line (shared by both arms)."""
    return {"workload": {"c2": "C2: 1k users, 6 apps, 1M calls, 5% abusive; profile + FS(W+I) replay + ACT",
                         "c3": "C3: 10k users, 12 apps, 10M calls; profile + FS(W+I) replay + ACT",
                         "c4": f"C4: app profile of {n_calls} calls sharded by user over {world} GPU(s) "
                               f"(NCCL u64 SUM all-reduce rounds)",
                         "c5": f"C5: profile + sweep of {scenarios} replays (throttle k x (alpha,beta,gamma) x "
                               f"E_abusive x tier_max) of a 1M-call trace"}[wl],
            "n_calls": n_calls, "n_users": n_users, "n_apps": n_apps, "scenarios_per_gpu": scenarios,
            "parallelism": (f"user-hash shards x{world}" if wl == "c4" else
                            f"one {scenarios}-scenario grid split over {world} GPUs (LPT, NCCL all_gather)" if split else
                            f"independent problem per GPU x{world}")}


def workload_cfg(name):
    from paper_2411_15997_b200 import tracegen as G
    c = G.CONFIGS[name]
    eng = dict(c["engine"] or {}, mode=1, tier_max=255, alpha=1, beta=2, gamma=1,
               act=dict(window_ms=60000, limits_from_profile=1, limit_mult_q8=0, count_mode=0))
    pcfg = dict(tier_max=c["profile"]["tier_max"], window_ms=60000, max_stage=64)
    return c, eng, pcfg


def sweep_scenarios(eng, total):
    """C5 grid: throttle k x (alpha,beta,gamma) x E_abusive x tier_max, first `total`."""
    ks = [128, 192, 256, 320, 384, 512, 640, 768, 1024, 1280, 1536, 2048, 2560, 4096, 8192, 0xFFFFFFFF]
    ws = [(1, 2, 1), (1, 1, 1), (1, 1, 2), (1, 0, 1), (2, 1, 1), (1, 2, 2), (1, 1, 4), (4, 1, 1)]
    out = []
    for k in ks:
        for (a, b, g) in ws:
            for E in (65536, 131072):
                for tm in range(16):
                    s = dict(eng, alpha=a, beta=b, gamma=g, prio_abusive_q16=E, tier_max=tm)
                    s["act"] = dict(eng["act"], limit_mult_q8=k)
                    out.append(s)
    # spread the first `total` across the grid deterministically
    idx = np.random.default_rng(5).permutation(len(out))[:total]
    return [out[i] for i in sorted(idx)]


# ALGORITHMIC bytes per call of the kernels that touch every call once per launch,
# reported for the C3 / C4 workloads (the C5 trace is L2-resident: its stage rates are cache rates)
ALGO_BYTES = {"prof_stream": 16, "act_flags": 21, "pack_records": 84,
              "radix_scatter": 16}   # radix pass: 4 B key + 4 B value read, the same written


def participating(meta, scen):
    """Participating calls of each scenario (tier <= tier_max): the units of requests/s (SURVEY
    §8(d): calls in the (filtered) trace).  Filtered users' calls never arrive (Q35)."""
    from paper_2411_15997_b200.fairserve import scenario_costs
    return scenario_costs(meta, scen)


def stratified_sample(scen):
    """One scenario per abuse mix (tier_max 0..15): the middle one of the grid's scenarios with
    that tier_max (throttle k, weights and E vary across the sample)."""
    out = []
    for tm in range(16):
        c = [s for s in scen if s["tier_max"] == tm]
        if c:
            out.append(c[len(c) // 2])
    return out


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def shard_device_trace(F, T, rank, world):
    """Rank's user-hash shard of a device-resident trace (sm64(user) mod world, the split of
    tracegen.shard_by_user), keeping (t_ms, id) order; interaction ids renumbered densely in
    id order.  Input plumbing on the device (untimed); none of the method's arithmetic."""
    import torch
    u = T.t["user"].long() & 0xFFFFFFFF
    M = (1 << 64) - 1

    def c64(v):                                  # u64 constant as a wrapped int64
        return v - (1 << 64) if v >= 1 << 63 else v

    def shr(x, k):                               # logical right shift of u64 bits held in int64
        return (x >> k) & ((1 << (64 - k)) - 1)
    x = u + c64(0x9E3779B97F4A7C15)
    x = (x ^ shr(x, 30)) * c64(0xBF58476D1CE4E5B9)
    x = (x ^ shr(x, 27)) * c64(0x94D049BB133111EB)
    x = x ^ shr(x, 31)
    # unsigned mod: (hi * 2^32 + lo) mod w
    hi, lo = shr(x, 32), x & 0xFFFFFFFF
    h = ((hi % world) * ((1 << 32) % world) + lo % world) % world
    keep = torch.nonzero(h == rank).squeeze(1)
    t = {k: T.t[k].index_select(0, keep).contiguous() for k in F.FIELDS}
    uniq, inv = torch.unique(t["inter"].long() & 0xFFFFFFFF, return_inverse=True)
    t["inter"] = inv.to(torch.int32).contiguous()
    del M
    meta = dict(n_calls=int(keep.numel()), n_users=T.U, n_apps=T.A, n_inters=int(uniq.numel()))
    return F.Trace(meta, tensors=t)


def profile_sha(prof):
    """sha256 over the finalised profile's tables (the G-invariance check of the sharded C4 line)."""
    import hashlib
    r = prof.read()
    h = hashlib.sha256()
    for k in sorted(x for x in r if hasattr(r[x], "tobytes")):
        h.update(k.encode())
        h.update(np.ascontiguousarray(r[k]).tobytes())
    return h.hexdigest()


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return reference(args, rank, world)
    import torch
    import torch.distributed as dist
    from paper_2411_15997_b200 import build as B
    from paper_2411_15997_b200 import fairserve as F
    from paper_2411_15997_b200 import tracegen as G

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if rank == 0:
        B.build()
    if world > 1:
        dist.barrier()
    ctx = F.Context(local)
    stream = torch.cuda.current_stream()
    wl = args.workload
    split = wl == "c5" and world > 1 and args.sweep_split != "off"
    c, eng, pcfg = workload_cfg("c2" if wl in ("c5", "c4") else wl)
    c4_sha = None
    if wl == "c4":
        # C4: ONE 100M-call trace (the same seed on every rank) sharded by user hash over the
        # ranks (strong scaling); NCCL SUM all-reduce rounds; every G finalises the
        # identical profile (config.profile_sha)
        c4 = G.CONFIGS["c4"]
        total = args.calls or c4["n_calls"]
        c4r = dict(c4, n_calls=total)
        if args.gen == "gpu":                       # NEXT-4 device generator (untimed setup)
            Tfull = F.generate_trace(ctx, c4r)
        else:
            Tfull = F.Trace(G.generate(c4r))
        T = shard_device_trace(F, Tfull, rank, world) if world > 1 else Tfull
        del Tfull
        tr = {k: T.t[k].cpu().numpy().view(np.uint32) for k in F.FIELDS}
        tr.update(n_calls=T.n, n_users=T.U, n_apps=T.A, n_inters=T.X)
        pcfg = dict(tier_max=0, window_ms=60000, max_stage=64)
    else:
        # c5 at N > 1 (default): one grid split over the ranks (strong scaling); --sweep-split off or
        # c2/c3: every rank gets its own independent problem (weak scaling; rank 0 = the BASELINE config)
        tr = G.generate(wl, seed=G.CONFIGS[wl]["seed"] + (0 if split else rank))
        T = F.Trace(tr)                                            # inputs resident in HBM before timing
    N = tr["n_calls"]
    host = {k: torch.from_numpy(np.ascontiguousarray(tr[k]).view(np.int32)).pin_memory() for k in F.FIELDS}
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.int8, device="cuda")   # > 126 MB L2
    scen = sweep_scenarios(eng, args.scenarios) if wl == "c5" else None
    outs = F.replay_outputs(ctx, T) if wl not in ("c4",) else None
    status = torch.empty(N, dtype=torch.uint8, device="cuda")

    def step(trace):
        if wl == "c4":                                                  # A1-A5 + A10
            if world > 1:
                return F.build_app_profiles_dist(ctx, trace, pcfg)
            return F.build_app_profiles(ctx, trace, pcfg)
        prof = F.build_app_profiles(ctx, trace, pcfg)                 # A1-A5
        if scen is not None:
            if split:                                                    # A9 over the ranks + A10 gather
                return F.sweep_dist(ctx, trace, prof, scen, tr["meta"])
            return F.sweep(ctx, trace, prof, scen)                       # A9 (A6-A7 inside every replay)
        o, s = F.wsc_replay(ctx, trace, prof, eng, out=outs)            # A7
        return F.act_throttle(ctx, trace, prof, eng["act"], overloaded=o["ovl"], t_ns_override=o["arrive_ns"],
                              status=status)                             # A6 on the replay's arrivals (P8)

    for _ in range(args.warmup):
        step(T)
    torch.cuda.synchronize()
    ctx.timing_reset()
    ctx.set_timing(True)
    evs = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    last = None
    with Clocks(local) as clk:
        for _ in range(args.steps):
            flush.zero_()                                  # L2 flush between timed steps (not timed)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            last = step(T)
            b.record(stream)
            evs.append((a, b))
        torch.cuda.synchronize()
    ctx.set_timing(False)
    ms = sum(a.elapsed_time(b) for a, b in evs)
    kt = ctx.timings()
    launches = sum(v[0] for v in kt.values())
    if wl == "c4":
        c4_sha = profile_sha(last)
    sweep_codes_ok = None
    if scen is not None:
        sweep_codes_ok = bool((np.asarray(last[1]) == 0).all())
    # end to end through the public API with host buffers: H2D of the trace, the step, D2H of the results
    e2e_steps = 1 if scen is not None else max(1, min(args.steps, 3))
    e2e_ms = 0.0
    d2h_c4 = 0
    d2h = torch.empty(N, dtype=torch.uint8).pin_memory()
    for _ in range(e2e_steps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        T2 = F.Trace.from_host_tensors(tr, host)
        res = step(T2)                                    # the sweep returns its summaries in host memory
        if wl == "c4":
            got = res.read()                              # D2H of the profile tables
            d2h_c4 = sum(v.nbytes for v in got.values() if hasattr(v, "nbytes"))
        elif scen is None:
            d2h.copy_(status, non_blocking=True)
        b.record(stream)
        torch.cuda.synchronize()
        e2e_ms += a.elapsed_time(b)
        del T2
    # one single replay of the C2 configuration on this trace (BASELINE configs[1]), for context
    single = None
    if scen is not None and rank == 0:
        prof = F.build_app_profiles(ctx, T, pcfg)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        F.wsc_replay(ctx, T, prof, eng, out=outs)
        b.record(stream)
        torch.cuda.synchronize()
        single = {"workload": "C2 single FS(W+I) replay (configs[1])", "ms": a.elapsed_time(b),
                  "value": N / (a.elapsed_time(b) / 1e3), "unit": "requests/s"}
    t = torch.tensor([ms, e2e_ms / e2e_steps], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, e2e_step_ms = float(t[0]), float(t[1])
    # requests/s counts the calls in the (filtered) trace: a sweep scenario's units
    # are its participating calls (tier <= tier_max); filtered users' calls never arrive
    units_per_rank = sum(participating(tr["meta"], scen)) if scen is not None else N
    calls_replayed_per_rank = N * len(scen) if scen is not None else N
    grids = 1 if split else world
    total_units = units_per_rank * grids               # c4: the ranks' shards sum to the one trace
    if wl == "c4":
        total_units = units_per_rank * world
    value = total_units * args.steps / (ms_max / 1e3)
    e2e_value = total_units / (e2e_step_ms / 1e3)
    if args.timings and rank == 0:
        for k, v in sorted(kt.items(), key=lambda kv: -kv[1][1]):
            sys.stderr.write(f"{k:28s} launches={v[0]:7d} total_ms={v[1]:10.3f} per_step_ms={v[1] / args.steps:9.3f}\n")
    hbm = None
    if rank == 0 and world == 1 and wl == "c5" and not args.no_hbm:
        del host
        hbm = hbm_lines(ctx, F, G, T, outs, eng, flush)
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    peaks, peak_src = load_peaks()
    dom_name, (dom_launches, dom_ms) = max(kt.items(), key=lambda kv: kv[1][1])
    roof = roofline(dom_name, dom_launches, dom_ms, N, peaks, peak_src, args, kt)
    S = len(scen) if scen is not None else 0
    cfg = dict(workload_config(wl, N * world if wl == "c4" else N, tr["n_users"], tr["n_apps"], S, world,
                               split=split),
               l2="flushed between timed steps (256 MB write, untimed)")
    if scen is not None:
        cfg.update(participating_calls_per_grid=units_per_rank, replayed_calls_per_grid=calls_replayed_per_rank,
                   all_scenario_codes_ok=sweep_codes_ok)
    if wl == "c4":
        cfg.update(profile_sha=c4_sha, trace="fs_generate_trace (device)" if args.gen == "gpu" else "tracegen.py")
    line = {
        "metric": "trace requests throttled+scheduled/sec",
        "value": value, "unit": "requests/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong" if wl == "c4" or split else "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": cfg,
        "e2e": {"value": e2e_value, "unit": "requests/s", "h2d_bytes_per_step": 32 * N,
                "d2h_bytes_per_step": d2h_c4 if wl == "c4" else (N if scen is None else 144 * S)},
        "gpu_launches": int(launches),
        "roofline": roof,
        "stage_ms": {k: v[1] / args.steps for k, v in sorted(kt.items(), key=lambda kv: -kv[1][1])[:8]},
        "clocks": clk.summary(),
    }
    if scen is not None:
        line["replayed_calls_per_s"] = calls_replayed_per_rank * grids * args.steps / (ms_max / 1e3)
    if single:
        line["single_replay"] = single
    if hbm:
        line["hbm"] = hbm
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(wl, tr)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# algorithmic bytes per call of the HBM-bound stages
PROFILE_ALGO_B = 56          # one read of user, t, meta, L_I, L_S, L_O (24 B) + per order 16 B (perm + (t, tau))
ACT_ALGO_B = 30              # user, t, meta, L_I, L_S, inter, overload (25 B) + perm (4 B) + status (1 B):
                             # one pass; the fixed-point passes the implementation adds are not credited


def _time_calls(ctx, fn, flush, stream, reps):
    """mean device ms of `reps` L2-flushed calls after one warm-up, and the library's per-kernel times"""
    import torch
    fn()
    torch.cuda.synchronize()
    ctx.timing_reset()
    ctx.set_timing(True)
    tot = 0.0
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    ctx.set_timing(False)
    return tot / reps, ctx.timings()


def _stage_line(name, ms, n, algo_b, peaks, kt, reps, ncu):
    gbs = algo_b * n / (ms / 1e3) / 1e9
    kern = []
    for k, (l, t) in sorted(kt.items(), key=lambda kv: -kv[1][1])[:12]:
        e = {"kernel": k, "ms": t / reps, "launches": l / reps}
        if ncu and k in ncu:
            e["ncu_dram_bytes_per_call"] = ncu[k]
        kern.append(e)
    return {"workload": name, "calls": n, "ms": ms, "calls_per_s": n / (ms / 1e3),
            "algorithmic_bytes_per_call": algo_b, "achieved_gbs": gbs, "peak_gbs": peaks["hbm_gbs"],
            "frac": gbs / peaks["hbm_gbs"], "kernels": kern}


NCU_TAGS = ("r02d", "r02c", "r02b", "r02")          # committed ncu captures, newest first (profiles/README.md)


def ncu_path(name):
    """The newest committed ncu capture `profiles/<tag>_<name>` (the same command bench.py times)."""
    for tag in NCU_TAGS:
        p = os.path.join(ROOT, "profiles", f"{tag}_{name}")
        if os.path.exists(p):
            return p
    return os.path.join(ROOT, "profiles", f"{NCU_TAGS[-1]}_{name}")


def ncu_bytes_per_call(path, n):
    """{kernel: DRAM bytes (read + write) per call per launch} from a committed ncu --csv capture."""
    import csv
    out = {}
    try:
        rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    except OSError:
        return out
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    acc = {}
    for r in rows[1:]:
        try:
            nm = r[ix["Kernel Name"]].split("(")[0].split("<")[0].replace("k_", "", 1)
            if r[ix["Metric Name"]] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                v = float(r[ix["Metric Value"]].replace(",", ""))
                unit = r[ix["Metric Unit"]]
                v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
                acc.setdefault((nm, r[ix["ID"]]), 0.0)
                acc[(nm, r[ix["ID"]])] += v
        except (KeyError, ValueError, IndexError):
            pass
    per = {}
    for (nm, _), v in acc.items():
        per.setdefault(nm, []).append(v)
    for nm, vs in per.items():
        out[nm] = sum(vs) / len(vs) / n
    return out


def hbm_lines(ctx, F, G, T5, outs, eng, flush):
    """The HBM half of the metric at full size (north_star: profile + ACT >= 50 % of HBM peak),
    in the default run: (1) the 100M-call C4 profile on a device-generated trace, (2) ACT on a
    device-generated 10M-call C3 trace with overload always on (the heavy worst-case screening
    path), (3) ACT on the C2/C5 trace with the single replay's recorded arrivals and overload
    flags.  Generation is untimed; each stage is the median-free mean of `reps` L2-flushed runs."""
    import torch
    stream = torch.cuda.current_stream()
    peaks, _ = load_peaks()
    res = {}
    reps = 3
    T4 = F.generate_trace(ctx, "c4")
    p4 = dict(tier_max=0, window_ms=60000, max_stage=64)
    ms, kt = _time_calls(ctx, lambda: F.build_app_profiles(ctx, T4, p4), flush, stream, reps)
    res["c4_profile"] = _stage_line("C4 fs_build_app_profiles, 100M calls (device-generated), tier_max 0",
                                    ms, T4.n, PROFILE_ALGO_B, peaks, kt, reps,
                                    ncu_bytes_per_call(ncu_path("c4_dram.csv"), T4.n))
    del T4
    torch.cuda.synchronize()
    T3 = F.generate_trace(ctx, "c3")
    _, e3, p3 = workload_cfg("c3")
    prof3 = F.build_app_profiles(ctx, T3, p3)
    st3 = torch.empty(T3.n, dtype=torch.uint8, device="cuda")
    summ = {}
    ms, kt = _time_calls(ctx, lambda: summ.update(F.act_throttle(ctx, T3, prof3, e3["act"], status=st3)[1]),
                         flush, stream, reps)
    res["c3_act_overload_always"] = _stage_line(
        "C3 fs_act_throttle, 10M calls (device-generated), overload always", ms, T3.n, ACT_ALGO_B, peaks, kt, reps,
        ncu_bytes_per_call(ncu_path("c3_act_dram.csv"), T3.n))
    res["c3_act_overload_always"]["summary"] = summ
    del T3, prof3, st3
    # ACT on the C2 trace with the single replay's recorded arrival times and overload flags
    _, e2, p2 = workload_cfg("c2")
    prof2 = F.build_app_profiles(ctx, T5, p2)
    st2 = torch.empty(T5.n, dtype=torch.uint8, device="cuda")
    summ = {}
    ms, kt = _time_calls(ctx, lambda: summ.update(F.act_throttle(ctx, T5, prof2, e2["act"], overloaded=outs["ovl"],
                                                                 t_ns_override=outs["arrive_ns"], status=st2)[1]),
                         flush, stream, reps)
    res["c2_act_replay_flags"] = _stage_line(
        "C2 fs_act_throttle, 1M calls, the replay's arrival times + overload flags", ms, T5.n, ACT_ALGO_B, peaks,
        kt, reps, None)
    res["c2_act_replay_flags"]["summary"] = summ
    res["c2_act_replay_flags"]["equals_replay_status"] = bool(torch.equal(st2, outs["status"]))
    return res


def ncu_csv(path):
    """{metric name: value} of the first kernel row of an ncu --csv --metrics log."""
    import csv
    try:
        rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    except OSError:
        return {}
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    out = {}
    for r in rows[1:]:
        try:
            out[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
        except (KeyError, ValueError, IndexError):
            pass
    return out


def roofline(name, launches, ms, N, peaks, src, args, kt):
    per_s = ms / max(launches, 1) / 1e3
    stages = []
    for k, b in (ALGO_BYTES.items() if args.workload in ("c3", "c4") else ()):
        if k in kt and kt[k][1] > 0:
            gbs = b * N * kt[k][0] / (kt[k][1] / 1e3) / 1e9
            stages.append({"kernel": k, "bound": "hbm", "bytes_per_call": b, "achieved": gbs,
                           "peak": peaks["hbm_gbs"], "frac": gbs / peaks["hbm_gbs"]})
    if name in ("wsc_replay", "wsc_sweep"):
        ghz = peaks.get("sm_max_mhz", 1965.0) / 1e3
        units = N
        if name == "wsc_replay":
            # dependent instruction chain: one engine warp (+ the head-prefetch warp) issuing at
            # most one warp-instruction per cycle each at the measured max SM clock.
            prof = ncu_csv(ncu_path("replay.csv")) if args.workload == "c2" else {}
            peak = 2 * ghz
            ncalls = 1_000_000
        else:
            # many independent one-lane replays: every SMSP can issue one warp-instruction per cycle
            prof = ncu_csv(ncu_path("sweep.csv"))
            peak = peaks.get("sm_count", 148) * 4 * ghz
            ncalls = 1_000_000 * int(prof.get("scenarios", 64))
            units = N * args.scenarios
        inst = prof.get("smsp__inst_executed.sum")
        achieved = inst / ncalls * units / per_s / 1e9 if inst else None
        traffic = None
        if prof.get("dram__bytes_read.sum") is not None:
            traffic = prof["dram__bytes_read.sum"] + prof.get("dram__bytes_write.sum", 0.0)
        return {"bound": "alu", "kernel": name, "achieved": achieved, "peak": peak, "unit": "Ginst/s",
                "frac": achieved / peak if achieved else None, "traffic": traffic, "ms_per_launch": per_s * 1e3,
                "peak_source": src + (" (2 issuing warps x 1 inst/cycle x sm_max_mhz)" if name == "wsc_replay" else " (148 SMs x 4 schedulers x 1 warp-inst/cycle x sm_max_mhz)"),
                "instructions_per_call": inst / ncalls if inst else None,
                "ns_per_call": per_s / N * 1e9, "hbm_stages": stages}
    b = ALGO_BYTES.get(name, 0) * N
    gbs = b / per_s / 1e9 if b else None
    traffic = None
    return {"bound": "hbm", "kernel": name, "ms_per_launch": per_s * 1e3, "achieved": gbs,
            "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": gbs / peaks["hbm_gbs"] if gbs else None,
            "traffic": traffic, "algorithmic_bytes_per_launch": b, "peak_source": src, "hbm_stages": stages}


def oracle_sweep_parallel(O, tr, p, scen, P):
    """the oracle's replays (oracle/, single-threaded C++ each) run side by side on P host threads
    (ctypes releases the GIL; the oracle keeps no global state): the P-core CPU baseline of
    BASELINE.md §5"""
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(P) as ex:
        return list(ex.map(lambda s: O.sweep(tr, p, [s]), sorted(scen, key=lambda s: -s["tier_max"])))


def cpu_baseline(workload, tr):
    """The oracle as it stands (oracle/, single-threaded C++) on a bounded sample of the
    same workload, timed on this host; the sweep's sample runs on all host cores."""
    import oracle as O
    from paper_2411_15997_b200 import tracegen as G
    c, eng, pcfg = workload_cfg("c2" if workload == "c5" else workload)
    sample, desc = tr, "full trace"
    cores = 1
    if workload == "c3":
        sample = G.generate(dict(G.CONFIGS["c3"], n_users=1000, n_calls=1_000_000, seed=3))
        desc = "C3-shaped 1M-call / 1k-user sample: profile + FS(W+I) replay + ACT"
    if workload == "c4":
        sample = G.generate(dict(G.CONFIGS["c4"], n_calls=2_000_000, n_users=2000, seed=4))
        desc = "C4-shaped 2M-call / 2k-user sample: profile"
    t0 = time.perf_counter()
    p = O.profile(sample, pcfg)
    n = sample["n_calls"]
    if workload == "c4":
        pass
    elif workload == "c5":
        picks = stratified_sample(sweep_scenarios(eng, 4096))
        cores = min(host_cores(), len(picks))
        oracle_sweep_parallel(O, sample, p, picks, cores)
        n = sum(participating(sample["meta"], picks))
        desc = (f"C5 trace: profile + {len(picks)} of the grid's replays (one per tier_max 0..15, "
                f"stratified) on {cores} host threads; units = participating calls")
    else:
        o, _ = O.replay(sample, p, eng)
        O.act(sample, p, eng["act"], overloaded=o["ovl"], t_ns_override=o["arrive_ns"])
        if workload == "c2":
            desc = "full C2 step: profile + FS(W+I) replay + ACT"
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "requests/s", "cores": cores, "kind": "oracle", "sample": desc, "seconds": dt,
            "cpu": cpu_model()}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def reference(args, rank, world):
    if rank != 0:
        return
    import oracle as O
    from paper_2411_15997_b200 import tracegen as G
    wl = args.workload
    c, eng, pcfg = workload_cfg("c2" if wl == "c5" else wl)
    cores = 1
    if wl == "c3":
        tr = G.generate(dict(G.CONFIGS["c3"], n_users=1000, n_calls=1_000_000, seed=3))
        desc = "C3-shaped 1M-call / 1k-user sample per step"
    elif wl == "c4":
        tr = G.generate(dict(G.CONFIGS["c4"], n_calls=2_000_000, n_users=2000, seed=4))
        desc = "C4-shaped 2M-call / 2k-user sample per step: profile"
    else:
        tr = G.generate("c2")
        desc = "full C2 step"
    O.build()
    picks = stratified_sample(sweep_scenarios(eng, 4096))
    if wl == "c5":
        cores = min(host_cores(), len(picks))
        desc = (f"C5 trace per step: profile + {len(picks)} of the grid's replays (one per tier_max 0..15, "
                f"stratified) on {cores} host threads; units = participating calls")

    def step():
        p = O.profile(tr, pcfg)
        if wl == "c4":
            return
        if wl == "c5":
            oracle_sweep_parallel(O, tr, p, picks, cores)
            return
        o, _ = O.replay(tr, p, eng)
        O.act(tr, p, eng["act"], overloaded=o["ovl"], t_ns_override=o["arrive_ns"])

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    n = sum(participating(tr["meta"], picks)) if wl == "c5" else tr["n_calls"]
    v = n * args.steps / dt
    split = wl == "c5" and world > 1 and args.sweep_split != "off"
    line = {"impl": "reference", "metric": "trace requests throttled+scheduled/sec", "value": v,
            "unit": "requests/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "strong" if wl == "c4" or split else "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": workload_config(wl, G.CONFIGS[wl]["n_calls"], G.CONFIGS[wl]["n_users"], n_apps_of(wl),
                                      args.scenarios if wl == "c5" else 0, world, split=split),
            "cpu_baseline": {"value": v, "unit": "requests/s", "cores": cores, "kind": "oracle", "sample": desc,
                             "cpu": cpu_model()},
            "e2e": {"value": v, "unit": "requests/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
