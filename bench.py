"""Benchmark of the FairServe trace-scale hot path on B200 (one JSON line on rank 0).

Default workload (BASELINE.json configs[4], the config the metric's "1/2/4/8 B200" is
quoted on): C5 -- a step is fs_build_app_profiles (A1-A5) on the 1M-call trace and an
fs_sweep of 4096 FS(W+I) replays over the grid throttle k x (alpha, beta, gamma) x
E_abusive x tier_max (A6-A9 inside every replay).  value = calls x scenarios / device
time of the step (requests throttled+scheduled/s).  One single C2 replay (configs[1])
is timed after the steps and reported as `single_replay`.

Other workloads: c2 / c3 (profile -> FS(W+I) replay -> ACT on the replay's arrival
times and overload flags), c4 (100M-call profile sharded by user, NCCL rounds).
N > 1: one process per GPU (torchrun).  c2/c3/c5 give every rank its own independent
problem (weak scaling; the replay itself does not shard -- DESIGN.md §8); c4 shards one
trace by user (strong scaling).  Time = max over ranks of CUDA-event time around the K steps.

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
    ap.add_argument("--sweep-split", action="store_true",
                    help="c5 at N>1: one grid split over the ranks (LPT, all_gather of summaries; strong scaling)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--gen", default="cpu", choices=["cpu", "gpu"],
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


# ALGORITHMIC bytes per call of the kernels that touch every call once per launch
ALGO_BYTES = {"prof_stream": 16, "win_scan": 28, "act_flags": 21, "pack_records": 84,
              "radix_scatter": 16}   # radix pass: 4 B key + 4 B value read, the same written


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
    c, eng, pcfg = workload_cfg("c2" if wl in ("c5", "c4") else wl)
    if wl == "c4":
        # C4: one 100M-call profile sharded by user over the ranks (strong scaling): rank r
        # holds users [r U/G, (r+1) U/G) with its share of the calls; NCCL SUM all-reduce rounds
        c4 = G.CONFIGS["c4"]
        total = args.calls or c4["n_calls"]
        Ur = c4["n_users"] // world
        c4r = dict(c4, n_calls=total // world, n_users=Ur, seed=c4["seed"] + rank)
        if args.gen == "gpu":                       # NEXT-4 device generator (untimed setup)
            Tg = F.generate_trace(ctx, c4r)
            tr = {k: Tg.t[k].cpu().numpy().view(np.uint32) for k in F.FIELDS}
            tr.update(n_calls=Tg.n, n_users=Tg.U, n_apps=Tg.A, n_inters=Tg.X)
            del Tg
        else:
            tr = G.generate(c4r)
        tr["user"] = (tr["user"] + np.uint32(rank * Ur)).astype(np.uint32)
        tr["n_users"] = Ur * world
        pcfg = dict(tier_max=0, window_ms=60000, max_stage=64)
    else:
        # weak scaling: every rank gets its own independent problem (rank 0 = the BASELINE config)
        split = wl == "c5" and args.sweep_split and world > 1
        tr = G.generate(wl, seed=G.CONFIGS[wl]["seed"] + (0 if split else rank))
    N = tr["n_calls"]
    T = F.Trace(tr)                                                # inputs resident in HBM before timing
    host = {k: torch.from_numpy(np.ascontiguousarray(tr[k]).view(np.int32)).pin_memory() for k in F.FIELDS}
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.int8, device="cuda")   # > 126 MB L2
    scen = sweep_scenarios(eng, args.scenarios) if wl == "c5" else None
    outs = F.replay_outputs(ctx, T) if wl != "c4" else None
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
    with Clocks(local) as clk:
        for _ in range(args.steps):
            flush.zero_()                                  # L2 flush between timed steps (not timed)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step(T)
            b.record(stream)
            evs.append((a, b))
        torch.cuda.synchronize()
    ctx.set_timing(False)
    ms = sum(a.elapsed_time(b) for a, b in evs)
    kt = ctx.timings()
    launches = sum(v[0] for v in kt.values())
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
    units_per_rank = N * (len(scen) if scen is not None else 1)
    total_units = units_per_rank * world               # c4: the ranks' shards sum to the one trace
    if wl == "c5" and args.sweep_split and world > 1:
        total_units = units_per_rank                   # one grid over all ranks
    value = total_units * args.steps / (ms_max / 1e3)
    e2e_value = total_units / (e2e_step_ms / 1e3)
    if args.timings and rank == 0:
        for k, v in sorted(kt.items(), key=lambda kv: -kv[1][1]):
            sys.stderr.write(f"{k:28s} launches={v[0]:7d} total_ms={v[1]:10.3f} per_step_ms={v[1] / args.steps:9.3f}\n")
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    peaks, peak_src = load_peaks()
    dom_name, (dom_launches, dom_ms) = max(kt.items(), key=lambda kv: kv[1][1])
    roof = roofline(dom_name, dom_launches, dom_ms, N, peaks, peak_src, args, kt)
    S = len(scen) if scen is not None else 0
    line = {
        "metric": "trace requests throttled+scheduled/sec",
        "value": value, "unit": "requests/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong" if wl == "c4" or (wl == "c5" and args.sweep_split and world > 1) else "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": dict(workload_config(wl, N * world if wl == "c4" else N, tr["n_users"], tr["n_apps"], S, world,
                                       split=wl == "c5" and args.sweep_split and world > 1),
                       l2="flushed between timed steps (256 MB write, untimed)"),
        "e2e": {"value": e2e_value, "unit": "requests/s", "h2d_bytes_per_step": 32 * N,
                "d2h_bytes_per_step": d2h_c4 if wl == "c4" else (N if scen is None else 144 * S)},
        "gpu_launches": int(launches),
        "roofline": roof,
        "stage_ms": {k: v[1] / args.steps for k, v in sorted(kt.items(), key=lambda kv: -kv[1][1])[:8]},
        "clocks": clk.summary(),
    }
    if single:
        line["single_replay"] = single
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(wl, tr)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()




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
    for k, b in ALGO_BYTES.items():
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
            prof = ncu_csv(os.path.join(ROOT, "profiles", "r01_replay.csv")) if args.workload == "c2" else {}
            peak = 2 * ghz
            ncalls = 1_000_000
        else:
            # many independent one-lane replays: every SMSP can issue one warp-instruction per cycle
            prof = ncu_csv(os.path.join(ROOT, "profiles", "r01_sweep.csv"))
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
    if name == "win_scan" and args.workload == "c4" and N == 100_000_000:
        # one ncu launch of the same kernel at this size (profiles/r01_c4_winscan.csv)
        prof = ncu_csv(os.path.join(ROOT, "profiles", "r01_c4_winscan.csv"))
        if prof.get("dram__bytes_read.sum") is not None:
            traffic = prof["dram__bytes_read.sum"] + prof.get("dram__bytes_write.sum", 0.0)
    return {"bound": "hbm", "kernel": name, "ms_per_launch": per_s * 1e3, "achieved": gbs,
            "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": gbs / peaks["hbm_gbs"] if gbs else None,
            "traffic": traffic, "algorithmic_bytes_per_launch": b, "peak_source": src, "hbm_stages": stages}


def cpu_baseline(workload, tr):
    """The oracle as it stands (oracle/, single-threaded C++) on a bounded sample of the
    same workload, timed on this host."""
    import oracle as O
    from paper_2411_15997_b200 import tracegen as G
    c, eng, pcfg = workload_cfg("c2" if workload == "c5" else workload)
    sample, desc = tr, "full trace"
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
        scen = sweep_scenarios(eng, 4096)
        picks = [scen[0], scen[len(scen) // 2]]
        O.sweep(sample, p, picks)
        n *= len(picks)
        desc = "C5 trace: profile + 2 of the grid's scenario replays"
    else:
        o, _ = O.replay(sample, p, eng)
        O.act(sample, p, eng["act"], overloaded=o["ovl"], t_ns_override=o["arrive_ns"])
        if workload == "c2":
            desc = "full C2 step: profile + FS(W+I) replay + ACT"
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "requests/s", "cores": 1, "kind": "oracle", "sample": desc, "seconds": dt}


def reference(args, rank, world):
    if rank != 0:
        return
    import oracle as O
    from paper_2411_15997_b200 import tracegen as G
    wl = args.workload
    c, eng, pcfg = workload_cfg("c2" if wl == "c5" else wl)
    if wl == "c3":
        tr = G.generate(dict(G.CONFIGS["c3"], n_users=1000, n_calls=1_000_000, seed=3))
        desc = "C3-shaped 1M-call / 1k-user sample per step"
    elif wl == "c4":
        tr = G.generate(dict(G.CONFIGS["c4"], n_calls=2_000_000, n_users=2000, seed=4))
        desc = "C4-shaped 2M-call / 2k-user sample per step: profile"
    else:
        tr = G.generate("c2")
        desc = "full C2 step" if wl == "c2" else "C5 trace: profile + 2 of the grid's scenario replays per step"
    O.build()

    scen = sweep_scenarios(eng, 4096)
    picks = [scen[0], scen[len(scen) // 2]]

    def step():
        p = O.profile(tr, pcfg)
        if wl == "c4":
            return
        if wl == "c5":
            O.sweep(tr, p, picks)
            return
        o, _ = O.replay(tr, p, eng)
        O.act(tr, p, eng["act"], overloaded=o["ovl"], t_ns_override=o["arrive_ns"])

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    n = tr["n_calls"] * (2 if wl == "c5" else 1)
    v = n * args.steps / dt
    line = {"impl": "reference", "metric": "trace requests throttled+scheduled/sec", "value": v,
            "unit": "requests/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "strong" if wl == "c4" else "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": workload_config(wl, G.CONFIGS[wl]["n_calls"], G.CONFIGS[wl]["n_users"], n_apps_of(wl),
                                      args.scenarios if wl == "c5" else 0, 1),
            "cpu_baseline": {"value": v, "unit": "requests/s", "cores": 1, "kind": "oracle", "sample": desc},
            "e2e": {"value": v, "unit": "requests/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
