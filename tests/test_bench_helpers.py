"""CPU checks of bench.py's host-side helpers (JSON fields, roofline arithmetic, the C5 grid)."""
import types

import bench


def test_sweep_grid_is_the_c5_grid():
    eng = dict(mode=1, act=dict(limit_mult_q8=0))
    s = bench.sweep_scenarios(eng, 4096)
    assert len(s) == 4096
    keys = {(x["alpha"], x["beta"], x["gamma"], x["prio_abusive_q16"], x["tier_max"], x["act"]["limit_mult_q8"])
            for x in s}
    assert len(keys) == 4096                       # 16 x 8 x 2 x 16 distinct scenarios


def test_roofline_fields():
    peaks = {"hbm_gbs": 6456.8, "sm_max_mhz": 1965.0}
    args = types.SimpleNamespace(workload="c5", scenarios=4096)
    kt = {"wsc_sweep": (1, 20000.0), "prof_stream": (1, 0.3), "pack_records": (1, 0.2)}
    r = bench.roofline("wsc_sweep", 1, 20000.0, 1_000_000, peaks, "measured", args, kt)
    assert r["bound"] == "alu" and r["peak"] > 0
    assert r["hbm_stages"] == []                   # the C5 trace is L2-resident: no cache rates as HBM rates
    args4 = types.SimpleNamespace(workload="c4", scenarios=4096)
    r4 = bench.roofline("wsc_sweep", 1, 20000.0, 1_000_000, peaks, "measured", args4, kt)
    assert {x["kernel"] for x in r4["hbm_stages"]} == {"prof_stream", "pack_records"}
    r2 = bench.roofline("prof_stream", 1, 0.3, 1_000_000, peaks, "measured", args, kt)
    assert r2["bound"] == "hbm" and abs(r2["achieved"] - 16e6 / 0.3e-3 / 1e9) < 1e-6
    assert r2["frac"] == r2["achieved"] / 6456.8


def test_ncu_csv_parser(tmp_path):
    p = tmp_path / "x.csv"
    p.write_text('==PROF== hello\n"ID","Kernel Name","Metric Name","Metric Unit","Metric Value"\n'
                 '"0","k","smsp__inst_executed.sum","inst","1,234"\n')
    assert bench.ncu_csv(str(p)) == {"smsp__inst_executed.sum": 1234.0}


def test_ncu_captures_newest_first():
    """bench.py reads the newest committed ncu capture of each kind (profiles/<tag>_<name>), and the
    sweep capture it reads carries the instruction count the C5 roofline divides by."""
    import os
    p = bench.ncu_path("sweep.csv")
    assert os.path.exists(p) and os.path.basename(p).startswith(bench.NCU_TAGS[0] + "_")
    m = bench.ncu_csv(p)
    assert m.get("smsp__inst_executed.sum", 0) > 0 and m.get("gpu__time_duration.sum", 0) > 0
    for name in ("c4_dram.csv", "c3_act_dram.csv", "replay.csv"):
        assert os.path.exists(bench.ncu_path(name)), name
