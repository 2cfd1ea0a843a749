"""Per-kernel table of an ncu --csv --metrics capture (gpu__time_duration, dram bytes):
launches, mean us per launch, DRAM bytes per launch and per call, achieved GB/s.
Usage: python tools/ncu_kernel_table.py capture.csv n_calls [top]"""
import csv
import sys

path, n = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
hdr = {h: i for i, h in enumerate(rows[0])}
units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}
launch = {}
for r in rows[1:]:
    key = (r[hdr["ID"]], r[hdr["Kernel Name"]].split("(")[0])
    v = float(r[hdr["Metric Value"]].replace(",", "")) * units.get(r[hdr["Metric Unit"]], 1.0)
    launch.setdefault(key, {})[r[hdr["Metric Name"]]] = v
agg = {}
for (lid, name), m in launch.items():
    a = agg.setdefault(name, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':48s} {'launches':>8s} {'us/launch':>10s} {'share':>6s} {'DRAM MB/launch':>14s} {'B/call':>7s} {'GB/s':>7s}")
for name, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{name[:48]:48s} {c:8d} {t / c * 1e6:10.1f} {100 * t / tot:5.1f}% {b / c / 1e6:14.1f} {b / c / n:7.1f} "
          f"{(b / t / 1e9) if t else 0:7.0f}")
print(f"total {tot * 1e3:.3f} ms over {sum(a[0] for a in agg.values())} launches (cold, serialised)")
