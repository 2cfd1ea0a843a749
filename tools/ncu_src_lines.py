"""Per-CUDA-line stall attribution from `ncu -i rep --page source --csv --print-source cuda,sass`:
top lines by stall samples with their instruction counts and two largest stall reasons.
Usage: python tools/ncu_src_lines.py dump.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 50
fname, hdr, out, T, I = "?", None, [], 0, 0
reasons = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        reasons = [(i, h) for i, h in enumerate(r) if h.startswith("stall_") and "Not Issued" not in h]
        ix_s = r.index("Warp Stall Sampling (All Samples)")
        ix_i = r.index("Instructions Executed")
        continue
    if hdr is None or not r[0]:
        continue
    try:
        s = int(r[ix_s] or 0)
        ins = int(r[ix_i] or 0)
    except (ValueError, IndexError):
        continue
    top = sorted(((int(r[i] or 0), h[6:]) for i, h in reasons), reverse=True)[:2]
    T += s
    I += ins
    out.append((s, ins, f"{fname}:{r[0]}", r[1].strip()[:80], top))
out.sort(reverse=True)
print(f"total stall samples {T}, warp instructions {I}")
for s, ins, loc, src, top in out[:N]:
    t = ", ".join(f"{h} {100 * v / max(s, 1):.0f}%" for v, h in top if v)
    print(f"{100 * s / max(T, 1):5.1f}% smp {100 * ins / max(I, 1):5.1f}% ins  {loc:18s} {src:80s} [{t}]")
