"""Aggregate an ncu `--page source --csv --print-source cuda,sass` dump by CUDA source line:
stall samples and executed warp instructions, top N lines.  Usage: ncu_lines.py dump.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, out, tot_s, tot_i = None, [], 0, 0
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if not r or not hdr or not r[0] or r[0] == "":
        continue
    try:
        s = int(r[hdr["Warp Stall Sampling (All Samples)"]])
        ins = int(r[hdr["Instructions Executed"]])
    except (ValueError, KeyError, IndexError):
        continue
    tot_s += s
    tot_i += ins
    out.append((s, ins, f"{fname}:{r[0]}", r[1].strip()[:90]))
out.sort(reverse=True)
print(f"total samples {tot_s}  total warp instructions {tot_i}")
for s, ins, loc, src in out[:N]:
    print(f"{100*s/tot_s:5.1f}% smp {100*ins/max(tot_i,1):5.1f}% inst  {loc:22s} {src}")
