"""Per CUDA-source-line totals (instructions, stall samples, threads/inst) from an ncu report
exported with --page source --print-source=cuda,sass --csv.  Usage: ncu_lines.py file.csv [func-substring]"""
import csv
import sys
from collections import defaultdict


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else ""
cur_file, cur_fn, hdr = None, None, None
agg = defaultdict(lambda: [0.0, 0.0, 0.0, ""])
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        cur_fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or want not in (cur_fn or ""):
        continue
    try:
        ie = hdr.index("Instructions Executed")
        te = hdr.index("Thread Instructions Executed")
        sm = hdr.index("Warp Stall Sampling (All Samples)")
    except ValueError:
        continue
    if r[0] == "":          # SASS row under a source line: the line row already aggregates it
        continue
    key = (cur_file, r[0])
    a = agg[key]
    a[0] += num(r[ie])
    a[1] += num(r[te])
    a[2] += num(r[sm])
    a[3] = r[1][:90]
tot_i = sum(a[0] for a in agg.values()) or 1
tot_s = sum(a[2] for a in agg.values()) or 1
print(f"total warp instr {tot_i / 1e6:.1f}M")
for (f, ln), a in sorted(agg.items(), key=lambda kv: -kv[1][2])[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    tpi = a[1] / a[0] if a[0] else 0
    print(f"{f[:14]:14s}:{ln:>4s} instr {100 * a[0] / tot_i:5.1f}% stall {100 * a[2] / tot_s:5.1f}% thr/inst {tpi:4.1f} | {a[3]}")
