"""Summarise an ncu report: SOL, occupancy, pipes, stall reasons, top SASS opcodes (stdout)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]


def page(name, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


raw = page("raw")
d = dict(zip(raw[0], raw[2]))
keys = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__inst_executed.sum"]
for k in keys:
    if k in d:
        print(f"{k:80s} {d[k]}")
print("-- stalls (per issue)")
st = []
for k, v in d.items():
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        try:
            st.append((float(v.replace(",", "")), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        except ValueError:
            pass
for v, k in sorted(st, reverse=True)[:8]:
    print(f"  {k:40s} {v:.3f}")
src = page("source", ["--print-source=sass"])
if len(src) > 2:
    h = src[1]
    ei, si = h.index("Instructions Executed"), h.index("Source")
    op = collections.Counter()
    tot = 0.0
    for r in src[2:]:
        t = r[si].strip().split()
        if not t:
            continue
        o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        x = float(r[ei] or 0)
        op[o] += x
        tot += x
    print(f"-- top opcodes of {tot / 1e6:.1f}M warp instructions")
    for o, c in op.most_common(14):
        print(f"  {o:10s} {c / 1e6:8.1f}M {100 * c / tot:5.1f}%")
