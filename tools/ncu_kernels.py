"""Per-kernel table from an ncu --set full report: duration, DRAM bytes, throughput, pipes, occupancy, stalls."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
cols = {
    "kernel": "Kernel Name", "dur_us": "gpu__time_duration.sum", "dram_rd_MB": "dram__bytes_read.sum",
    "dram_wr_MB": "dram__bytes_write.sum", "dram_%": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_%": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_%": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_%": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "fp64_%": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "fma_%": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "alu_%": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "lsu_%": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
}
idx = {k: (h.index(v) if v in h else None) for k, v in cols.items()}
units = rows[1]
print("| " + " | ".join(cols) + " | top stall |")
print("|" + "---|" * (len(cols) + 1))
for r in rows[2:]:
    vals = []
    for k, i in idx.items():
        if i is None:
            vals.append("-")
            continue
        v = r[i]
        if k == "kernel":
            v = v.split("(")[0].replace("void ", "").replace("puv::", "")[:24]
        elif k in ("dram_rd_MB", "dram_wr_MB"):
            x = float(v.replace(",", ""))
            u = units[i]
            mult = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "B": 1e-6, "KB": 1e-3, "MB": 1.0,
                    "GB": 1e3}.get(u, 1.0)
            v = f"{x * mult:.1f}"
        elif k == "dur_us":
            x = float(v.replace(",", ""))
            u = units[i]
            v = f"{x * {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3}.get(u, 1.0):.1f}"
        else:
            try:
                v = f"{float(v.replace(',', '')):.1f}"
            except ValueError:
                pass
        vals.append(v)
    st = []
    for j, name in enumerate(h):
        if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(r[j].replace(",", "")), name[34:-23]))
            except ValueError:
                pass
    st.sort(reverse=True)
    top = ", ".join(f"{n} {x:.2f}" for x, n in st[:3] if n not in ("selected",))
    print("| " + " | ".join(vals) + f" | {top} |")
