"""dram bytes (read + write) per launch of each captured kernel -> profiles/traffic.json (the bench's
roofline `traffic`).  Usage: ncu_traffic.py OUT.json NAME=report.ncu-rep:VIEWS_PER_LAUNCH ..."""
import csv
import io
import json
import statistics
import subprocess
import sys

out = {"_what": "dram__bytes_read.sum + dram__bytes_write.sum per launch (median over the captured launches) from "
                "`ncu --set full --clock-control none` captures of `python bench.py --steps 1 --warmup 1 --views 8 "
                "--no-e2e --no-cpu-baseline --no-serial` (C3) with the round-2 kernels (tools/gpu_validate.sh)",
       "config": "C3", "bytes_per_launch": {}, "views_per_launch": {}}
for arg in sys.argv[2:]:
    name, rest = arg.split("=", 1)
    rep, views = rest.rsplit(":", 1)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        continue
    h, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    vals = []
    for r in rows[2:]:
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(m)
            b += float(r[i].replace(",", "")) * scale.get(units[i], 1)
        vals.append(b)
    out["bytes_per_launch"][name] = statistics.median(vals)
    out["views_per_launch"][name] = int(views)
json.dump(out, open(sys.argv[1], "w"), indent=2)
print(json.dumps(out))
