# Measurements of the "next" rows (tools/bench_extra.py) on one B200, through gpurun.
mkdir -p gpurun_out
touch paper_2602_23040_b200/csrc/*.cu; make -s -C paper_2602_23040_b200/csrc > /dev/null 2>&1
timeout 1500 python tools/bench_extra.py rho lpo objective label > gpurun_out/extra.jsonl 2> gpurun_out/extra.err
