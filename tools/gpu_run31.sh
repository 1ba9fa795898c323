mkdir -p gpurun_out
touch paper_2602_23040_b200/csrc/*.cu; make -s -C paper_2602_23040_b200/csrc > /dev/null 2>&1
timeout 600 python bench.py > gpurun_out/r31_bench.json 2> gpurun_out/r31_bench.err
