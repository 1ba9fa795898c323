mkdir -p gpurun_out
M="make -s -C paper_2602_23040_b200/csrc"
run() { timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r9_bench_$1.json 2> gpurun_out/r9_bench_$1.err; }
touch paper_2602_23040_b200/csrc/k_raster*.cu; $M > /dev/null 2>&1; run base
touch paper_2602_23040_b200/csrc/k_raster*.cu; $M EXTRA="-DPUV_FWD_PPT=4" > /dev/null 2>&1; run fwd4
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c1 or c2 or cap or edge" > gpurun_out/r9_pytest_fwd4.log 2>&1
touch paper_2602_23040_b200/csrc/k_raster*.cu; $M EXTRA="-DPUV_BWD_MINB=10" > /dev/null 2>&1; run bwd10
touch paper_2602_23040_b200/csrc/k_raster*.cu; $M > /dev/null 2>&1
