mkdir -p gpurun_out
M="make -s -C paper_2602_23040_b200/csrc"
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2602_23040_b200/csrc tools/value_path_check.cu -o /tmp/vpc && /tmp/vpc > gpurun_out/r11_value_path_check.json 2>&1
run() { timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r11_bench_$1.json 2> gpurun_out/r11_bench_$1.err; }
touch paper_2602_23040_b200/csrc/k_raster*.cu; $M > /dev/null 2>&1; run base
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -x -q > gpurun_out/r11_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r11_pytest.log
touch paper_2602_23040_b200/csrc/k_raster*.cu; $M EXTRA="-DPUV_BWD_MINB=7" > /dev/null 2>&1; run minb7
touch paper_2602_23040_b200/csrc/k_raster*.cu; $M > /dev/null 2>&1
