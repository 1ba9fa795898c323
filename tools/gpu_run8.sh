mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r8_bench_ppt2.json 2> gpurun_out/r8_bench_ppt2.err
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c1 or c2 or cap or edge" > gpurun_out/r8_pytest_ppt2.log 2>&1
touch paper_2602_23040_b200/csrc/k_raster_bwd.cu && make -s -C paper_2602_23040_b200/csrc EXTRA=-DPUV_BWD_PPT=4 > /dev/null 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r8_bench_ppt4.json 2> gpurun_out/r8_bench_ppt4.err
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c1 or c2 or cap or edge" > gpurun_out/r8_pytest_ppt4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_raster_bwd -c 1 -o gpurun_out/r8_bwd_ppt4 python bench.py --steps 1 --warmup 0 --views 8 --no-e2e --no-cpu-baseline > gpurun_out/r8_ncu.log 2>&1
touch paper_2602_23040_b200/csrc/k_raster_bwd.cu && make -s -C paper_2602_23040_b200/csrc > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_raster_bwd -c 1 -o gpurun_out/r8_bwd_ppt2 python bench.py --steps 1 --warmup 0 --views 8 --no-e2e --no-cpu-baseline >> gpurun_out/r8_ncu.log 2>&1
