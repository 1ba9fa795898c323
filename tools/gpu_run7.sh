mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rho.py -x -q > gpurun_out/r7_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r7_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r7_bench.json 2> gpurun_out/r7_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_raster_fwd -c 1 -o gpurun_out/r7_fwd python bench.py --steps 1 --warmup 0 --views 8 --no-e2e --no-cpu-baseline > gpurun_out/r7_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_raster_bwd -c 1 -o gpurun_out/r7_bwd python bench.py --steps 1 --warmup 0 --views 8 --no-e2e --no-cpu-baseline >> gpurun_out/r7_ncu.log 2>&1
