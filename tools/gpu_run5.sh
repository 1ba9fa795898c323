mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r5_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r5_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r5_bench.json 2> gpurun_out/r5_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r5_ncu_launch.log 2>&1
