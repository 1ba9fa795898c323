mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r6_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r6_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r6_bench.json 2> gpurun_out/r6_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r6_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r6_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_seg_walk|k_tile_scatter|k_tile_count" -c 4 -o gpurun_out/r6_bin python bench.py --steps 1 --warmup 0 --views 8 --no-e2e --no-cpu-baseline > gpurun_out/r6_ncu.log 2>&1
