mkdir -p gpurun_out
touch paper_2602_23040_b200/csrc/*.cu; make -s -C paper_2602_23040_b200/csrc > /dev/null 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r18_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r18_pytest.log
timeout 600 python bench.py > gpurun_out/r18_bench.json 2> gpurun_out/r18_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r18_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r18_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_raster_bwd" -c 1 -o gpurun_out/r18_bwd python bench.py --steps 1 --warmup 0 --views 8 --no-e2e --no-cpu-baseline > gpurun_out/r18_ncu.log 2>&1
