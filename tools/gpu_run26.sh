mkdir -p gpurun_out
touch paper_2602_23040_b200/csrc/*.cu; make -s -C paper_2602_23040_b200/csrc > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r26_pytest_parity.log 2>&1; echo "pytest exit $?" >> gpurun_out/r26_pytest_parity.log
for r in 1 2; do timeout 300 python tools/ab_raster.py --reps 4 --tag quadtree >> gpurun_out/r26_ab.jsonl 2>> gpurun_out/r26_ab.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r26_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r26_ncu_launch.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r26_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r26_pytest.log
timeout 600 python bench.py > gpurun_out/r26_bench.json 2> gpurun_out/r26_bench.err
