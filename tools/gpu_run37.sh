mkdir -p gpurun_out
touch paper_2602_23040_b200/csrc/*.cu; make -s -C paper_2602_23040_b200/csrc > /dev/null 2>&1
timeout 2000 python -m pytest tests -m gpu -x -q > gpurun_out/r37_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r37_pytest.log
timeout 600 python bench.py > gpurun_out/r37_bench.json 2> gpurun_out/r37_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r37_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r37_ncu_launch.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r37_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r37_smoke.log
