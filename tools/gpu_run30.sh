mkdir -p gpurun_out
touch paper_2602_23040_b200/csrc/*.cu; make -s -C paper_2602_23040_b200/csrc > /dev/null 2>&1
timeout 2000 python -m pytest tests -m gpu -x -q > gpurun_out/r30_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r30_pytest.log
timeout 600 python bench.py > gpurun_out/r30_bench.json 2> gpurun_out/r30_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r30_bench_ref.json 2> gpurun_out/r30_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r30_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r30_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_raster_bwd" -c 1 -o /tmp/r30_bwd python bench.py --steps 1 --warmup 0 --views 8 --no-e2e --no-cpu-baseline > gpurun_out/r30_ncu.log 2>&1
python tools/ncu_kernels.py /tmp/r30_bwd.ncu-rep > gpurun_out/r30_ncu_bwd.md 2>&1; python tools/ncu_summary.py /tmp/r30_bwd.ncu-rep > gpurun_out/r30_ncu_bwd_detail.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_raster_fwd" -c 1 -o /tmp/r30_fwd python bench.py --steps 1 --warmup 0 --views 8 --no-e2e --no-cpu-baseline >> gpurun_out/r30_ncu.log 2>&1
python tools/ncu_kernels.py /tmp/r30_fwd.ncu-rep > gpurun_out/r30_ncu_fwd.md 2>&1; python tools/ncu_summary.py /tmp/r30_fwd.ncu-rep > gpurun_out/r30_ncu_fwd_detail.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r30_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r30_smoke.log
