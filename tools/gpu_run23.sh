mkdir -p gpurun_out
touch paper_2602_23040_b200/csrc/*.cu; make -s -C paper_2602_23040_b200/csrc > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "more_views" > gpurun_out/r23_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r23_pytest.log
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_run.py 1 > gpurun_out/r23_san_${tool}_c1.log 2>&1; echo "exit $?" >> gpurun_out/r23_san_${tool}_c1.log
done
timeout 1200 $CS --tool memcheck --error-exitcode 9 --print-limit 20 python tools/sanitize_run.py 2 2 > gpurun_out/r23_san_memcheck_c2.log 2>&1; echo "exit $?" >> gpurun_out/r23_san_memcheck_c2.log
timeout 1200 $CS --tool racecheck --error-exitcode 9 --print-limit 20 python tools/sanitize_run.py 2 1 > gpurun_out/r23_san_racecheck_c2.log 2>&1; echo "exit $?" >> gpurun_out/r23_san_racecheck_c2.log
