mkdir -p gpurun_out
touch paper_2602_23040_b200/csrc/*.cu; make -s -C paper_2602_23040_b200/csrc > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_shard.py -x -q > gpurun_out/r25_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r25_pytest.log
for r in 1 2 3; do timeout 300 python tools/ab_raster.py --reps 4 --fused --tag fused >> gpurun_out/r25_ab.jsonl 2>> gpurun_out/r25_ab.err; done
timeout 600 python bench.py > gpurun_out/r25_bench.json 2> gpurun_out/r25_bench.err
source tools/gpu_ab.sh
build chk "-DPUV_DEBUG_CHECKS"
touch $C/*.cu; make -s -C $C > /dev/null 2>&1
PUV_LIB=/tmp/ab_chk.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_shard.py -x -q > gpurun_out/r25_pytest_checks.log 2>&1; echo "pytest exit $?" >> gpurun_out/r25_pytest_checks.log
