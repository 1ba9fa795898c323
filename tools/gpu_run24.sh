source tools/gpu_ab.sh
build chk "-DPUV_DEBUG_CHECKS"
touch $C/*.cu; make -s -C $C > /dev/null 2>&1
PUV_LIB=/tmp/ab_chk.so timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r24_pytest_checks.log 2>&1; echo "pytest exit $?" >> gpurun_out/r24_pytest_checks.log
PUV_LIB=/tmp/ab_chk.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/r24_bench_checks.json 2>&1
