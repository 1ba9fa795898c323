source tools/gpu_ab.sh
build cur ""
build fm8 "-DPUV_FWD_MINB=8"
build bppt2 "-DPUV_BWD_PPT=2"
touch $C/k_raster*.cu; make -s -C $C > /dev/null 2>&1
for r in 1 2; do for v in cur fm8 bppt2; do
  PUV_LIB=/tmp/ab_$v.so timeout 300 python tools/ab_raster.py --reps 4 --tag $v >> gpurun_out/r15_ab.jsonl 2>> gpurun_out/r15_ab.err
done; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rho.py tests/test_gpu_shard.py -x -q > gpurun_out/r15_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r15_pytest.log
