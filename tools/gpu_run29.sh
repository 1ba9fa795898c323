source tools/gpu_ab.sh
build on ""
build off "-DPUV_DMASK=0"
build cap384 "-DPUV_DMASK_CAP=384"
touch $C/*.cu; make -s -C $C > /dev/null 2>&1
for r in 1 2; do for v in off on cap384; do
  PUV_LIB=/tmp/ab_$v.so timeout 300 python tools/ab_raster.py --reps 4 --tag $v >> gpurun_out/r29_ab.jsonl 2>> gpurun_out/r29_ab.err
done; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -x -q > gpurun_out/r29_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r29_pytest.log
