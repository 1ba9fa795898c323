source tools/gpu_ab.sh
build fp4 ""
build fp0 "-DPUV_FIRST_PROJECT=0"
build fp2 "-DPUV_FIRST_PROJECT=2"
build fp8 "-DPUV_FIRST_PROJECT=8"
touch $C/k_raster*.cu $C/api.cu; make -s -C $C > /dev/null 2>&1
for r in 1 2; do for v in fp4 fp0 fp2 fp8; do
  PUV_LIB=/tmp/ab_$v.so timeout 300 python tools/ab_raster.py --reps 4 --tag $v >> gpurun_out/r21_ab.jsonl 2>> gpurun_out/r21_ab.err
done; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_configs.py -x -q > gpurun_out/r21_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r21_pytest.log
timeout 1500 ncu --set full --clock-control none -o /tmp/r21_all python bench.py --steps 1 --warmup 0 --views 4 --no-e2e --no-cpu-baseline > gpurun_out/r21_ncu.log 2>&1
python tools/ncu_kernels.py /tmp/r21_all.ncu-rep > gpurun_out/r21_all_kernels.md 2>&1
ncu -i /tmp/r21_all.ncu-rep --page raw --csv > /tmp/r21_raw.csv 2>/dev/null; gzip -c /tmp/r21_raw.csv > gpurun_out/r21_all_raw.csv.gz
