source tools/gpu_ab.sh
build cur ""
build bb32 "-DPUV_BWD_BATCH=32"
build shfl "-DPUV_BWD_SHFL"
build shflbb32 "-DPUV_BWD_SHFL -DPUV_BWD_BATCH=32"
build bb128 "-DPUV_BWD_BATCH=128"
touch $C/k_raster*.cu; make -s -C $C > /dev/null 2>&1
for r in 1 2; do for v in cur bb32 shfl shflbb32 bb128; do
  PUV_LIB=/tmp/ab_$v.so timeout 300 python tools/ab_raster.py --reps 4 --tag $v >> gpurun_out/r14_ab.jsonl 2>> gpurun_out/r14_ab.err
done; done
