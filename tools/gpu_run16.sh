source tools/gpu_ab.sh
build lean ""
build leanm10 "-DPUV_BWD_MINB=10"
build leanm9 "-DPUV_BWD_MINB=9"
touch $C/k_raster*.cu; make -s -C $C > /dev/null 2>&1
for r in 1 2; do for v in lean leanm10 leanm9; do
  PUV_LIB=/tmp/ab_$v.so timeout 300 python tools/ab_raster.py --reps 4 --tag $v >> gpurun_out/r16_ab.jsonl 2>> gpurun_out/r16_ab.err
done; done
