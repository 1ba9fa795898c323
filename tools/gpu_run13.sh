source tools/gpu_ab.sh
build cur ""
build minb0 "-DPUV_BWD_MINB=0"
build bb64 "-DPUV_BWD_BATCH=64"
build m0bb64 "-DPUV_BWD_MINB=0 -DPUV_BWD_BATCH=64"
build fb64 "-DPUV_FWD_BATCH=64"
build fb256 "-DPUV_FWD_BATCH=256"
touch $C/k_raster*.cu; make -s -C $C > /dev/null 2>&1
for r in 1 2; do for v in cur minb0 bb64 m0bb64 fb64 fb256; do
  PUV_LIB=/tmp/ab_$v.so timeout 300 python tools/ab_raster.py --reps 4 --tag $v >> gpurun_out/r13_ab.jsonl 2>> gpurun_out/r13_ab.err
done; done
