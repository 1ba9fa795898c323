source tools/gpu_ab.sh
build cur ""
build minb7 "-DPUV_BWD_MINB=7"
build old "" variants/k_raster_bwd_c8eed76.cu
touch $C/k_raster*.cu; make -s -C $C > /dev/null 2>&1
for r in 1 2; do for v in cur minb7 old; do
  PUV_LIB=/tmp/ab_$v.so timeout 300 python tools/ab_raster.py --reps 5 --tag $v >> gpurun_out/r12_ab.jsonl 2>> gpurun_out/r12_ab.err
done; done
