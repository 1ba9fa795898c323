source tools/gpu_ab.sh
build cur ""
build ks1 "-DPUV_BWD_KSKIP=1"
build ks2 "-DPUV_BWD_KSKIP=2"
touch $C/k_raster*.cu $C/api.cu; make -s -C $C > /dev/null 2>&1
for r in 1 2; do for v in cur ks1 ks2; do
  PUV_LIB=/tmp/ab_$v.so timeout 300 python tools/ab_raster.py --reps 4 --tag $v >> gpurun_out/r19_ab.jsonl 2>> gpurun_out/r19_ab.err
done; done
