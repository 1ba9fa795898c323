source tools/gpu_ab.sh
build g1 ""
build g2 "-DPUV_FWD_GROUP=2"
build g4 "-DPUV_FWD_GROUP=4"
touch $C/k_raster*.cu $C/api.cu; make -s -C $C > /dev/null 2>&1
for r in 1 2; do for v in g1 g2 g4; do
  PUV_LIB=/tmp/ab_$v.so timeout 300 python tools/ab_raster.py --reps 4 --tag $v >> gpurun_out/r17_ab.jsonl 2>> gpurun_out/r17_ab.err
done; done
