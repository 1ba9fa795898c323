source tools/gpu_ab.sh
build base ""
build fm6 "-DPUV_FWD_MINB=6"
build fm5 "-DPUV_FWD_MINB=5"
touch $C/*.cu; make -s -C $C > /dev/null 2>&1
for r in 1 2; do for v in base fm6 fm5; do
  PUV_LIB=/tmp/ab_$v.so timeout 300 python tools/ab_raster.py --reps 4 --tag $v >> gpurun_out/r27_ab.jsonl 2>> gpurun_out/r27_ab.err
done; done
