source tools/gpu_ab.sh
build base ""
build seg256 "-DPUV_SEG_MIN=256"
build seg1k "-DPUV_SEG_MIN=1024"
build os8 "-DPUV_OS_ITEMS=8"
touch $C/*.cu; make -s -C $C > /dev/null 2>&1
for r in 1 2; do for v in base seg256 seg1k os8; do
  PUV_LIB=/tmp/ab_$v.so timeout 300 python tools/ab_raster.py --reps 4 --tag $v >> gpurun_out/r34_ab.jsonl 2>> gpurun_out/r34_ab.err
done; done
