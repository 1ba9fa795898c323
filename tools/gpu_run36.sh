source tools/gpu_ab.sh
build base ""
build bs2 "-DPUV_BIN_STREAMS=2"
build bs8 "-DPUV_BIN_STREAMS=8"
touch $C/*.cu; make -s -C $C > /dev/null 2>&1
for r in 1 2; do for v in base bs2 bs8; do
  PUV_LIB=/tmp/ab_$v.so timeout 300 python tools/ab_raster.py --reps 4 --tag $v >> gpurun_out/r36_ab.jsonl 2>> gpurun_out/r36_ab.err
done; done
