source tools/gpu_ab.sh
build base ""
build pm4 "-DPUV_PROJ_MINB=4"
build pm3 "-DPUV_PROJ_MINB=3"
build wk16 "-DPUV_WALK_CTAS_PER_SM=16"
touch $C/*.cu; make -s -C $C > /dev/null 2>&1
for r in 1 2; do for v in base pm4 pm3 wk16; do
  PUV_LIB=/tmp/ab_$v.so timeout 300 python tools/ab_raster.py --reps 4 --tag $v >> gpurun_out/r35_ab.jsonl 2>> gpurun_out/r35_ab.err
done; done
