source tools/gpu_ab.sh
build base ""
build t128 "-DPUV_BIN_THREADS=128 -DPUV_BIN_CTAS_PER_SM=16 -DPUV_BIN_BAND_TILES=512 -DPUV_BIN_ITEM_CACHE=1024"
build t256 "-DPUV_BIN_THREADS=256 -DPUV_BIN_CTAS_PER_SM=8 -DPUV_BIN_BAND_TILES=512 -DPUV_BIN_ITEM_CACHE=1024"
build t512b "-DPUV_BIN_BAND_TILES=512 -DPUV_BIN_ITEM_CACHE=1024 -DPUV_BIN_CTAS_PER_SM=6"
touch $C/*.cu; make -s -C $C > /dev/null 2>&1
for r in 1 2; do for v in base t128 t256 t512b; do
  PUV_LIB=/tmp/ab_$v.so timeout 300 python tools/ab_raster.py --reps 4 --tag $v >> gpurun_out/r32_ab.jsonl 2>> gpurun_out/r32_ab.err
done; done
