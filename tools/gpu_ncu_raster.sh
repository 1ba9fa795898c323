# ncu --set full capture of the raster kernels (one launch each) with source correlation, summarised
# here (through gpurun).  TAG names the outputs.
set -u
mkdir -p gpurun_out
make -s -C paper_2602_23040_b200/csrc > /dev/null 2>&1; make -s -C oracle > /dev/null 2>&1
TAG=${TAG:-r2}
for k in k_raster_fwd k_raster_bwd; do
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:$k -c 1 -o /tmp/ncu_$k \
    python bench.py --steps 1 --warmup 1 --views 8 --no-e2e --no-cpu-baseline --no-serial > gpurun_out/ncu_${TAG}_$k.log 2>&1
  python tools/ncu_summary.py /tmp/ncu_$k.ncu-rep > gpurun_out/ncu_${TAG}_${k}_detail.txt 2>&1
  ncu -i /tmp/ncu_$k.ncu-rep --page source --csv --print-source=cuda,sass > /tmp/src_$k.csv 2>/dev/null
  python tools/ncu_lines.py /tmp/src_$k.csv "" 45 > gpurun_out/ncu_${TAG}_${k}_lines.txt 2>&1
done
