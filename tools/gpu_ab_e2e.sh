# A/B of the end-to-end (host-buffer) step between library builds, like gpu_ab_bench.sh but timing
# the bench's e2e leg too.  Usage: VARIANTS="c4:-DPUV_TEXEL_CHUNKS=4 c8:-DPUV_TEXEL_CHUNKS=8" bash tools/gpu_ab_e2e.sh
set -u
mkdir -p gpurun_out
C=paper_2602_23040_b200/csrc
make -s -C oracle > /dev/null 2>&1
for v in $VARIANTS; do
  name=${v%%:*}; flags=${v#*:}; flags=${flags//,/ }
  touch $C/*.cu; make -s -C $C EXTRA="$flags" > /tmp/ab_build_$name.log 2>&1 || { cat /tmp/ab_build_$name.log; exit 1; }
  cp paper_2602_23040_b200/libpuv.so /tmp/ab_$name.so
done
for r in $(seq ${ROUNDS:-2}); do
  for v in $VARIANTS; do
    name=${v%%:*}
    PUV_LIB=/tmp/ab_$name.so timeout 600 python bench.py --no-cpu-baseline --no-serial ${BENCH_ARGS:-} > /tmp/ab_out.json 2>/tmp/ab_err.txt
    python -c "import json; d=json.loads(open('/tmp/ab_out.json').read().strip().splitlines()[-1]); print('$name', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1))" | tee -a gpurun_out/ab_e2e.log
  done
done
