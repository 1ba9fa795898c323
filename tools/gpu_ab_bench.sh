# A/B of whole-step time between library builds (through gpurun): builds each variant with EXTRA
# nvcc defines into /tmp/ab_NAME.so, then runs the bench interleaved (PUV_LIB), ROUNDS times.
# Usage: VARIANTS="base:-DPUV_BIN_PRIORITY=0 prio: two:-DA=1,-DB=2" bash tools/gpu_ab_bench.sh
# (a variant's flags are comma-separated)
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
    PUV_LIB=/tmp/ab_$name.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-serial ${BENCH_ARGS:-} > /tmp/ab_out.json 2>/tmp/ab_err.txt
    python -c "import json,sys; d=json.loads(open('/tmp/ab_out.json').read().strip().splitlines()[-1]); print('$name', round(d['ms_per_step'],2), {k: v for k, v in d['stage_ms_per_step'].items() if k in ('raster_fwd','raster_bwd','project','project_bwd')})" | tee -a gpurun_out/ab.log
  done
done
