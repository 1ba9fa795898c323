# C4 and C5 bench lines (through gpurun, from the repo root).
set -u
mkdir -p gpurun_out
make -s -C paper_2602_23040_b200/csrc > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
make -s -C oracle >> gpurun_out/build.log 2>&1
for c in ${CONFIGS:-4 5}; do
  timeout 1500 python bench.py --config $c ${BENCH_ARGS:-} > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo "bench c$c exit $?"
  tail -c 2500 gpurun_out/bench_c$c.json; tail -3 gpurun_out/bench_c$c.err
done
