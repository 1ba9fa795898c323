# GPU test suite + default bench (through gpurun, from the repo root).
set -u
mkdir -p gpurun_out
make -s -C paper_2602_23040_b200/csrc > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
make -s -C oracle >> gpurun_out/build.log 2>&1
T=${PYTEST_TIMEOUT:-2400}
timeout $T python -m pytest tests -m gpu -q -x --durations=25 ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -40 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
