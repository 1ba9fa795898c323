# Round validation on one B200 (run through gpurun from the repo root):
#   gpurun --timeout 3600 -- 'bash tools/gpu_validate.sh'
# Builds libpuv for sm_100a, runs the GPU parity suite, the bench (ours + the reference arm), the
# ncu launch list of one bench step, one ncu --set full capture of each raster kernel (summaries
# only: full reports exceed gpurun's copy-back limit), and smoke().
set -u
mkdir -p gpurun_out
touch paper_2602_23040_b200/csrc/*.cu; make -s -C paper_2602_23040_b200/csrc > /dev/null 2>&1
timeout 2000 python -m pytest tests -m gpu -x -q > gpurun_out/val_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/val_pytest.log
timeout 600 python bench.py > gpurun_out/val_bench.json 2> gpurun_out/val_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/val_bench_ref.json 2> gpurun_out/val_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/val_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/val_ncu_launch.log 2>&1
for k in k_raster_bwd k_raster_fwd; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o /tmp/val_$k \
    python bench.py --steps 1 --warmup 0 --views 8 --no-e2e --no-cpu-baseline >> gpurun_out/val_ncu.log 2>&1
  python tools/ncu_kernels.py /tmp/val_$k.ncu-rep > gpurun_out/val_ncu_$k.md 2>&1
  python tools/ncu_summary.py /tmp/val_$k.ncu-rep > gpurun_out/val_ncu_${k}_detail.txt 2>&1
done
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/val_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/val_smoke.log
