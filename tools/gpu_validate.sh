# Round validation on one B200 (run through gpurun from the repo root):
#   gpurun --timeout 3600 -- 'TAG=r02 bash tools/gpu_validate.sh'
# Builds libpuv for sm_100a, runs the GPU parity suite, the bench (ours + the reference arm), the
# ncu launch list of one bench step, one ncu --set full capture of each main kernel (summaries and
# per-launch DRAM traffic -> traffic.json; full reports exceed gpurun's copy-back limit), and smoke().
set -u
TAG=${TAG:-val}
O=gpurun_out
mkdir -p $O
touch paper_2602_23040_b200/csrc/*.cu; make -s -C paper_2602_23040_b200/csrc > /dev/null 2>&1; make -s -C oracle > /dev/null 2>&1
if [ -z "${SKIP_TESTS:-}" ]; then
  timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > $O/${TAG}_pytest.log 2>&1; echo "pytest exit $?" >> $O/${TAG}_pytest.log
fi
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/${TAG}_bench_ref.json 2> $O/${TAG}_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-serial > $O/${TAG}_ncu_launch.log 2>&1
python tools/launch_summary.py $O/${TAG}_launches.csv > $O/${TAG}_launches_summary.txt 2>&1
REPS=""
for k in k_raster_fwd k_raster_bwd k_project k_project_bwd k_seg_walk k_tile_scatter; do
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:$k -c 1 -o /tmp/${TAG}_$k \
    python bench.py --steps 1 --warmup 1 --views 8 --no-e2e --no-cpu-baseline --no-serial >> $O/${TAG}_ncu.log 2>&1
  python tools/ncu_summary.py /tmp/${TAG}_$k.ncu-rep > $O/${TAG}_ncu_${k}_detail.txt 2>&1
done
python tools/ncu_kernels.py /tmp/${TAG}_k_raster_fwd.ncu-rep > $O/${TAG}_ncu_kernels.md 2>&1
for k in k_raster_bwd k_project k_project_bwd k_seg_walk k_tile_scatter; do
  python tools/ncu_kernels.py /tmp/${TAG}_$k.ncu-rep | tail -n +3 >> $O/${TAG}_ncu_kernels.md 2>&1
done
python tools/ncu_traffic.py $O/${TAG}_traffic.json raster_fwd=/tmp/${TAG}_k_raster_fwd.ncu-rep:1 \
  raster_bwd=/tmp/${TAG}_k_raster_bwd.ncu-rep:8 project=/tmp/${TAG}_k_project.ncu-rep:8 \
  project_bwd=/tmp/${TAG}_k_project_bwd.ncu-rep:8 > /dev/null 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke exit $?" >> $O/${TAG}_smoke.log
tail -3 $O/${TAG}_pytest.log 2>/dev/null; tail -c 400 $O/${TAG}_bench.json; tail -2 $O/${TAG}_smoke.log
