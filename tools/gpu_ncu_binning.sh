# ncu --set full of one view's binning chain (depth sort K3 + level-1 tile pass K2/K4) and the loss
# kernel K10: the first 16 launches of those kernels in a short bench run, summarised per kernel.
set -u
mkdir -p gpurun_out
make -s -C paper_2602_23040_b200/csrc > /dev/null 2>&1; make -s -C oracle > /dev/null 2>&1
TAG=${TAG:-r2}
K='regex:k_os_|k_bin_prep|k_koff_|k_block_starts|k_tile_count|k_col_scan|k_tile_ranges|k_tile_scatter|k_view_finalize2|k_scan_bsum|k_l2_loss'
timeout 1200 ncu -f --set full --clock-control none -k "$K" -c 16 -o /tmp/${TAG}_bin \
  python bench.py --steps 1 --warmup 1 --views 8 --no-e2e --no-cpu-baseline --no-serial > gpurun_out/${TAG}_ncu_bin.log 2>&1
python tools/ncu_kernels.py /tmp/${TAG}_bin.ncu-rep > gpurun_out/${TAG}_ncu_binning.md 2>&1
cat gpurun_out/${TAG}_ncu_binning.md
