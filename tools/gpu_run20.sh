mkdir -p gpurun_out
touch paper_2602_23040_b200/csrc/*.cu; make -s -C paper_2602_23040_b200/csrc > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none -o gpurun_out/r20_all python bench.py --steps 1 --warmup 0 --views 4 --no-e2e --no-cpu-baseline > gpurun_out/r20_ncu.log 2>&1
echo "ncu exit $?" >> gpurun_out/r20_ncu.log
