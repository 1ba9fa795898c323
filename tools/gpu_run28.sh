mkdir -p gpurun_out
C=paper_2602_23040_b200/csrc
touch $C/*.cu; make -s -C $C > /dev/null 2>&1; cp paper_2602_23040_b200/libpuv.so /tmp/ab_cur.so
mkdir -p /tmp/keep; for f in contract.cuh k_raster.cu k_raster_bwd.cu; do cp $C/$f /tmp/keep/$f; cp variants/head/$f $C/$f; done
touch $C/*.cu; make -s -C $C > /dev/null 2>&1; cp paper_2602_23040_b200/libpuv.so /tmp/ab_head.so
for f in contract.cuh k_raster.cu k_raster_bwd.cu; do cp /tmp/keep/$f $C/$f; done
touch $C/*.cu; make -s -C $C > /dev/null 2>&1
for r in 1 2; do for v in head cur; do
  PUV_LIB=/tmp/ab_$v.so timeout 300 python tools/ab_raster.py --reps 4 --tag $v >> gpurun_out/r28_ab.jsonl 2>> gpurun_out/r28_ab.err
done; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r28_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r28_pytest.log
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I $C tools/value_path_check.cu -o /tmp/vpc && /tmp/vpc > gpurun_out/r28_vpc.json 2>&1
