# A/B helper, sourced by a driver script run through gpurun: `build NAME "FLAGS" [SRC]` compiles libpuv with
# extra nvcc defines (or a replacement k_raster_bwd.cu) into /tmp/ab_NAME.so; time each with
#   PUV_LIB=/tmp/ab_NAME.so python tools/ab_raster.py --tag NAME   (interleave builds to cancel box drift)
set -u
mkdir -p gpurun_out
C=paper_2602_23040_b200/csrc
build() {  # name, extra flags, optional replacement source for k_raster_bwd.cu
  if [ -n "${3:-}" ]; then cp $C/k_raster_bwd.cu /tmp/bwd_keep.cu; cp $3 $C/k_raster_bwd.cu; fi
  touch $C/*.cu; make -s -C $C EXTRA="$2" > /tmp/ab_build_$1.log 2>&1; cp paper_2602_23040_b200/libpuv.so /tmp/ab_$1.so
  if [ -n "${3:-}" ]; then cp /tmp/bwd_keep.cu $C/k_raster_bwd.cu; fi
}
