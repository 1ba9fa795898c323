"""PackUV-GS view-parallel differentiable splat render for B200 (sm_100a).

The hot path (atlas unpack, EWA projection, tile binning, compositing and the
backward onto atlas texels) is hand-written CUDA in `csrc/` behind the C ABI
of `include/puv.h`; `puv` is its ctypes binding and `shard` the view-sharding
layer over torch.distributed.  See DESIGN.md.
"""
from . import puv  # noqa: F401
