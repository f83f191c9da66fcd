"""B200-native candidate-evaluation backend for the implementation-space search
of arXiv 1904.03383 (reference: "ispace", /root/reference/proj).

Layers:
  csrc/   libispc.so       C-ABI backend: sm_100a CUDA emitter, NVRTC, timed
                           launches, on-device checks (include/ispc.h)
  host/   libispc_host.so  reference-side host: reference search space linked
                           unchanged, reconstruct -> flat nest adapter, walks
                           (include/ispc_host.h)
  api.py                   Python mirror used by tests and bench.py
"""
from .api import (Candidate, DeadEnd, Device, EmitError, Measurement, Module, NestHandle, Search, Space,  # noqa: F401
                  compile_sources, tile_cuda)
from . import _native  # noqa: F401
