#!/usr/bin/env python
"""Read-bandwidth ceiling for the gemv shape: a hand-written kernel that only
streams A (64 MiB) and reduces it, launched through the same runtime and
rotation timing as the searched gemv kernels, over several grid shapes.
Development tool (no output check)."""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SRC = r"""
extern "C" __global__ void __launch_bounds__(%(T)d) k_read(const float* __restrict__ g_a, const float* __restrict__ g_x,
                                                       float* __restrict__ g_y) {
  const float4* a = (const float4*)g_a;
  const long long n4 = %(N4)dLL;
  const long long stride = (long long)gridDim.x * %(T)d;
  float s = 0.f;
  long long i = (long long)blockIdx.x * %(T)d + threadIdx.x;
  #pragma unroll 1
  for (; i + %(U1)d * stride < n4; i += %(U)d * stride) {
    float4 v[%(U)d];
    #pragma unroll
    for (int u = 0; u < %(U)d; ++u) v[u] = __ldcs(a + i + u * stride);
    #pragma unroll
    for (int u = 0; u < %(U)d; ++u) s += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  for (; i < n4; i += stride) { float4 v = __ldcs(a + i); s += v.x + v.y + v.z + v.w; }
  if (s == 123.456f) g_y[threadIdx.x] = s;
}
"""


def main():
    from paper_1904_03383_b200 import Device, Space, compile_sources, tile_cuda
    from paper_1904_03383_b200.measure import rotation
    m = n = 4096
    space = Space("gemv", m=m, n=n)
    dev = Device(0)
    dev.bind(space.problem())
    rot = rotation(space, dev.info()["l2_bytes"])
    base = space.root().first_leaf().tiles()
    _, L0 = tile_cuda(base, "k_base")
    for T in (256, 512, 1024):
        for per_sm in (1, 2, 4, 8, 16):
            if T * per_sm > 2048:
                continue
            for U in (2, 4, 8):
                src = SRC % dict(T=T, N4=m * n // 4, U=U, U1=U - 1)
                mod = compile_sources([src])
                h = dev.load(mod)
                L = L0
                L.name = b"k_read"
                L.grid_x = 148 * per_sm
                L.block[0], L.block[1], L.block[2] = T, 1, 1
                L.static_smem = 0
                L.cluster[0] = L.cluster[1] = L.cluster[2] = 0
                L.num_tmaps = 0
                r = dev.launch(h, L, warmup=3, reps=24, check=False, rotate=rot)
                us = r.median_ns / 1e3
                print(json.dumps({"T": T, "ctas_per_sm": per_sm, "unroll": U, "status": r.status, "us": round(us, 2),
                                  "GBs": round(m * n * 4 / (us * 1e-6) / 1e9, 1)}), flush=True)
                dev.unload(h)
    dev.close()


if __name__ == "__main__":
    main()
