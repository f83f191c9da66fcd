#!/usr/bin/env python
"""Diagnoses the tcgen05 sgemm on a B200: runs the emitted kernel (and
descriptor variants made by textual substitution) on random inputs and saves
A, B, C for offline least-squares analysis (C pinv(B) recovers the A the tensor
core actually used). Development tool."""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_1904_03383_b200 import Device, Space, compile_sources, tile_cuda
    out = {}
    dev = Device(0)
    for (m, n, k) in [(128, 64, 32), (128, 64, 64), (256, 128, 128)]:
        space = Space("sgemm_tc", m=m, n=n, k=k)
        c = space.root()
        c.decide("engine", ["kernel"], "TF32")
        c.decide("tile", ["bn"], "64")
        c.decide("tile", ["stages"], "2")
        t = c.first_leaf().tiles()
        src, L = tile_cuda(t, "k_dbg")
        variants = {"v0": src, "v1_swap_a_lbo_sbo": src.replace("4096u, 1024u)", "1024u, 4096u)")}
        p = space.problem()
        dev.bind(p)
        a = dev.read("a", m * k)
        b = dev.read("b", k * n)
        out[f"{m}_{n}_{k}_a"] = a
        out[f"{m}_{n}_{k}_b"] = b
        out[f"{m}_{n}_{k}_exp"] = dev.read("c", m * n, expected=True)
        for name, s in variants.items():
            mod = compile_sources([s])
            h = dev.load(mod)
            r = dev.launch(h, L, warmup=0, reps=1, check=True, bit_exact=False, rtol=4e-3)
            out[f"{m}_{n}_{k}_{name}"] = dev.read("c", m * n)
            print(m, n, k, name, r.status, r.max_err, r.mismatches, flush=True)
            dev.unload(h)
    dev.close()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    np.savez(os.path.join(ROOT, "gpurun_out", "tc_debug.npz"), **out)


if __name__ == "__main__":
    main()
