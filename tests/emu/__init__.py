"""Runs an emitted ispc kernel on the CPU (one std::thread per CUDA thread,
std::barrier for __syncthreads) — TEST INFRASTRUCTURE ONLY. Lets the CPU test
suite check emitted CUDA semantics (value flow, barriers, vector lanes)
against the oracle without a GPU; the GPU tests then check the same kernels
on a B200."""
from __future__ import annotations

import ctypes as C
import hashlib
import os
import subprocess
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
CACHE = os.path.join(tempfile.gettempdir(), "ispc_emu_cache")


def _entry(launch) -> str:
    args = []
    for i in range(launch.num_params):
        p = launch.params[i]
        if p.kind == 0:
            args.append(f"(float*)a[{i}]")
        elif p.kind == 1:
            args.append(f"*(float*)a[{i}]")
        else:
            args.append(f"*(unsigned long long*)a[{i}]")
    name = launch.name.decode()
    b = list(launch.block)
    return (f'extern "C" int emu_entry(void** a) {{\n'
            f'  return emu_launch({launch.grid_x}u, {b[0]}u, {b[1]}u, {b[2]}u, [&] {{ {name}({", ".join(args)}); }});\n'
            f'}}\n')


def build(src: str, launch) -> C.CDLL:
    text = f'#include "{HERE}/cuda_emu.hpp"\n' + src + "\n" + _entry(launch)
    key = hashlib.sha1(text.encode()).hexdigest()[:16]
    os.makedirs(CACHE, exist_ok=True)
    so = os.path.join(CACHE, f"k_{key}.so")
    if not os.path.exists(so):
        cpp = os.path.join(CACHE, f"k_{key}.cpp")
        with open(cpp, "w") as f:
            f.write(text)
        subprocess.run(["g++", "-std=c++20", "-O1", "-fPIC", "-shared", "-pthread", "-ffp-contract=off",
                        "-Wno-unknown-pragmas", "-w", "-o", so + ".tmp", cpp], check=True)
        os.replace(so + ".tmp", so)
    lib = C.CDLL(so)
    lib.emu_entry.argtypes = [C.POINTER(C.c_void_p)]
    lib.emu_entry.restype = C.c_int
    return lib


def run(src: str, launch, regions: dict[str, np.ndarray], alpha: float = 1.5) -> dict[str, np.ndarray]:
    """Executes the kernel; `regions` maps problem region names to float32
    arrays (outputs are modified in place). Temporaries get NaN scratch."""
    lib = build(src, launch)
    keep = []
    ptrs = (C.c_void_p * max(launch.num_params, 1))()
    for i in range(launch.num_params):
        p = launch.params[i]
        if p.kind == 0:
            name = p.name.decode()
            if p.is_input:
                arr = regions[name]
            else:
                arr = np.full(p.elems, np.nan, dtype=np.float32)
            keep.append(arr)
            ptrs[i] = arr.ctypes.data
        elif p.kind == 1:
            v = C.c_float(alpha)
            keep.append(v)
            ptrs[i] = C.cast(C.pointer(v), C.c_void_p)
        else:
            v = C.c_uint64(2 ** 63)
            keep.append(v)
            ptrs[i] = C.cast(C.pointer(v), C.c_void_p)
    rc = lib.emu_entry(ptrs)
    if rc == 1:
        raise RuntimeError("emulated kernel deadlocked at a barrier")
    if rc == 2:
        raise TooLong("kernel exceeds the emulation budget of barrier phases")
    return regions


class TooLong(Exception):
    pass
