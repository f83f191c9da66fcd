"""Host-side cost of the evaluation runtime's calls on the B200 (development
probe): module load / unload and ispc_launch_batch over a batch of 8 copies
of the searched-best axpy 2^26 schedule, wall clock per call against the
device time of the kernels it ran.

  python tools/launch_overhead.py [kernel.cu]
"""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1904_03383_b200 import Device, Space, _native as N  # noqa: E402
from paper_1904_03383_b200.api import compile_sources  # noqa: E402


def main():
    sp = Space("axpy", n=1 << 26, factors=[[2, 4], [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024]])
    # a fused leaf: the first leaf of a greedy descent is good enough to probe costs
    import random
    best = None
    root = sp.root()
    for seed in range(1, 400):
        try:
            leaf, _, _ = root.random_leaf(seed=seed, max_restarts=0)
            b = leaf.bound()["total"]
            src, L = leaf.nest().cuda(watchdog=1)
        except Exception:
            continue
        if best is None or b < best[0]:
            best = (b, leaf)
    leaf = best[1]
    dev = Device(0)
    dev.bind(sp.problem())
    srcs, launches = [], []
    for i in range(8):
        s, L = leaf.nest().cuda(fn_name=f"probe_k{i}", watchdog=1)
        srcs.append(s)
        launches.append(L)
    mod = compile_sources(srcs)
    out = {}
    for trial in range(6):
        t0 = time.perf_counter()
        h = dev.load(mod)
        t1 = time.perf_counter()
        items = (N.BatchItem * 8)()
        for i in range(8):
            items[i].launch = C.pointer(launches[i])
            items[i].opts = N.TimeOpts(warmup=1, reps=3, check=1, bit_exact=1, rtol=1e-5, budget_ns=50e6)
        res = (N.TimeResult * 8)()
        t2 = time.perf_counter()
        rc = N.ispc().ispc_launch_batch(dev._h, h, 8, items, float("inf"), res)
        t3 = time.perf_counter()
        rc2 = N.ispc().ispc_launch_batch(dev._h, h, 8, items, 0.0, res)  # screen only
        t4 = time.perf_counter()
        dev.unload(h)
        t5 = time.perf_counter()
        first = sum(r.first_ns for r in res) / 1e3
        out = {"load_ms": (t1 - t0) * 1e3, "batch_refine_ms": (t3 - t2) * 1e3, "batch_screen_ms": (t4 - t3) * 1e3,
               "unload_ms": (t5 - t4) * 1e3, "kernel_us_sum": first, "status": [r.status for r in res],
               "rc": (rc, rc2)}
        print({k: (round(v, 3) if isinstance(v, float) else v) for k, v in out.items()}, flush=True)


def block_dispatch():
    """Time of empty grids (each block exits at once): the per-block dispatch
    cost that makes huge grids of tiny blocks slow whatever they compute."""
    sp = Space("axpy", n=1 << 20, factors=[[2], [2]])
    dev = Device(0)
    dev.bind(sp.problem())
    src = ('extern "C" __global__ void empty_k(const unsigned long long d) '
           '{ if (ispc_now() > (d ? d : ispc_deadline_at)) ispc_timeout_flag = 1; }\n')
    mod = compile_sources([src])
    h = dev.load(mod)
    for threads in (32, 128, 1024):
        for lg in (10, 14, 16, 18, 20, 22):
            L = N.Launch()
            L.name = b"empty_k"
            L.grid_x = 1 << lg
            L.block[0], L.block[1], L.block[2] = threads, 1, 1
            L.num_params = 1
            L.params[0].kind = 2  # ISPC_PARAM_DEADLINE
            m = dev.launch(h, L, warmup=1, reps=5, check=False, budget_ns=1e9)
            print(f"empty grid 2^{lg} x {threads} threads: {m.median_ns / 1e3:.1f} us "
                  f"({m.median_ns / (1 << lg):.3f} ns/block)", flush=True)


if __name__ == "__main__":
    block_dispatch()
    main()
