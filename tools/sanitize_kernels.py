#!/usr/bin/env python
"""Runs one small kernel of every family once through the C-ABI, for
compute-sanitizer (memcheck / racecheck / synccheck). Development tool:

  compute-sanitizer --tool racecheck python tools/sanitize_kernels.py [family ...]

Families: parity (a loop-nest schedule with shared-memory temporaries and
barriers), gemv_tma (TMA ring with full/empty mbarriers), gemv_cluster
(DSMEM split), sgemm_split (split-K over a cluster through DSMEM),
sgemm_wt (warp-tiled FFMA2 cp.async ring), tc_pair (tcgen05 cta_group::2),
tc_persistent (tcgen05 persistent grid, double-buffered TMEM accumulator).
Prints one line per kernel with its status; the sanitizer writes its own
report."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1904_03383_b200 import Device, Space  # noqa: E402


def tiles_leaf(space, decisions):
    c = space.root()
    for (choice, arg), value in decisions.items():
        c.decide(choice, [arg], str(value))
    return c.first_leaf().tiles()


def parity(dev):
    """A small axpy schedule of the reference space (bound 1 us) that stages
    a temporary in shared memory behind __syncthreads: seeded uniform descent
    28293 in the paper's decision order (found by scanning seeds)."""
    space = Space("axpy", n=1 << 12, factors=[[2, 4], [2, 4, 8, 16, 32, 64]])
    leaf, _, _ = space.root().random_leaf(28293, order="size,dim_kind,thread_level,mem_space,order,cache")
    nest = leaf.nest()
    src, _ = nest.cuda("probe")
    assert "__syncthreads()" in src and "__shared__" in src
    dev.bind(space.problem())
    return dev.evaluate(nest, watchdog=0, reps=1, warmup=0)


def first_emittable(space, decisions, tries=400):
    """The first seeded random leaf under `decisions` the emitter accepts."""
    from paper_1904_03383_b200 import DeadEnd, EmitError, tile_cuda
    root = space.root()
    for (choice, arg), value in decisions.items():
        root.decide(choice, [arg], str(value))
    for seed in range(tries):
        try:
            t = root.random_leaf(seed)[0].tiles()
            tile_cuda(t, "probe")
            return t
        except (DeadEnd, EmitError):
            continue
    raise RuntimeError(f"no emittable leaf under {decisions}")


def gemv_tma(dev):
    space = Space("gemv", m=1024, n=512)
    dev.bind(space.problem())
    t = first_emittable(space, {("staging", "kernel"): "TMA"})
    return dev.evaluate_tiles(t, reps=1, warmup=0)


def gemv_cluster(dev):
    space = Space("gemv", m=512, n=256)
    dev.bind(space.problem())
    t = tiles_leaf(space, {("staging", "kernel"): "DIRECT", ("tile", "split"): 4, ("tile", "warps_n"): 2})
    return dev.evaluate_tiles(t, reps=1, warmup=0)


def sgemm_split(dev):
    space = Space("sgemm", m=128, n=128, k=128)
    dev.bind(space.problem())
    t = tiles_leaf(space, {("staging", "kernel"): "CP_ASYNC", ("tile", "split"): 2, ("tile", "thr_m"): 8,
                            ("tile", "thr_n"): 8, ("tile", "tm"): 4, ("tile", "tn"): 4, ("tile", "vec"): 4,
                            ("tile", "bk"): 16, ("tile", "stages"): 2})
    return dev.evaluate_tiles(t, reps=1, warmup=0)


def sgemm_wt(dev):
    space = Space("sgemm", m=128, n=128, k=128)
    dev.bind(space.problem())
    t = tiles_leaf(space, {("staging", "kernel"): "CP_ASYNC", ("tile", "split"): 1, ("tile", "thr_m"): 16,
                            ("tile", "thr_n"): 8, ("tile", "tm"): 8, ("tile", "tn"): 8, ("tile", "vec"): 4,
                            ("tile", "bk"): 16, ("tile", "stages"): 3})
    return dev.evaluate_tiles(t, reps=1, warmup=0)


def tc_pair(dev):
    space = Space("sgemm_tc", m=256, n=256, k=64)
    dev.bind(space.problem())
    t = tiles_leaf(space, {("engine", "kernel"): "TF32", ("staging", "kernel"): "TMA", ("tile", "split"): 2,
                            ("tile", "bn"): 64, ("tile", "stages"): 2})
    return dev.evaluate_tiles(t, reps=1, warmup=0)


def tc_persistent(dev):
    space = Space("sgemm_tc", m=2048, n=1024, k=64)
    dev.bind(space.problem())
    t = tiles_leaf(space, {("engine", "kernel"): "TF32", ("staging", "kernel"): "TMA", ("tile", "split"): 1,
                            ("tile", "bn"): 64, ("tile", "stages"): 2, ("tile", "grid"): 148})
    return dev.evaluate_tiles(t, reps=1, warmup=0)


FAMILIES = {f.__name__: f for f in (parity, gemv_tma, gemv_cluster, sgemm_split, sgemm_wt, tc_pair, tc_persistent)}


def main():
    want = sys.argv[1:] or list(FAMILIES)
    dev = Device(0)
    for name in want:
        try:
            m = FAMILIES[name](dev)
            print(f"KERNEL {name}: status={m.status} mismatches={m.mismatches} kernel={m.launch.name.decode()} "
                  f"grid={m.launch.grid_x} block={m.launch.block[0]} cluster={m.launch.cluster[0]}", flush=True)
        except Exception as e:  # noqa: BLE001 - report and continue with the next family
            print(f"KERNEL {name}: error {e}", flush=True)
    dev.close()


if __name__ == "__main__":
    main()
