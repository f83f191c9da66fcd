#!/usr/bin/env python
"""Times a few leaves of the reference's matmul 1024^3 gpu.space
(make_matmul(1024, 1024, 1024, {{2..32}, {2, 4}})) on the B200 without a
watchdog: the lowest-bound leaf of a greedy descent and seeded descents in
the paper's decision order. Development tool."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_1904_03383_b200 import DeadEnd, Device, EmitError, Space
    space = Space("matmul", m=1024, n=1024, k=1024, factors=[[2, 4, 8, 16, 32], [2, 4]])
    order = "size,dim_kind,thread_level,mem_space,order,cache"
    dev = Device(0)
    dev.bind(space.problem())
    leaves = []
    leaf, b = space.root().greedy_leaf(order)
    leaves.append(("greedy", leaf))
    for seed in range(1, 400):
        if len(leaves) >= 8:
            break
        try:
            l2, _, _ = space.root().random_leaf(seed, order=order)
            if l2.bound()["total"] < 1.0:
                leaves.append((f"seed{seed}", l2))
        except DeadEnd:
            continue
    for tag, l in leaves:
        try:
            src, L = l.nest().cuda()
        except (EmitError, ValueError) as e:
            print(json.dumps({"leaf": tag, "emit": str(e)[:120]}), flush=True)
            continue
        t0 = time.perf_counter()
        m = dev.evaluate(l.nest(), watchdog=0, reps=1, warmup=0)
        print(json.dumps({"leaf": tag, "status": m.status, "us": round(m.median_ns / 1e3, 1),
                          "bound_us": round(l.bound()["total"] * 1e6, 1), "grid": int(L.grid_x),
                          "block": list(L.block), "wall_s": round(time.perf_counter() - t0, 2)}), flush=True)
    dev.close()


if __name__ == "__main__":
    main()
