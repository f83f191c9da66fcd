#!/usr/bin/env python
"""Re-runs the best kernel bench.py saved for a configuration
(gpurun_out/best_<kind>.json) through the C-ABI: 1 checked launch, 3 warm-up
launches, `--reps` timed launches, each after an L2 flush. Meant to run
under ncu, filtered to the emitted kernel (names ispc_k* / ispc_t*):

  ncu --set full --import-source on -k regex:^ispc_[kt] -s 2 -c 1 \\
      -o gpurun_out/prof_gemv python tools/profile_best.py gemv
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("kind")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--file", default=None)
    a = ap.parse_args()
    from paper_1904_03383_b200 import Device, Space
    path = a.file or os.path.join(ROOT, "gpurun_out", f"best_{a.kind}.json")
    d = json.load(open(path))
    space = Space(d["kind"], **d["space"])
    cand = space.deserialize(d["candidate"])
    dev = Device(0)
    dev.bind(space.problem())
    if space.tiles:
        m = dev.evaluate_tiles(cand.tiles(), reps=a.reps, warmup=3, flush_l2=True)
    else:
        m = dev.evaluate(cand.nest(), watchdog=0, reps=a.reps, warmup=3, flush_l2=True)
    dev.close()
    print(json.dumps({"kind": a.kind, "status": m.status, "median_us": m.median_ns / 1e3,
                      "kernel": m.launch.name.decode()}))


if __name__ == "__main__":
    main()
