#!/usr/bin/env python
"""Times every tcgen05 sgemm variant (staging x engine x pair x bn x stages)
at one shape on a B200 and checks each against the golden kernel.
Development tool: python tools/tc_variants.py 4096 4096 4096"""
from __future__ import annotations

import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_1904_03383_b200 import DeadEnd, Device, Space
    m, n, k = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (4096, 4096, 4096)
    engines = sys.argv[4].split(",") if len(sys.argv) > 4 else ["TF32", "TF32X3"]
    space = Space("sgemm_tc", m=m, n=n, k=k)
    dev = Device(0)
    dev.bind(space.problem())
    rows = []
    grids = sys.argv[5].split(",") if len(sys.argv) > 5 else ["0", "148"]
    pairs = sys.argv[6].split(",") if len(sys.argv) > 6 else ["1", "2"]
    for st, eng, pair, bn, stg, grid in itertools.product(["TMA", "SHARED"], engines, pairs, ["128", "256"],
                                                          ["2", "3", "4", "6", "8"], grids):
        c = space.root()
        try:
            c.decide("staging", ["kernel"], st).decide("engine", ["kernel"], eng).decide("tile", ["split"], pair)
            c.decide("tile", ["bn"], bn).decide("tile", ["stages"], stg).decide("tile", ["grid"], grid)
            t = c.first_leaf().tiles()
        except (DeadEnd, ValueError):
            continue
        runs = [dev.evaluate_tiles(t, reps=5, warmup=2, rotate=3) for _ in range(2)]
        r = runs[-1]
        us = min(x.median_ns for x in runs) / 1e3 if all(x.status == "ok" for x in runs) else None
        tf = 2.0 * m * n * k / (us * 1e-6) / 1e12 if us else None
        row = dict(staging=st, engine=eng, pair=pair, bn=bn, stages=stg, grid=grid, status=r.status, us=us,
                   tflops=tf and round(tf, 1), mismatches=r.mismatches, max_err=r.max_err)
        if r.status not in ("ok", "illegal"):
            row["error"] = dev.error()
        print(json.dumps(row), flush=True)
        rows.append(row)
    dev.close()


if __name__ == "__main__":
    main()
