#!/usr/bin/env python
"""Runs one tcgen05 sgemm variant (decisions on the command line) for ncu:
  ncu --set full -k regex:^ispc_t -s 3 -c 1 -o out python tools/profile_tc.py \\
      4096 4096 4096 staging=SHARED engine=TF32 split=1 bn=256 stages=2
Development tool."""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_1904_03383_b200 import Device, Space
    m, n, k = (int(x) for x in sys.argv[1:4])
    space = Space("sgemm_tc", m=m, n=n, k=k)
    c = space.root()
    for kv in sys.argv[4:]:
        key, val = kv.split("=")
        if key in ("staging", "engine"):
            c.decide(key, ["kernel"], val)
        else:
            c.decide("tile", [key], val)
    t = c.first_leaf().tiles()
    dev = Device(0)
    dev.bind(space.problem())
    r = dev.evaluate_tiles(t, reps=3, warmup=2, rotate=3)
    dev.close()
    print(json.dumps({"status": r.status, "median_us": r.median_ns / 1e3, "kernel": r.launch.name.decode(),
                      "mismatches": r.mismatches}))


if __name__ == "__main__":
    main()
