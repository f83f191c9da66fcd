#!/usr/bin/env python
"""Runs one FFMA sgemm configuration (decisions on the command line) for ncu:
  ncu --set full -k regex:^ispc_t -s 2 -c 1 -o out python tools/profile_sgemm.py \\
      1024 1024 1024 staging=CP_ASYNC thr_m=16 thr_n=16 tm=8 tn=8 bk=16 stages=2 vec=4 split=2
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
    space = Space("sgemm", m=m, n=n, k=k)
    c = space.root()
    for kv in sys.argv[4:]:
        key, val = kv.split("=")
        if key in ("staging", "engine", "cache", "xreduce"):
            c.decide(key, ["kernel"], val)
        else:
            c.decide("tile", [key], val)
    t = c.first_leaf().tiles()
    dev = Device(0)
    dev.bind(space.problem())
    r = dev.evaluate_tiles(t, reps=3, warmup=1)
    dev.close()
    print(json.dumps({"status": r.status, "median_us": r.median_ns / 1e3, "kernel": r.launch.name.decode()}))


if __name__ == "__main__":
    main()
