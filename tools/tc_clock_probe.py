#!/usr/bin/env python
"""Runs one tcgen05 sgemm variant back to back for a few seconds while
nvidia-smi samples the SM clock and power (does a smaller persistent grid run
at a higher clock?). Development tool:
  python tools/tc_clock_probe.py grid=128 split=2 bn=256 stages=6"""
from __future__ import annotations

import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_1904_03383_b200 import Device, Space
    space = Space("sgemm_tc", m=4096, n=4096, k=4096)
    c = space.root().decide("engine", ["kernel"], "TF32").decide("staging", ["kernel"], "TMA")
    for kv in sys.argv[1:]:
        k, v = kv.split("=")
        c.decide("tile", [k], v)
    t = c.first_leaf().tiles()
    dev = Device(0)
    dev.bind(space.problem())
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                            "-lms", "100"], stdout=subprocess.PIPE, text=True)
    t0 = time.time()
    times = []
    while time.time() - t0 < 6:
        r = dev.evaluate_tiles(t, reps=48, warmup=2, rotate=3)
        times.append(r.median_ns / 1e3)
    smi.terminate()
    rows = [l.split(",") for l in smi.stdout.read().strip().splitlines()[5:]]
    clk = sorted(float(r[0]) for r in rows if len(r) == 2)
    pw = sorted(float(r[1]) for r in rows if len(r) == 2)
    dev.close()
    print(json.dumps({"args": sys.argv[1:], "us_median": round(sorted(times)[len(times) // 2], 1),
                      "sm_mhz_median": clk[len(clk) // 2] if clk else None,
                      "power_w_median": pw[len(pw) // 2] if pw else None, "samples": len(clk)}))


if __name__ == "__main__":
    main()
