#!/usr/bin/env python
"""Development probe: the headline's best axpy 2^26 schedule (gpurun_out/
best_axpy.json, or the smoke's fused vectorised schedule) re-timed with and
without programmatic dependent launch (ISPC_PARITY_PDL=1), rotation timing."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    from paper_1904_03383_b200 import Device, Space
    from paper_1904_03383_b200.measure import rotation
    space = Space("axpy", n=bench.N_AXPY, factors=bench.FACTORS)
    best = json.load(open(os.path.join(ROOT, "profiles", "r2x_best_axpy.json")))
    cand = space.deserialize(best["candidate"])
    dev = Device(0)
    dev.bind(space.problem())
    rot = rotation(space, dev.info()["l2_bytes"])
    for rep in range(3):
        for mode in ("0", "1"):
            os.environ["ISPC_PARITY_PDL"] = mode
            m = dev.evaluate(cand.nest(), watchdog=0, reps=40, warmup=3, rotate=rot)
            m2 = dev.evaluate(cand.nest(), reps=40, warmup=3, rotate=rot)
            print(json.dumps({"pdl": mode, "no_watchdog": [m.status, round(m.median_ns / 1e3, 2)],
                              "watchdog": [m2.status, round(m2.median_ns / 1e3, 2)]}), flush=True)
    dev.close()


if __name__ == "__main__":
    main()
