#!/usr/bin/env python
"""Times hand-picked FFMA sgemm building-block configurations at 1024^3
(rotation timing) to map what the emitter can reach (development tool)."""
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_1904_03383_b200 import DeadEnd, Device, Space
    from paper_1904_03383_b200.measure import rotation
    space = Space("sgemm", m=1024, n=1024, k=1024)
    dev = Device(0)
    dev.bind(space.problem())
    rot = rotation(space, dev.info()["l2_bytes"])
    shapes = [(16, 16, 8, 8), (16, 8, 8, 8), (8, 16, 8, 8), (8, 8, 8, 8), (32, 8, 4, 8), (16, 16, 4, 8),
              (16, 4, 16, 8), (32, 4, 8, 8), (16, 16, 8, 4)]
    bks = tuple(int(x) for x in os.environ.get("PROBE_BK", "8,16").split(","))
    for (tx, ty, tm, tn), bk, st, split, staging in itertools.product(shapes, bks, (2, 3), (1, 2, 4),
                                                                       ("CP_ASYNC", "SHARED")):
        if staging == "SHARED" and st != 2:
            continue
        c = space.root()
        try:
            c.decide("staging", ["kernel"], staging)
            for k, v in dict(thr_m=tx, thr_n=ty, tm=tm, tn=tn, bk=bk, stages=st if staging == "CP_ASYNC" else 1,
                             vec=4, split=split).items():
                c.decide("tile", [k], str(v))
            t = c.first_leaf().tiles()
        except (DeadEnd, ValueError) as e:
            continue
        m = dev.evaluate_tiles(t, reps=16, warmup=2, rotate=rot)
        us = m.median_ns / 1e3
        print(json.dumps({"thr": [tx, ty], "t": [tm, tn], "bk": bk, "stages": st, "split": split, "staging": staging,
                          "status": m.status, "us": round(us, 2), "tflops": round(2 * 1024 ** 3 / us / 1e6, 1)}),
              flush=True)
    dev.close()


if __name__ == "__main__":
    main()
