#!/usr/bin/env python
"""Times hand-picked batched-sgemm building-block configurations
(512 x 32x32x64, rotation timing) to map the achievable region
(development tool)."""
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_1904_03383_b200 import DeadEnd, Device, Space
    from paper_1904_03383_b200.measure import rotation
    space = Space("batched", m=32, n=32, k=64, batch=512)
    dev = Device(0)
    dev.bind(space.problem())
    rot = rotation(space, dev.info()["l2_bytes"])
    for staging, (tm, tn), pc, vec, cache, bk in itertools.product(
            ("CP_ASYNC", "SHARED", "DIRECT"), ((1, 1), (1, 2), (2, 2), (2, 4), (4, 4), (2, 8)), (1, 2, 4),
            (2, 4), ("L1", "L2"), (16, 64)):
        if staging == "CP_ASYNC" and bk != 64:
            continue
        c = space.root()
        try:
            c.decide("staging", ["kernel"], staging).decide("cache", ["kernel"], cache)
            for k, v in dict(tm=tm, tn=tn, per_cta=pc, vec=vec, bk=bk).items():
                c.decide("tile", [k], str(v))
            t = c.first_leaf().tiles()
        except (DeadEnd, ValueError):
            continue
        m = dev.evaluate_tiles(t, reps=32, warmup=3, rotate=rot)
        print(json.dumps({"staging": staging, "t": [tm, tn], "per_cta": pc, "vec": vec, "cache": cache, "bk": bk,
                          "status": m.status, "us": round(m.median_ns / 1e3, 2)}), flush=True)
    dev.close()


if __name__ == "__main__":
    main()
