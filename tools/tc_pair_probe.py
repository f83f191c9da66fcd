#!/usr/bin/env python
"""Development probe: tcgen05 pair kernels with the peer's TMA completion
relayed by a lane (default) or signalled straight to the leader's barrier
(ISPC_TC_PAIR_TMA=direct, cta_group::2 TMA); small shape read back against
the oracle first, then 4096^3 timing (round 2)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

CFGS = [dict(staging="TMA", engine="TF32", bn=256, stages=7, split=2, grid=148),
        dict(staging="TMA", engine="TF32", bn=256, stages=7, split=2, grid=128),
        dict(staging="TMA", engine="TF32", bn=256, stages=7, split=4, grid=128),
        dict(staging="TMA", engine="TF32", bn=256, stages=7, split=2, grid=0),
        dict(staging="TMA", engine="TF32", bn=256, stages=4, split=2, grid=0),
        dict(staging="TMA", engine="TF32", bn=256, stages=5, split=2, grid=148),
        dict(staging="TMA", engine="TF32", bn=256, stages=6, split=2, grid=128),
        dict(staging="TMA", engine="TF32", bn=256, stages=6, split=2, grid=148),
        dict(staging="TMA", engine="TF32", bn=128, stages=6, split=2, grid=148),
        dict(staging="TMA", engine="TF32", bn=256, stages=6, split=4, grid=128)]


def main():
    import numpy as np

    from paper_1904_03383_b200 import Device, Space
    from paper_1904_03383_b200 import _native as N
    from paper_1904_03383_b200.measure import rotation
    from pdl_probe import config
    dev = Device(0)
    l2 = dev.info()["l2_bytes"]
    for shape, reps in ((dict(m=512, n=512, k=256), 2), (dict(m=4096, n=4096, k=4096), 6)):
        space = Space("sgemm_tc", **shape)
        dev.bind(space.problem())
        rot = rotation(space, l2)
        for f in CFGS:
            row = {"shape": shape["m"], **f}
            for mode in os.environ.get("TC_MODES", "relay,direct").split(","):
                os.environ["ISPC_TC_PAIR_TMA"] = mode
                m = dev.evaluate_tiles(config(N, "sgemm_tc", shape, f, 1), reps=reps, warmup=2, rotate=rot)
                row[mode] = [m.status, round(m.median_ns / 1e3, 2), m.max_err]
            print(json.dumps(row), flush=True)
    dev.close()


if __name__ == "__main__":
    main()
