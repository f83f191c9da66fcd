#!/usr/bin/env python
"""Runs TMA-staged gemv configurations on a B200 and prints the failing ones
with their per-row error pattern (development tool)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_1904_03383_b200 import DeadEnd, Device, Space
    space = Space("gemv", m=4096, n=4096)
    dev = Device(0)
    dev.bind(space.problem())
    exp = dev.read("y", 4096, expected=True)
    root = space.root().decide("staging", ["kernel"], "TMA")
    bad = 0
    for seed in range(80):
        try:
            leaf, _, _ = root.random_leaf(seed)
        except DeadEnd:
            continue
        t = leaf.tiles()
        m = dev.evaluate_tiles(t, reps=1, warmup=0)
        if m.status == "illegal":
            continue
        y = dev.read("y", 4096)
        rows = np.nonzero(np.abs(y - exp) > 1e-3 * (np.abs(exp) + 1))[0]
        d = t.as_dict()
        print(json.dumps({"status": m.status, "bad_rows": int(rows.size), "first": rows[:8].tolist(),
                          **{k: d[k] for k in ("vec", "lanes_m", "lanes_n", "warps_m", "warps_n", "split", "bk",
                                               "stages", "xreduce")}}), flush=True)
        bad += m.status != "ok"
    # the two configurations that failed before the proxy fence, ten times each
    for cfg in ({"vec": "2", "lanes_m": "1", "warps_m": "8", "warps_n": "1", "split": "2", "bk": "64", "stages": "4"},
                {"vec": "4", "lanes_m": "2", "warps_m": "4", "warps_n": "8", "split": "8", "bk": "128", "stages": "3"}):
        c = space.root().decide("staging", ["kernel"], "TMA").decide("xreduce", ["kernel"], "SHUFFLE")
        for k, v in cfg.items():
            c.decide("tile", [k], v)
        t = c.first_leaf().tiles()
        res = []
        for _ in range(10):
            m = dev.evaluate_tiles(t, reps=1, warmup=0)
            res.append((m.status, m.mismatches))
        print(json.dumps({"cfg": cfg, "runs": res}), flush=True)
    dev.close()
    print("bad", bad)


if __name__ == "__main__":
    main()
