#!/usr/bin/env python
"""Times hand-picked gemv building-block configurations (rotation timing) to
map the achievable region of the space on a B200 (development tool)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CFGS = [
    # the r16-r22 searches' best (DIRECT, one-tile-per-CTA)
    dict(staging="DIRECT", cache="NONE", vec=2, lanes_m=8, warps_m=1, warps_n=32, split=1, unroll=8),
    dict(staging="DIRECT", cache="L1", xreduce="SHARED", vec=4, lanes_m=16, warps_m=2, warps_n=16, split=8, unroll=2),
    # balanced row blocks: 37 clusters (x 8 or x 4) of ceil(4096 / 37) -> 112 rows
    dict(staging="DIRECT", cache="NONE", vec=4, lanes_m=32, warps_m=1, warps_n=32, split=8, unroll=4, grid=296),
    dict(staging="DIRECT", cache="NONE", vec=4, lanes_m=32, warps_m=1, warps_n=32, split=8, unroll=8, grid=296),
    dict(staging="DIRECT", cache="NONE", vec=4, lanes_m=32, warps_m=1, warps_n=32, split=8, unroll=16, grid=296),
    dict(staging="DIRECT", cache="STREAM", vec=4, lanes_m=32, warps_m=1, warps_n=32, split=8, unroll=8, grid=296),
    dict(staging="DIRECT", cache="L1", vec=4, lanes_m=32, warps_m=1, warps_n=32, split=8, unroll=8, grid=296),
    dict(staging="DIRECT", cache="NONE", vec=4, lanes_m=32, warps_m=1, warps_n=16, split=8, unroll=8, grid=296),
    dict(staging="DIRECT", cache="NONE", vec=2, lanes_m=32, warps_m=2, warps_n=16, split=8, unroll=8, grid=296),
    dict(staging="DIRECT", cache="NONE", vec=1, lanes_m=32, warps_m=4, warps_n=8, split=8, unroll=16, grid=296),
    dict(staging="DIRECT", cache="NONE", vec=4, lanes_m=32, warps_m=1, warps_n=32, split=4, unroll=8, grid=148),
    dict(staging="DIRECT", cache="NONE", vec=4, lanes_m=32, warps_m=1, warps_n=32, split=4, unroll=16, grid=148),
    dict(staging="DIRECT", cache="NONE", vec=2, lanes_m=32, warps_m=1, warps_n=32, split=8, unroll=8, grid=592),
    dict(staging="DIRECT", cache="NONE", vec=2, lanes_m=32, warps_m=1, warps_n=16, split=8, unroll=8, grid=592),
]


def main():
    from paper_1904_03383_b200 import DeadEnd, Device, Space
    from paper_1904_03383_b200.measure import roofline, rotation
    space = Space("gemv", m=4096, n=4096)
    dev = Device(0)
    dev.bind(space.problem())
    rot = rotation(space, dev.info()["l2_bytes"])
    for cfg in CFGS:
        c = space.root()
        try:
            for k, v in cfg.items():
                if k in ("staging", "cache", "xreduce"):
                    c.decide(k, ["kernel"], v)
                else:
                    c.decide("tile", [k], str(v))
            t = c.first_leaf().tiles()
        except DeadEnd as e:
            print(json.dumps({"cfg": cfg, "dead_end": str(e)}))
            continue
        m = dev.evaluate_tiles(t, reps=24, warmup=3, rotate=rot)
        r = roofline(space, m.median_ns) if m.status == "ok" else {}
        print(json.dumps({"cfg": {k: v for k, v in t.as_dict().items() if k not in ("m", "n", "k", "batch")},
                          "status": m.status, "us": round(m.median_ns / 1e3, 2), "frac": r.get("frac")}), flush=True)
    dev.close()


if __name__ == "__main__":
    main()
