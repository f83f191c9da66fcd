#!/usr/bin/env python
"""Development probe: each building-block family's best configurations timed
with and without programmatic dependent launch (tile parameter `pdl`), with
the rotation timing the search uses and the on-device check (round 2)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

BASE = dict(staging="DIRECT", engine="FFMA", xreduce="SHUFFLE", cache="L2")
CASES = [
    ("sgemm", dict(m=1024, n=1024, k=1024), dict(staging="CP_ASYNC", cache="STREAM", thr_m=32, thr_n=8, tm=8, tn=8,
                                                 bk=16, stages=3, vec=4, split=2)),
    ("sgemm", dict(m=1024, n=1024, k=1024), dict(staging="CP_ASYNC", cache="STREAM", thr_m=16, thr_n=8, tm=8, tn=8,
                                                 bk=16, stages=3, vec=4, split=2)),
    ("sgemm", dict(m=1024, n=1024, k=1024), dict(staging="CP_ASYNC", cache="STREAM", thr_m=16, thr_n=8, tm=8, tn=8,
                                                 bk=16, stages=3, vec=4, split=1)),
    ("sgemm", dict(m=1024, n=1024, k=1024), dict(staging="CP_ASYNC", cache="STREAM", thr_m=32, thr_n=8, tm=8, tn=8,
                                                 bk=16, stages=4, vec=4, split=2)),
    ("sgemm", dict(m=1024, n=1024, k=1024), dict(staging="CP_ASYNC", cache="STREAM", thr_m=32, thr_n=8, tm=8, tn=8,
                                                 bk=16, stages=4, vec=4, split=2, lds=1)),
    ("sgemm", dict(m=1024, n=1024, k=1024), dict(staging="CP_ASYNC", cache="STREAM", thr_m=16, thr_n=8, tm=8, tn=8,
                                                 bk=16, stages=3, vec=4, split=1, lds=1)),
    ("sgemm", dict(m=1024, n=1024, k=1024), dict(staging="CP_ASYNC", cache="STREAM", thr_m=16, thr_n=8, tm=8, tn=8,
                                                 bk=16, stages=4, vec=4, split=2, lds=1)),
    ("gemv", dict(m=4096, n=4096), dict(cache="STREAM", bk=1, stages=1, vec=4, lanes_m=16, lanes_n=2, warps_m=1,
                                        warps_n=32, split=4, unroll=16)),
    ("gemv", dict(m=4096, n=4096), dict(cache="STREAM", bk=1, stages=1, vec=4, lanes_m=32, lanes_n=1, warps_m=1,
                                        warps_n=16, split=4, unroll=16)),
    ("gemv", dict(m=4096, n=4096), dict(cache="STREAM", bk=1, stages=1, vec=4, lanes_m=16, lanes_n=2, warps_m=1,
                                        warps_n=16, split=8, unroll=8)),
    ("gemv", dict(m=4096, n=4096), dict(cache="STREAM", bk=1, stages=1, vec=4, lanes_m=32, lanes_n=1, warps_m=1,
                                        warps_n=32, split=4, unroll=16)),
    ("gemv", dict(m=4096, n=4096), dict(cache="STREAM", bk=1, stages=1, vec=4, lanes_m=32, lanes_n=1, warps_m=2,
                                        warps_n=16, split=4, unroll=16)),
    ("gemv", dict(m=4096, n=4096), dict(cache="STREAM", bk=1, stages=1, vec=4, lanes_m=32, lanes_n=1, warps_m=4,
                                        warps_n=8, split=8, unroll=16)),
    ("gemv", dict(m=4096, n=4096), dict(cache="STREAM", bk=1, stages=1, vec=4, lanes_m=16, lanes_n=2, warps_m=1,
                                        warps_n=32, split=8, unroll=8)),
    ("gemv", dict(m=4096, n=4096), dict(cache="STREAM", bk=1, stages=1, vec=4, lanes_m=16, lanes_n=2, warps_m=2,
                                        warps_n=16, split=4, unroll=16)),
    ("gemv", dict(m=4096, n=4096), dict(cache="STREAM", bk=1, stages=1, vec=4, lanes_m=8, lanes_n=4, warps_m=1,
                                        warps_n=32, split=4, unroll=16)),
    ("gemv", dict(m=4096, n=4096), dict(cache="STREAM", bk=1, stages=1, vec=4, lanes_m=16, lanes_n=2, warps_m=1,
                                        warps_n=32, split=2, unroll=16)),
    ("gemv", dict(m=4096, n=4096), dict(cache="STREAM", bk=1, stages=1, vec=4, lanes_m=32, lanes_n=1, warps_m=1,
                                        warps_n=32, split=2, unroll=16)),
    ("gemv", dict(m=4096, n=4096), dict(cache="STREAM", bk=1, stages=1, vec=4, lanes_m=16, lanes_n=2, warps_m=1,
                                        warps_n=16, split=4, unroll=16)),
    ("batched", dict(m=32, n=32, k=64, batch=512), dict(staging="CP_ASYNC", tm=2, tn=8, bk=16, vec=4, per_cta=1)),
    ("batched", dict(m=32, n=32, k=64, batch=512), dict(staging="CP_ASYNC", tm=4, tn=4, bk=32, vec=4, per_cta=1)),
    ("axpy_stream", dict(n=1 << 26), dict(vec=2, unroll=2, threads=512)),
    ("axpy_stream", dict(n=1 << 26), dict(vec=4, unroll=1, threads=256)),
    ("sgemm_tc", dict(m=4096, n=4096, k=4096), dict(staging="TMA", engine="TF32", bn=256, stages=6, split=4,
                                                    grid=128)),
    ("sgemm_tc", dict(m=4096, n=4096, k=4096), dict(staging="TMA", engine="TF32", bn=256, stages=4, split=2,
                                                    grid=0)),
]


def config(N, kind, shape, fields, pdl):
    c = N.TileConfig()
    c.kind = {"gemv": N.TILE_GEMV, "sgemm": N.TILE_SGEMM, "batched": N.TILE_BATCHED, "sgemm_tc": N.TILE_SGEMM_TC,
              "axpy_stream": N.TILE_AXPY}[kind]
    f = dict(BASE, **fields)
    c.staging, c.engine = N.STAGINGS.index(f.pop("staging")), N.ENGINES.index(f.pop("engine"))
    c.xreduce, c.cache = N.XREDUCES.index(f.pop("xreduce")), N.CACHES.index(f.pop("cache"))
    for k, v in dict(shape, batch=shape.get("batch", 1)).items():
        setattr(c, k, v)
    for k, v in f.items():
        setattr(c, k, v)
    c.pdl = pdl
    return c


def main():
    from paper_1904_03383_b200 import Device, Space
    from paper_1904_03383_b200 import _native as N
    from paper_1904_03383_b200.measure import rotation
    dev = Device(0)
    l2 = dev.info()["l2_bytes"]
    kinds = os.environ.get("PROBE_KINDS")
    for kind, shape, fields in CASES:
        if kinds and kind not in kinds.split(","):
            continue
        space = Space(kind, **shape)
        dev.bind(space.problem())
        rot = rotation(space, l2)
        row = {"kind": kind, **fields}
        for pdl in (0, 1):
            m = dev.evaluate_tiles(config(N, kind, shape, fields, pdl), reps=16, warmup=3, rotate=rot)
            row[f"pdl{pdl}"] = [m.status, round(m.median_ns / 1e3, 2)]
        print(json.dumps(row), flush=True)
    dev.close()


if __name__ == "__main__":
    main()
