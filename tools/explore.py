#!/usr/bin/env python
"""Runs the bound-pruned search on one building-block space on a B200 and
prints the best kernel found, its re-timed speed and the cuBLAS reference on
the same shape (torch -> cuBLAS, fp32, TF32 off). Development tool; the
judged numbers come from bench.py.

  python tools/explore.py gemv 4096 4096 --evals 96
  python tools/explore.py sgemm 1024 1024 1024 --evals 96
  python tools/explore.py batched 32 32 64 --batch 512
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("kind")
    ap.add_argument("dims", type=int, nargs="+")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--evals", type=int, default=64)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--log", default=None)
    a = ap.parse_args()
    from paper_1904_03383_b200 import Search, Space
    from paper_1904_03383_b200.measure import retime_best, cublas_reference

    m, n = a.dims[0], a.dims[1]
    k = a.dims[2] if len(a.dims) > 2 else 0
    space = Space(a.kind, m=m, n=n, k=k, batch=a.batch)
    s = Search(space, device=0, seed=a.seed, reps=3, warmup=1, log_path=a.log,
               flush_l2=a.kind in ("gemv", "batched", "axpy"))
    s.step(a.evals)
    st = s.stats()
    best = s.best()
    src = s.best_source()
    s.close()
    out = {"kind": a.kind, "shape": [m, n, k, a.batch], "stats": {x: st[x] for x in (
        "evaluations", "ok", "mismatches", "timeouts", "launch_errors", "illegal", "compile_errors",
        "duplicates", "rollouts", "dead_rollouts", "pruned_children", "bound_violations", "best_ns",
        "best_bound_ns", "time_to_best_s", "elapsed_s", "exhausted")}}
    if best is not None:
        out["best"] = retime_best(space, best)
        out["best"]["config"] = best.tiles().as_dict()
    out["cublas"] = cublas_reference(space)
    print(json.dumps(out))
    if src:
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        with open(os.path.join(ROOT, "gpurun_out", f"best_{a.kind}.cu"), "w") as f:
            f.write(src)


if __name__ == "__main__":
    main()
