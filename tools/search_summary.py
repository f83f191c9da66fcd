#!/usr/bin/env python
"""Summarises tools/search_experiment.sh output: per setting the median and
spread of the best kernel time, evaluations/s and time to best."""
import json
import statistics
import sys

cur, res = None, {}
for line in open(sys.argv[1]):
    if line.startswith("setting="):
        cur = line.split(" seed=")[0][len("setting="):]
    elif line.startswith("{"):
        res.setdefault(cur, []).append(json.loads(line))
for k, v in res.items():
    b = sorted(d["best_us"] for d in v)
    print(f"{k:45s} n={len(v)} best_us median {statistics.median(b):7.1f} all {[round(x) for x in b]} "
          f"evals/s {statistics.mean(d.get('evals_per_s', 0) for d in v):5.1f} "
          f"ttb_s {statistics.median(d['time_to_best_s'] for d in v):4.1f}")
