#!/usr/bin/env python
"""Collects one GPU round's evidence into profiles/ (tracked): the bench JSON
line, the ncu launch list aggregated per kernel family, and per-kernel ncu
summaries (tools/ncu_summary.py) of the best kernels. Runs here, no GPU.

  python tools/summarize_round.py r01
"""
from __future__ import annotations

import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def bench_line(tag: str) -> dict | None:
    p = os.path.join(OUT, f"{tag}_bench.log")
    if not os.path.exists(p):
        return None
    for line in reversed(open(p).read().splitlines()):
        if line.startswith("{"):
            return json.loads(line)
    return None


def launch_shares(tag: str) -> dict | None:
    p = os.path.join(OUT, f"{tag}_launches.csv")
    if not os.path.exists(p):
        return None
    rows = [r for r in csv.reader(open(p)) if r]
    head = None
    per = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            head = r
            continue
        if head is None or len(r) != len(head):
            continue
        d = dict(zip(head, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"]
        fam = "emitted candidate kernels (ispc_k*/ispc_t*)" if name.startswith("ispc_") else name.split("(")[0]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "nsecond")
        ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        per[fam][0] += 1
        per[fam][1] += ns
    total = sum(t for _, t in per.values()) or 1
    return {k: {"launches": n, "total_us": round(t / 1e3, 1), "share": round(t / total, 4)}
            for k, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1])}


def main():
    tag = sys.argv[1]
    os.makedirs(PROF, exist_ok=True)
    res = {"tag": tag}
    b = bench_line(tag)
    if b:
        res["bench"] = b
        json.dump(b, open(os.path.join(PROF, f"{tag}_bench.json"), "w"), indent=1)
    sh = launch_shares(tag)
    if sh:
        res["launch_shares"] = sh
        json.dump(sh, open(os.path.join(PROF, f"{tag}_launch_shares.json"), "w"), indent=1)
    for f in sorted(os.listdir(OUT)):
        if f.startswith(f"{tag}_prof_") and f.endswith(".ncu-rep"):
            k = f[len(f"{tag}_prof_"):-len(".ncu-rep")]
            rep = os.path.join(OUT, f)
            dst = os.path.join(PROF, f"{tag}_{k}_ncu.json")
            subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep, dst], check=False)
    # the bench line is written before this round's ncu captures; when one of
    # them is the headline kernel, record its DRAM traffic beside the line
    if b and b.get("roofline") and b["roofline"].get("traffic") is None:
        for f in sorted(os.listdir(PROF)):
            if f.startswith(f"{tag}_") and f.endswith("_ncu.json"):
                try:
                    j = json.load(open(os.path.join(PROF, f)))
                except (OSError, ValueError):
                    continue
                if j.get("kernel") == b["roofline"].get("kernel") and j.get("dram_bytes_per_launch"):
                    b["roofline"]["traffic"] = j["dram_bytes_per_launch"]
                    b["roofline"]["traffic_source"] = f"profiles/{f} (ncu --set full after the bench run)"
                    json.dump(b, open(os.path.join(PROF, f"{tag}_bench.json"), "w"), indent=1)
                    break
    print(json.dumps({k: v for k, v in res.items() if k != "bench"}, indent=1))


if __name__ == "__main__":
    main()
