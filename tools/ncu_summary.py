#!/usr/bin/env python
"""Summarises an ncu report (`ncu -i <rep> --page raw --csv`) into the JSON
kept under profiles/: per-launch duration, DRAM bytes, throughput fractions,
pipe utilisation, occupancy. Runs here (no GPU needed).

  python tools/ncu_summary.py gpurun_out/prof_gemv.ncu-rep profiles/r01_gemv_ncu.json
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic", "launch__cluster_dim_x",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum",
    "sm__cycles_elapsed.avg.per_second", "dram__cycles_elapsed.avg.per_second",
]


def rows(rep: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    lines = [l for l in out.stdout.splitlines() if l.startswith('"')]
    rd = list(csv.reader(io.StringIO("\n".join(lines))))
    head, units, data = rd[0], rd[1], rd[2:]
    res = []
    for r in data:
        d = {}
        for k in KEYS:
            for i, h in enumerate(head):
                if h == k or h.startswith(k):
                    v = r[i].replace(",", "")
                    try:
                        v = float(v)
                    except ValueError:
                        pass
                    d[h] = {"value": v, "unit": units[i]} if units[i] else v
                    break
        res.append(d)
    return res


def main():
    rep, out = sys.argv[1], sys.argv[2]
    rs = rows(rep)
    summary = {"report": rep, "launches": rs}
    if rs:
        r = rs[0]

        def val(k):
            x = r.get(k)
            return x["value"] if isinstance(x, dict) else x

        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}

        def nbytes(k):
            x = r.get(k)
            if not isinstance(x, dict):
                return None
            return x["value"] * scale.get(x["unit"], 1)

        rd, wr = nbytes("dram__bytes_read.sum"), nbytes("dram__bytes_write.sum")
        if rd is not None and wr is not None:
            summary["dram_bytes_per_launch"] = rd + wr
        t = r.get("gpu__time_duration.sum")
        if isinstance(t, dict):
            summary["duration_us"] = t["value"] * {"ns": 1e-3, "us": 1, "ms": 1e3, "s": 1e6}.get(t["unit"], 1)
        summary["kernel"] = val("Kernel Name")
    json.dump(summary, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k != "launches"}))


if __name__ == "__main__":
    main()
