"""Roofline bookkeeping for the BASELINE configurations: algorithmic bytes /
flops per launch, the measured peaks (MEASURED_PEAKS.json), re-timing of a
search's best kernel through the C-ABI, and cuBLAS on the same shapes (torch
-> cuBLAS, fp32 with TF32 off unless asked) for reference."""
from __future__ import annotations

import json
import os
import statistics

from . import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SMS, FP32_LANES, F_MAX_HZ = 148, 128, 1.965e9


def peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"], "sm_max_mhz": d.get("sm_max_mhz", 1965.0),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0,
            "source": "fallback (B200_PROFILING.md)"}


def work(space) -> dict:
    """Algorithmic bytes and flops of one launch of the space's kernel."""
    m, n, k, b = space.m, space.n, space.k, max(space.batch, 1)
    kind = space.kind
    if kind == "axpy":
        return {"bytes": 12 * n, "flops": 2 * n, "bound": "hbm"}
    if kind == "gemv":
        return {"bytes": 4 * (m * n + m + n), "flops": 2 * m * n, "bound": "hbm"}
    if kind == "batched":
        return {"bytes": 4 * b * (m * k + k * n + m * n), "flops": 2 * b * m * n * k, "bound": "hbm"}
    if kind in ("sgemm", "matmul"):
        return {"bytes": 4 * (m * k + k * n + m * n), "flops": 2 * m * n * k, "bound": "fp32"}
    if kind in ("sgemm_tc", "sgemm_tc_x3"):
        return {"bytes": 4 * (m * k + k * n + m * n), "flops": 2 * m * n * k, "bound": "tensor"}
    raise ValueError(kind)


def roofline(space, ns: float) -> dict:
    pk = peaks()
    w = work(space)
    if w["bound"] == "hbm":
        ach = w["bytes"] / ns  # GB/s
        return {"bound": "hbm", "achieved": round(ach, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": round(ach / pk["hbm_gbs"], 4), "algorithmic_bytes_per_launch": w["bytes"],
                "peak_source": pk["source"]}
    tf = w["flops"] / ns / 1e3  # TFLOP/s
    if w["bound"] == "fp32":
        peak = SMS * FP32_LANES * 2 * pk["sm_max_mhz"] * 1e6 / 1e12
        src = "148 SM x 128 FFMA x 2 x max SM clock (derived)"
    else:
        peak = pk["bf16_tflops"] / 2  # dense TF32 runs at half the bf16 rate
        src = "measured bf16 cuBLAS / 2 (TF32 rate)"
    return {"bound": "tensor" if w["bound"] == "tensor" else "fp32", "achieved": round(tf, 2), "peak": round(peak, 2),
            "unit": "TFLOP/s", "frac": round(tf / peak, 4), "algorithmic_flops_per_launch": w["flops"],
            "peak_source": src}


def retime_best(space, cand, reps: int = 20, dev=None, ordinal: int = 0) -> dict:
    """Re-times a candidate through the C-ABI (L2 flushed before every launch)."""
    from .api import Device
    own = dev is None
    dev = dev or Device(ordinal)
    dev.bind(space.problem())
    if space.tiles:
        m = dev.evaluate_tiles(cand.tiles(), reps=reps, warmup=3, flush_l2=True)
    else:
        m = dev.evaluate(cand.nest(), watchdog=0, reps=reps, warmup=3, flush_l2=True)
    if own:
        dev.close()
    if m.status != "ok":
        return {"status": m.status}
    r = {"status": "ok", "kernel_us": round(m.median_ns / 1e3, 3), "min_us": round(m.min_ns / 1e3, 3),
         "max_err": m.max_err, "grid": int(m.launch.grid_x), "block": list(m.launch.block)[:1][0],
         "smem": int(m.launch.static_smem), "cluster": int(m.launch.cluster[0]),
         "kernel": m.launch.name.decode()}
    r["traffic"] = traffic_of(r["kernel"])
    r["roofline"] = roofline(space, m.median_ns)
    return r


def traffic_of(kernel: str) -> float | None:
    """DRAM read+write bytes per launch of `kernel` from an ncu --set full
    capture summarised under profiles/ (None when this exact kernel was not
    captured)."""
    d = os.path.join(ROOT, "profiles")
    if not os.path.isdir(d):
        return None
    for f in sorted(os.listdir(d), reverse=True):
        if f.endswith("_ncu.json"):
            try:
                j = json.load(open(os.path.join(d, f)))
            except (OSError, ValueError):
                continue
            if j.get("kernel") == kernel:
                return j.get("dram_bytes_per_launch")
    return None


def _flush_buf():
    import torch
    return torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def _time(fn, reps=20, flush=None) -> float:
    import torch
    times = []
    for i in range(reps + 3):
        if flush is not None:  # same flush as the runtime: write, then read back (clean L2)
            flush.fill_(i & 0xff)
            flush.view(torch.int32).max()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        if i >= 3:
            times.append(s.elapsed_time(e) * 1e6)
    return statistics.median(times)


def cublas_reference(space, reps: int = 20) -> dict | None:
    """cuBLAS (through torch) on the same shape, L2 flushed before each call."""
    try:
        import torch
    except ImportError:
        return None
    if not torch.cuda.is_available():
        return None
    m, n, k, b = space.m, space.n, space.k, max(space.batch, 1)
    torch.backends.cuda.matmul.allow_tf32 = False
    flush = _flush_buf()
    out = {}
    kind = space.kind
    if kind == "axpy":
        x = torch.rand(n, device="cuda")
        y = torch.rand(n, device="cuda")
        ns = _time(lambda: y.add_(x, alpha=1.5), reps, flush)
        out["axpy"] = ns
    elif kind == "gemv":
        at = torch.rand(n, m, device="cuda")  # column-major m x n
        x = torch.rand(n, device="cuda")
        out["sgemv"] = _time(lambda: torch.mv(at.t(), x), reps, flush)
    elif kind == "sgemm":
        a, bb = torch.rand(k, m, device="cuda"), torch.rand(n, k, device="cuda")
        out["sgemm"] = _time(lambda: torch.mm(a.t(), bb.t()), reps, flush)
    elif kind == "batched":
        a, bb = torch.rand(b, k, m, device="cuda"), torch.rand(b, n, k, device="cuda")
        out["sgemm_strided_batched"] = _time(lambda: torch.bmm(a.transpose(1, 2), bb.transpose(1, 2)), reps, flush)
    elif kind in ("sgemm_tc", "sgemm_tc_x3"):
        a, bb = torch.rand(k, m, device="cuda"), torch.rand(n, k, device="cuda")
        out["sgemm_fp32"] = _time(lambda: torch.mm(a.t(), bb.t()), reps, flush)
        torch.backends.cuda.matmul.allow_tf32 = True
        out["sgemm_tf32"] = _time(lambda: torch.mm(a.t(), bb.t()), reps, flush)
        torch.backends.cuda.matmul.allow_tf32 = False
    res = {}
    for name, ns in out.items():
        res[name] = {"us": round(ns / 1e3, 3), "roofline": roofline(space, ns)}
    return res
