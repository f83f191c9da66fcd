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
    if kind in ("axpy", "axpy_stream"):
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


def rotation(space, l2_bytes: int) -> int:
    """Copies of the inputs so that consecutive launches never find their
    inputs in L2: aggregate input footprint >= 2 x L2 (at least 2)."""
    w = work(space)
    inputs = w["bytes"] - output_bytes(space)
    return int(max(2, min(16, -(-2 * l2_bytes // max(inputs, 1)) + 1)))


def output_bytes(space) -> int:
    m, n, b = space.m, space.n, max(space.batch, 1)
    if space.kind in ("axpy", "axpy_stream"):
        return 4 * n
    if space.kind == "gemv":
        return 4 * m
    if space.kind == "batched":
        return 4 * b * m * n
    return 4 * m * n


def retime_best(space, cand, reps: int = 20, dev=None, ordinal: int = 0) -> dict:
    """Re-times a candidate through the C-ABI: batches of back-to-back launches
    over rotating copies of the inputs (each launch reads inputs that are not
    in L2; the launch overhead is amortised), mean per launch."""
    from .api import Device
    own = dev is None
    dev = dev or Device(ordinal)
    dev.bind(space.problem())
    rot = rotation(space, dev.info()["l2_bytes"])
    reps = max(reps, 8 * rot)  # at least 8 groups of back-to-back launches (median over groups)
    if space.tiles:
        m = dev.evaluate_tiles(cand.tiles(), reps=reps, warmup=3, rotate=rot)
    else:
        m = dev.evaluate(cand.nest(), watchdog=0, reps=reps, warmup=3, rotate=rot)
    if own:
        dev.close()
    if m.status != "ok":
        return {"status": m.status}
    r = {"status": "ok", "kernel_us": round(m.median_ns / 1e3, 3), "min_us": round(m.min_ns / 1e3, 3),
         "timing": f"batches of {rot} back-to-back launches over {rot} input copies (inputs not L2-resident)",
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


def _time_rotating(make_call, rot: int, batches: int = 8) -> float:
    """Mean ns per call of `rot` back-to-back calls, each on its own copy of
    the inputs (the same rotation the runtime uses for our kernels); median
    over batches."""
    import torch
    calls = [make_call() for _ in range(rot)]
    for c in calls:  # warm-up (and cuBLAS heuristics / workspace)
        c()
    torch.cuda.synchronize()
    times = []
    for _ in range(batches):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for c in calls:
            c()
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e) * 1e6 / rot)
    return statistics.median(times)


def cublas_reference(space, reps: int = 20) -> dict | None:
    """cuBLAS (through torch) on the same shape, timed like our kernels:
    back-to-back calls over rotating input copies (not L2-resident)."""
    try:
        import torch
    except ImportError:
        return None
    if not torch.cuda.is_available():
        return None
    m, n, k, b = space.m, space.n, space.k, max(space.batch, 1)
    torch.backends.cuda.matmul.allow_tf32 = False
    rot = rotation(space, torch.cuda.get_device_properties(0).L2_cache_size)
    out = {}
    kind = space.kind

    def mk(shapes, fn):
        def make():
            ts = [torch.rand(*sh, device="cuda") for sh in shapes]
            return lambda: fn(*ts)
        return make

    if kind in ("axpy", "axpy_stream"):
        out["axpy"] = _time_rotating(mk([(n,), (n,)], lambda x, y: y.add_(x, alpha=1.5)), rot)
    elif kind == "gemv":
        out["sgemv"] = _time_rotating(mk([(n, m), (n,)], lambda at, x: torch.mv(at.t(), x)), rot)
    # our problem's layout: A column-major M x K (storage = a (k, m) row-major),
    # B column-major K x N (storage = bb (n, k)), C column-major M x N; in torch
    # C's storage is torch.mm(bb, a) of shape (n, m): cuBLAS then solves
    # exactly C = A B with A m-contiguous ("nn"). The "_tt" entries time the
    # transposed product torch.mm(a.t(), bb.t()) (both operands k-contiguous
    # for cuBLAS, kernel name ..._ttn_...): same flops, an easier layout for
    # the TF32 tensor cores, reported for context only.
    nn = lambda a, bb: torch.mm(bb, a)  # noqa: E731
    tt = lambda a, bb: torch.mm(a.t(), bb.t())  # noqa: E731
    if kind in ("sgemm", "matmul"):
        out["sgemm"] = _time_rotating(mk([(k, m), (n, k)], nn), rot)
        out["sgemm_tt"] = _time_rotating(mk([(k, m), (n, k)], tt), rot)
    elif kind == "batched":
        out["sgemm_strided_batched"] = _time_rotating(mk([(b, k, m), (b, n, k)], lambda a, bb: torch.bmm(bb, a)), rot)
    elif kind in ("sgemm_tc", "sgemm_tc_x3"):
        out["sgemm_fp32"] = _time_rotating(mk([(k, m), (n, k)], nn), rot, 3)
        torch.backends.cuda.matmul.allow_tf32 = True
        out["sgemm_tf32"] = _time_rotating(mk([(k, m), (n, k)], nn), rot)
        out["sgemm_tf32_tt"] = _time_rotating(mk([(k, m), (n, k)], tt), rot)
        torch.backends.cuda.matmul.allow_tf32 = False
    res = {}
    for name, ns in out.items():
        res[name] = {"us": round(ns / 1e3, 3), "roofline": roofline(space, ns),
                     "timing": f"batches of {rot} back-to-back calls over {rot} input copies"}
    return res
