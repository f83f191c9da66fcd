#!/usr/bin/env python
"""Headline benchmark: candidate evaluation on B200 for arXiv 1904.03383.

Metric (BASELINE.json): best-kernel GB/s vs roofline and candidates evaluated
per second. A step = STEP_EVALS candidates of the axpy n=2^26 search space
(paper factors {2,4} x {2..1024}, the reference's parity space) taken from
this rank's disjoint subtrees by the bound-pruned search, each one emitted as
sm_100a CUDA, NVRTC-compiled, launched (1 checked + warmup + reps timed) and
checked on device. `value` = candidates evaluated / s over the timed steps
(device-timeline marks, max over ranks); `e2e` = the same with the problem's
inputs uploaded from pinned host memory and its output read back every step
through the C-ABI. `roofline` = the best kernel found, re-timed without the
watchdog. `cpu_baseline` = the reference's own CPU search + simulated
evaluation (oracle/_ref/ref_cpu_bench) on this host.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_AXPY = 1 << 26
FACTORS = [[2, 4], [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024]]
BYTES_PER_RUN = 12 * N_AXPY  # x, y read + z written, fp32
METRIC = "candidates evaluated/s (best-kernel GB/s vs HBM roofline in `roofline`)"
WORKLOAD = "axpy fp32 n=2^26: full search + evaluation (paper factors {2,4}x{2..1024}, reference gpu.space)"
REF_CPU_BENCH = os.path.join(ROOT, "oracle", "_ref", "ref_cpu_bench")
PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "r01_axpy_best_ncu.json")


def peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d["hbm_gbs"], "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback"}


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    return world, rank, local


def allreduce(vals: list[float], op: str, world: int) -> list[float]:
    if world == 1:
        return vals
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return t.tolist()


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def cpu_baseline(seconds: float, threads: int) -> dict | None:
    """The reference's own CPU search + evaluation (oracle/_ref), bounded sample."""
    if not os.path.exists(REF_CPU_BENCH):
        return None
    args = [REF_CPU_BENCH, "axpy", "0", str(N_AXPY), "0", f"{seconds}", str(threads)]
    args += [",".join(str(v) for v in u) for u in FACTORS]
    out = subprocess.run(args, capture_output=True, text=True, timeout=seconds * 4 + 120)
    if out.returncode != 0:
        return None
    return json.loads(out.stdout.strip().splitlines()[-1])


def cublas_axpy_gbs() -> float | None:
    """cuBLAS Saxpy on the same n (reads x, y, writes y: the same 12 B/element)."""
    try:
        import ctypes as C

        import torch
        lib = C.CDLL("libcublas.so.12")
        h = C.c_void_p()
        lib.cublasCreate_v2(C.byref(h))
        x = torch.rand(N_AXPY, device="cuda")
        y = torch.rand(N_AXPY, device="cuda")
        alpha = C.c_float(1.5)
        stream = torch.cuda.current_stream().cuda_stream
        lib.cublasSetStream_v2(h, C.c_void_p(stream))
        times = []
        for i in range(13):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            lib.cublasSaxpy_v2(h, N_AXPY, C.byref(alpha), C.c_void_p(x.data_ptr()), 1, C.c_void_p(y.data_ptr()), 1)
            e.record()
            torch.cuda.synchronize()
            if i >= 3:
                times.append(s.elapsed_time(e))
        lib.cublasDestroy_v2(h)
        return BYTES_PER_RUN / (statistics.median(times) * 1e-3) / 1e9
    except Exception:
        return None


def run_reference(args, world, rank):
    """`--impl reference`: the reference's CPU search + simulated evaluation on
    this host's cores (rank 0 only), on our metric/config."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    per_step = 2.0
    res = cpu_baseline(per_step * args.steps, threads)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_cpu_bench not built"}))
        return
    v = res["leaves_per_s"]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "candidates/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "evaluator": "reference simulate() (analytic cycles)"},
        "cpu_baseline": {"value": v, "unit": "candidates/s", "cores": threads, "kind": "reference",
                         "sample": f"{res['leaves']} leaves of seeded uniform descents in {res['seconds']:.1f}s"},
        "e2e": {"value": v, "unit": "candidates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_detail": res,
    }
    print(json.dumps(line))


def run_ours(args, world, rank, local):
    import numpy as np
    import torch

    from paper_1904_03383_b200 import Device, Search, Space

    torch.cuda.set_device(local)
    space = Space("axpy", n=N_AXPY, factors=FACTORS)
    port = os.environ.get("MASTER_PORT", "0")
    shm = f"/ispc_inc_{port}_{os.getppid()}" if world > 1 else None
    log = os.path.join(ROOT, "gpurun_out", f"search_r{rank}.jsonl") if os.path.isdir(
        os.path.join(ROOT, "gpurun_out")) else None
    search = Search(space, device=local, seed=0x1904 + rank, shard_index=rank, shard_count=world,
                    reps=3, warmup=1, batch=args.batch, incumbent_shm=shm, log_path=log)
    E = args.per_step
    for _ in range(args.warmup):
        search.step(E)

    # ---- timed steps (inputs resident in HBM) ----
    barrier(world)
    torch.cuda.synchronize()
    dev_ms = []
    t_wall = time.perf_counter()
    with Clocks(local) as clk:
        for _ in range(args.steps):
            search.step(E)
            dev_ms.append(search.stats()["device_step_ms"])
    wall = time.perf_counter() - t_wall
    torch.cuda.synchronize()
    barrier(world)
    dev_s = sum(dev_ms) * 1e-3
    (dev_s_max,) = allreduce([dev_s], "max", world)
    (evals_total,) = allreduce([float(E * args.steps)], "sum", world)
    value = evals_total / dev_s_max

    # ---- end to end: host buffers through the C-ABI every step ----
    xh = torch.empty(N_AXPY, dtype=torch.float32, pin_memory=True)
    yh = torch.empty(N_AXPY, dtype=torch.float32, pin_memory=True)
    zh = torch.empty(N_AXPY, dtype=torch.float32, pin_memory=True)
    search.read_region("x", xh.data_ptr(), xh.nbytes)
    search.read_region("y", yh.data_ptr(), yh.nbytes)
    e2e_steps = max(2, args.steps // 2)
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        search.write_region("x", xh.data_ptr(), xh.nbytes)
        search.write_region("y", yh.data_ptr(), yh.nbytes)
        search.step(E)
        search.read_region("z", zh.data_ptr(), zh.nbytes)
    e2e_wall = time.perf_counter() - t0
    (e2e_max,) = allreduce([e2e_wall], "max", world)
    (e2e_evals,) = allreduce([float(E * e2e_steps)], "sum", world)
    e2e_value = e2e_evals / e2e_max

    st = search.stats()
    best = search.best()
    best_src = search.best_source()
    search.close()

    if rank != 0:
        return

    # ---- roofline: the best kernel, re-timed without the watchdog ----
    pk = peaks()
    roofline = None
    best_info = {}
    if best is not None:
        dev = Device(local)
        dev.bind(space.problem())
        m = dev.evaluate(best.nest(), watchdog=0, reps=20, warmup=3)
        dev.close()
        if m.status == "ok":
            gbs = BYTES_PER_RUN / m.median_ns
            traffic = None
            if os.path.exists(PROFILE_SUMMARY):
                traffic = json.load(open(PROFILE_SUMMARY)).get("dram_bytes_per_launch")
            roofline = {"bound": "hbm", "achieved": round(gbs, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                        "frac": round(gbs / pk["hbm_gbs"], 4), "traffic": traffic,
                        "algorithmic_bytes_per_launch": BYTES_PER_RUN, "kernel_us": round(m.median_ns / 1e3, 2),
                        "peak_source": pk["source"]}
            best_info = {"kernel_us": m.median_ns / 1e3, "gbs": gbs, "search_median_us": st["best_ns"] / 1e3,
                         "bound_us": st["best_bound_ns"] / 1e3, "time_to_best_s": st["time_to_best_s"]}
    cub = cublas_axpy_gbs()
    cpu = None
    if not args.no_cpu_baseline:
        res = cpu_baseline(args.cpu_seconds, os.cpu_count() or 1)
        if res:
            cpu = {"value": res["leaves_per_s"], "unit": "candidates/s", "cores": res["threads"],
                   "kind": "reference",
                   "sample": f"reference CPU search+simulate: {res['leaves']} leaves in {res['seconds']:.1f}s"}
    per_eval_launches = 1 + 1 + 3 + 1  # checked launch, warmup, reps, compare kernel
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "candidates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dev_s_max / args.steps * 1e3, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": WORKLOAD, "evals_per_step": E,
                                        "l2": "inputs 768 MB > 126 MB L2 (no flush needed)",
                                        "parallelism": f"shards{world}"},
        "e2e": {"value": round(e2e_value, 2), "unit": "candidates/s",
                "h2d_bytes_per_step": 2 * 4 * N_AXPY, "d2h_bytes_per_step": 4 * N_AXPY},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "gpu_launches": int(evals_total * per_eval_launches),
        "clocks": clk.summary(),
        "best_kernel": best_info,
        "cublas_saxpy_gbs": round(cub, 1) if cub else None,
        "search": {k: st[k] for k in ("evaluations", "ok", "mismatches", "timeouts", "launch_errors", "illegal",
                                      "compile_errors", "duplicates", "rollouts", "dead_rollouts",
                                      "pruned_children", "bound_violations", "frontier", "t_rollout_s",
                                      "t_compile_s", "t_gpu_s")},
        "wall_s": round(wall, 3),
    }
    print(json.dumps(line))
    if os.path.isdir(os.path.join(ROOT, "gpurun_out")) and best_src:
        with open(os.path.join(ROOT, "gpurun_out", "best_axpy_kernel.cu"), "w") as f:
            f.write(best_src)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--per-step", type=int, default=48, help="candidates evaluated per step")
    ap.add_argument("--batch", type=int, default=8, help="kernels per NVRTC program")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
