"""Python mirror of the reference's evaluation-path API over the two C ABIs.

``Space`` / ``Candidate`` drive the reference search space (libispc_host:
build_gpu_space, make_root, apply_decision, reconstruct). ``Device`` is the
B200 backend (libispc: emit sm_100a CUDA, NVRTC, timed launch, on-device
check). ``Device.evaluate(nest)`` is the drop-in for the reference's
``evaluate(kernel, nest, machine)`` (proj/core/include/ispace/simulate.hpp:33):
same input (a reconstructed schedule), a measured time instead of simulated
cycles.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

from . import _native as N


def explore_spec(space: "Space", budget: int, *, seed: int = 1, order: str | None = None, pruning: bool = True,
                 evaluator: str = "bound", delta: float = 0.05, bucket: int = 20, max_rollouts: int = 0,
                 log_path: str | None = None, resume_log: str | None = None) -> dict:
    """Deterministic single-threaded TAG-MCTS with a CPU
    evaluator: "bound" (the B200 bound x a digest-hashed factor in [1, 1.5),
    admissible by construction) or "simulate" (the reference's cycles).
    `resume_log`: the log of an earlier run is its checkpoint; it is replayed
    (ValueError if a record differs) and the search continues to `budget`."""
    keep = [x.encode() if x else None for x in (order, log_path, resume_log)]
    cfg = N.SpecConfig(budget=budget, max_rollouts=max_rollouts, seed=seed, order=keep[0], pruning=int(pruning),
                       evaluator={"bound": N.SPEC_EVAL_BOUND, "simulate": N.SPEC_EVAL_SIMULATE}[evaluator],
                       delta=delta, bucket=bucket, log_path=keep[1], resume_log=keep[2])
    r = N.SpecResult()
    buf = C.create_string_buffer(1 << 20)
    n = C.c_size_t(0)
    if N.host().ispc_explore_spec(space._h, C.byref(cfg), C.byref(r), buf, len(buf), C.byref(n)) != 0:
        raise ValueError(N.host_error())
    text = buf.value.decode()
    out = {f: getattr(r, f) for f, _ in N.SpecResult._fields_ if f != "_pad"}
    out["exhausted"] = bool(out["exhausted"])
    out["best"] = space.deserialize(text) if text else None
    return out


def tag_select(s: list[float], t: list[float], total: int, excluded: list[bool] | None = None,
               delta: float = 0.05, bucket: int = 20) -> int:
    """The TAG selection rule (ispc_tag_select); -1 when every child is excluded."""
    k = len(s)
    ex = (C.c_ubyte * k)(*[int(x) for x in (excluded or [False] * k)])
    return N.host().ispc_tag_select(k, (C.c_double * k)(*s), (C.c_double * k)(*t), ex, total, delta, bucket)


# ---------------------------------------------------------------- search space
class Space:
    """A kernel backbone bound to the GPU decision space (gpu_space.hpp:15-18)."""

    TILE_KINDS = ("gemv", "sgemm", "batched", "sgemm_tc", "sgemm_tc_x3", "axpy_stream")

    def __init__(self, kind: str, *, m: int = 0, n: int = 0, k: int = 0, a_stride: int = 1,
                 factors: list[list[int]] | None = None, mode: int = N.SPACE_PARITY, batch: int = 1):
        factors = factors or []
        spec = N.KernelSpec()
        self._kind = kind.encode()
        spec.kind = self._kind
        spec.m, spec.n, spec.k, spec.a_stride = m, n, k, a_stride
        if len(factors) > 4:
            raise ValueError("at most 4 strip-mining universes")
        spec.num_factors = len(factors)
        for i, u in enumerate(factors):
            if not 0 < len(u) <= 32:
                raise ValueError("a universe holds 1..32 sizes")
            spec.factor_len[i] = len(u)
            for j, v in enumerate(u):
                spec.factors[i][j] = v
        spec.mode = mode
        spec.batch = batch
        self.kind, self.m, self.n, self.k, self.a_stride, self.factors, self.mode = (
            kind, m, n, k, a_stride, factors, mode)
        self.batch = batch
        self.tiles = kind in self.TILE_KINDS
        h = C.c_void_p()
        rc = N.host().ispc_space_create(C.byref(spec), C.byref(h))
        if rc != 0:
            raise ValueError(N.host_error())
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            N.host().ispc_space_free(self._h)
            self._h = None

    def stats(self) -> dict:
        s = N.SpaceStats()
        N.host().ispc_space_stats_get(self._h, C.byref(s))
        return {f: getattr(s, f) for f, _ in N.SpaceStats._fields_}

    def problem(self) -> N.Problem:
        p = N.Problem()
        if N.host().ispc_space_problem(self._h, C.byref(p)) != 0:
            raise ValueError(N.host_error())
        return p

    def root(self) -> "Candidate":
        h = C.c_void_p()
        N.host().ispc_cand_root(self._h, C.byref(h))
        return Candidate(self, h)

    def deserialize(self, text: str) -> "Candidate":
        h = C.c_void_p()
        if N.host().ispc_cand_deserialize(self._h, text.encode(), C.byref(h)) != 0:
            raise ValueError(N.host_error())
        return Candidate(self, h)


class DeadEnd(Exception):
    pass


class Candidate:
    """A (partially) specified implementation (candidate.hpp:54-59)."""

    def __init__(self, space: Space, h):
        self.space, self._h = space, h

    def __del__(self):
        if getattr(self, "_h", None):
            N.host().ispc_cand_free(self._h)
            self._h = None

    def clone(self) -> "Candidate":
        return Candidate(self.space, C.c_void_p(N.host().ispc_cand_clone(self._h)))

    def decide(self, choice: str, args: list[str], value: str) -> "Candidate":
        a0 = args[0].encode() if len(args) > 0 else None
        a1 = args[1].encode() if len(args) > 1 else None
        rc = N.host().ispc_cand_decide(self.space._h, self._h, choice.encode(), a0, a1, value.encode())
        if rc == 1:
            raise DeadEnd(f"{choice}({', '.join(args)}) = {value}")
        if rc != 0:
            raise ValueError(N.host_error())
        return self

    @property
    def open_count(self) -> int:
        return N.host().ispc_cand_open_count(self.space._h, self._h)

    @property
    def fully_specified(self) -> bool:
        return bool(N.host().ispc_cand_fully_specified(self.space._h, self._h))

    @property
    def digest(self) -> int:
        return N.host().ispc_cand_digest(self.space._h, self._h)

    @property
    def fired(self) -> int:
        return N.host().ispc_cand_fired(self._h)

    def first_leaf(self, budget: int = 100000) -> "Candidate":
        h = C.c_void_p()
        if N.host().ispc_cand_first_leaf(self.space._h, self._h, budget, C.byref(h)) != 0:
            raise DeadEnd("no leaf within budget")
        return Candidate(self.space, h)

    def random_leaf(self, seed: int, max_restarts: int = 1000, order: str | None = None
                    ) -> tuple["Candidate", int, int]:
        h = C.c_void_p()
        dec, dead = C.c_int64(), C.c_int64()
        rc = N.host().ispc_cand_random_leaf_ordered(self.space._h, self._h, seed, order.encode() if order else None,
                                                    max_restarts, C.byref(h), C.byref(dec), C.byref(dead))
        if rc != 0:
            raise DeadEnd("random descent gave up")
        return Candidate(self.space, h), dec.value, dead.value

    def estimate_tree(self, probes: int = 1000, seed: int = 1, order: str | None = None) -> dict:
        """Knuth's estimate of the subtree below this candidate."""
        out = (C.c_double * 5)()
        rc = N.host().ispc_estimate_tree(self.space._h, self._h, probes, seed, order.encode() if order else None, out)
        if rc != 0:
            raise ValueError(N.host_error())
        return dict(zip(("leaves", "leaves_stderr", "nodes", "dead_probe_ratio", "probes"), list(out)))

    def count_leaves(self, cap: int = 10 ** 7) -> int:
        return N.host().ispc_count_leaves(self.space._h, self._h, cap)

    def estimate(self, method: str = "knuth", iterations: int = 1000, seed: int = 1, order: str | None = None,
                 stratifier: str = "depth_remaining") -> dict:
        """Knuth's or Chen's estimate of the subtree below this candidate
        (SPEC.md:516-567); ValueError for a stratifier that does not strictly
        decrease along the tree."""
        e = N.TreeEstimate()
        rc = N.host().ispc_estimate(self.space._h, self._h, method.encode(), iterations, seed,
                                    order.encode() if order else None, stratifier.encode(), C.byref(e))
        if rc != 0:
            raise ValueError(N.host_error())
        return _estimate_dict(e)

    def enumerate(self, node_budget: int = 10 ** 6, order: str | None = None, depth_cap: int = 64) -> dict:
        """Exact node / leaf / dead-end counts and nodes per depth; ValueError
        (a refusal) past `node_budget` nodes."""
        r = N.EnumReport()
        per = (C.c_int64 * depth_cap)()
        rc = N.host().ispc_enumerate(self.space._h, self._h, order.encode() if order else None, node_budget,
                                     C.byref(r), per, depth_cap)
        if rc != 0:
            raise ValueError(N.host_error())
        return _enum_dict(r, per)

    def deadend_rate(self, trials: int = 1000, seed: int = 1, order: str | None = None) -> dict:
        """Share of uniform random descents ending at a dead end, 95% Wilson CI
        (paper section 5.2)."""
        r = N.DeadendReport()
        rc = N.host().ispc_deadend_rate(self.space._h, self._h, trials, seed, order.encode() if order else None,
                                        C.byref(r))
        if rc != 0:
            raise ValueError(N.host_error())
        return {"trials": r.trials, "dead_ends": r.dead_ends, "ratio": r.ratio, "ci95": [r.ci_lo, r.ci_hi],
                "mean_decisions": r.mean_decisions}

    def greedy_leaf(self, order: str | None = None) -> tuple["Candidate", float]:
        """The lowest-bound descent from here: (leaf, its bound in seconds)."""
        h = C.c_void_p()
        b = C.c_double()
        rc = N.host().ispc_greedy_leaf(self.space._h, self._h, order.encode() if order else None, C.byref(h),
                                       C.byref(b))
        if rc == 1:
            raise DeadEnd("greedy descent met a dead end")
        if rc != 0:
            raise ValueError(N.host_error())
        return Candidate(self.space, h), b.value

    def walk_digests(self, seed: int, walks: int) -> list[int]:
        """Leaf digests of `walks` seeded uniform first-open descents sharing
        one generator (oracle/ref_cpu_bench.cpp's walk); 0 = dead end."""
        out = (C.c_uint64 * walks)()
        if N.host().ispc_walk_digests(self.space._h, self._h, seed, walks, out) != 0:
            raise ValueError(N.host_error())
        return list(out)

    def descend(self, steps: int, seed: int = 1, order: str | None = None) -> "Candidate":
        """A uniform partial descent of `steps` decisions; DeadEnd when it
        meets a dead end or a leaf first."""
        h = C.c_void_p()
        rc = N.host().ispc_cand_descend(self.space._h, self._h, order.encode() if order else None, seed, steps,
                                        C.byref(h))
        if rc == 1:
            raise DeadEnd("partial descent ended early")
        if rc != 0:
            raise ValueError(N.host_error())
        return Candidate(self.space, h)

    def order_round_trip(self, node_budget: int = 10 ** 6) -> dict:
        """derive_orders over every leaf below here against the leaves' order
        decisions (nest_test.cpp:309-334)."""
        lv, pr, bad = C.c_int64(), C.c_int64(), C.c_int64()
        if N.host().ispc_order_round_trip(self.space._h, self._h, node_budget, C.byref(lv), C.byref(pr),
                                          C.byref(bad)) != 0:
            raise ValueError(N.host_error())
        return {"leaves": lv.value, "pairs": pr.value, "mismatches": bad.value}

    def deadend_exact(self, node_budget: int = 10 ** 6, order: str | None = None) -> float:
        """Exact dead-end probability of a uniform random descent from here."""
        p = C.c_double()
        if N.host().ispc_deadend_exact(self.space._h, self._h, order.encode() if order else None, node_budget,
                                       C.byref(p)) != 0:
            raise ValueError(N.host_error())
        return p.value

    def prune_profile(self, threshold_s: float, depth_cap: int, order: str | None = None,
                      node_budget: int = 10 ** 6) -> dict:
        """Nodes per depth of the first `depth_cap` levels and how many the B200
        bound prunes against incumbent `threshold_s` (paper section 5.4)."""
        nodes = (C.c_int64 * depth_cap)()
        pruned = (C.c_int64 * depth_cap)()
        rc = N.host().ispc_prune_profile(self.space._h, self._h, order.encode() if order else None, threshold_s,
                                         depth_cap, node_budget, nodes, pruned)
        if rc != 0:
            raise ValueError(N.host_error())
        return {"nodes": list(nodes), "pruned": list(pruned),
                "fraction": [p / n if n else None for p, n in zip(pruned, nodes)]}

    def tiles(self) -> N.TileConfig:
        """Decided building-block configuration (tiles.space candidates)."""
        t = N.TileConfig()
        if N.host().ispc_cand_to_tiles(self.space._h, self._h, C.byref(t)) != 0:
            raise ValueError(N.host_error())
        return t

    def nest(self) -> "NestHandle":
        h = C.c_void_p()
        if N.host().ispc_cand_to_nest(self.space._h, self._h, C.byref(h)) != 0:
            raise ValueError(N.host_error())
        return NestHandle(h)

    def reference_source(self) -> str:
        return N.read_text(N.host().ispc_cand_reference_source, self.space._h, self._h)

    def simulate(self) -> dict:
        out = (C.c_int64 * 5)()
        if N.host().ispc_cand_simulate(self.space._h, self._h, out) != 0:
            raise ValueError(N.host_error())
        return dict(zip(("compute", "memory", "sync", "block_serial", "total"), list(out)))

    def serialize(self) -> str:
        return N.read_text(N.host().ispc_cand_serialize, self.space._h, self._h)

    def bound(self, l2_flushed: bool = False) -> dict:
        """B200 lower bound in seconds (host/bound.hpp)."""
        r = N.BoundReport()
        if N.host().ispc_bound(self.space._h, self._h, int(l2_flushed), C.byref(r)) != 0:
            raise ValueError(N.host_error())
        return {f: getattr(r, f) for f, _ in N.BoundReport._fields_}


def _estimate_dict(e) -> dict:
    z = 1.959963984540054
    return {"method": ("knuth", "chen")[e.method], "iterations": e.iterations, "leaves": e.leaves,
            "leaves_stderr": e.leaves_stderr, "leaves_ci95": [e.leaves - z * e.leaves_stderr,
                                                             e.leaves + z * e.leaves_stderr],
            "nodes": e.nodes, "nodes_stderr": e.nodes_stderr, "dead_ratio": e.dead_ratio}


def _enum_dict(r, per) -> dict:
    depth = [int(v) for v in per]
    while depth and depth[-1] == 0:
        depth.pop()
    return {"nodes": r.nodes, "leaves": r.leaves, "dead_ends": r.dead_ends, "max_depth": r.max_depth,
            "nodes_per_depth": depth}


def estimate_synthetic(tree: str, method: str = "knuth", iterations: int = 1000, seed: int = 1,
                       stratifier: str = "depth_remaining") -> dict:
    """The estimators on a closed-form tree ("uniform:B,D", "caterpillar:D,H",
    "random:S,B,D"): their known answers."""
    e = N.TreeEstimate()
    rc = N.host().ispc_estimate_synthetic(tree.encode(), method.encode(), iterations, seed, stratifier.encode(),
                                          C.byref(e))
    if rc != 0:
        raise ValueError(N.host_error())
    return _estimate_dict(e)


def enumerate_synthetic(tree: str, node_budget: int = 10 ** 7, depth_cap: int = 64) -> dict:
    r = N.EnumReport()
    per = (C.c_int64 * depth_cap)()
    if N.host().ispc_enumerate_synthetic(tree.encode(), node_budget, C.byref(r), per, depth_cap) != 0:
        raise ValueError(N.host_error())
    return _enum_dict(r, per)


class NestHandle:
    """Flat ispc_nest of a reconstructed schedule (owned by libispc_host)."""

    def __init__(self, h):
        self._h = h
        self.nest = N.host().ispc_nest_buf_get(h)

    def __del__(self):
        if getattr(self, "_h", None):
            N.host().ispc_nest_buf_free(self._h)
            self._h = None

    def pseudo(self) -> str:
        return N.read_text(N.ispc().ispc_emit_pseudo, self.nest)

    def cuda(self, fn_name: str | None = None, watchdog: int = 2) -> tuple[str, N.Launch]:
        opts = N.EmitOpts(watchdog=watchdog)
        L = N.Launch()
        n = C.c_size_t()
        nm = fn_name.encode() if fn_name else None
        rc = N.ispc().ispc_emit_cuda(self.nest, C.byref(opts), nm, None, 0, C.byref(n), C.byref(L))
        if rc != 0:
            raise EmitError(rc, N.last_error())
        buf = C.create_string_buffer(n.value + 1)
        rc = N.ispc().ispc_emit_cuda(self.nest, C.byref(opts), nm, buf, n.value + 1, C.byref(n), C.byref(L))
        if rc != 0:
            raise EmitError(rc, N.last_error())
        return buf.value.decode(), L


def tile_cuda(cfg: N.TileConfig, fn_name: str | None = None) -> tuple[str, N.Launch]:
    """sm_100a source of a building-block configuration (ispc_emit_tiles)."""
    L = N.Launch()
    n = C.c_size_t()
    nm = fn_name.encode() if fn_name else None
    rc = N.ispc().ispc_emit_tiles(C.byref(cfg), nm, None, 0, C.byref(n), C.byref(L))
    if rc != 0:
        raise EmitError(rc, N.last_error())
    buf = C.create_string_buffer(n.value + 1)
    rc = N.ispc().ispc_emit_tiles(C.byref(cfg), nm, buf, n.value + 1, C.byref(n), C.byref(L))
    if rc != 0:
        raise EmitError(rc, N.last_error())
    return buf.value.decode(), L


class EmitError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{N.STATUS.get(code, code)}: {msg}")
        self.code = code


# ---------------------------------------------------------------- compilation
class Module:
    def __init__(self, h):
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            N.ispc().ispc_module_free(self._h)
            self._h = None

    def cubin(self) -> bytes:
        p, n = C.c_void_p(), C.c_size_t()
        N.ispc().ispc_module_cubin(self._h, C.byref(p), C.byref(n))
        return C.string_at(p, n.value)


def compile_sources(srcs: list[str], arch: str = "sm_100a") -> Module:
    arr = (C.c_char_p * len(srcs))(*[s.encode() for s in srcs])
    h = C.c_void_p()
    rc = N.ispc().ispc_compile(arr, len(srcs), arch.encode(), C.byref(h))
    if rc != 0:
        raise EmitError(rc, N.last_error())
    return Module(h)


# ---------------------------------------------------------------- device
@dataclass
class Measurement:
    status: str
    median_ns: float
    min_ns: float
    first_ns: float
    max_err: float
    mismatches: int
    launch: N.Launch | None = field(default=None, repr=False)


class Device:
    """One B200 (ispc_dev)."""

    def __init__(self, ordinal: int = 0):
        h = C.c_void_p()
        rc = N.ispc().ispc_dev_open(ordinal, C.byref(h))
        if rc != 0:
            raise RuntimeError(f"ispc_dev_open({ordinal}): {N.last_error()}")
        self._h = h
        self.ordinal = ordinal

    def close(self):
        if getattr(self, "_h", None):
            N.ispc().ispc_dev_close(self._h)
            self._h = None

    __del__ = close

    def error(self) -> str:
        return N.last_error(self._h)

    def info(self) -> dict:
        sm, l2, hbm, clk = C.c_int(), C.c_int64(), C.c_int64(), C.c_int()
        N.ispc().ispc_dev_info(self._h, C.byref(sm), C.byref(l2), C.byref(hbm), C.byref(clk))
        return {"sm_count": sm.value, "l2_bytes": l2.value, "hbm_bytes": hbm.value, "sm_clock_khz": clk.value}

    def bind(self, problem: N.Problem):
        rc = N.ispc().ispc_bind_problem(self._h, C.byref(problem))
        if rc != 0:
            raise RuntimeError(self.error())

    def read(self, name: str, count: int, expected: bool = False):
        import numpy as np
        out = np.empty(count, dtype=np.float32)
        fn = N.ispc().ispc_read_expected if expected else N.ispc().ispc_read_region
        rc = fn(self._h, name.encode(), out.ctypes.data_as(C.c_void_p), out.nbytes)
        if rc != 0:
            raise RuntimeError(self.error())
        return out

    def load(self, module: Module) -> int:
        h = C.c_int()
        rc = N.ispc().ispc_module_load(self._h, module._h, C.byref(h))
        if rc != 0:
            raise RuntimeError(self.error())
        return h.value

    def unload(self, handle: int):
        N.ispc().ispc_module_unload(self._h, handle)

    @staticmethod
    def _opts(warmup, reps, flush_l2, check, bit_exact, rtol, budget_ns, rotate=0):
        return N.TimeOpts(warmup=warmup, reps=reps, flush_l2=int(flush_l2), check=int(check),
                          bit_exact=int(bit_exact), rtol=rtol, budget_ns=budget_ns, rotate=rotate)

    def launch(self, handle: int, launch: N.Launch, *, warmup=1, reps=3, flush_l2=False, check=True,
               bit_exact=True, rtol=1e-5, budget_ns=2e9, rotate=0) -> Measurement:
        r = N.TimeResult()
        rc = N.ispc().ispc_launch_timed(self._h, handle, C.byref(launch),
                                        C.byref(self._opts(warmup, reps, flush_l2, check, bit_exact, rtol,
                                                           budget_ns, rotate)), C.byref(r))
        if rc != 0:
            return Measurement(N.STATUS.get(rc, str(rc)), float("inf"), float("inf"), float("inf"), 0.0, -1,
                               launch)
        return Measurement(N.STATUS.get(r.status, str(r.status)), r.median_ns, r.min_ns, r.first_ns, r.max_err,
                           r.mismatches, launch)

    def evaluate(self, nest: NestHandle, *, watchdog=2, warmup=1, reps=3, flush_l2=False, check=True,
                 bit_exact=True, rtol=1e-5, budget_ns=2e9, rotate=0) -> Measurement:
        r = N.TimeResult()
        L = N.Launch()
        eo = N.EmitOpts(watchdog=watchdog)
        rc = N.ispc().ispc_evaluate(self._h, nest.nest, C.byref(eo),
                                    C.byref(self._opts(warmup, reps, flush_l2, check, bit_exact, rtol, budget_ns,
                                                       rotate)),
                                    C.byref(r), C.byref(L))
        if rc != 0:
            return Measurement(N.STATUS.get(rc, str(rc)), float("inf"), float("inf"), float("inf"), 0.0, -1, L)
        return Measurement(N.STATUS.get(r.status, str(r.status)), r.median_ns, r.min_ns, r.first_ns, r.max_err,
                           r.mismatches, L)


    def evaluate_tiles(self, cfg: N.TileConfig, *, warmup=1, reps=3, flush_l2=False, check=True,
                       bit_exact=None, rtol=None, rotate=0) -> Measurement:
        """Emit + compile + timed launch + on-device check of a building-block
        configuration. Default checking: bit-exact for the FFMA sgemm and
        batched kernels (k ascending per output), norm-wise rtol otherwise."""
        exact_default = (cfg.kind == N.TILE_SGEMM and cfg.split <= 1) or cfg.kind in (N.TILE_BATCHED, N.TILE_AXPY)
        if bit_exact is None:
            bit_exact = exact_default
        if rtol is None:
            rtol = 4e-3 if (cfg.kind == N.TILE_SGEMM_TC and cfg.engine == 1) else 1e-5
        r = N.TimeResult()
        L = N.Launch()
        rc = N.ispc().ispc_evaluate_tiles(self._h, C.byref(cfg),
                                          C.byref(self._opts(warmup, reps, flush_l2, check, bit_exact, rtol, 2e9,
                                                             rotate)),
                                          C.byref(r), C.byref(L))
        if rc != 0:
            return Measurement(N.STATUS.get(rc, str(rc)), float("inf"), float("inf"), float("inf"), 0.0, -1, L)
        return Measurement(N.STATUS.get(r.status, str(r.status)), r.median_ns, r.min_ns, r.first_ns, r.max_err,
                           r.mismatches, L)


def explore_spec(space: "Space", budget: int, *, seed: int = 1, order: str | None = None, pruning: bool = True,
                 evaluator: str = "bound", delta: float = 0.05, bucket: int = 20, max_rollouts: int = 0,
                 log_path: str | None = None, resume_log: str | None = None) -> dict:
    """Deterministic single-threaded TAG-MCTS with a CPU
    evaluator: "bound" (the B200 bound x a digest-hashed factor in [1, 1.5),
    admissible by construction) or "simulate" (the reference's cycles).
    `resume_log`: the log of an earlier run is its checkpoint; it is replayed
    (ValueError if a record differs) and the search continues to `budget`."""
    keep = [x.encode() if x else None for x in (order, log_path, resume_log)]
    cfg = N.SpecConfig(budget=budget, max_rollouts=max_rollouts, seed=seed, order=keep[0], pruning=int(pruning),
                       evaluator={"bound": N.SPEC_EVAL_BOUND, "simulate": N.SPEC_EVAL_SIMULATE}[evaluator],
                       delta=delta, bucket=bucket, log_path=keep[1], resume_log=keep[2])
    r = N.SpecResult()
    buf = C.create_string_buffer(1 << 20)
    n = C.c_size_t(0)
    if N.host().ispc_explore_spec(space._h, C.byref(cfg), C.byref(r), buf, len(buf), C.byref(n)) != 0:
        raise ValueError(N.host_error())
    text = buf.value.decode()
    out = {f: getattr(r, f) for f, _ in N.SpecResult._fields_ if f != "_pad"}
    out["exhausted"] = bool(out["exhausted"])
    out["best"] = space.deserialize(text) if text else None
    return out


def tag_select(s: list[float], t: list[float], total: int, excluded: list[bool] | None = None,
               delta: float = 0.05, bucket: int = 20) -> int:
    """The TAG selection rule (ispc_tag_select); -1 when every child is excluded."""
    k = len(s)
    ex = (C.c_ubyte * k)(*[int(x) for x in (excluded or [False] * k)])
    return N.host().ispc_tag_select(k, (C.c_double * k)(*s), (C.c_double * k)(*t), ex, total, delta, bucket)


# ---------------------------------------------------------------- search
class Search:
    """Bound-pruned Monte-Carlo search with measured evaluation on one B200
    (libispc_host ispc_search_*). The pipeline keeps running between step()s."""

    PAPER_ORDER = "size,dim_kind,thread_level,mem_space,order,cache"

    def __init__(self, space: Space, *, device: int = 0, seed: int = 1, shard_index: int = 0, shard_count: int = 1,
                 pruning: bool = True, rollout_threads: int = 0, compile_threads: int = 0, batch: int = 8,
                 reps: int = 3, warmup: int = 1, flush_l2: bool = False, watchdog: int = 1,
                 budget_factor: float = 3.0, max_budget_ns: float = 50e6, max_unrolled: int = 512,
                 decision_order: str | None = None, incumbent_shm: str | None = None, log_path: str | None = None,
                 tree_depth: int = 0, rotate: int = 0, refine_factor: float = 0.0, walk: str = "search"):
        self.space = space
        self._keep = [x.encode() if x else None for x in (decision_order, incumbent_shm, log_path)]
        cfg = N.SearchConfig(device=device, rollout_threads=rollout_threads, compile_threads=compile_threads,
                             batch=batch, seed=seed, shard_index=shard_index, shard_count=shard_count,
                             pruning=int(pruning), watchdog=watchdog, reps=reps, warmup=warmup,
                             flush_l2=int(flush_l2), max_unrolled=max_unrolled, budget_factor=budget_factor,
                             max_budget_ns=max_budget_ns, decision_order=self._keep[0],
                             incumbent_shm=self._keep[1], log_path=self._keep[2], tree_depth=tree_depth,
                             rotate=rotate, refine_factor=refine_factor,
                             walk={"search": N.WALK_SEARCH, "uniform": N.WALK_UNIFORM}[walk])
        h = C.c_void_p()
        if N.host().ispc_search_create(space._h, C.byref(cfg), C.byref(h)) != 0:
            raise RuntimeError(N.host_error())
        self._h = h

    def step(self, evaluations: int, max_seconds: float = 0.0) -> bool:
        """Measures `evaluations` more kernels; False when `max_seconds`
        passed first (the pipeline could not produce them in time)."""
        rc = N.host().ispc_search_step_for(self._h, evaluations, max_seconds)
        if rc == N.E_TIMEOUT:
            return False
        if rc != 0:
            raise RuntimeError(N.host().ispc_search_error(self._h).decode())
        return True

    def stats(self) -> dict:
        s = N.SearchStats()
        N.host().ispc_search_stats_get(self._h, C.byref(s))
        return {f: getattr(s, f) for f, _ in N.SearchStats._fields_}

    def best(self) -> Candidate | None:
        text = N.read_text(N.host().ispc_search_best, self._h)
        return self.space.deserialize(text) if text else None

    def elites(self) -> list[Candidate]:
        """The best measured leaves kept for elite-guided rollouts, fastest
        first (building-block spaces; empty for the loop-nest spaces)."""
        out = []
        for i in range(64):
            text = N.read_text(N.host().ispc_search_elite, self._h, i)
            if not text:
                break
            out.append(self.space.deserialize(text))
        return out

    def best_source(self) -> str:
        return N.read_text(N.host().ispc_search_best_source, self._h)

    def write_region(self, name: str, ptr: int, nbytes: int):
        if N.host().ispc_search_write_region(self._h, name.encode(), C.c_void_p(ptr), nbytes) != 0:
            raise RuntimeError(N.last_error())

    def read_region(self, name: str, ptr: int, nbytes: int):
        if N.host().ispc_search_read_region(self._h, name.encode(), C.c_void_p(ptr), nbytes) != 0:
            raise RuntimeError(N.last_error())

    def frontier(self) -> list[int]:
        """Digests of this shard's subtree roots."""
        n = N.host().ispc_search_frontier(self._h, None, 0)
        buf = (C.c_uint64 * max(n, 1))()
        N.host().ispc_search_frontier(self._h, buf, n)
        return list(buf)[:n]

    def offer(self, ns: float) -> bool:
        """CAS-min a measured time into the shared incumbent."""
        return bool(N.host().ispc_search_offer(self._h, ns))

    def close(self):
        if getattr(self, "_h", None):
            N.host().ispc_search_free(self._h)
            self._h = None

    __del__ = close
