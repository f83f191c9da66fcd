"""ctypes bindings of the two C-ABI libraries (include/ispc.h, include/ispc_host.h).

The libraries are built in-tree by ``__graft_entry__.build()`` (``make`` in
``csrc/`` and ``host/``). There is no fallback: importing a binding whose
shared object is missing raises, so a GPU run can never silently evaluate
candidates anywhere but on the device.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIBISPC_PATH = os.path.join(_HERE, "csrc", "libispc.so")
LIBHOST_PATH = os.path.join(_HERE, "host", "libispc_host.so")

ISPC_NONE = 0xFFFFFFFF
ABI_VERSION = 2

STATUS = {0: "ok", -1: "arg", -2: "cuda", -3: "nvrtc", -4: "launch", -5: "mismatch",
          -6: "timeout", -7: "illegal", -8: "nomem", -9: "sticky"}
OK, E_ARG, E_CUDA, E_NVRTC, E_LAUNCH, E_MISMATCH, E_TIMEOUT, E_ILLEGAL, E_NOMEM, E_STICKY = (
    0, -1, -2, -3, -4, -5, -6, -7, -8, -9)

PROB_AXPY, PROB_OUTER, PROB_MATMUL, PROB_GEMV, PROB_BATCHED = range(5)
SPACE_PARITY, SPACE_B200 = 0, 1
TILE_GEMV, TILE_SGEMM, TILE_BATCHED, TILE_SGEMM_TC, TILE_AXPY = range(5)
STAGINGS = ("DIRECT", "SHARED", "CP_ASYNC", "TMA")
ENGINES = ("FFMA", "TF32", "TF32X3")
XREDUCES = ("SHUFFLE", "SHARED")
CACHES = ("L1", "L2", "READ_ONLY", "NONE", "STREAM")


class AddrTerm(C.Structure):
    _fields_ = [("dim", C.c_uint32), ("size_dims_begin", C.c_uint32), ("size_dims_count", C.c_uint32),
                ("_pad", C.c_uint32), ("base", C.c_int64)]


class IVar(C.Structure):
    _fields_ = [("offset", C.c_int64), ("terms_begin", C.c_uint32), ("terms_count", C.c_uint32)]


class Operand(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("input", C.c_uint32), ("ivar", C.c_uint32), ("producer", C.c_uint32),
                ("init", C.c_uint32), ("comm", C.c_uint32), ("pairs_begin", C.c_uint32),
                ("pairs_count", C.c_uint32), ("reduce_begin", C.c_uint32), ("reduce_count", C.c_uint32),
                ("value", C.c_int64)]


class Inst(C.Structure):
    _fields_ = [("obj", C.c_uint32), ("op", C.c_uint32), ("region", C.c_uint32), ("ivar", C.c_uint32),
                ("operands_begin", C.c_uint32), ("operands_count", C.c_uint32), ("dims_begin", C.c_uint32),
                ("dims_count", C.c_uint32), ("live", C.c_uint32), ("cache", C.c_uint32)]


class Region(C.Structure):
    _fields_ = [("obj", C.c_uint32), ("input", C.c_uint32), ("live", C.c_uint32), ("mem_space", C.c_uint32),
                ("elems", C.c_int64), ("elem_bytes", C.c_int64)]


class Dim(C.Structure):
    _fields_ = [("obj", C.c_uint32), ("logical", C.c_uint32), ("is_static", C.c_uint32), ("_pad", C.c_uint32),
                ("size", C.c_int64)]


class Comm(C.Structure):
    _fields_ = [("producer", C.c_uint32), ("consumer", C.c_uint32), ("region", C.c_uint32),
                ("store", C.c_uint32), ("load", C.c_uint32), ("pairs_begin", C.c_uint32),
                ("pairs_count", C.c_uint32), ("fired", C.c_uint32)]


class Node(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("dim_kind", C.c_uint32), ("thread_level", C.c_int32),
                ("block_level", C.c_int32), ("inst", C.c_uint32), ("dims_begin", C.c_uint32),
                ("dims_count", C.c_uint32), ("children_begin", C.c_uint32), ("children_count", C.c_uint32),
                ("_pad", C.c_uint32), ("size", C.c_int64)]


class Nest(C.Structure):
    _fields_ = [("abi_version", C.c_uint32), ("kernel_name", C.c_char_p), ("num_objects", C.c_uint32),
                ("object_names", C.POINTER(C.c_char_p)),
                ("num_insts", C.c_uint32), ("insts", C.POINTER(Inst)),
                ("num_regions", C.c_uint32), ("regions", C.POINTER(Region)),
                ("num_dims", C.c_uint32), ("dims", C.POINTER(Dim)),
                ("num_ivars", C.c_uint32), ("ivars", C.POINTER(IVar)),
                ("num_terms", C.c_uint32), ("terms", C.POINTER(AddrTerm)),
                ("num_operands", C.c_uint32), ("operands", C.POINTER(Operand)),
                ("num_comms", C.c_uint32), ("comms", C.POINTER(Comm)),
                ("num_inputs", C.c_uint32), ("input_names", C.POINTER(C.c_char_p)),
                ("pool_size", C.c_uint32), ("pool", C.POINTER(C.c_uint32)),
                ("num_nodes", C.c_uint32), ("nodes", C.POINTER(Node)),
                ("roots_begin", C.c_uint32), ("roots_count", C.c_uint32),
                ("num_thread_levels", C.c_uint32), ("num_block_levels", C.c_uint32),
                ("thread_shape", C.c_int64 * 3), ("block_shape", C.c_int64 * 3)]


class Param(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("index", C.c_uint32), ("is_input", C.c_uint32), ("_pad", C.c_uint32),
                ("elems", C.c_int64), ("name", C.c_char * 24)]


class TMap(C.Structure):
    _fields_ = [("param", C.c_uint32), ("rank", C.c_uint32), ("swizzle", C.c_uint32), ("_pad", C.c_uint32),
                ("region", C.c_char * 24), ("dims", C.c_uint64 * 3), ("strides", C.c_uint64 * 2),
                ("box", C.c_uint32 * 3), ("_pad2", C.c_uint32)]


class Launch(C.Structure):
    _fields_ = [("name", C.c_char * 64), ("grid_x", C.c_uint64), ("block", C.c_uint32 * 3),
                ("static_smem", C.c_uint32), ("num_params", C.c_uint32), ("pdl", C.c_uint32), ("params", Param * 32),
                ("watchdog", C.c_uint32), ("reg_elems", C.c_uint32), ("source_hash", C.c_uint64),
                ("cluster", C.c_uint32 * 3), ("num_tmaps", C.c_uint32), ("tmaps", TMap * 4)]


class TileConfig(C.Structure):
    _fields_ = ([(f, C.c_uint32) for f in ("kind", "staging", "engine", "xreduce", "cache", "lds")]
                + [(f, C.c_int64) for f in ("m", "n", "k", "batch")]
                + [(f, C.c_int32) for f in ("thr_m", "thr_n", "tm", "tn", "bk", "bn", "stages", "vec", "lanes_m",
                                            "lanes_n", "warps_m", "warps_n", "split", "unroll", "per_cta",
                                            "threads", "grid", "pdl")])

    def as_dict(self) -> dict:
        d = {f: getattr(self, f) for f, _ in self._fields_ if not f.startswith("_")}
        d["staging"], d["engine"] = STAGINGS[self.staging], ENGINES[self.engine]
        d["xreduce"], d["cache"] = XREDUCES[self.xreduce], CACHES[self.cache]
        return d


class EmitOpts(C.Structure):
    _fields_ = [("watchdog", C.c_uint32), ("max_reg_elems", C.c_uint32), ("max_unrolled", C.c_uint32),
                ("_pad", C.c_uint32)]


class Problem(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("_pad", C.c_uint32), ("m", C.c_int64), ("n", C.c_int64),
                ("k", C.c_int64), ("batch", C.c_int64), ("a_stride", C.c_int64), ("seed", C.c_uint64),
                ("alpha", C.c_float), ("_pad2", C.c_float)]


class TimeOpts(C.Structure):
    _fields_ = [("warmup", C.c_uint32), ("reps", C.c_uint32), ("flush_l2", C.c_uint32), ("check", C.c_uint32),
                ("bit_exact", C.c_uint32), ("rotate", C.c_uint32), ("rtol", C.c_double),
                ("budget_ns", C.c_double)]


class TimeResult(C.Structure):
    _fields_ = [("status", C.c_int), ("_pad", C.c_int), ("median_ns", C.c_double), ("min_ns", C.c_double),
                ("first_ns", C.c_double), ("max_err", C.c_double), ("mismatches", C.c_int64)]


class BatchItem(C.Structure):
    _fields_ = [("launch", C.POINTER(Launch)), ("opts", TimeOpts)]


class KernelSpec(C.Structure):
    _fields_ = [("kind", C.c_char_p), ("m", C.c_int64), ("n", C.c_int64), ("k", C.c_int64),
                ("a_stride", C.c_int64), ("num_factors", C.c_int32), ("factor_len", C.c_int32 * 4),
                ("factors", (C.c_int64 * 32) * 4), ("mode", C.c_int32), ("_pad", C.c_int32),
                ("batch", C.c_int64)]


class SpaceStats(C.Structure):
    _fields_ = [("instances", C.c_uint64), ("enum_instances", C.c_uint64), ("int_instances", C.c_uint64),
                ("counter_instances", C.c_uint64), ("objects", C.c_uint64), ("lowerings", C.c_uint64),
                ("root_open", C.c_uint64), ("root_digest", C.c_uint64), ("build_seconds", C.c_double)]


class BoundReport(C.Structure):
    _fields_ = [(f, C.c_double) for f in ("total", "dram", "sm_mem", "issue", "thread", "launch", "dram_bytes",
                                          "blocks_max", "threads_per_block_max", "dispatch", "l1", "lsu")]


class SearchConfig(C.Structure):
    _fields_ = [("device", C.c_int32), ("rollout_threads", C.c_int32), ("compile_threads", C.c_int32),
                ("batch", C.c_int32), ("seed", C.c_uint64), ("shard_index", C.c_int32), ("shard_count", C.c_int32),
                ("pruning", C.c_int32), ("watchdog", C.c_int32), ("reps", C.c_int32), ("warmup", C.c_int32),
                ("flush_l2", C.c_int32), ("max_unrolled", C.c_int32), ("budget_factor", C.c_double),
                ("max_budget_ns", C.c_double), ("decision_order", C.c_char_p), ("incumbent_shm", C.c_char_p),
                ("log_path", C.c_char_p), ("tree_depth", C.c_int32), ("rotate", C.c_int32),
                ("refine_factor", C.c_double), ("walk", C.c_int32), ("_pad", C.c_int32)]

WALK_SEARCH, WALK_UNIFORM = 0, 1


class SearchStats(C.Structure):
    _fields_ = ([(f, C.c_int64) for f in ("evaluations", "ok", "mismatches", "timeouts", "launch_errors",
                                           "illegal", "compile_errors", "duplicates", "rollouts", "dead_rollouts",
                                           "pruned_children", "bound_violations")]
                + [(f, C.c_double) for f in ("best_ns", "incumbent_ns", "best_bound_ns", "time_to_best_s",
                                             "elapsed_s", "device_step_ms", "t_rollout_s", "t_compile_s",
                                             "t_gpu_s")]
                + [("best_hash", C.c_uint64), ("frontier", C.c_int64), ("exhausted", C.c_int64),
                   ("refined", C.c_int64), ("device_busy_ms", C.c_double), ("t_launch_host_s", C.c_double),
                   ("frontier_total", C.c_int64), ("stealing_since", C.c_int64)])


# Every symbol include/ispc.h declares, with its ctypes signature.
ISPC_SYMBOLS = {
    "ispc_dev_inject_fault": (C.c_int, [C.c_void_p]),
    "ispc_emit_cuda": (C.c_int, [C.POINTER(Nest), C.POINTER(EmitOpts), C.c_char_p, C.c_char_p, C.c_size_t,
                                 C.POINTER(C.c_size_t), C.POINTER(Launch)]),
    "ispc_cuda_prelude": (C.c_char_p, []),
    "ispc_emit_pseudo": (C.c_int, [C.POINTER(Nest), C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "ispc_compile": (C.c_int, [C.POINTER(C.c_char_p), C.c_int, C.c_char_p, C.POINTER(C.c_void_p)]),
    "ispc_module_cubin": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]),
    "ispc_module_log": (C.c_char_p, [C.c_void_p]),
    "ispc_module_free": (None, [C.c_void_p]),
    "ispc_dev_open": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "ispc_dev_close": (None, [C.c_void_p]),
    "ispc_last_error": (C.c_char_p, [C.c_void_p]),
    "ispc_dev_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                C.POINTER(C.c_int)]),
    "ispc_bind_problem": (C.c_int, [C.c_void_p, C.POINTER(Problem)]),
    "ispc_problem_region": (C.c_int, [C.c_void_p, C.c_char_p, C.POINTER(C.c_uint64), C.POINTER(C.c_int64)]),
    "ispc_module_load": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_int)]),
    "ispc_module_unload": (C.c_int, [C.c_void_p, C.c_int]),
    "ispc_launch_timed": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(Launch), C.POINTER(TimeOpts),
                                    C.POINTER(TimeResult)]),
    "ispc_launch_batch": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(BatchItem), C.c_double,
                                    C.POINTER(TimeResult)]),
    "ispc_check": (C.c_int, [C.c_void_p, C.c_double, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                             C.POINTER(C.c_int)]),
    "ispc_read_region": (C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.c_size_t]),
    "ispc_write_region": (C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.c_size_t]),
    "ispc_read_expected": (C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.c_size_t]),
    "ispc_dev_mark": (C.c_int, [C.c_void_p, C.c_int]),
    "ispc_dev_mark_elapsed": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double)]),
    "ispc_host_register": (C.c_int, [C.c_void_p, C.c_size_t]),
    "ispc_host_unregister": (C.c_int, [C.c_void_p]),
    "ispc_evaluate": (C.c_int, [C.c_void_p, C.POINTER(Nest), C.POINTER(EmitOpts), C.POINTER(TimeOpts),
                                C.POINTER(TimeResult), C.POINTER(Launch)]),
    "ispc_emit_tiles": (C.c_int, [C.POINTER(TileConfig), C.c_char_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t),
                                  C.POINTER(Launch)]),
    "ispc_evaluate_tiles": (C.c_int, [C.c_void_p, C.POINTER(TileConfig), C.POINTER(TimeOpts),
                                      C.POINTER(TimeResult), C.POINTER(Launch)]),
}

class TreeEstimate(C.Structure):
    _fields_ = [("leaves", C.c_double), ("leaves_stderr", C.c_double), ("nodes", C.c_double),
                ("nodes_stderr", C.c_double), ("dead_ratio", C.c_double), ("iterations", C.c_int64),
                ("method", C.c_int32), ("_pad", C.c_int32)]


class EnumReport(C.Structure):
    _fields_ = [("nodes", C.c_int64), ("leaves", C.c_int64), ("dead_ends", C.c_int64), ("max_depth", C.c_int64)]


class DeadendReport(C.Structure):
    _fields_ = [("trials", C.c_int64), ("dead_ends", C.c_int64), ("ratio", C.c_double), ("ci_lo", C.c_double),
                ("ci_hi", C.c_double), ("mean_decisions", C.c_double)]


class SpecConfig(C.Structure):
    _fields_ = [("budget", C.c_int64), ("max_rollouts", C.c_int64), ("seed", C.c_uint64), ("order", C.c_char_p),
                ("pruning", C.c_int32), ("evaluator", C.c_int32), ("delta", C.c_double), ("bucket", C.c_int32),
                ("_pad", C.c_int32), ("log_path", C.c_char_p), ("resume_log", C.c_char_p)]


class SpecResult(C.Structure):
    _fields_ = [("evaluations", C.c_int64), ("rollouts", C.c_int64), ("dead_rollouts", C.c_int64),
                ("expanded", C.c_int64), ("duplicates", C.c_int64), ("time_to_best_evals", C.c_int64),
                ("replayed", C.c_int64),
                ("exhausted", C.c_int32), ("_pad", C.c_int32), ("best_cost", C.c_double),
                ("best_digest", C.c_uint64)]


SPEC_EVAL_BOUND, SPEC_EVAL_SIMULATE = 0, 1


HOST_SYMBOLS = {
    "ispc_space_create": (C.c_int, [C.POINTER(KernelSpec), C.POINTER(C.c_void_p)]),
    "ispc_space_free": (None, [C.c_void_p]),
    "ispc_space_stats_get": (C.c_int, [C.c_void_p, C.POINTER(SpaceStats)]),
    "ispc_space_problem": (C.c_int, [C.c_void_p, C.POINTER(Problem)]),
    "ispc_host_last_error": (C.c_char_p, []),
    "ispc_cand_root": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "ispc_cand_clone": (C.c_void_p, [C.c_void_p]),
    "ispc_cand_free": (None, [C.c_void_p]),
    "ispc_cand_decide": (C.c_int, [C.c_void_p, C.c_void_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p]),
    "ispc_cand_open_count": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ispc_cand_fully_specified": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ispc_cand_digest": (C.c_uint64, [C.c_void_p, C.c_void_p]),
    "ispc_cand_fired": (C.c_uint64, [C.c_void_p]),
    "ispc_cand_first_leaf": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    "ispc_cand_random_leaf": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.POINTER(C.c_void_p),
                                        C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "ispc_cand_random_leaf_ordered": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_char_p, C.c_int,
                                                C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "ispc_count_leaves": (C.c_int64, [C.c_void_p, C.c_void_p, C.c_int64]),
    "ispc_estimate_tree": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_uint64, C.c_char_p,
                                     C.POINTER(C.c_double)]),
    "ispc_estimate": (C.c_int, [C.c_void_p, C.c_void_p, C.c_char_p, C.c_int64, C.c_uint64, C.c_char_p,
                                C.c_char_p, C.POINTER(TreeEstimate)]),
    "ispc_estimate_synthetic": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int64, C.c_uint64, C.c_char_p,
                                          C.POINTER(TreeEstimate)]),
    "ispc_enumerate": (C.c_int, [C.c_void_p, C.c_void_p, C.c_char_p, C.c_int64, C.POINTER(EnumReport),
                                 C.POINTER(C.c_int64), C.c_int]),
    "ispc_enumerate_synthetic": (C.c_int, [C.c_char_p, C.c_int64, C.POINTER(EnumReport), C.POINTER(C.c_int64),
                                           C.c_int]),
    "ispc_deadend_rate": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_uint64, C.c_char_p,
                                    C.POINTER(DeadendReport)]),
    "ispc_deadend_exact": (C.c_int, [C.c_void_p, C.c_void_p, C.c_char_p, C.c_int64, C.POINTER(C.c_double)]),
    "ispc_cand_descend": (C.c_int, [C.c_void_p, C.c_void_p, C.c_char_p, C.c_uint64, C.c_int,
                                    C.POINTER(C.c_void_p)]),
    "ispc_order_round_trip": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64),
                                        C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "ispc_greedy_leaf": (C.c_int, [C.c_void_p, C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p),
                                   C.POINTER(C.c_double)]),
    "ispc_prune_profile": (C.c_int, [C.c_void_p, C.c_void_p, C.c_char_p, C.c_double, C.c_int, C.c_int64,
                                     C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "ispc_explore_spec": (C.c_int, [C.c_void_p, C.POINTER(SpecConfig), C.POINTER(SpecResult), C.c_char_p,
                                    C.c_size_t, C.POINTER(C.c_size_t)]),
    "ispc_tag_select": (C.c_int, [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_ubyte),
                                  C.c_int64, C.c_double, C.c_int]),
    "ispc_walk_digests": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int64, C.POINTER(C.c_uint64)]),
    "ispc_cand_to_nest": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
    "ispc_cand_to_tiles": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(TileConfig)]),
    "ispc_nest_buf_get": (C.POINTER(Nest), [C.c_void_p]),
    "ispc_nest_buf_free": (None, [C.c_void_p]),
    "ispc_cand_reference_source": (C.c_int, [C.c_void_p, C.c_void_p, C.c_char_p, C.c_size_t,
                                             C.POINTER(C.c_size_t)]),
    "ispc_cand_simulate": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]),
    "ispc_cand_serialize": (C.c_int, [C.c_void_p, C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "ispc_cand_deserialize": (C.c_int, [C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p)]),
    "ispc_bound": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(BoundReport)]),
    "ispc_search_create": (C.c_int, [C.c_void_p, C.POINTER(SearchConfig), C.POINTER(C.c_void_p)]),
    "ispc_search_step": (C.c_int, [C.c_void_p, C.c_int64]),
    "ispc_search_step_for": (C.c_int, [C.c_void_p, C.c_int64, C.c_double]),
    "ispc_search_stats_get": (C.c_int, [C.c_void_p, C.POINTER(SearchStats)]),
    "ispc_search_best": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "ispc_search_best_source": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "ispc_search_elite": (C.c_int, [C.c_void_p, C.c_int, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "ispc_search_error": (C.c_char_p, [C.c_void_p]),
    "ispc_search_free": (None, [C.c_void_p]),
    "ispc_search_write_region": (C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.c_size_t]),
    "ispc_search_read_region": (C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.c_size_t]),
    "ispc_search_frontier": (C.c_int64, [C.c_void_p, C.POINTER(C.c_uint64), C.c_int64]),
    "ispc_search_offer": (C.c_int, [C.c_void_p, C.c_double]),
}

_libs: dict[str, C.CDLL] = {}


def _load(path: str, symbols: dict) -> C.CDLL:
    if path in _libs:
        return _libs[path]
    if not os.path.exists(path):
        raise ImportError(f"{path} is not built; run __graft_entry__.build() (no CPU fallback exists)")
    lib = C.CDLL(path, mode=C.RTLD_GLOBAL)
    for name, (res, args) in symbols.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _libs[path] = lib
    return lib


def ispc() -> C.CDLL:
    return _load(LIBISPC_PATH, ISPC_SYMBOLS)


def host() -> C.CDLL:
    ispc()  # the host library links libispc; load it first with its signatures
    return _load(LIBHOST_PATH, HOST_SYMBOLS)


def read_text(fn, *args) -> str:
    """Calls a (..., char* buf, size_t cap, size_t* len) entry point twice."""
    n = C.c_size_t(0)
    rc = fn(*args, None, 0, C.byref(n))
    if rc != 0:
        raise RuntimeError(last_error())
    buf = C.create_string_buffer(n.value + 1)
    rc = fn(*args, buf, n.value + 1, C.byref(n))
    if rc != 0:
        raise RuntimeError(last_error())
    return buf.value.decode()


def last_error(dev=None) -> str:
    e = ispc().ispc_last_error(dev)
    return e.decode() if e else ""


def host_error() -> str:
    e = host().ispc_host_last_error()
    return e.decode() if e else ""
