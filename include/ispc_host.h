/*
 * ispc_host.h — C-ABI of the reference-side host library (libispc_host.so).
 *
 * This library lives on the CALLER side of the boundary declared in ispc.h:
 * it links the reference search-space library (namespace ispace) unchanged
 * and exposes, as plain C, what a driver needs to walk the space and hand
 * fully specified candidates to the B200 backend:
 *
 *   kernel builders       make_axpy / make_matmul / make_outer_product
 *                         (proj/core/include/ispace/kernels.hpp:110-121)
 *   space construction    build_gpu_space (gpu_space.hpp:18) with MachineParams
 *                         (machine.hpp:17-34)
 *   candidates            make_root / apply_decision / open_choices /
 *                         fully_specified / digest (candidate.hpp:69-95)
 *   reconstruction        reconstruct (loop_nest.hpp:52) -> flat ispc_nest
 *   reference evaluation  emit_source (loop_nest.hpp:62), evaluate
 *                         (simulate.hpp:33) for cross-checks
 *   B200 lower bound      ispc_bound (the reference's bound.cpp is a stub;
 *                         contract SPEC.md:416-457, re-parameterised in seconds)
 *   branch and bound      ispc_search_run (the reference's search.cpp is a stub;
 *                         contract SPEC.md:459-514) sharding subtrees over GPUs
 *
 * Status convention as in ispc.h. Decisions return 0 (ok), 1 (dead end).
 */
#ifndef ISPC_HOST_H
#define ISPC_HOST_H

#include <stddef.h>
#include <stdint.h>

#include "ispc.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ispc_space ispc_space;
typedef struct ispc_cand ispc_cand;
typedef struct ispc_nest_buf ispc_nest_buf;

/* Space modes: PARITY = the reference's gpu.space and default MachineParams
 * (candidate counts equal the reference's); B200 = the same space bound to
 * B200 machine limits (227 KiB shared memory per block). */
enum ispc_space_mode { ISPC_SPACE_PARITY = 0, ISPC_SPACE_B200 = 1 };

typedef struct {
  const char* kind;       /* reference gpu.space: "axpy" | "outer_product" | "matmul";
                             building blocks (tiles.space): "gemv" | "sgemm" |
                             "batched" | "sgemm_tc"                                  */
  int64_t m, n, k;        /* axpy uses n                                          */
  int64_t a_stride;       /* matmul: element stride of A (1 = dense)              */
  int32_t num_factors;    /* strip-mining universes, outermost first              */
  int32_t factor_len[4];  /* values per universe                                  */
  int64_t factors[4][32];
  int32_t mode;           /* ispc_space_mode                                      */
  int32_t _pad;
  int64_t batch;          /* batched: number of independent problems              */
} ispc_kernel_spec;

typedef struct {
  uint64_t instances;       /* choice instances (enum + integer + counter)        */
  uint64_t enum_instances, int_instances, counter_instances;
  uint64_t objects;         /* backbone objects                                   */
  uint64_t lowerings;
  uint64_t root_open;       /* open choices at the root                           */
  uint64_t root_digest;
  double build_seconds;
} ispc_space_stats;

int ispc_space_create(const ispc_kernel_spec* spec, ispc_space** out);
void ispc_space_free(ispc_space* s);
int ispc_space_stats_get(const ispc_space* s, ispc_space_stats* out);
int ispc_space_problem(const ispc_space* s, ispc_problem* out); /* matching ispc_problem */
const char* ispc_host_last_error(void);

int ispc_cand_root(const ispc_space* s, ispc_cand** out);
ispc_cand* ispc_cand_clone(const ispc_cand* c);
void ispc_cand_free(ispc_cand* c);
/* Named decision, in the orientation the names are given (antisymmetric
 * choices resolved like nest_test.cpp:36-55). 0 ok, 1 dead end, <0 error. */
int ispc_cand_decide(const ispc_space* s, ispc_cand* c, const char* choice, const char* arg0,
                     const char* arg1, const char* value);
int ispc_cand_open_count(const ispc_space* s, const ispc_cand* c);
int ispc_cand_fully_specified(const ispc_space* s, const ispc_cand* c);
uint64_t ispc_cand_digest(const ispc_space* s, const ispc_cand* c);
uint64_t ispc_cand_fired(const ispc_cand* c);

/* First-open depth-first descent, values in index order (nest_test.cpp:57-75). */
int ispc_cand_first_leaf(const ispc_space* s, const ispc_cand* from, int budget, ispc_cand** out);
/* Uniform random descent with restart on dead ends: at each step the first
 * open instance in `order` (NULL: declaration order) gets a uniformly drawn
 * value. Reports decisions applied and dead ends met. 0 ok, 1 gave up. */
int ispc_cand_random_leaf(const ispc_space* s, const ispc_cand* from, uint64_t seed, int max_restarts,
                          ispc_cand** out, int64_t* decisions, int64_t* dead_ends);
/* Same, deciding the open instance that comes first in `order` (comma
 * separated choice names, e.g. the paper's "size,dim_kind,thread_level,
 * mem_space,order,cache"). */
int ispc_cand_random_leaf_ordered(const ispc_space* s, const ispc_cand* from, uint64_t seed, const char* order,
                                  int max_restarts, ispc_cand** out, int64_t* decisions, int64_t* dead_ends);
/* Knuth's tree-size estimator (the reference's tree_size.cpp is a stub;
 * SPEC.md:516-567): `probes` random descents from `from` branching like
 * ispc_count_leaves (or by `order`). out = {leaves, leaves_stderr, nodes,
 * dead-end probe ratio, probes}. */
int ispc_estimate_tree(const ispc_space* s, const ispc_cand* from, int64_t probes, uint64_t seed, const char* order,
                       double out[5]);
/* Exhaustive first-open enumeration; returns the number of leaves (capped). */
int64_t ispc_count_leaves(const ispc_space* s, const ispc_cand* from, int64_t cap);

/* ---- tree-size estimators, enumeration, dead ends, prune profile ----------
 * The reference's tree_size.cpp is a stub (proj/core/src/tree_size.cpp:1);
 * contract SPEC.md:516-567 and paper sections 5.2-5.4. The tree below `from`
 * branches on the first open instance (or the first in `order`, comma
 * separated choice names); children are the values surviving apply_decision. */
typedef struct {
  double leaves, leaves_stderr;  /* estimate of the leaf count, its standard error */
  double nodes, nodes_stderr;    /* estimate of the node count                    */
  double dead_ratio;             /* knuth: probes ending at a dead end;
                                    chen: runs reaching no leaf                   */
  int64_t iterations;            /* knuth probes / chen runs                      */
  int32_t method;                /* 0 knuth, 1 chen                               */
  int32_t _pad;
} ispc_tree_estimate;
/* method "knuth" (random descents, product of branching factors) or "chen"
 * (heuristic sampling over strata; stratifier "depth_remaining" = the paper's
 * (depth, remaining open instances) pair, "depth", "remaining", or "constant",
 * which violates strict decrease and is reported as ISPC_E_ARG). */
int ispc_estimate(const ispc_space* s, const ispc_cand* from, const char* method, int64_t iterations,
                  uint64_t seed, const char* order, const char* stratifier, ispc_tree_estimate* out);
/* The same estimators on closed-form trees (their known answers):
 * "uniform:B,D", "caterpillar:D,H", "random:S,B,D". */
int ispc_estimate_synthetic(const char* tree, const char* method, int64_t iterations, uint64_t seed,
                            const char* stratifier, ispc_tree_estimate* out);
typedef struct {
  int64_t nodes, leaves, dead_ends, max_depth;
} ispc_enum_report;
/* Exact depth-first enumeration; ISPC_E_ARG (refusal) past node_budget nodes.
 * per_depth[d] (d < depth_cap) = nodes at depth d. */
int ispc_enumerate(const ispc_space* s, const ispc_cand* from, const char* order, int64_t node_budget,
                   ispc_enum_report* out, int64_t* per_depth, int depth_cap);
int ispc_enumerate_synthetic(const char* tree, int64_t node_budget, ispc_enum_report* out, int64_t* per_depth,
                             int depth_cap);
typedef struct {
  int64_t trials, dead_ends;
  double ratio, ci_lo, ci_hi;  /* 95% Wilson score interval */
  double mean_decisions;
} ispc_deadend_report;
/* Uniform random descents without pruning (paper section 5.2, Table 2). */
int ispc_deadend_rate(const ispc_space* s, const ispc_cand* from, int64_t trials, uint64_t seed, const char* order,
                      ispc_deadend_report* out);
/* A uniform partial descent of `steps` decisions among the surviving
 * children (subtrees for the estimator oracles). 1: dead end or leaf first. */
int ispc_cand_descend(const ispc_space* s, const ispc_cand* from, const char* order, uint64_t seed, int steps,
                      ispc_cand** out);
/* Exact probability that such a descent meets a dead end (small trees;
 * ISPC_E_ARG past node_budget nodes): the oracle of ispc_deadend_rate. */
int ispc_deadend_exact(const ispc_space* s, const ispc_cand* from, const char* order, int64_t node_budget,
                       double* p_dead);
/* The lowest-bound descent: children in ascending B200 bound (ties: value
 * order), backtracking out of dead ends and infinite-bound subtrees; 1 when
 * no leaf is found within its node budget. */
int ispc_greedy_leaf(const ispc_space* s, const ispc_cand* from, const char* order, ispc_cand** out,
                     double* bound_s);
/* The reference's order round trip (nest_test.cpp:309-334) over every leaf
 * below `from`: derive_orders(reconstruct(leaf)) against the leaf's order
 * decisions. Counts leaves, derived pairs and pairs that disagree. */
int ispc_order_round_trip(const ispc_space* s, const ispc_cand* from, int64_t node_budget, int64_t* leaves,
                          int64_t* pairs, int64_t* mismatches);
/* Paper section 5.4: nodes per depth of the first depth_cap levels and how
 * many have a B200 bound >= threshold_s (prunable against incumbent T). */
int ispc_prune_profile(const ispc_space* s, const ispc_cand* from, const char* order, double threshold_s,
                       int depth_cap, int64_t node_budget, int64_t* nodes_per_depth, int64_t* pruned_per_depth);

/* Building-block spaces: the decided tile configuration (ispc.h). */
int ispc_cand_to_tiles(const ispc_space* s, const ispc_cand* c, ispc_tile_config* out);

/* reconstruct() + flatten. */
int ispc_cand_to_nest(const ispc_space* s, const ispc_cand* c, ispc_nest_buf** out);
const ispc_nest* ispc_nest_buf_get(const ispc_nest_buf* b);
void ispc_nest_buf_free(ispc_nest_buf* b);

/* Reference-side renderings / costs of the same candidate. */
int ispc_cand_reference_source(const ispc_space* s, const ispc_cand* c, char* buf, size_t cap, size_t* len);
/* evaluate(): out = {compute, memory, sync, block_serial, total} cycles. */
int ispc_cand_simulate(const ispc_space* s, const ispc_cand* c, int64_t out[5]);
int ispc_cand_serialize(const ispc_space* s, const ispc_cand* c, char* buf, size_t cap, size_t* len);
int ispc_cand_deserialize(const ispc_space* s, const char* text, ispc_cand** out);

/* ---- deterministic TAG-MCTS ------------------------------
 * Single-threaded, no clocks: the same seed and configuration give the same
 * evaluations, best candidate and byte-identical JSONL log (one record per
 * rollout: seed, path of decision values, cost or DEADEND, ancestor bounds).
 * Evaluators: BOUND = the B200 bound x (1 + u), u in [0, 0.5) hashed from the
 * leaf digest (admissible by construction: pruning on and off must agree on
 * the optimum); SIMULATE = the reference's reconstruct + evaluate cycles
 * (simulate.cpp:131-133) with a zero bound. */
enum ispc_spec_evaluator { ISPC_SPEC_EVAL_BOUND = 0, ISPC_SPEC_EVAL_SIMULATE = 1 };
typedef struct {
  int64_t budget;        /* evaluations (distinct leaves)                      */
  int64_t max_rollouts;  /* 0: unlimited                                       */
  uint64_t seed;
  const char* order;     /* comma separated choice names; NULL: first open     */
  int32_t pruning;       /* exclude / zero-weight children with bound >= T     */
  int32_t evaluator;     /* ispc_spec_evaluator                                */
  double delta;          /* TAG confidence (0: 0.05)                           */
  int32_t bucket;        /* TAG top-s set size (0: 20)                         */
  int32_t _pad;
  const char* log_path;  /* JSONL per rollout, NULL: none                      */
  const char* resume_log; /* checkpoint: a log of an earlier run (same seed and
                             configuration); its records are re-derived and must
                             match, then the run continues to `budget` (NULL: none) */
} ispc_spec_config;
typedef struct {
  int64_t evaluations, rollouts, dead_rollouts, expanded, duplicates;
  int64_t time_to_best_evals;  /* evaluations when the best was first met     */
  int64_t replayed;            /* resume-log records re-derived and matched    */
  int32_t exhausted;           /* the whole tree was evaluated or excluded     */
  int32_t _pad;
  double best_cost;            /* seconds (BOUND) or cycles (SIMULATE); inf: none */
  uint64_t best_digest;
} ispc_spec_result;
int ispc_explore_spec(const ispc_space* s, const ispc_spec_config* cfg, ispc_spec_result* out, char* best_text,
                      size_t cap, size_t* len);
/* The TAG rule: unvisited (t <= 0) non-excluded children first, lowest index;
 * then argmax (s + a + sqrt(2 s a + a^2)) / t with a = ln(2 total k / delta);
 * -1 when every child is excluded. */
int ispc_tag_select(int k, const double* s, const double* t, const unsigned char* excluded, int64_t total,
                    double delta, int bucket);
/* Seeded uniform first-open descents sharing one mt19937_64(seed), the walk of
 * oracle/ref_cpu_bench.cpp: leaf digest per walk, 0 for a dead end. */
int ispc_walk_digests(const ispc_space* s, const ispc_cand* from, uint64_t seed, int64_t walks, uint64_t* digests);

/* ---- B200 lower bound (seconds) ------------------------------------------- */
typedef struct {
  double total, dram, sm_mem, issue, thread, launch; /* seconds */
  double dram_bytes, blocks_max, threads_per_block_max;
  double dispatch, l1;      /* seconds: block dispatch floor, L1 lines of scattered warp accesses */
  double lsu;               /* seconds: memory warp-instructions at 1 per SM cycle */
} ispc_bound_report;
/* l2_flushed: inputs start outside L2 (the timing flushes L2 between runs). */
int ispc_bound(const ispc_space* s, const ispc_cand* c, int l2_flushed, ispc_bound_report* out);

/* ---- bound-pruned search with measured evaluation ------------------------- */
typedef struct ispc_search ispc_search;

typedef struct {
  int32_t device;           /* CUDA ordinal of this worker's B200; -1 dry run (NVRTC,
                               no device), -2 dry run without NVRTC (host pipeline) */
  int32_t rollout_threads;  /* 0: auto                                          */
  int32_t compile_threads;  /* 0: auto                                          */
  int32_t batch;            /* kernels per NVRTC program (0: 8)                 */
  uint64_t seed;
  int32_t shard_index;      /* this worker's share of the frontier              */
  int32_t shard_count;
  int32_t pruning;          /* 1: bound pruning + p ~ max(T-b,0) rollouts, 0: uniform */
  int32_t watchdog;         /* emit option (1: always)                          */
  int32_t reps, warmup;     /* timed / untimed launches per candidate           */
  int32_t flush_l2;         /* L2 flush before each launch                      */
  int32_t max_unrolled;     /* emit budget (0: 512)                             */
  double budget_factor;     /* watchdog budget = factor x incumbent (0: 3)      */
  double max_budget_ns;     /* budget before any incumbent (0: 50 ms)           */
  const char* decision_order; /* comma separated choice names; NULL: paper order */
  const char* incumbent_shm;  /* POSIX shm name shared by ranks; NULL: process-local */
  const char* log_path;       /* JSONL evaluation log; NULL: none              */
  int32_t tree_depth;         /* TAG-MCTS tree over the first decisions (0: 12, <0: off) */
  int32_t rotate;             /* > 1: time each candidate over this many input copies
                                 (ispc_time_opts.rotate) instead of L2 flushes */
  double refine_factor;       /* re-time (warmup + reps) only the kernels whose screened
                                 first launch is <= factor x incumbent (0: 1.25); the
                                 others keep their single checked launch's time */
  int32_t walk;               /* ISPC_WALK_SEARCH (default) or ISPC_WALK_UNIFORM          */
  int32_t _pad;
} ispc_search_config;

/* ISPC_WALK_UNIFORM: seeded uniform first-open descents from the root, every
 * leaf evaluated - the walk of the reference's CPU baseline
 * (oracle/ref_cpu_bench.cpp), so the two arms measure the same candidates'
 * evaluation; no bound, incumbent pruning, tree or aspiration band. */
enum { ISPC_WALK_SEARCH = 0, ISPC_WALK_UNIFORM = 1 };

typedef struct {
  int64_t evaluations;      /* kernels launched on the device                   */
  int64_t ok, mismatches, timeouts, launch_errors;
  int64_t illegal, compile_errors, duplicates;
  int64_t rollouts, dead_rollouts, pruned_children, bound_violations;
  double best_ns;           /* best measured median (this worker's view)        */
  double incumbent_ns;      /* shared incumbent (all ranks)                     */
  double best_bound_ns;     /* bound of the best leaf                           */
  double time_to_best_s, elapsed_s;
  double device_step_ms;    /* device-timeline duration of the last step()      */
  double t_rollout_s, t_compile_s, t_gpu_s; /* busy time per stage (summed over threads) */
  uint64_t best_hash;
  int64_t frontier;         /* subtree roots owned by this shard                */
  int64_t exhausted;        /* 1: no new kernel survives pruning in this shard  */
  int64_t refined;          /* kernels re-timed after their screening launch    */
  double device_busy_ms;    /* device time of the timed launches in the last step */
  double t_launch_host_s;   /* launch thread: host time spent per batch outside the
                               device waits (binding, enqueue, result processing) */
  int64_t frontier_total;   /* subtree roots of the whole (all-shard) frontier     */
  int64_t stealing_since;   /* rollouts when this shard's own subtrees were spent and
                               it began stealing from the whole frontier (-1: never) */
} ispc_search_stats;

int ispc_search_create(const ispc_space* s, const ispc_search_config* cfg, ispc_search** out);
/* Runs until `evaluations` more kernels were measured (the pipeline keeps
 * running between calls). Records device-timeline marks around the step. */
int ispc_search_step(ispc_search* h, int64_t evaluations);
/* Same with a wall-clock deadline: returns ISPC_E_TIMEOUT when fewer kernels
 * could be produced and measured in `max_seconds` (0: no deadline). */
int ispc_search_step_for(ispc_search* h, int64_t evaluations, double max_seconds);
int ispc_search_stats_get(const ispc_search* h, ispc_search_stats* out);
/* Best candidate (reference text serialization) and its CUDA source. */
int ispc_search_best(const ispc_search* h, char* buf, size_t cap, size_t* len);
int ispc_search_best_source(const ispc_search* h, char* buf, size_t cap, size_t* len);
/* The i-th best measured leaf the search keeps for its elite-guided rollouts
 * (fastest first; at most 8, only when elite guidance is on: the building-block
 * spaces), reference text serialization; "" past the last. */
int ispc_search_elite(const ispc_search* h, int i, char* buf, size_t cap, size_t* len);
const char* ispc_search_error(const ispc_search* h);
/* Host <-> device copies of the search's bound problem between steps (the
 * end-to-end measurement uploads inputs and reads the output every step). */
int ispc_search_write_region(ispc_search* h, const char* name, const void* host, size_t bytes);
int ispc_search_read_region(ispc_search* h, const char* name, void* host, size_t bytes);
void ispc_search_free(ispc_search* h);
/* Digests of this shard's subtree roots (disjoint across shards); returns the
 * count, writes at most `cap`. */
int64_t ispc_search_frontier(const ispc_search* h, uint64_t* digests, int64_t cap);
/* Offers a measured time to the shared incumbent (CAS-min across ranks);
 * 1 when it became the new incumbent. Used by external evaluators and tests. */
int ispc_search_offer(ispc_search* h, double ns);

#ifdef __cplusplus
}
#endif
#endif /* ISPC_HOST_H */
