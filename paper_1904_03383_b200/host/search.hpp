// Bound-pruned Monte-Carlo search over the reference's decision space with
// measured evaluation on a B200 (the reference's search.cpp is a stub,
// proj/core/src/search.cpp:1; contract SPEC.md:459-514).
//
// Pipeline (one process per GPU):
//   rollout threads   descend from this shard's subtree roots in the fixed
//                     decision order (size, dim_kind, thread_level, mem_space,
//                     order, cache). At each decision every
//                     child is propagated (apply_decision) and bounded; children
//                     with bound >= incumbent T are pruned and the rest drawn with
//                     p ~ max(T - b, 0). Leaves are
//                     reconstructed, flattened and emitted as sm_100a CUDA.
//   compile threads   batch emitted kernels into NVRTC programs (sm_100a cubins)
//   launch thread     loads each cubin on the device, times every kernel with a
//                     watchdog budget of max(T x factor) and checks it on device,
//                     then CAS-mins the incumbent
// Sharding: the first levels of the tree are expanded deterministically into a
// frontier; shard i owns frontier nodes i, i+S, i+2S, ... (disjoint subtrees,
// no collective). The incumbent is one 64-bit cell in POSIX shared memory
// (pinned through libispc), read by every rank before pruning.
#pragma once

#include <atomic>
#include <limits>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <memory>
#include <mutex>
#include <shared_mutex>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "adapter.hpp"
#include "bound.hpp"
#include "host_internal.hpp"
#include "ispc.h"
#include "ispc_host.h"

namespace ispc_host {

struct Incumbent {
  std::atomic<uint64_t>* cell = nullptr;  // best measured time, ns (0: none yet)
  void* map = nullptr;
  size_t map_bytes = 0;
  bool pinned = false;
  std::string name;
  std::unique_ptr<std::atomic<uint64_t>> local;
  void open(const char* shm_name);
  void pin();
  void repin();
  ~Incumbent();
  double seconds() const;
  bool offer(uint64_t ns);  // true when it became the new best
};

// One node of the Monte-Carlo tree over the first `tree_depth` decisions of
// a shard. Children are the propagated
// values of the node's next decision that survived pruning; per child the
// search keeps the visit count and the measured times of the leaves below
// it, for the TAG (threshold ascent on graphs) selection rule.
struct MctsNode {
  ispace::Candidate cand;
  bool expanded = false, dead = false;
  std::vector<ispace::Candidate> kid_cand;
  std::vector<double> kid_bound;
  std::vector<std::unique_ptr<MctsNode>> kids;
  std::vector<int64_t> visits;
  std::vector<std::vector<double>> times;  // measured ns of leaves below each child
  std::vector<double> leaf_min;             // smallest leaf bound (s) produced below each child
  int64_t total = 0;
};

struct Work {
  ispace::Candidate leaf;
  std::vector<std::pair<MctsNode*, int>> path;  // tree edges taken (TAG back-propagation)
  std::unique_ptr<NestBuf> nest;
  std::string src;
  ispc_launch launch{};
  double bound_s = 0;
  uint64_t digest = 0;
  size_t root = 0;  // index of the shard subtree the leaf came from
  int tid = 0;             // rollout thread that produced it
  int64_t rollout_no = 0;  // that thread's rollout counter
  bool bit_exact = true;  // parity-mode and FFMA sgemm outputs: identical bits
  double rtol = 1e-5;     // otherwise: |out - exp| <= rtol * sum |products|
};

struct CompiledBatch {
  std::vector<std::unique_ptr<Work>> items;
  ispc_module* module = nullptr;
  int handle = 0;       // loaded on the device by the compile thread (0: not loaded)
  int load_rc = 0;      // ispc_module_load status
  std::string load_err;
};

// Digests of partial candidates every completion of which is pruned or was
// already produced (a dead end a rollout ran into, or a leaf it emitted).
// The pruning threshold only falls, so membership is permanent; descents skip
// such children instead of walking into them again. Sharded for the rollout
// threads.
class DeadSet {
 public:
  bool has(uint64_t d) {
    Shard& s = shards_[d % kShards];
    std::lock_guard<std::mutex> lk(s.mu);
    return s.set.count(d) != 0;
  }
  void add(uint64_t d) {
    Shard& s = shards_[d % kShards];
    std::lock_guard<std::mutex> lk(s.mu);
    s.set.insert(d);
  }
  size_t size() {
    size_t n = 0;
    for (Shard& s : shards_) {
      std::lock_guard<std::mutex> lk(s.mu);
      n += s.set.size();
    }
    return n;
  }

 private:
  static constexpr size_t kShards = 64;
  struct Shard {
    std::mutex mu;
    std::unordered_set<uint64_t> set;
  };
  Shard shards_[kShards];
};

class Search {
 public:
  Search(const ispc_space* space, const ispc_search_config& cfg);
  ~Search();
  int step(int64_t evaluations, double max_seconds = 0);
  ispc_search_stats stats() const;
  std::string best_candidate() const;
  // the i-th of the best measured leaves (elite-guided rollouts keep 8), "" past the end
  std::string elite_candidate(size_t i) const;
  std::string best_source() const;
  ispc_launch best_launch() const;
  std::string error() const { return err_; }
  std::vector<uint64_t> frontier_digests() const;
  bool offer(double ns) { return inc_.offer(uint64_t(ns < 1 ? 1 : ns)); }
  // host <-> device copy of a problem region while the device is idle
  int region_io(const char* name, void* host, size_t bytes, bool upload);

 private:
  const ispc_space* space_;
  ispc_search_config cfg_;
  std::string order_text_, shm_text_, log_text_;
  B200Machine machine_;
  std::unique_ptr<BoundModel> model_;
  DecisionOrder order_;
  // every rank computes the same frontier; this shard owns the indices in
  // mine_ and, once those are spent (exhausted), steals: its rollouts start
  // from any frontier subtree (stealing_), so no GPU idles while others work
  std::vector<ispace::Candidate> subtrees_;  // the whole frontier
  std::vector<size_t> mine_;
  std::atomic<bool> stealing_{false};
  std::atomic<int64_t> stealing_since_{-1};  // rollout count when stealing began (-1: never)
  Incumbent inc_;
  ispc_dev* dev_ = nullptr;
  std::shared_mutex dev_mu_;          // module loads (shared) against device replacement
  int64_t inject_fault_at_ = -1;     // ISPC_INJECT_FAULT_AT: batch number (fault-handling tests)
  int64_t batches_launched_ = 0;     // launch thread only
  std::string err_;
  FILE* log_ = nullptr;

  // pipeline
  std::mutex mu_;
  std::condition_variable cv_work_, cv_batch_, cv_done_;
  std::deque<std::unique_ptr<Work>> work_q_;
  std::deque<std::unique_ptr<CompiledBatch>> batch_q_;
  std::unordered_set<uint64_t> seen_hash_;
  // digests of every leaf a rollout has produced: a rollout that reaches one
  // again backtracks to an untried sibling instead of re-emitting it
  std::unordered_set<uint64_t> seen_leaf_;
  std::mutex seen_leaf_mu_;
  DeadSet dead_;
  static constexpr int kRolloutExpansions = 96;  // node expansions one rollout may spend backtracking
  std::vector<std::thread> threads_;
  std::atomic<bool> stop_{false};
  std::atomic<int64_t> target_{0};
  std::atomic<uint64_t> subtree_cursor_{0};
  bool pipeline_started_ = false;
  bool launching_ = false;  // guarded by mu_
  bool step_open_ = false;  // guarded by mu_: device mark 0 recorded for this step
  bool trace_ = false;      // ISPC_TRACE: one stderr line per launch
  // ISPC_ROLLOUT: what a rollout does at a dead end or an already produced
  // leaf: 0 "restart" from the tree (the paper's rollout), 1 "deep" (resume
  // from the deepest frame with an untried child), 2 "ancestor" (resume from
  // a uniformly drawn ancestor frame)
  int rollout_mode_ = 0;
  // ISPC_GREEDY: the greedy half of the rollout draws takes the lowest-bound
  // child; ties (many children share the DRAM floor) go to 0 "first" in value
  // order, 1 "random"; 2 "off" samples every draw p ~ max(T - b, 0)
  int greedy_mode_ = 1;
  double greedy_p_ = 0.9;  // ISPC_GREEDY_P: share of greedy draws (0.5 in the first version)
  // ISPC_LEAFB_P: share of in-tree selections (once every child was visited)
  // that take the child with the smallest leaf bound produced below it; the
  // rest use the TAG score. Leaves of low bound are rare and run fast (the
  // fused axpy schedules: bound 88 µs, measured 117-125 µs), which a score of
  // measured top-16 times alone learns slowly.
  double leafb_p_ = 0.5;
  // ISPC_SHARP (gamma): the sampled draws weight a child by
  // max(T - b, 0) * exp(-gamma (b - b_min) / b_min), b_min the lowest bound
  // among the siblings; 0 = the paper's p ~ max(T - b, 0)
  double sharp_ = 8.0;
  bool lazy_greedy_ = true;  // ISPC_LAZY=0: greedy draws expand every child
  // ISPC_ASPIRE (kappa, 0 = off; 1.5 by default on loop-nest spaces): a leaf
  // whose bound exceeds kappa x the lowest leaf bound produced so far is not
  // evaluated (a heuristic filter on top of the admissible b >= T pruning)
  double aspire_ = 0.0;
  std::atomic<double> min_leaf_bound_{std::numeric_limits<double>::infinity()};
  double prune_threshold() const;
  // elite-guided rollouts (ISPC_ELITE_Q, ISPC_ELITE_MUT): a share q of the
  // rollouts copies the decisions of one of the kElite best measured leaves,
  // deviating at ~mut randomly drawn decisions (local search around the
  // incumbents; the rest explore through the tree as before)
  static constexpr size_t kElite = 8;
  double elite_q_ = 0.0, elite_mut_ = 2.0;  // tiles 0.5, loop nests off (constructor)
  struct Elite {
    double ns;
    size_t root;
    ispace::Candidate leaf;
  };
  std::vector<Elite> elites_;  // ascending ns, under elite_mu_
  std::mutex elite_mu_;
  std::atomic<int64_t> decisions_per_leaf_{0};  // running estimate of the decisions below a subtree root
  void note_elite(double ns, size_t root, const ispace::Candidate& leaf);

  // statistics (guarded by mu_ unless atomic)
  ispc_search_stats st_{};
  std::atomic<int64_t> rollouts_{0}, dead_rollouts_{0}, pruned_{0}, illegal_{0}, duplicates_{0};
  std::atomic<int64_t> compile_errors_{0};
  // consecutive rollouts (all threads) that queued no new kernel: dead ends,
  // illegal or duplicate leaves. Past kExhaust the shard's subtrees are
  // exhausted under the current incumbent and step() returns early.
  static constexpr int64_t kExhaust = 3000;
  std::atomic<int64_t> fruitless_{0};
  std::atomic<bool> exhausted_{false};
  std::atomic<int> compiling_{0};  // batches inside NVRTC right now
  void note_fruitless();
  std::atomic<double> t_rollout_{0}, t_compile_{0};
  double t_launch_host_ = 0;     // launch thread outside device waits (under mu_)
  double step_busy_ms_ = 0;      // device time of timed launches in the open step (under mu_)
  int64_t refined_ = 0;          // under mu_
  double refine_factor_ = 1.25;
  bool uniform_ = false;         // ISPC_WALK_UNIFORM
  std::vector<int> retired_;     // loaded modules already evaluated (launch thread only)
  static constexpr size_t kMaxRetired = 4096;
  bool log_dead_ = false;        // ISPC_LOG_DEADENDS=1: JSONL records of rollouts that queued no kernel
  bool uniform_walk(std::mt19937_64& rng, ispace::Candidate& leaf);
  double t0_ = 0;
  std::string best_text_, best_src_;
  ispc_launch best_launch_{};

  double bound_total(const ispace::Candidate& c) const;
  void expand_frontier();
  bool rollout(std::mt19937_64& rng, ispace::Candidate& leaf, double& leaf_bound,
               std::vector<std::pair<MctsNode*, int>>& path, size_t& root_out);
  bool descend(std::mt19937_64& rng, ispace::Candidate cur, const ispace::Candidate* guide, double p_mut,
               ispace::Candidate& leaf, double& leaf_bound, MctsNode* node);
  // TAG-MCTS state (guarded by tree_mu_)
  std::mutex tree_mu_;
  std::vector<std::unique_ptr<MctsNode>> tree_roots_;
  std::vector<double> top_;  // the kTop best measured times (ns), ascending
  static constexpr size_t kTop = 16;
  int tree_depth_ = 12;
  int select_child(MctsNode& n, double T, std::mt19937_64& rng);
  void backprop(const std::vector<std::pair<MctsNode*, int>>& path, double ns);
  void worker(int tid);
  void rollout_one(int tid, std::mt19937_64& rng, int64_t& k_roll, const ispc_emit_opts& eo);
  void compile_items(std::vector<std::unique_ptr<Work>> items);
  int workers_ = 1;  // host threads sharing rollouts and NVRTC
  void launch_worker();
  void close_step();
  void log_eval(const Work& w, const ispc_time_result& r, int rc, const std::string& status, double t_now,
                bool improved);
  void log_dead(int tid, int64_t rollout_no, const char* reason);  // from the rollout threads (stdio locks)
  void start();
  double now() const;
};

}  // namespace ispc_host
