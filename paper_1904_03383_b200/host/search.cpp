#include "search.hpp"

#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <limits>
#include <sstream>

#include "adapter.hpp"
#include "ispace/loop_nest.hpp"

namespace ispc_host {

using namespace ispace;

// ---- incumbent -------------------------------------------------------------

void Incumbent::open(const char* shm_name) {
  if (shm_name && *shm_name) {
    int fd = shm_open(shm_name, O_CREAT | O_RDWR, 0600);
    if (fd >= 0) {
      map_bytes = 4096;
      if (ftruncate(fd, off_t(map_bytes)) == 0) {
        void* p = mmap(nullptr, map_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        if (p != MAP_FAILED) {
          map = p;
          name = shm_name;
          cell = static_cast<std::atomic<uint64_t>*>(p);  // zero-filled when created: no incumbent yet
        }
      }
      close(fd);
    }
  }
  if (!cell) {
    local = std::make_unique<std::atomic<uint64_t>>(0);
    cell = local.get();
  }
}

// Page-locks the shared page once the worker's device is selected (so the
// registration creates no context on another GPU).
void Incumbent::pin() {
  if (map && !pinned) pinned = ispc_host_register(map, map_bytes) == ISPC_OK;
}

// after a device reset the registration died with the old context
void Incumbent::repin() {
  pinned = false;
  pin();
}

Incumbent::~Incumbent() {
  if (map) {
    if (pinned) ispc_host_unregister(map);
    munmap(map, map_bytes);
    // every rank unlinks at exit: the name never outlives the job, so a later
    // job reusing it starts from an empty (zero) cell, not a stale incumbent
    if (!name.empty()) shm_unlink(name.c_str());
  }
}

double Incumbent::seconds() const {
  uint64_t v = cell->load(std::memory_order_acquire);
  return v == 0 ? std::numeric_limits<double>::infinity() : double(v) * 1e-9;
}

bool Incumbent::offer(uint64_t ns) {
  if (ns == 0) ns = 1;
  uint64_t cur = cell->load(std::memory_order_acquire);
  while (cur == 0 || ns < cur)
    if (cell->compare_exchange_weak(cur, ns, std::memory_order_acq_rel)) return true;
  return false;
}

// ---- search ------------------------------------------------------------------

namespace {

std::vector<std::string> split(const std::string& s) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, ','))
    if (!tok.empty()) out.push_back(tok);
  return out;
}

const char* kPaperOrder = "size,dim_kind,thread_level,mem_space,order,cache";

// Structural key of a candidate inside this process (domains, counters,
// fired lowerings): the rollouts' memo key. The reference's digest()
// (candidate.cpp:413) hashes the canonical names and values character by
// character - 68 us per call on the axpy space, more than a propagation -
// and stays the key of logs and serializations.
uint64_t fast_key(const Candidate& c) {
  auto mix = [](uint64_t h, uint64_t w) {
    h ^= w + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
    h *= 0xff51afd7ed558ccdull;
    return h ^ (h >> 32);
  };
  uint64_t h = mix(0x1904033830ull, c.fired);
  const size_t n = c.dom.size();
  size_t i = 0;
  for (; i + 1 < n; i += 2) h = mix(h, uint64_t(c.dom[i]) | (uint64_t(c.dom[i + 1]) << 32));
  if (i < n) h = mix(h, c.dom[i]);
  for (const Interval& v : c.cnt) h = mix(mix(h, uint64_t(v.lo)), uint64_t(v.hi));
  return h;
}
// building-block spaces: the engine and staging shape everything below them
const char* kTileOrder = "engine,staging,tile,xreduce,cache";

}  // namespace

double Search::now() const {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

Search::Search(const ispc_space* space, const ispc_search_config& cfg) : space_(space), cfg_(cfg) {
  order_text_ = cfg.decision_order ? cfg.decision_order : space->tiles ? kTileOrder : kPaperOrder;
  shm_text_ = cfg.incumbent_shm ? cfg.incumbent_shm : "";
  log_text_ = cfg.log_path ? cfg.log_path : "";
  cfg_.decision_order = order_text_.c_str();
  if (cfg_.shard_count <= 0) cfg_.shard_count = 1;
  if (cfg_.batch <= 0) cfg_.batch = 8;
  if (cfg_.budget_factor <= 0) cfg_.budget_factor = 3.0;
  if (cfg_.max_budget_ns <= 0) cfg_.max_budget_ns = 50e6;
  if (cfg_.reps <= 0) cfg_.reps = 3;
  if (cfg_.max_unrolled <= 0) cfg_.max_unrolled = B200Machine::kDefaultMaxUnrolled;
  unsigned hw = std::max(2u, std::thread::hardware_concurrency());
  // one process per GPU: the ranks of this node share its cores
  if (const char* lws = std::getenv("LOCAL_WORLD_SIZE")) {
    const int ranks = std::atoi(lws);
    if (ranks > 1) hw = std::max(2u, hw / unsigned(ranks));
  }
  // one launch thread; every other core alternates rollouts and NVRTC by
  // need (worker()); rollout_threads + compile_threads, when given, set the total
  workers_ = cfg_.rollout_threads > 0 || cfg_.compile_threads > 0
                 ? std::max(1, std::max(0, cfg_.rollout_threads) + std::max(0, cfg_.compile_threads))
                 : int(std::max(1u, hw));  // the launch thread mostly waits on the device
  machine_.l2_flushed = cfg_.flush_l2 != 0;
  machine_.max_unrolled = cfg_.max_unrolled;
  if (!space_->tiles) model_ = std::make_unique<BoundModel>(space_->kernel, *space_->ctx, machine_);
  order_ = DecisionOrder::from_names(*space_->ctx, split(order_text_));
  inc_.open(shm_text_.empty() ? nullptr : shm_text_.c_str());
  trace_ = std::getenv("ISPC_TRACE") != nullptr;
  if (const char* e = std::getenv("ISPC_INJECT_FAULT_AT")) inject_fault_at_ = std::atoll(e);
  if (const char* ld = std::getenv("ISPC_LOG_DEADENDS")) log_dead_ = std::atoi(ld) != 0;
  if (const char* g = std::getenv("ISPC_GREEDY")) {
    const std::string v(g);
    greedy_mode_ = v == "first" ? 0 : v == "off" ? 2 : 1;
  }
  if (const char* gp = std::getenv("ISPC_GREEDY_P")) greedy_p_ = std::clamp(std::atof(gp), 0.0, 1.0);
  if (const char* lp = std::getenv("ISPC_LEAFB_P")) leafb_p_ = std::clamp(std::atof(lp), 0.0, 1.0);
  if (const char* sh = std::getenv("ISPC_SHARP")) sharp_ = std::max(0.0, std::atof(sh));
  if (const char* lz = std::getenv("ISPC_LAZY")) lazy_greedy_ = std::atoi(lz) != 0;
  // default: on for the reference's loop-nest spaces (where a leaf's bound
  // separates fused from unfused schedules), off for the building-block
  // spaces (whose leaves mostly share one bound)
  aspire_ = space_->tiles ? 0.0 : 1.5;
  if (const char* as = std::getenv("ISPC_ASPIRE")) aspire_ = std::max(0.0, std::atof(as));
  // elite-guided rollouts (local search around the best measured leaves): on
  // for the building-block spaces, whose leaves share one bound, so the tree
  // statistics alone choose among ~10^5 of them (sgemm 1024^3: 53.3 us with
  // q = 0.5 against 56.5 us without, same seed and budget; batched unchanged;
  // profiles/r2h_elite.log); off for the loop-nest spaces (measured worse,
  // section 5 of DESIGN.md)
  // (q 0.5-0.9 with 1.5-3 expected deviations: profiles/r2m_sweep_*.log; the
  // spread between settings is within the run-to-run spread of one setting)
  elite_q_ = space_->tiles ? 0.5 : 0.0;
  if (const char* q = std::getenv("ISPC_ELITE_Q")) elite_q_ = std::clamp(std::atof(q), 0.0, 1.0);
  if (const char* mu = std::getenv("ISPC_ELITE_MUT")) elite_mut_ = std::max(0.0, std::atof(mu));
  if (const char* r = std::getenv("ISPC_ROLLOUT")) {
    const std::string v(r);
    rollout_mode_ = v == "deep" ? 1 : v == "ancestor" ? 2 : 0;
  }
  tree_depth_ = cfg_.tree_depth < 0 ? 0 : cfg_.tree_depth == 0 ? 12 : cfg_.tree_depth;
  refine_factor_ = cfg_.refine_factor > 0 ? cfg_.refine_factor : 1.25;
  uniform_ = cfg_.walk == ISPC_WALK_UNIFORM;
  if (uniform_) {  // the reference baseline's walk: no bound, tree or band
    cfg_.pruning = 0;
    tree_depth_ = 0;
    aspire_ = 0;
  }
  if (!log_text_.empty()) log_ = std::fopen(log_text_.c_str(), "w");
  expand_frontier();

  st_.best_ns = std::numeric_limits<double>::infinity();
  t0_ = now();
  if (cfg_.device < 0) return;  // dry run: rollouts + emission + NVRTC, no device
  int rc = ispc_dev_open(cfg_.device, &dev_);
  if (rc) throw std::runtime_error(std::string("ispc_dev_open: ") + ispc_last_error(nullptr));
  inc_.pin();
  ispc_problem p{};
  if (ispc_space_problem(space_, &p) != 0) throw std::runtime_error("no problem for this space");
  if ((rc = ispc_bind_problem(dev_, &p))) throw std::runtime_error(std::string("bind: ") + ispc_last_error(dev_));
  st_.best_ns = std::numeric_limits<double>::infinity();
  t0_ = now();
}

Search::~Search() {
  stop_ = true;
  cv_work_.notify_all();
  cv_batch_.notify_all();
  cv_done_.notify_all();
  for (auto& t : threads_) t.join();
  for (auto& b : batch_q_) {
    if (dev_ && b->handle) ispc_module_unload(dev_, b->handle);
    ispc_module_free(b->module);
  }
  if (dev_)
    for (int h : retired_) ispc_module_unload(dev_, h);
  if (dev_) ispc_dev_close(dev_);
  if (log_) std::fclose(log_);
}

// Deterministic breadth-first expansion of the first decisions; shard i keeps
// frontier nodes i, i + S, ... Every rank computes the same frontier.
void Search::expand_frontier() {
  const SpaceContext& ctx = *space_->ctx;
  std::vector<Candidate> frontier{space_->root};
  const size_t want = size_t(16) * size_t(cfg_.shard_count);
  for (int depth = 0; depth < 64 && frontier.size() < want; ++depth) {
    std::vector<Candidate> next;
    bool grew = false;
    for (const Candidate& c : frontier) {
      std::uint32_t inst = order_.pick(ctx, c);
      if (inst == kNoInstance) {
        next.push_back(c);
        continue;
      }
      Mask m = c.dom[inst];
      for (int v = 0; v < kMaxDomainBits; ++v) {
        if (!mask_has(m, v)) continue;
        Candidate child;
        if (apply_decision(ctx, c, inst, v, child) != PropStatus::Ok) continue;
        // unrunnable subtrees (infinite bound, e.g. a ring beyond 227 KiB)
        // never enter the frontier
        if (cfg_.pruning && !std::isfinite(bound_total(child))) continue;
        next.push_back(std::move(child));
      }
      grew = true;
    }
    if (!grew || next.empty()) break;
    frontier = std::move(next);
  }
  subtrees_ = std::move(frontier);
  for (size_t i = size_t(cfg_.shard_index); i < subtrees_.size(); i += size_t(cfg_.shard_count)) mine_.push_back(i);
  if (mine_.empty()) {  // tiny spaces: every shard searches all
    for (size_t i = 0; i < subtrees_.size(); ++i) mine_.push_back(i);
  }
  st_.frontier = int64_t(mine_.size());
  st_.frontier_total = int64_t(subtrees_.size());
}

double Search::bound_total(const Candidate& c) const {
  if (space_->tiles) return tile_bound(*space_->tiles, *space_->ctx, c).total;
  return model_->bound(c).total;
}

// TAG selection (threshold ascent): with s_i the number of child i's
// samples among the kTop best times seen by the shard, n_i its visits and
// alpha = ln(2 N kTop / delta), pick argmax (s_i + alpha + sqrt(2 s_i alpha +
// alpha^2)) / n_i; unvisited children first (drawn by bound, p ~ 1/b).
// Children whose bound reached the incumbent are skipped.
int Search::select_child(MctsNode& n, double T, std::mt19937_64& rng) {
  const double thr = top_.size() >= kTop ? top_.back() : std::numeric_limits<double>::infinity();
  const double alpha = std::log(2.0 * double(std::max<int64_t>(n.total, 1)) * double(kTop) / 0.01);
  std::vector<int> fresh;
  std::vector<double> fresh_w;
  int best = -1;
  double best_h = -1;
  for (size_t i = 0; i < n.kid_cand.size(); ++i) {
    if (!(n.kid_bound[i] < T)) continue;
    if (n.kids[i] && n.kids[i]->dead) continue;
    if (n.visits[i] == 0) {
      fresh.push_back(int(i));
      fresh_w.push_back(1.0 / std::max(n.kid_bound[i], 1e-12));
      continue;
    }
    double si = 0;
    for (double t : n.times[i]) si += (t <= thr) ? 1 : 0;
    double h = (si + alpha + std::sqrt(2 * si * alpha + alpha * alpha)) / double(n.visits[i]);
    if (h > best_h) best_h = h, best = int(i);
  }
  if (fresh.empty() && leafb_p_ > 0 && double(rng() % 4096) < leafb_p_ * 4096.0) {
    // the child whose subtree produced the lowest-bound leaf (ties at random)
    double lb = std::numeric_limits<double>::infinity();
    std::vector<int> at;
    for (size_t i = 0; i < n.kid_cand.size(); ++i) {
      if (!(n.kid_bound[i] < T) || (n.kids[i] && n.kids[i]->dead) || !std::isfinite(n.leaf_min[i])) continue;
      if (n.leaf_min[i] < lb * (1 - 1e-9)) lb = n.leaf_min[i], at.clear();
      if (n.leaf_min[i] <= lb * (1 + 1e-9)) at.push_back(int(i));
    }
    if (!at.empty()) return at[size_t(rng() % at.size())];
  }
  if (!fresh.empty()) {  // the lowest bound first half of the time, else p ~ 1/b
    if (rng() & 1) return fresh[size_t(std::max_element(fresh_w.begin(), fresh_w.end()) - fresh_w.begin())];
    std::discrete_distribution<size_t> pick(fresh_w.begin(), fresh_w.end());
    return fresh[pick(rng)];
  }
  return best;
}

void Search::backprop(const std::vector<std::pair<MctsNode*, int>>& path, double ns) {
  std::lock_guard<std::mutex> lk(tree_mu_);
  if (std::isfinite(ns)) {
    top_.insert(std::upper_bound(top_.begin(), top_.end(), ns), ns);
    if (top_.size() > kTop) top_.pop_back();
  }
  for (auto& [node, i] : path) {
    if (std::isfinite(ns)) node->times[size_t(i)].push_back(ns);
  }
}

bool Search::rollout(std::mt19937_64& rng, Candidate& leaf, double& leaf_bound,
                     std::vector<std::pair<MctsNode*, int>>& path, size_t& root_out) {
  const SpaceContext& ctx = *space_->ctx;
  const uint64_t cur_i = subtree_cursor_++;
  size_t root_i = stealing_ ? size_t(cur_i % subtrees_.size()) : mine_[size_t(cur_i % mine_.size())];
  const bool prune = cfg_.pruning != 0;
  path.clear();
  Candidate cur;
  // ---- elite-guided: follow a measured leaf's decisions, deviate at a few ----
  Candidate elite;
  bool guided = false;
  double p_mut = 0;
  if (elite_q_ > 0 && double(rng() % 4096) < elite_q_ * 4096.0) {
    std::lock_guard<std::mutex> lk(elite_mu_);
    if (!elites_.empty()) {
      // rank-biased pick: the incumbent half of the time, else any elite
      const size_t e = (rng() & 1) ? 0 : size_t(rng() % elites_.size());
      elite = elites_[e].leaf;
      root_i = elites_[e].root;
      guided = true;
      const double depth = double(std::max<int64_t>(decisions_per_leaf_.load(), 1));
      p_mut = std::min(1.0, elite_mut_ / depth);
    }
  }
  root_out = root_i;
  if (guided) return descend(rng, subtrees_[root_i], &elite, p_mut, leaf, leaf_bound, nullptr);
  // ---- in-tree descent (TAG) over the first tree_depth_ decisions ----
  MctsNode* node = nullptr;
  if (tree_depth_ > 0) {
    std::lock_guard<std::mutex> lk(tree_mu_);
    if (tree_roots_.size() != subtrees_.size()) {
      tree_roots_.clear();
      for (const Candidate& c : subtrees_) {
        tree_roots_.push_back(std::make_unique<MctsNode>());
        tree_roots_.back()->cand = c;
      }
    }
    node = tree_roots_[root_i].get();
  }
  int depth = 0;
  while (node && depth < tree_depth_) {
    const double T = prune ? prune_threshold() : std::numeric_limits<double>::infinity();
    if (!node->expanded) {
      // expand outside the lock (propagation dominates), install under it
      std::uint32_t inst = order_.pick(ctx, node->cand);
      std::vector<Candidate> kc;
      std::vector<double> kb;
      if (inst != kNoInstance) {
        Mask m = node->cand.dom[inst];
        for (int v = 0; v < kMaxDomainBits; ++v) {
          if (!mask_has(m, v)) continue;
          Candidate child;
          if (apply_decision(ctx, node->cand, inst, v, child) != PropStatus::Ok) continue;
          double b = bound_total(child);
          if (!std::isfinite(b)) {
            ++pruned_;
            continue;
          }
          kc.push_back(std::move(child));
          kb.push_back(b);
        }
      }
      std::lock_guard<std::mutex> lk(tree_mu_);
      if (!node->expanded) {
        if (inst == kNoInstance) {  // a leaf inside the tree
          node->expanded = true;
        } else {
          node->kid_cand = std::move(kc);
          node->kid_bound = std::move(kb);
          node->kids.resize(node->kid_cand.size());
          node->visits.assign(node->kid_cand.size(), 0);
          node->times.assign(node->kid_cand.size(), {});
          node->leaf_min.assign(node->kid_cand.size(), std::numeric_limits<double>::infinity());
          node->expanded = true;
          if (node->kid_cand.empty()) node->dead = true;
        }
      }
    }
    std::lock_guard<std::mutex> lk(tree_mu_);
    if (node->kid_cand.empty()) {
      if (node->dead) return false;
      break;  // fully specified inside the tree
    }
    int i = select_child(*node, T, rng);
    if (i < 0) {  // every child dead, or pruned by the incumbent (which only falls): for good
      node->dead = true;
      ++pruned_;
      return false;
    }
    ++node->visits[size_t(i)];
    ++node->total;
    path.emplace_back(node, i);
    if (!node->kids[size_t(i)]) {
      node->kids[size_t(i)] = std::make_unique<MctsNode>();
      node->kids[size_t(i)]->cand = node->kid_cand[size_t(i)];
    }
    node = node->kids[size_t(i)].get();
    ++depth;
  }
  if (node) {
    std::lock_guard<std::mutex> lk(tree_mu_);
    cur = node->cand;
  } else {
    cur = subtrees_[root_i];
  }
  const bool ok = descend(rng, std::move(cur), nullptr, 0.0, leaf, leaf_bound, node);
  if (ok && !path.empty()) {
    std::lock_guard<std::mutex> lk(tree_mu_);
    for (auto& [pn, i] : path) pn->leaf_min[size_t(i)] = std::min(pn->leaf_min[size_t(i)], leaf_bound);
  }
  return ok;
}

// ---- rollout below the tree: p ~ max(T - b, 0), with backtracking ----
  // A descent that dead-ends (every child infeasible or bound >= incumbent)
  // or reaches a leaf it already produced returns to the deepest frame with
  // an untried child instead of starting over from the root, so the prefix's
  // propagation is reused; siblings are re-checked against the incumbent
  // when they are taken. A subtree the walk exhausts within its expansion
  // budget is marked dead in the tree above it.
// With `guide`, each decision takes the guide leaf's value when that child
// is still feasible and unpruned, except with probability p_mut (and always
// when it is not), where it samples like an exploring rollout.
bool Search::descend(std::mt19937_64& rng, Candidate cur, const Candidate* guide, double p_mut, Candidate& leaf,
                     double& leaf_bound, MctsNode* node) {
  const SpaceContext& ctx = *space_->ctx;
  const bool prune = cfg_.pruning != 0;
  int64_t decisions = 0;
  struct Frame {
    std::vector<Candidate> kids;
    std::vector<double> w, b;
  };
  std::vector<Frame> stack;
  int budget = rollout_mode_ == 0 ? std::numeric_limits<int>::max() : kRolloutExpansions;
  bool cut = false, dead_end = false;
  double cur_b = -1;  // bound of `cur` when known (the child a lazy greedy draw took)
  for (;;) {
    std::uint32_t inst = order_.pick(ctx, cur);
    const double T = prune ? prune_threshold() : std::numeric_limits<double>::infinity();
    if (inst == kNoInstance) {
      const uint64_t d = fast_key(cur);
      bool fresh;
      {
        std::lock_guard<std::mutex> lk(seen_leaf_mu_);
        fresh = seen_leaf_.insert(d).second;
      }
      dead_.add(d);  // produced: no later rollout needs to reach it again
      if (fresh) {
        if (!guide) {  // running estimate of the decisions a rollout makes below its start
          const int64_t old = decisions_per_leaf_.load();
          decisions_per_leaf_.store(old == 0 ? decisions : (3 * old + decisions + 2) / 4);
        }
        leaf_bound = bound_total(cur);
        leaf = std::move(cur);
        return true;
      }
      dead_end = rollout_mode_ == 0;  // produced before: a restart treats it as a dead end
      if (decisions == 0 && node) {  // the tree node itself is that leaf: never select it again
        std::lock_guard<std::mutex> lk(tree_mu_);
        node->dead = true;
      }
    } else if (budget > 0) {
      --budget;
      Mask m = cur.dom[inst];
      ++decisions;
      // guided: the guide's value alone (one propagation) unless this
      // decision mutates or that child is infeasible / pruned
      const int want = guide ? decided_value(*guide, inst) : -1;
      if (want >= 0 && mask_has(m, want) && double(rng() % 4096) >= p_mut * 4096.0) {
        Candidate child;
        if (apply_decision(ctx, cur, inst, want, child) == PropStatus::Ok) {
          const double b = prune ? bound_total(child) : 0.0;
          if (!prune || (std::isfinite(b) && b < T)) {
            cur = std::move(child);
            continue;
          }
        }
      }
      // lazy greedy draw (restart mode): children in random order; the bound
      // is monotone, so a child whose bound equals the parent's is a minimum
      // and ends the scan early (most decisions leave the bound unchanged);
      // otherwise the lowest-bound child seen, ties kept at random
      if (rollout_mode_ == 0 && prune && greedy_mode_ != 2 && lazy_greedy_ &&
          double(rng() % 4096) < greedy_p_ * 4096.0) {
        int vals[kMaxDomainBits], nv = 0;
        for (int v = 0; v < kMaxDomainBits; ++v)
          if (mask_has(m, v)) vals[nv++] = v;
        for (int k = nv - 1; k > 0; --k) std::swap(vals[k], vals[size_t(rng() % uint64_t(k + 1))]);
        const double b_parent = cur_b >= 0 ? cur_b : bound_total(cur);
        Candidate best_child;
        double best_b = std::numeric_limits<double>::infinity();
        for (int k = 0; k < nv; ++k) {
          Candidate child;
          if (apply_decision(ctx, cur, inst, vals[k], child) != PropStatus::Ok) continue;
          const double b = bound_total(child);
          if (!std::isfinite(b) || b >= T || dead_.has(fast_key(child))) {
            ++pruned_;
            continue;
          }
          if (b < best_b) best_b = b, best_child = std::move(child);
          if (best_b <= b_parent * (1 + 1e-12)) break;
        }
        if (!std::isfinite(best_b)) {  // dead end: remember it, restart
          dead_.add(fast_key(cur));
          break;
        }
        cur = std::move(best_child);
        cur_b = best_b;
        continue;
      }
      Frame f;
      for (int v = 0; v < kMaxDomainBits; ++v) {
        if (!mask_has(m, v)) continue;
        Candidate child;
        if (apply_decision(ctx, cur, inst, v, child) != PropStatus::Ok) continue;
        double weight = 1.0, b = 0.0;
        if (prune) {
          b = bound_total(child);
          // unrunnable, cannot beat the incumbent, or spent by earlier rollouts
          if (!std::isfinite(b) || b >= T || dead_.has(fast_key(child))) {
            ++pruned_;
            continue;
          }
          // p ~ max(T - b, 0); before the first measurement
          // there is no T, and the bound itself ranks the children (p ~ 1/b)
          weight = std::isfinite(T) ? T - b : 1.0 / std::max(b, 1e-12);
        }
        f.kids.push_back(std::move(child));
        f.w.push_back(weight);
        f.b.push_back(b);
      }
      if (!f.kids.empty()) {
        stack.push_back(std::move(f));
      } else {
        if (prune) dead_.add(fast_key(cur));  // every child pruned or spent: so is this node
        dead_end = true;
      }
    } else {
      cut = true;
      break;
    }
    // a dead end resumes from a uniformly drawn ancestor frame (diversity
    // close to a restart, prefix propagation reused); a leaf produced before
    // resumes from the deepest frame (a live region: its siblings)
    if (rollout_mode_ == 0 && dead_end) break;  // restart: a fresh descent from the tree next time
    if (dead_end && rollout_mode_ == 2 && stack.size() > 1) stack.resize(1 + size_t(rng() % stack.size()));
    dead_end = false;
    // take an untried child of the deepest frame that still has one
    bool took = false;
    while (!stack.empty() && !took) {
      Frame& f = stack.back();
      if (prune) {  // drop siblings the incumbent has overtaken since the frame was built
        for (size_t k = f.kids.size(); k-- > 0;)
          if (f.b[k] >= T) {
            f.kids.erase(f.kids.begin() + long(k)), f.w.erase(f.w.begin() + long(k)), f.b.erase(f.b.begin() + long(k));
            ++pruned_;
          }
      }
      if (f.kids.empty()) {
        stack.pop_back();
        continue;
      }
      // half of the draws follow the bound greedily (the most promising child,
      // lowest b), the other half sample p ~ max(T - b, 0) / 1/b
      size_t choice;
      // (with lazy greedy draws the greedy share was drawn above; this is the sampled rest)
      const bool lazy_drawn = rollout_mode_ == 0 && lazy_greedy_ && greedy_mode_ != 2;
      if (prune && greedy_mode_ != 2 && !lazy_drawn && double(rng() % 4096) < greedy_p_ * 4096.0) {
        choice = size_t(std::max_element(f.w.begin(), f.w.end()) - f.w.begin());
        if (greedy_mode_ == 1) {  // uniformly among the children tied at the best weight
          const double top = f.w[choice];
          size_t ties = 0;
          for (double x : f.w) ties += x >= top;
          size_t r = size_t(rng() % ties);
          for (size_t k = 0; k < f.w.size(); ++k)
            if (f.w[k] >= top && r-- == 0) {
              choice = k;
              break;
            }
        }
      } else if (prune && sharp_ > 0) {
        const double bmin = std::max(*std::min_element(f.b.begin(), f.b.end()), 1e-12);
        std::vector<double> w2(f.w.size());
        for (size_t k = 0; k < w2.size(); ++k) w2[k] = f.w[k] * std::exp(-sharp_ * (f.b[k] - bmin) / bmin);
        std::discrete_distribution<size_t> pick(w2.begin(), w2.end());
        choice = pick(rng);
      } else {
        std::discrete_distribution<size_t> pick(f.w.begin(), f.w.end());
        choice = pick(rng);
      }
      cur = std::move(f.kids[choice]);
      cur_b = prune ? f.b[choice] : -1;
      f.kids.erase(f.kids.begin() + long(choice));
      f.w.erase(f.w.begin() + long(choice));
      f.b.erase(f.b.begin() + long(choice));
      took = true;
    }
    if (!took) break;  // the whole subtree below the tree node is spent
  }
  if (rollout_mode_ != 0 && !cut && node && tree_depth_ > 0) {  // exhausted exactly: skip it from now on
    std::lock_guard<std::mutex> lk(tree_mu_);
    node->dead = true;
  }
  return false;
}

// Pruning threshold of the rollouts: the incumbent (admissible B&B), and
// with the aspiration filter also kappa x the lowest leaf bound produced so
// far, applied to partial candidates too (their bounds never exceed their
// leaves'), so descents leave the band as early as the bound shows it. Both
// terms only fall, so what they prune stays pruned.
double Search::prune_threshold() const {
  double T = inc_.seconds();
  if (aspire_ > 0) T = std::min(T, aspire_ * min_leaf_bound_.load());
  return T;
}

void Search::note_elite(double ns, size_t root, const Candidate& leaf) {
  std::lock_guard<std::mutex> lk(elite_mu_);
  if (elites_.size() >= kElite && ns >= elites_.back().ns) return;
  auto at = std::upper_bound(elites_.begin(), elites_.end(), ns, [](double x, const Elite& e) { return x < e.ns; });
  elites_.insert(at, Elite{ns, root, leaf});
  if (elites_.size() > kElite) elites_.pop_back();
}

void Search::note_fruitless() {
  if (++fruitless_ < kExhaust) return;
  if (cfg_.shard_count > 1 && mine_.size() < subtrees_.size() && !stealing_.exchange(true)) {
    fruitless_ = 0;  // own shard spent: steal from the whole frontier before giving up
    stealing_since_ = rollouts_.load();
    if (trace_) std::fprintf(stderr, "[ispc] shard %d spent, stealing from %zu subtrees\n", cfg_.shard_index,
                             subtrees_.size());
    return;
  }
  if (!exhausted_.exchange(true)) {
    std::lock_guard<std::mutex> lk(mu_);
    cv_done_.notify_all();
  }
}

// One rollout: descend to a leaf (or a dead end), emit its kernel and queue it.
void Search::rollout_one(int tid, std::mt19937_64& rng, int64_t& k_roll, const ispc_emit_opts& eo) {
  double t = now();
  auto w = std::make_unique<Work>();
  w->tid = tid;
  w->rollout_no = k_roll++;
  bool ok;
  const char* dead_reason = "deadend";
  if (uniform_) {
    ok = uniform_walk(rng, w->leaf);
    if (ok) w->bound_s = bound_total(w->leaf);  // not used to prune: counts bound violations
  } else {
    ok = rollout(rng, w->leaf, w->bound_s, w->path, w->root);
  }
  if (ok && aspire_ > 0) {
    double lo = min_leaf_bound_.load();
    while (w->bound_s < lo && !min_leaf_bound_.compare_exchange_weak(lo, w->bound_s)) {
    }
    if (w->bound_s > aspire_ * std::min(lo, w->bound_s)) {  // outside the aspiration band
      ok = false;
      dead_reason = "aspiration";
    }
  }
  ++rollouts_;
  if (!ok) {
    ++dead_rollouts_;
    if (log_ && log_dead_) log_dead(tid, w->rollout_no, dead_reason);
    t_rollout_.fetch_add(now() - t);
    note_fruitless();
    if (exhausted_) std::this_thread::sleep_for(std::chrono::milliseconds(1));
    return;
  }
  int rc = ISPC_OK;
  size_t len = 0;
  if (space_->tiles) {
    // building-block leaf: decided tile configuration -> sm_100a kernel
    ispc_tile_config tc{};
    try {
      tc = tile_config(*space_->tiles, *space_->ctx, w->leaf);
    } catch (const std::exception& e) {
      if (trace_) std::fprintf(stderr, "[ispc] leaf without a tile config: %s\n", e.what());
      ++illegal_;
      if (log_ && log_dead_) log_dead(tid, w->rollout_no, "illegal");
      t_rollout_.fetch_add(now() - t);
      note_fruitless();
      return;
    }
    w->bit_exact = tile_bit_exact(tc);
    w->rtol = tc.kind == ISPC_TILE_SGEMM_TC && tc.engine == ISPC_ENGINE_TF32X3 ? 1e-5 : space_->tiles->rtol();
    rc = ispc_emit_tiles(&tc, nullptr, nullptr, 0, &len, &w->launch);
    if (rc == ISPC_OK) {
      w->src.assign(len + 1, '\0');
      rc = ispc_emit_tiles(&tc, nullptr, w->src.data(), w->src.size(), &len, &w->launch);
      w->src.resize(len);
    }
  } else {
    try {
      LoopNest l = reconstruct(space_->kernel, *space_->ctx, w->leaf);
      w->nest = flatten(space_->kernel, l);
    } catch (const std::exception&) {
      ++illegal_;
      if (log_ && log_dead_) log_dead(tid, w->rollout_no, "illegal");
      t_rollout_.fetch_add(now() - t);
      note_fruitless();
      return;
    }
    rc = ispc_emit_cuda(&w->nest->nest, &eo, nullptr, nullptr, 0, &len, &w->launch);
    if (rc == ISPC_OK) {
      w->src.assign(len + 1, '\0');
      rc = ispc_emit_cuda(&w->nest->nest, &eo, nullptr, w->src.data(), w->src.size(), &len, &w->launch);
      w->src.resize(len);
    }
  }
  t_rollout_.fetch_add(now() - t);
  if (rc != ISPC_OK) {
    if (trace_) std::fprintf(stderr, "[ispc] illegal leaf: %s\n", ispc_last_error(nullptr));
    ++illegal_;
    if (log_ && log_dead_) log_dead(tid, w->rollout_no, "illegal");
    note_fruitless();
    return;
  }
  w->digest = digest(*space_->ctx, w->leaf);
  std::unique_lock<std::mutex> lk(mu_);
  if (!seen_hash_.insert(w->launch.source_hash).second) {
    ++duplicates_;
    lk.unlock();
    if (log_ && log_dead_) log_dead(tid, w->rollout_no, "duplicate");
    note_fruitless();
    if (exhausted_) std::this_thread::sleep_for(std::chrono::milliseconds(1));
    return;
  }
  fruitless_ = 0;
  exhausted_ = false;
  work_q_.push_back(std::move(w));
  cv_batch_.notify_all();
}

// Compiles a batch of emitted kernels into one NVRTC program (isolating a
// failing kernel) and loads the cubin on the device.
void Search::compile_items(std::vector<std::unique_ptr<Work>> items) {
  double t = now();
  std::vector<const char*> srcs;
  for (auto& w : items) srcs.push_back(w->src.c_str());
  ispc_module* m = nullptr;
  // device -2: a dry run of the host pipeline alone (no NVRTC, no device):
  // the tests of sharding and stealing
  int rc = cfg_.device == -2 ? ISPC_OK : ispc_compile(srcs.data(), int(srcs.size()), "sm_100a", &m);
  if (const char* dir = std::getenv("ISPC_DUMP_DIR")) {  // the compiled programs, for compile-cost studies
    static std::atomic<int> seq{0};
    if (FILE* f = std::fopen((std::string(dir) + "/prog" + std::to_string(seq++) + ".cu").c_str(), "w")) {
      for (const char* x : srcs) std::fputs(x, f);
      std::fclose(f);
    }
  }
  if (trace_) {
    size_t bytes = 0;
    for (auto& w : items) bytes += w->src.size();
    std::fprintf(stderr, "[ispc] compile %zu kernels (%zu B of source) in %.3f s rc=%d first=%s\n", items.size(), bytes,
                 now() - t, rc, items.front()->launch.name);
    std::fflush(stderr);
  }
  std::vector<std::unique_ptr<CompiledBatch>> out;
  if (rc == ISPC_OK) {
    auto b = std::make_unique<CompiledBatch>();
    b->items = std::move(items);
    b->module = m;
    out.push_back(std::move(b));
  } else {
    // isolate the failing kernel(s)
    for (auto& w : items) {
      const char* one[] = {w->src.c_str()};
      ispc_module* m1 = nullptr;
      if (ispc_compile(one, 1, "sm_100a", &m1) != ISPC_OK) {
        ++compile_errors_;
        continue;
      }
      auto b = std::make_unique<CompiledBatch>();
      b->items.push_back(std::move(w));
      b->module = m1;
      out.push_back(std::move(b));
    }
  }
  // load the cubins here, off the launch thread (module load and the eager
  // upload of its kernels overlap the device's work on earlier batches)
  {
    std::shared_lock<std::shared_mutex> dl(dev_mu_);
    if (dev_)
      for (auto& b : out) {
        b->load_rc = ispc_module_load(dev_, b->module, &b->handle);
        if (b->load_rc != ISPC_OK) b->load_err = ispc_last_error(dev_);
      }
  }
  t_compile_.fetch_add(now() - t);
  std::lock_guard<std::mutex> lk(mu_);
  for (auto& b : out) batch_q_.push_back(std::move(b));
  --compiling_;
  cv_done_.notify_all();
}

// Every host thread but the launch thread alternates between the two CPU
// stages by need: it compiles when a whole batch of emitted kernels waits (or
// any kernel waits while the device has nothing queued), otherwise it runs a
// rollout while the emitted-kernel queue has room. The split adapts to the
// walk: pruned rollouts cost ~2-3x the CPU of NVRTC per kernel, uniform
// leaves the reverse (r2 measurements), so fixed pools left cores idle.
void Search::worker(int tid) {
  // uniform walk: thread tid's descents are those of the reference baseline's
  // thread tid (oracle/ref_cpu_bench.cpp seeds 0x190403383 + 7919 tid)
  std::mt19937_64 rng(cfg_.seed + 7919ull * uint64_t(tid) + 104729ull * uint64_t(cfg_.shard_index));
  int64_t k_roll = 0;
  ispc_emit_opts eo{};
  eo.watchdog = uint32_t(cfg_.watchdog);
  eo.max_unrolled = uint32_t(cfg_.max_unrolled);
  eo.max_reg_elems = B200Machine::kMaxRegElems;  // register arrays beyond this spill on a 255-register thread anyway
  const size_t batch = size_t(cfg_.batch);
  const size_t cap_w = batch * size_t(workers_) * 2;  // emitted kernels waiting for NVRTC
  const size_t cap_b = size_t(workers_) / 2 + 4;      // compiled batches waiting for the device
  while (!stop_) {
    std::vector<std::unique_ptr<Work>> items;
    {
      std::unique_lock<std::mutex> lk(mu_);
      for (;;) {
        if (stop_) return;
        const bool room_b = batch_q_.size() < cap_b;
        const bool starving = batch_q_.empty() && compiling_.load() == 0;
        if (!work_q_.empty() && room_b && (work_q_.size() >= batch || starving || work_q_.size() >= cap_w)) {
          // a backlog compiles in bigger programs: NVRTC's fixed cost per
          // program (~25 ms) is then shared by up to 2 x batch kernels
          const size_t take = work_q_.size() >= 2 * batch ? 2 * batch : batch;
          while (!work_q_.empty() && items.size() < take) {
            items.push_back(std::move(work_q_.front()));
            work_q_.pop_front();
          }
          ++compiling_;
          break;
        }
        if (work_q_.size() < cap_w) break;  // room: run a rollout
        cv_work_.wait_for(lk, std::chrono::milliseconds(5));
      }
    }
    if (!items.empty()) {
      compile_items(std::move(items));
      cv_work_.notify_all();
    } else {
      rollout_one(tid, rng, k_roll, eo);
    }
  }
}


bool Search::uniform_walk(std::mt19937_64& rng, Candidate& leaf) {
  return random_walk(*space_->ctx, space_->root, rng, leaf, nullptr).ok;
}

void Search::log_dead(int tid, int64_t rollout_no, const char* reason) {
  std::fprintf(log_, "{\"status\": \"%s\", \"seed\": %llu, \"tid\": %d, \"rollout\": %lld, \"t\": %.4f}\n",
               reason, (unsigned long long)cfg_.seed, tid, (long long)rollout_no, now() - t0_);
}


void Search::launch_worker() {
  bool& step_open = step_open_;
  while (!stop_) {
    std::unique_ptr<CompiledBatch> b;
    {
      std::unique_lock<std::mutex> lk(mu_);
      // the device only works inside step(): outside it the rollouts and
      // compiles keep filling their bounded queues while the GPU idles
      while (!(stop_ || (!batch_q_.empty() && st_.evaluations < target_.load())))
        cv_done_.wait_for(lk, std::chrono::milliseconds(20));
      if (stop_) return;
      launching_ = true;
      b = std::move(batch_q_.front());
      batch_q_.pop_front();
      cv_batch_.notify_all();
      if (dev_ && !step_open) {
        ispc_dev_mark(dev_, 0);
        step_open = true;
      }
    }
    const double t_busy = now();
    const int64_t n = int64_t(b->items.size());
    if (!dev_ || b->load_rc != ISPC_OK) {
      // dry run: the compiled kernels count as evaluated; a module that did
      // not load: every kernel of it is a launch error (a sticky fault ends
      // the search, as in ispc_launch_batch)
      bool sticky_load = false;
      {
      std::lock_guard<std::mutex> lk(mu_);
      if (!dev_ && log_) {
        for (int64_t i = 0; i < n; ++i) {
          const Work& w = *b->items[size_t(i)];
          std::fprintf(log_, "{\"i\": %lld, \"status\": \"dry\", \"digest\": \"%016llx\", \"subtree\": %zu, \"shard\": %d}\n",
                       (long long)(st_.evaluations + i + 1), (unsigned long long)w.digest, w.root, cfg_.shard_index);
        }
        std::fflush(log_);
      }
      st_.evaluations += n;
      if (dev_) {
        st_.launch_errors += n;
        if (b->load_rc == ISPC_E_STICKY) {
          err_ = b->load_err;
          sticky_load = true;
        }
      }
      ispc_module_free(b->module);
      }
      if (sticky_load) {  // the context is dead for this process (see stop below)
        std::lock_guard<std::mutex> lk(mu_);
        stop_ = true;
      }
      {
        std::lock_guard<std::mutex> lk(mu_);
        launching_ = false;
      }
      cv_done_.notify_all();
      continue;
    }
    const double T = inc_.seconds();
    std::vector<ispc_batch_item> items(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      Work& w = *b->items[size_t(i)];
      if (trace_) {
        std::fprintf(stderr, "[ispc] launch %s grid=%llu block=%u,%u,%u smem=%u wd=%u\n", w.launch.name,
                     (unsigned long long)w.launch.grid_x, w.launch.block[0], w.launch.block[1], w.launch.block[2],
                     w.launch.static_smem, w.launch.watchdog);
        if (const char* dir = std::getenv("ISPC_TRACE_DIR")) {  // the kernel source, for post-mortems
          if (FILE* f = std::fopen((std::string(dir) + "/" + w.launch.name + ".cu").c_str(), "w")) {
            std::fputs(w.src.c_str(), f);
            std::fclose(f);
          }
        }
      }
      ispc_time_opts& to = items[size_t(i)].opts;
      items[size_t(i)].launch = &w.launch;
      to.warmup = uint32_t(std::max(0, cfg_.warmup));
      to.reps = uint32_t(cfg_.reps);
      to.flush_l2 = uint32_t(cfg_.flush_l2);
      to.rotate = cfg_.rotate > 1 ? uint32_t(cfg_.rotate) : 0u;
      to.check = 1;
      to.bit_exact = w.bit_exact ? 1 : 0;
      to.rtol = w.rtol;
      // before the first measurement: 50x the leaf's own bound (>= 2 ms) for
      // the first 64 evaluations, then the cap (a schedule 50x off its bound
      // is not worth waiting 50 ms for while any incumbent is missing); a
      // caller that raised the cap above the default (the reference's matmul
      // space, whose schedules run for seconds ~100x above their bounds) gets
      // the cap from the start
      const bool long_cap = cfg_.max_budget_ns > 50e6;
      to.budget_ns = std::isfinite(T) ? std::min(cfg_.max_budget_ns, std::max(T * 1e9 * cfg_.budget_factor,
                                                                              T * 1e9 + 20e3))
                     : st_.evaluations < 64 && !long_cap
                         ? std::min(cfg_.max_budget_ns, std::max(2e6, 50.0 * w.bound_s * 1e9))
                         : cfg_.max_budget_ns;
    }
    // screened kernels slower than factor x incumbent cannot become the
    // incumbent: their single checked launch is their time
    const double refine_below = std::isfinite(T) ? T * 1e9 * refine_factor_ : std::numeric_limits<double>::infinity();
    std::vector<ispc_time_result> res(static_cast<size_t>(n));
    const double t_dev0 = now();
    ++batches_launched_;
    const int brc = batches_launched_ == inject_fault_at_
                        ? ispc_dev_inject_fault(dev_)  // test hook: the batch dies with the context
                        : ispc_launch_batch(dev_, b->handle, int(n), items.data(), refine_below, res.data());
    const double t_dev = now() - t_dev0;
    const std::string berr = brc ? ispc_last_error(dev_) : std::string();
    // cuModuleUnload measured 1.4-231 ms per call on the B200 (it waits on
    // the context): modules stay loaded (a few hundred KiB of device memory
    // each) and are unloaded in bulk, between steps or at close
    retired_.push_back(b->handle);
    ispc_module_free(b->module);
    b->module = nullptr;
    if (retired_.size() >= kMaxRetired) {
      for (size_t k = 0; k < kMaxRetired / 2; ++k) ispc_module_unload(dev_, retired_[k]);
      retired_.erase(retired_.begin(), retired_.begin() + long(kMaxRetired / 2));
    }
    bool sticky_batch = false;
    {
      std::lock_guard<std::mutex> lk(mu_);
      for (int64_t i = 0; i < n; ++i) {
        Work& w = *b->items[size_t(i)];
        const ispc_time_result& r = res[size_t(i)];
        // a device-level failure of the batch fails every item of it
        const int rc = brc ? brc : (r.status == ISPC_OK || r.status == ISPC_E_TIMEOUT || r.status == ISPC_E_MISMATCH)
                                       ? ISPC_OK
                                       : r.status;
        const double t_now = now() - t0_;
        std::string status;
        bool improved = false;
        if (rc == ISPC_E_ILLEGAL) {  // the compiled kernel cannot run its block (registers): never launched
          ++illegal_;
          continue;
        }
        ++st_.evaluations;
        if (rc != ISPC_OK) {
          ++st_.launch_errors;
          status = rc == ISPC_E_STICKY ? "sticky" : "launch_error";
          if (rc == ISPC_E_STICKY) {
            err_ = berr;
            sticky_batch = true;
          }
        } else {
          step_busy_ms_ += r.first_ns * 1e-6;
          if (r.median_ns != r.first_ns || r.min_ns != r.first_ns) ++refined_;
          if (r.status == ISPC_E_MISMATCH) {
            ++st_.mismatches;
            status = "mismatch";
          } else if (r.status == ISPC_E_TIMEOUT) {
            ++st_.timeouts;
            status = "timeout";
          } else {
            ++st_.ok;
            status = "ok";
            if (w.bound_s * 1e9 > r.median_ns * (1 + 1e-9)) ++st_.bound_violations;
            inc_.offer(uint64_t(std::llround(r.median_ns)));
            if (r.median_ns < st_.best_ns) {
              improved = true;
              st_.best_ns = r.median_ns;
              st_.best_bound_ns = w.bound_s * 1e9;
              st_.time_to_best_s = t_now;
              st_.best_hash = w.launch.source_hash;
              best_text_ = serialize_text(*space_->ctx, w.leaf);
              best_src_ = w.src;
              best_launch_ = w.launch;
            }
          }
        }
        if (rc == ISPC_OK && r.status == ISPC_OK && std::isfinite(r.median_ns)) note_elite(r.median_ns, w.root, w.leaf);
        if (!w.path.empty()) {
          const double ns = (rc == ISPC_OK && r.status == ISPC_OK) ? r.median_ns : std::numeric_limits<double>::infinity();
          backprop(w.path, ns);
        }
        if (log_) log_eval(w, r, rc, status, t_now, improved);
      }
      if (log_) std::fflush(log_);  // once per batch
      if (step_open && st_.evaluations >= target_.load() && !sticky_batch) close_step();
      t_launch_host_ += (now() - t_busy) - t_dev;
      st_.t_gpu_s += now() - t_busy;
      if (!sticky_batch) launching_ = false;
    }
    if (sticky_batch) {
      // a context-killing fault ends this shard's search: on the B200 boxes
      // the faulted process cannot create a new context (cudaDeviceReset +
      // cudaFree report cudaErrorDevicesUnavailable, tools/respawn_probe.py),
      // while a fresh process can - the caller's recovery is a new worker
      // process (bench.py's config searches already run as children)
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      step_open = false;
      launching_ = false;
    }
    cv_done_.notify_all();
    if (trace_) std::fflush(stderr);
  }
}

// One JSONL record per evaluated kernel (under mu_): where the rollout came
// from (rollout thread, its rollout number, shard subtree, the tree edges
// taken with the bound of each child on the path), what was measured, and
// the candidate text whenever it improved the best. -1 = no value.
void Search::log_eval(const Work& w, const ispc_time_result& r, int rc, const std::string& status, double t_now,
                      bool improved) {
  std::string path = "[", anc = "[";
  {
    std::lock_guard<std::mutex> lk(tree_mu_);
    for (size_t k = 0; k < w.path.size(); ++k) {
      const auto& [node, i] = w.path[k];
      path += (k ? ", " : "") + std::to_string(i);
      char b[48];
      std::snprintf(b, sizeof(b), "%s%.1f", k ? ", " : "", node->kid_bound[size_t(i)] * 1e9);
      anc += b;
    }
  }
  path += "]";
  anc += "]";
  // the candidate text rides along when it improved the best, and on every
  // mismatch / launch error (bench.py replays those on the CPU emulator)
  const bool failed = status == "mismatch" || status == "launch_error" || status == "sticky";
  const bool with_cand = improved || failed;
  std::string compact = improved ? best_text_ : failed ? serialize_text(*space_->ctx, w.leaf) : std::string();
  std::replace(compact.begin(), compact.end(), '\n', ' ');
  if (status == "launch_error" || status == "sticky") {  // the device's last error message rides along
    std::string e;
    for (const char* q = dev_ ? ispc_last_error(dev_) : nullptr; q && *q && e.size() < 300; ++q)
      e += (*q == '"' || *q == '\\') ? '\'' : (static_cast<unsigned char>(*q) < 0x20) ? ' ' : *q;
    compact += (compact.empty() ? "" : ", ") + std::string("\"error\": \"") + e + "\"";
  }
  const bool timed = rc == ISPC_OK;
  std::fprintf(log_,
               "{\"i\": %lld, \"t\": %.4f, \"status\": \"%s\", \"median_ns\": %.1f, \"first_ns\": %.1f, "
               "\"min_ns\": %.1f, \"bound_ns\": %.1f, \"incumbent_ns\": %.1f, \"hash\": \"%016llx\", "
               "\"digest\": \"%016llx\", \"grid\": %llu, \"block\": %u, \"seed\": %llu, \"tid\": %d, \"rollout\": %lld, \"subtree\": %zu, "
               "\"path\": %s, \"path_bounds_ns\": %s, \"best\": %s%s%s}\n",
               (long long)st_.evaluations, t_now, status.c_str(), timed ? r.median_ns : -1.0,
               timed ? r.first_ns : -1.0, timed ? r.min_ns : -1.0, w.bound_s * 1e9,
               std::isfinite(inc_.seconds()) ? inc_.seconds() * 1e9 : -1.0, (unsigned long long)w.launch.source_hash,
               (unsigned long long)w.digest, (unsigned long long)w.launch.grid_x,
               w.launch.block[0] * w.launch.block[1] * w.launch.block[2], (unsigned long long)cfg_.seed, w.tid, (long long)w.rollout_no, w.root,
               path.c_str(), anc.c_str(), improved ? "true" : "false", with_cand ? ", \"candidate\": " : "",
               compact.c_str());
}

// Records the device-timeline end of the open step (under mu_).
void Search::close_step() {
  ispc_dev_mark(dev_, 1);
  double ms = 0;
  ispc_dev_mark_elapsed(dev_, 0, 1, &ms);
  st_.device_step_ms = ms;
  st_.device_busy_ms = step_busy_ms_;
  step_busy_ms_ = 0;
  step_open_ = false;
}

int Search::region_io(const char* name, void* host, size_t bytes, bool upload) {
  std::unique_lock<std::mutex> lk(mu_);
  cv_done_.wait(lk, [&] { return stop_ || !launching_; });  // device idle between steps
  return upload ? ispc_write_region(dev_, name, host, bytes) : ispc_read_region(dev_, name, host, bytes);
}

void Search::start() {
  for (int i = 0; i < workers_; ++i) threads_.emplace_back([this, i] { worker(i); });
  threads_.emplace_back([this] { launch_worker(); });
  pipeline_started_ = true;
}

int Search::step(int64_t evaluations, double max_seconds) {
  {
    std::lock_guard<std::mutex> lk(mu_);
    target_ = st_.evaluations + evaluations;
  }
  // wake the launch thread: it sleeps on cv_done_ between steps, and with
  // full queues nothing else would notify it
  cv_done_.notify_all();
  if (!pipeline_started_) start();
  std::unique_lock<std::mutex> lk(mu_);
  auto drained = [&] {
    return exhausted_ && work_q_.empty() && batch_q_.empty() && compiling_.load() == 0 && !launching_;
  };
  const double t_end = max_seconds > 0 ? now() + max_seconds : std::numeric_limits<double>::infinity();
  bool late = false;
  while (!(stop_ || st_.evaluations >= target_.load() || drained())) {
    if (now() > t_end) {  // the pipeline starved (rollouts/compiles slower than the deadline)
      late = true;
      break;
    }
    cv_done_.wait_for(lk, std::chrono::milliseconds(50));
  }
  // lower the target first: the launch thread then stops at its next batch
  // boundary and releases launching_ (else it could keep taking batches while
  // evaluations < the old target and starve this wait past the deadline)
  target_ = st_.evaluations;
  cv_done_.notify_all();
  if (late) cv_done_.wait(lk, [&] { return stop_ || !launching_; });
  if (step_open_) close_step();  // the device-timeline end of an exhausted / late step
  target_ = st_.evaluations;
  if (stop_ && !err_.empty()) return ISPC_E_STICKY;
  return late ? ISPC_E_TIMEOUT : ISPC_OK;
}

ispc_search_stats Search::stats() const {
  std::lock_guard<std::mutex> lk(const_cast<std::mutex&>(mu_));
  ispc_search_stats s = st_;
  s.rollouts = rollouts_;
  s.dead_rollouts = dead_rollouts_;
  s.pruned_children = pruned_;
  s.illegal = illegal_;
  s.duplicates = duplicates_;
  s.compile_errors = compile_errors_;
  s.t_rollout_s = t_rollout_;
  s.t_compile_s = t_compile_;
  s.incumbent_ns = inc_.seconds() * 1e9;
  s.exhausted = exhausted_ ? 1 : 0;
  s.stealing_since = stealing_since_;
  s.elapsed_s = now() - t0_;
  s.refined = refined_;
  s.t_launch_host_s = t_launch_host_;
  return s;
}

std::vector<uint64_t> Search::frontier_digests() const {
  std::vector<uint64_t> d;
  for (size_t i : mine_) d.push_back(digest(*space_->ctx, subtrees_[i]));
  return d;
}

std::string Search::best_candidate() const {
  std::lock_guard<std::mutex> lk(const_cast<std::mutex&>(mu_));
  return best_text_;
}

std::string Search::elite_candidate(size_t i) const {
  std::lock_guard<std::mutex> lk(const_cast<std::mutex&>(elite_mu_));
  return i < elites_.size() ? serialize_text(*space_->ctx, elites_[i].leaf) : std::string();
}

std::string Search::best_source() const {
  std::lock_guard<std::mutex> lk(const_cast<std::mutex&>(mu_));
  return best_src_;
}

}  // namespace ispc_host

// ---- C-ABI -----------------------------------------------------------------------

using namespace ispc_host;

struct ispc_search {
  std::unique_ptr<Search> s;
  std::string err;
};

extern "C" {

int ispc_bound(const ispc_space* s, const ispc_cand* c, int l2_flushed, ispc_bound_report* out) {
  try {
    if (!s || !c || !out) return set_err(ISPC_E_ARG, "null argument");
    if (s->tiles) {
      TileBoundReport r = tile_bound(*s->tiles, *s->ctx, c->c);
      std::memset(out, 0, sizeof(*out));
      out->total = r.total;
      out->dram = r.dram;
      out->issue = r.compute;
      out->launch = r.launch;
      out->dram_bytes = r.dram_bytes;
      out->blocks_max = r.ctas;
      return ISPC_OK;
    }
    B200Machine m;
    m.l2_flushed = l2_flushed != 0;
    BoundModel bm(s->kernel, *s->ctx, m);
    BoundReport r = bm.bound(c->c);
    out->total = r.total;
    out->dram = r.dram;
    out->sm_mem = r.sm_mem;
    out->issue = r.issue;
    out->thread = r.thread;
    out->launch = r.launch;
    out->dram_bytes = r.dram_bytes;
    out->blocks_max = r.blocks_max;
    out->threads_per_block_max = r.threads_per_block_max;
    out->dispatch = r.dispatch;
    out->l1 = r.l1;
    out->lsu = r.lsu;
    return ISPC_OK;
  } catch (const std::exception& e) {
    return set_err(ISPC_E_ARG, e.what());
  }
}

int ispc_search_create(const ispc_space* s, const ispc_search_config* cfg, ispc_search** out) {
  try {
    if (!s || !cfg || !out) return set_err(ISPC_E_ARG, "null argument");
    auto h = std::make_unique<ispc_search>();
    h->s = std::make_unique<Search>(s, *cfg);
    *out = h.release();
    return ISPC_OK;
  } catch (const std::exception& e) {
    return set_err(ISPC_E_CUDA, e.what());
  }
}

int ispc_search_step(ispc_search* h, int64_t evaluations) { return ispc_search_step_for(h, evaluations, 0); }

int ispc_search_step_for(ispc_search* h, int64_t evaluations, double max_seconds) {
  if (!h) return set_err(ISPC_E_ARG, "null search");
  int rc = h->s->step(evaluations, max_seconds);
  if (rc == ISPC_E_TIMEOUT) h->err = "step deadline reached before the evaluation target";
  else if (rc) h->err = h->s->error();
  return rc;
}

int ispc_search_stats_get(const ispc_search* h, ispc_search_stats* out) {
  if (!h || !out) return set_err(ISPC_E_ARG, "null argument");
  *out = h->s->stats();
  return ISPC_OK;
}

static int put(const std::string& s, char* buf, size_t cap, size_t* len) {
  if (len) *len = s.size();
  if (buf && cap) {
    size_t k = s.size() < cap - 1 ? s.size() : cap - 1;
    std::memcpy(buf, s.data(), k);
    buf[k] = 0;
  }
  return ISPC_OK;
}

int ispc_search_best(const ispc_search* h, char* buf, size_t cap, size_t* len) {
  if (!h) return set_err(ISPC_E_ARG, "null search");
  return put(h->s->best_candidate(), buf, cap, len);
}

int ispc_search_elite(const ispc_search* h, int i, char* buf, size_t cap, size_t* len) {
  if (!h || i < 0) return set_err(ISPC_E_ARG, "null search or negative index");
  return put(h->s->elite_candidate(size_t(i)), buf, cap, len);
}

int ispc_search_best_source(const ispc_search* h, char* buf, size_t cap, size_t* len) {
  if (!h) return set_err(ISPC_E_ARG, "null search");
  return put(h->s->best_source(), buf, cap, len);
}

const char* ispc_search_error(const ispc_search* h) { return h ? h->err.c_str() : ""; }

int ispc_search_write_region(ispc_search* h, const char* name, const void* host, size_t bytes) {
  if (!h || !name || !host) return set_err(ISPC_E_ARG, "null argument");
  return h->s->region_io(name, const_cast<void*>(host), bytes, true);
}

int ispc_search_read_region(ispc_search* h, const char* name, void* host, size_t bytes) {
  if (!h || !name || !host) return set_err(ISPC_E_ARG, "null argument");
  return h->s->region_io(name, host, bytes, false);
}

void ispc_search_free(ispc_search* h) { delete h; }

int64_t ispc_search_frontier(const ispc_search* h, uint64_t* digests, int64_t cap) {
  if (!h) return set_err(ISPC_E_ARG, "null search");
  std::vector<uint64_t> d = h->s->frontier_digests();
  for (int64_t i = 0; i < cap && i < int64_t(d.size()); ++i) digests[i] = d[size_t(i)];
  return int64_t(d.size());
}

int ispc_search_offer(ispc_search* h, double ns) {
  if (!h) return set_err(ISPC_E_ARG, "null search");
  return h->s->offer(ns) ? 1 : 0;
}

}  // extern "C"
