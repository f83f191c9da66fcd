// Deterministic, single-threaded TAG-MCTS exactly as SPEC.md:459-514 states
// it (the reference's search.cpp is a stub, proj/core/src/search.cpp:1):
// the bit-comparable counterpart of the production pipeline in search.cpp,
// whose pruning depends on measured times and on thread interleaving.
//
//   tree       SearchNode = candidate, children keyed by the values of the
//              next decision (fixed DecisionOrder; SPEC "DecisionOrder"),
//              one child per value, children failing propagation kept as
//              DeadEnd markers; per child the visit count t, the costs of the
//              rollouts through it (s = how many rank in the global best-
//              `bucket` set), its cached bound
//   select     TAG: unvisited children first (lowest index), then
//              argmax (s + a + sqrt(2 s a + a^2)) / t, a = ln(2 N k / delta);
//              children with bound >= T excluded (pruning on), ties to the
//              lowest index (ispc_tag_select)
//   expand     the first unexpanded node met: all its children materialised
//   rollout    below it: the next open instance per order, a value drawn with
//              p ~ max(T - b(child), 0) (uniform while T is infinite or
//              pruning is off); a dead end is recorded, not raised
//   evaluate   fully specified leaves: "bound" = the B200 bound x (1 + u),
//              u in [0, 0.5) from the leaf digest (admissible by
//              construction: the pruning-safety oracle), or "simulate" = the
//              reference's reconstruct + evaluate cycles (simulate.cpp:131-133)
//              with a zero bound (nothing is pruned: the reference has no bound)
//   log        one JSONL record per rollout: seed, path (decision values),
//              cost or DEADEND, the bounds of every ancestor; no clocks, so the
//              same seed and configuration give a byte-identical log
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <random>
#include <string>
#include <unordered_map>

#include "bound.hpp"
#include "host_internal.hpp"
#include "ispace/loop_nest.hpp"
#include "ispace/simulate.hpp"

namespace ispc_host {

using namespace ispace;

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

double tag_score(double s, double t, double alpha) {
  return (s + alpha + std::sqrt(2 * s * alpha + alpha * alpha)) / t;
}

struct SNode {
  Candidate cand;
  double bound = 0;
  bool dead_end = false;    // failed propagation (a DeadEnd marker)
  bool leaf = false;        // fully specified
  bool exhausted = false;   // every completion evaluated or excluded
  bool expanded = false;
  std::vector<int> values;  // decision value of each child
  std::vector<std::unique_ptr<SNode>> kids;
  int64_t t = 0;
  std::vector<double> costs;  // of the rollouts through this node
};

class SpecExplorer {
 public:
  SpecExplorer(const ispc_space* s, const ispc_spec_config& cfg)
      : s_(s), cfg_(cfg), rng_(cfg.seed), bm_(s->kernel, *s->ctx, B200Machine{}) {
    if (cfg.order && *cfg.order) {
      std::vector<std::string> names;
      std::string cur;
      for (const char* p = cfg.order;; ++p) {
        if (*p == ',' || *p == 0) {
          if (!cur.empty()) names.push_back(cur);
          cur.clear();
          if (!*p) break;
        } else {
          cur += *p;
        }
      }
      order_ = DecisionOrder::from_names(*s->ctx, names);
      has_order_ = true;
    }
    delta_ = cfg.delta > 0 ? cfg.delta : 0.05;
    bucket_ = cfg.bucket > 0 ? size_t(cfg.bucket) : 20;
    // resume: the log of an earlier run with the same seed and configuration
    // is the checkpoint; its records are re-derived (and must match byte for
    // byte) before new ones are appended
    if (cfg.resume_log && *cfg.resume_log) {
      FILE* f = std::fopen(cfg.resume_log, "r");
      if (!f) throw std::invalid_argument(std::string("cannot read resume log ") + cfg.resume_log);
      char buf[1 << 16];
      while (std::fgets(buf, sizeof(buf), f)) resume_.emplace_back(buf);
      std::fclose(f);
    }
    if (cfg.log_path && *cfg.log_path) log_ = std::fopen(cfg.log_path, "w");
    root_ = std::make_unique<SNode>();
    root_->cand = s->root;
    root_->bound = bound(root_->cand);
    root_->leaf = next(root_->cand) == kNoInstance;
  }
  ~SpecExplorer() {
    if (log_) std::fclose(log_);
  }

  void run(ispc_spec_result& res) {
    while ((st_.evaluations < cfg_.budget || replayed_ < resume_.size()) && !root_->exhausted) {
      if (cfg_.max_rollouts > 0 && st_.rollouts >= cfg_.max_rollouts) break;
      iterate();
    }
    if (replayed_ < resume_.size() || diverged_)
      throw std::runtime_error("resume log does not replay under this seed and configuration (record " +
                               std::to_string(diverged_ ? first_diverged_ : replayed_ + 1) + ")");
    st_.replayed = int64_t(replayed_);
    st_.exhausted = root_->exhausted ? 1 : 0;
    st_.best_cost = best_;
    st_.best_digest = best_digest_;
    res = st_;
  }
  std::string best_text() const { return best_text_; }

 private:
  const ispc_space* s_;
  ispc_spec_config cfg_;
  std::mt19937_64 rng_;
  BoundModel bm_;
  DecisionOrder order_;
  bool has_order_ = false;
  double delta_ = 0.05;
  size_t bucket_ = 20;
  FILE* log_ = nullptr;
  std::unique_ptr<SNode> root_;
  std::vector<double> top_;  // the best `bucket_` rollout costs, ascending
  std::unordered_map<uint64_t, double> evaluated_;
  double best_ = kInf;
  uint64_t best_digest_ = 0;
  std::string best_text_;
  ispc_spec_result st_{};
  std::vector<std::string> resume_;
  size_t replayed_ = 0;
  bool diverged_ = false;
  size_t first_diverged_ = 0;

  double T() const { return cfg_.pruning ? best_ : kInf; }

  std::uint32_t next(const Candidate& c) const {
    if (has_order_) return order_.pick(*s_->ctx, c);
    std::vector<std::uint32_t> open = open_choices(*s_->ctx, c);
    return open.empty() ? kNoInstance : open.front();
  }

  double bound(const Candidate& c) const {
    if (cfg_.evaluator == ISPC_SPEC_EVAL_SIMULATE) return 0.0;
    return bm_.bound(c).total;
  }

  double evaluate(const Candidate& leaf) {
    const uint64_t d = digest(*s_->ctx, leaf);
    auto it = evaluated_.find(d);
    if (it != evaluated_.end()) {
      ++st_.duplicates;
      return it->second;
    }
    double cost;
    if (cfg_.evaluator == ISPC_SPEC_EVAL_SIMULATE) {
      LoopNest l = reconstruct(s_->kernel, *s_->ctx, leaf);
      cost = double(ispace::evaluate(s_->kernel, l, s_->mp).total);
    } else {
      // admissible by construction: cost >= the leaf's bound >= every ancestor's
      uint64_t h = d * 0x9e3779b97f4a7c15ull;
      h ^= h >> 29;
      cost = bm_.bound(leaf).total * (1.0 + double(h % 1000003) / 1000003.0 * 0.5);
    }
    evaluated_.emplace(d, cost);
    ++st_.evaluations;
    if (std::isfinite(cost)) {
      top_.insert(std::upper_bound(top_.begin(), top_.end(), cost), cost);
      if (top_.size() > bucket_) top_.pop_back();
    }
    if (cost < best_) {
      best_ = cost;
      best_digest_ = d;
      best_text_ = serialize_text(*s_->ctx, leaf);
      st_.time_to_best_evals = st_.evaluations;
    }
    return cost;
  }

  void expand(SNode& n) {
    n.expanded = true;
    const std::uint32_t inst = next(n.cand);
    if (inst == kNoInstance) {
      n.leaf = true;
      return;
    }
    const Mask m = n.cand.dom[inst];
    for (int v = 0; v < kMaxDomainBits; ++v) {
      if (!mask_has(m, v)) continue;
      auto ch = std::make_unique<SNode>();
      if (apply_decision(*s_->ctx, n.cand, inst, v, ch->cand) != PropStatus::Ok) {
        ch->dead_end = true;
        ch->exhausted = true;
        ch->bound = kInf;
      } else {
        ch->bound = bound(ch->cand);
        ch->leaf = next(ch->cand) == kNoInstance;
      }
      n.values.push_back(v);
      n.kids.push_back(std::move(ch));
    }
  }

  // TAG over the node's live children (-1: none)
  int select(const SNode& n) const {
    const size_t k = n.kids.size();
    std::vector<double> s(k, 0), t(k, 0);
    std::vector<unsigned char> excl(k, 0);
    const double thr = top_.size() >= bucket_ ? top_.back() : kInf;
    for (size_t i = 0; i < k; ++i) {
      const SNode& c = *n.kids[i];
      excl[i] = c.exhausted || !(c.bound < T());
      t[i] = double(c.t);
      for (double x : c.costs) s[i] += x <= thr ? 1 : 0;
    }
    return ispc_tag_select(int(k), s.data(), t.data(), excl.data(), n.t, delta_, int(bucket_));
  }

  void refresh_exhausted(SNode& n) const {
    if (!n.expanded) return;
    bool all = true;
    for (auto& c : n.kids)
      if (!(c->exhausted || !(c->bound < T()))) all = false;
    if (all) n.exhausted = true;
  }

  void iterate() {
    ++st_.rollouts;
    std::vector<SNode*> path{root_.get()};
    std::vector<int> values;
    std::vector<double> bounds{root_->bound};  // of every node on the path, root first
    SNode* n = root_.get();
    // selection through expanded nodes
    while (n->expanded && !n->leaf) {
      const int i = select(*n);
      if (i < 0) {
        n->exhausted = true;
        for (size_t p = path.size(); p-- > 1;) refresh_exhausted(*path[p - 1]);
        ++st_.dead_rollouts;
        log_rollout(values, bounds, kInf, "PRUNED");
        return;
      }
      values.push_back(n->values[size_t(i)]);
      n = n->kids[size_t(i)].get();
      path.push_back(n);
      bounds.push_back(n->bound);
    }
    double cost;
    if (n->leaf) {  // a tree leaf: evaluated once, then exhausted
      cost = evaluate(n->cand);
      n->exhausted = true;
    } else {
      expand(*n);
      ++st_.expanded;
      cost = rollout(n->cand, values, bounds);
    }
    for (SNode* p : path) {
      ++p->t;
      if (std::isfinite(cost)) p->costs.push_back(cost);
    }
    for (size_t p = path.size(); p-- > 0;) refresh_exhausted(*path[p]);
    if (!std::isfinite(cost)) ++st_.dead_rollouts;
    log_rollout(values, bounds, cost, std::isfinite(cost) ? nullptr : "DEADEND");
  }

  // Monte-Carlo descent below the tree: p ~ max(T - b, 0) over the values
  double rollout(Candidate cur, std::vector<int>& values, std::vector<double>& bounds) {
    const SpaceContext& ctx = *s_->ctx;
    for (;;) {
      const std::uint32_t inst = next(cur);
      if (inst == kNoInstance) return evaluate(cur);
      const Mask m = cur.dom[inst];
      std::vector<Candidate> kids;
      std::vector<int> vals;
      std::vector<double> w, bs;
      const double Tv = T();
      for (int v = 0; v < kMaxDomainBits; ++v) {
        if (!mask_has(m, v)) continue;
        Candidate ch;
        if (apply_decision(ctx, cur, inst, v, ch) != PropStatus::Ok) continue;
        const double b = bound(ch);
        double weight;
        if (!std::isfinite(Tv)) weight = std::isfinite(b) || cfg_.evaluator == ISPC_SPEC_EVAL_SIMULATE ? 1.0 : 0.0;
        else weight = std::max(Tv - b, 0.0);
        if (weight <= 0) continue;
        kids.push_back(std::move(ch));
        vals.push_back(v);
        w.push_back(weight);
        bs.push_back(b);
      }
      if (kids.empty()) return kInf;  // all children infeasible or provably worse than T
      std::discrete_distribution<size_t> pick(w.begin(), w.end());
      const size_t i = pick(rng_);
      values.push_back(vals[i]);
      bounds.push_back(bs[i]);
      cur = std::move(kids[i]);
    }
  }

  void log_rollout(const std::vector<int>& values, const std::vector<double>& bounds, double cost,
                   const char* tag) {
    if (!log_ && resume_.empty()) return;
    std::string p = "[", b = "[";
    for (size_t i = 0; i < values.size(); ++i) p += (i ? "," : "") + std::to_string(values[i]);
    for (size_t i = 0; i < bounds.size(); ++i) {
      char x[40];
      std::snprintf(x, sizeof(x), "%s%.9g", i ? "," : "", bounds[i]);
      b += x;
    }
    char head[160], tail[160];
    std::snprintf(head, sizeof(head), "{\"rollout\": %lld, \"seed\": %llu, \"path\": ", (long long)st_.rollouts,
                  (unsigned long long)cfg_.seed);
    if (tag)
      std::snprintf(tail, sizeof(tail), "\"cost\": \"%s\", ", tag);
    else
      std::snprintf(tail, sizeof(tail), "\"cost\": %.9g, ", cost);
    char fin[96];
    std::snprintf(fin, sizeof(fin), "\"best\": %.9g, \"evaluations\": %lld}\n", best_, (long long)st_.evaluations);
    const std::string rec = std::string(head) + p + "], \"ancestor_bounds\": " + b + "], " + tail + fin;
    if (replayed_ < resume_.size()) {
      if (resume_[replayed_] != rec && !diverged_) diverged_ = true, first_diverged_ = replayed_ + 1;
      ++replayed_;
    }
    if (log_) std::fputs(rec.c_str(), log_);
  }
};

}  // namespace
}  // namespace ispc_host

using namespace ispc_host;

extern "C" {

int ispc_tag_select(int k, const double* s, const double* t, const unsigned char* excluded, int64_t total,
                    double delta, int bucket) {
  if (k <= 0 || !s || !t) return -1;
  for (int i = 0; i < k; ++i)  // unvisited first, lowest index
    if (!(excluded && excluded[i]) && t[i] <= 0) return i;
  const double alpha = std::log(2.0 * double(std::max<int64_t>(total, 1)) * double(k) / (delta > 0 ? delta : 0.05));
  (void)bucket;
  int best = -1;
  double best_h = -kInf;
  for (int i = 0; i < k; ++i) {
    if (excluded && excluded[i]) continue;
    const double h = tag_score(s[i], t[i], alpha);
    if (h > best_h) best_h = h, best = i;  // strict: ties keep the lowest index
  }
  return best;
}

int ispc_explore_spec(const ispc_space* s, const ispc_spec_config* cfg, ispc_spec_result* out, char* best_text,
                      size_t cap, size_t* len) {
  try {
    if (!s || !cfg || !out) return set_err(ISPC_E_ARG, "null argument");
    if (s->tiles) return set_err(ISPC_E_ARG, "spec explorer: loop-nest (gpu.space) kinds only");
    if (cfg->evaluator != ISPC_SPEC_EVAL_BOUND && cfg->evaluator != ISPC_SPEC_EVAL_SIMULATE)
      return set_err(ISPC_E_ARG, "evaluator must be ISPC_SPEC_EVAL_BOUND or ISPC_SPEC_EVAL_SIMULATE");
    SpecExplorer x(s, *cfg);
    x.run(*out);
    const std::string t = x.best_text();
    if (len) *len = t.size();
    if (best_text && cap > 0) {
      const size_t n = std::min(cap - 1, t.size());
      std::memcpy(best_text, t.data(), n);
      best_text[n] = 0;
    }
    return ISPC_OK;
  } catch (const std::exception& e) {
    return set_err(ISPC_E_ARG, e.what());
  }
}

// Seeded uniform first-open descents with one generator across walks, the
// walk oracle/ref_cpu_bench.cpp runs per thread (mt19937_64(0x190403383 +
// 7919 tid), rng() % count over the domain's values): digest of each leaf,
// 0 for a walk that met a dead end.
int ispc_walk_digests(const ispc_space* s, const ispc_cand* from, uint64_t seed, int64_t walks, uint64_t* digests) {
  try {
    if (!s || !from || !digests || walks < 0) return set_err(ISPC_E_ARG, "bad argument");
    std::mt19937_64 rng(seed);
    for (int64_t i = 0; i < walks; ++i) {
      Candidate leaf;
      WalkResult w = random_walk(*s->ctx, from->c, rng, leaf, nullptr);
      digests[i] = w.ok ? digest(*s->ctx, leaf) : 0;
    }
    return ISPC_OK;
  } catch (const std::exception& e) {
    return set_err(ISPC_E_ARG, e.what());
  }
}

}  // extern "C"
