// Tree-size estimators, exact enumeration, dead-end rate and the decision-
// order prune profile (the reference's tree_size.cpp is a stub,
// proj/core/src/tree_size.cpp:1; contract SPEC.md:516-567, paper §5.2-5.4,
// PAPER.md:1101-1133, 1192-1202).
//
// Every estimator is written once over a tree interface (root, ordered
// children, stratum key, SPEC.md "TreeInterface" / "Stratifier"):
//   SpaceTree      the reference's decision space: the children of a node are
//                  the values of its next open instance (first open, or first
//                  in a DecisionOrder) that survive apply_decision
//                  (candidate.hpp:75-95); leaves are fully specified
//                  candidates, nodes with no surviving child are dead ends
//   SyntheticTree  closed-form trees for the estimators' known answers:
//                  uniform:B,D (B-ary, depth D), caterpillar:D,H (a spine of D
//                  nodes, each with one leaf beside it, ending in a complete
//                  binary tree of height H: Knuth's worst case), random:S,B,D
//                  (0..B children per node drawn from a hash of the node id)
// Keys are lexicographic pairs that must strictly decrease along every edge
// (SPEC.md: "child key < parent key"; checked on every edge, a violation is
// reported instead of producing an estimate).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <limits>
#include <map>
#include <sstream>
#include <string>

#include "bound.hpp"
#include "host_internal.hpp"
#include "ispace/loop_nest.hpp"

namespace ispc_host {

using namespace ispace;

namespace {

enum class Strat { DepthRemaining, Depth, Remaining, Constant };

Strat parse_strat(const char* s) {
  if (!s || !*s || !std::strcmp(s, "depth_remaining")) return Strat::DepthRemaining;
  if (!std::strcmp(s, "depth")) return Strat::Depth;
  if (!std::strcmp(s, "remaining")) return Strat::Remaining;
  if (!std::strcmp(s, "constant")) return Strat::Constant;
  throw std::invalid_argument(std::string("unknown stratifier '") + s +
                              "' (depth_remaining | depth | remaining | constant)");
}

using Key = std::pair<int64_t, int64_t>;

// (-depth, remaining): the paper's "lexicographic pair of the depth in the
// tree and number of remaining choices", depth negated so the key decreases
//
Key make_key(Strat s, int64_t depth, int64_t remaining) {
  switch (s) {
    case Strat::DepthRemaining: return {-depth, remaining};
    case Strat::Depth: return {-depth, 0};
    case Strat::Remaining: return {0, remaining};
    case Strat::Constant: return {0, 0};
  }
  return {0, 0};
}

struct SpaceNode {
  Candidate c;
  int64_t depth = 0;
};

class SpaceTree {
 public:
  using Node = SpaceNode;
  SpaceTree(const SpaceContext& ctx, const Candidate& from, const DecisionOrder* order)
      : ctx_(ctx), from_(from), order_(order) {}
  Node root() const { return Node{from_, 0}; }
  // false at a leaf; true with the surviving children otherwise (empty: dead end)
  bool children(const Node& n, std::vector<Node>& out) const {
    out.clear();
    std::uint32_t inst = next(n.c);
    if (inst == kNoInstance) return false;
    Mask m = n.c.dom[inst];
    for (int v = 0; v < kMaxDomainBits; ++v) {
      if (!mask_has(m, v)) continue;
      Node ch;
      ch.depth = n.depth + 1;
      if (apply_decision(ctx_, n.c, inst, v, ch.c) == PropStatus::Ok) out.push_back(std::move(ch));
    }
    return true;
  }
  int64_t remaining(const Node& n) const { return int64_t(open_choices(ctx_, n.c).size()); }

 private:
  std::uint32_t next(const Candidate& c) const {
    if (order_) return order_->pick(ctx_, c);
    std::vector<std::uint32_t> open = open_choices(ctx_, c);
    return open.empty() ? kNoInstance : open.front();
  }
  const SpaceContext& ctx_;
  const Candidate& from_;
  const DecisionOrder* order_;
};

uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

struct SynNode {
  int kind = 0;  // uniform/random: 0; caterpillar: 0 spine, 1 leaf, 2 bush
  int64_t depth = 0, height = 0;
  uint64_t id = 1;
};

class SyntheticTree {
 public:
  using Node = SynNode;
  explicit SyntheticTree(const std::string& spec) {
    const size_t colon = spec.find(':');
    kind_ = spec.substr(0, colon);
    std::vector<int64_t> p;
    if (colon != std::string::npos) {
      std::stringstream ss(spec.substr(colon + 1));
      std::string tok;
      while (std::getline(ss, tok, ',')) p.push_back(std::stoll(tok));
    }
    auto need = [&](size_t n) {
      if (p.size() != n) throw std::invalid_argument("synthetic tree '" + spec + "': wrong parameter count");
    };
    if (kind_ == "uniform") {
      need(2);
      b_ = p[0], d_ = p[1];
    } else if (kind_ == "caterpillar") {
      need(2);
      d_ = p[0], h_ = p[1];
    } else if (kind_ == "random") {
      need(3);
      seed_ = uint64_t(p[0]), b_ = p[1], d_ = p[2];
    } else {
      throw std::invalid_argument("synthetic tree '" + spec + "': uniform:B,D | caterpillar:D,H | random:S,B,D");
    }
    if (b_ < 0 || d_ < 0 || h_ < 0 || b_ > 64 || d_ > 62 || h_ > 40)
      throw std::invalid_argument("synthetic tree '" + spec + "': parameter out of range");
  }
  Node root() const {
    Node n;
    n.height = kind_ == "caterpillar" ? d_ + h_ : d_;
    n.id = mix64(seed_ ^ 0x51ed);
    return n;
  }
  bool children(const Node& n, std::vector<Node>& out) const {
    out.clear();
    if (kind_ == "uniform") {
      if (n.depth >= d_ || b_ == 0) return false;
      for (int64_t i = 0; i < b_; ++i) out.push_back(Node{0, n.depth + 1, d_ - n.depth - 1, 0});
      return true;
    }
    if (kind_ == "random") {
      if (n.depth >= d_) return false;
      const int64_t k = int64_t(mix64(n.id) % uint64_t(b_ + 1));
      if (k == 0) return false;  // an early leaf
      for (int64_t i = 0; i < k; ++i) out.push_back(Node{0, n.depth + 1, d_ - n.depth - 1, mix64(n.id * 31 + uint64_t(i) + 1)});
      return true;
    }
    // caterpillar
    if (n.kind == 1) return false;
    if (n.kind == 2) {
      if (n.height == 0) return false;
      for (int i = 0; i < 2; ++i) out.push_back(Node{2, n.depth + 1, n.height - 1, 0});
      return true;
    }
    if (n.depth < d_) {
      out.push_back(Node{1, n.depth + 1, 0, 0});
      out.push_back(Node{0, n.depth + 1, d_ - n.depth - 1 + h_, 0});
      return true;
    }
    if (h_ == 0) return false;
    for (int i = 0; i < 2; ++i) out.push_back(Node{2, n.depth + 1, h_ - 1, 0});
    return true;
  }
  int64_t remaining(const Node& n) const { return n.height; }

 private:
  std::string kind_;
  int64_t b_ = 0, d_ = 0, h_ = 0;
  uint64_t seed_ = 0;
};

// ---- Knuth: one random descent per probe, the product
// of the branching factors estimates the leaves (0 at a dead end), the sum of
// the partial products the nodes. rng() % children, as knuth_estimate always drew.
template <class Tree>
ispc_tree_estimate knuth(const Tree& t, int64_t probes, std::mt19937_64& rng) {
  double sum = 0, sum2 = 0, nsum = 0, nsum2 = 0;
  int64_t dead = 0;
  std::vector<typename Tree::Node> kids;
  for (int64_t p = 0; p < probes; ++p) {
    typename Tree::Node cur = t.root();
    double w = 1, nd = 1, leaves = 0;
    for (;;) {
      if (!t.children(cur, kids)) {
        leaves = w;
        break;
      }
      if (kids.empty()) {
        ++dead;
        break;
      }
      w *= double(kids.size());
      nd += w;
      cur = std::move(kids[size_t(rng() % kids.size())]);
    }
    sum += leaves, sum2 += leaves * leaves, nsum += nd, nsum2 += nd * nd;
  }
  ispc_tree_estimate e{};
  const double n = double(std::max<int64_t>(probes, 1));
  e.method = 0;
  e.iterations = probes;
  e.leaves = sum / n;
  e.nodes = nsum / n;
  const double vl = probes > 1 ? std::max(0.0, (sum2 / n - e.leaves * e.leaves) / (n - 1)) : 0;
  const double vn = probes > 1 ? std::max(0.0, (nsum2 / n - e.nodes * e.nodes) / (n - 1)) : 0;
  e.leaves_stderr = std::sqrt(vl);
  e.nodes_stderr = std::sqrt(vn);
  e.dead_ratio = double(dead) / n;
  return e;
}

// ---- Chen's heuristic sampling: strata processed in
// decreasing key order; a child joining an occupied stratum adds its weight
// and replaces the representative with probability weight / stratum weight.
// One run estimates the leaves by the weights reaching leaves and the nodes
// by all weights processed; repetitions give the CI.
template <class Tree>
ispc_tree_estimate chen(const Tree& t, int64_t runs, std::mt19937_64& rng, Strat strat, std::string* err) {
  double sum = 0, sum2 = 0, nsum = 0, nsum2 = 0;
  int64_t dead_runs = 0;
  std::vector<typename Tree::Node> kids;
  for (int64_t r = 0; r < runs; ++r) {
    struct Entry {
      typename Tree::Node rep;
      double w;
    };
    std::map<Key, Entry> queue;
    typename Tree::Node root = t.root();
    queue.emplace(make_key(strat, root.depth, t.remaining(root)), Entry{root, 1.0});
    double leaves = 0, nodes = 0;
    bool any_leaf = false;
    while (!queue.empty()) {
      auto top = std::prev(queue.end());
      const Key pk = top->first;
      Entry e = std::move(top->second);
      queue.erase(top);
      nodes += e.w;
      if (!t.children(e.rep, kids)) {
        leaves += e.w;
        any_leaf = true;
        continue;
      }
      for (auto& ch : kids) {
        const Key ck = make_key(strat, ch.depth, t.remaining(ch));
        if (!(ck < pk)) {
          if (err) *err = "stratifier is not strictly decreasing along an edge (SPEC.md: child key < parent key)";
          return ispc_tree_estimate{};
        }
        auto it = queue.find(ck);
        if (it == queue.end()) {
          queue.emplace(ck, Entry{std::move(ch), e.w});
        } else {
          it->second.w += e.w;
          std::uniform_real_distribution<double> u(0.0, 1.0);
          if (u(rng) * it->second.w < e.w) it->second.rep = std::move(ch);
        }
      }
    }
    if (!any_leaf) ++dead_runs;
    sum += leaves, sum2 += leaves * leaves, nsum += nodes, nsum2 += nodes * nodes;
  }
  ispc_tree_estimate e{};
  const double n = double(std::max<int64_t>(runs, 1));
  e.method = 1;
  e.iterations = runs;
  e.leaves = sum / n;
  e.nodes = nsum / n;
  e.leaves_stderr = runs > 1 ? std::sqrt(std::max(0.0, (sum2 / n - e.leaves * e.leaves) / (n - 1))) : 0;
  e.nodes_stderr = runs > 1 ? std::sqrt(std::max(0.0, (nsum2 / n - e.nodes * e.nodes) / (n - 1))) : 0;
  e.dead_ratio = double(dead_runs) / n;
  return e;
}

// ---- exact enumeration (SPEC.md "exact_count"): depth-first, refusing past
// the node budget; per-depth node counts for the §5.4 experiments.
template <class Tree>
bool exact(const Tree& t, int64_t budget, ispc_enum_report& rep, int64_t* per_depth, int depth_cap) {
  std::vector<typename Tree::Node> stack{t.root()};
  std::vector<typename Tree::Node> kids;
  while (!stack.empty()) {
    typename Tree::Node n = std::move(stack.back());
    stack.pop_back();
    if (++rep.nodes > budget) return false;
    if (per_depth && n.depth < depth_cap) ++per_depth[n.depth];
    rep.max_depth = std::max<int64_t>(rep.max_depth, n.depth);
    if (!t.children(n, kids)) {
      ++rep.leaves;
      continue;
    }
    if (kids.empty()) {
      ++rep.dead_ends;
      continue;
    }
    for (auto it = kids.rbegin(); it != kids.rend(); ++it) stack.push_back(std::move(*it));
  }
  return true;
}

DecisionOrder parse_order(const SpaceContext& ctx, const char* order) {
  std::vector<std::string> names;
  std::string cur;
  for (const char* p = order;; ++p) {
    if (*p == ',' || *p == 0) {
      if (!cur.empty()) names.push_back(cur);
      cur.clear();
      if (!*p) break;
    } else {
      cur += *p;
    }
  }
  return DecisionOrder::from_names(ctx, names);
}

}  // namespace

TreeEstimate knuth_estimate(const SpaceContext& ctx, const Candidate& from, int64_t probes, std::mt19937_64& rng,
                            const DecisionOrder* order) {
  ispc_tree_estimate k = knuth(SpaceTree(ctx, from, order), probes, rng);
  TreeEstimate e;
  e.probes = probes;
  e.leaves = k.leaves;
  e.leaves_stderr = k.leaves_stderr;
  e.nodes = k.nodes;
  e.dead_probe_ratio = k.dead_ratio;
  return e;
}

}  // namespace ispc_host

using namespace ispc_host;

extern "C" {

int ispc_estimate(const ispc_space* s, const ispc_cand* from, const char* method, int64_t iterations,
                  uint64_t seed, const char* order, const char* stratifier, ispc_tree_estimate* out) {
  try {
    if (!s || !from || !out || iterations <= 0) return set_err(ISPC_E_ARG, "bad argument");
    std::mt19937_64 rng(seed);
    DecisionOrder ord;
    if (order) ord = parse_order(*s->ctx, order);
    SpaceTree t(*s->ctx, from->c, order ? &ord : nullptr);
    const std::string m = method ? method : "knuth";
    if (m == "knuth") {
      *out = knuth(t, iterations, rng);
    } else if (m == "chen") {
      std::string err;
      *out = chen(t, iterations, rng, parse_strat(stratifier), &err);
      if (!err.empty()) return set_err(ISPC_E_ARG, err);
    } else {
      return set_err(ISPC_E_ARG, "method must be knuth or chen");
    }
    return ISPC_OK;
  } catch (const std::exception& e) {
    return set_err(ISPC_E_ARG, e.what());
  }
}

int ispc_estimate_synthetic(const char* tree, const char* method, int64_t iterations, uint64_t seed,
                            const char* stratifier, ispc_tree_estimate* out) {
  try {
    if (!tree || !out || iterations <= 0) return set_err(ISPC_E_ARG, "bad argument");
    SyntheticTree t(tree);
    std::mt19937_64 rng(seed);
    const std::string m = method ? method : "knuth";
    if (m == "knuth") {
      *out = knuth(t, iterations, rng);
    } else if (m == "chen") {
      std::string err;
      *out = chen(t, iterations, rng, parse_strat(stratifier), &err);
      if (!err.empty()) return set_err(ISPC_E_ARG, err);
    } else {
      return set_err(ISPC_E_ARG, "method must be knuth or chen");
    }
    return ISPC_OK;
  } catch (const std::exception& e) {
    return set_err(ISPC_E_ARG, e.what());
  }
}

int ispc_enumerate(const ispc_space* s, const ispc_cand* from, const char* order, int64_t node_budget,
                   ispc_enum_report* out, int64_t* per_depth, int depth_cap) {
  try {
    if (!s || !from || !out || node_budget <= 0) return set_err(ISPC_E_ARG, "bad argument");
    *out = ispc_enum_report{};
    if (per_depth) std::fill(per_depth, per_depth + std::max(depth_cap, 0), int64_t(0));
    DecisionOrder ord;
    if (order) ord = parse_order(*s->ctx, order);
    if (!exact(SpaceTree(*s->ctx, from->c, order ? &ord : nullptr), node_budget, *out, per_depth, depth_cap))
      return set_err(ISPC_E_ARG, "enumeration refused: the tree has more than " + std::to_string(node_budget) +
                                       " nodes (raise the node budget)");
    return ISPC_OK;
  } catch (const std::exception& e) {
    return set_err(ISPC_E_ARG, e.what());
  }
}

int ispc_enumerate_synthetic(const char* tree, int64_t node_budget, ispc_enum_report* out, int64_t* per_depth,
                             int depth_cap) {
  try {
    if (!tree || !out || node_budget <= 0) return set_err(ISPC_E_ARG, "bad argument");
    *out = ispc_enum_report{};
    if (per_depth) std::fill(per_depth, per_depth + std::max(depth_cap, 0), int64_t(0));
    if (!exact(SyntheticTree(tree), node_budget, *out, per_depth, depth_cap))
      return set_err(ISPC_E_ARG, "enumeration refused: more than " + std::to_string(node_budget) + " nodes");
    return ISPC_OK;
  } catch (const std::exception& e) {
    return set_err(ISPC_E_ARG, e.what());
  }
}

// Paper §5.2's dead-end probability: uniform random descents (unweighted, no
// bound pruning) in the decision order; 95% Wilson score interval.
int ispc_deadend_rate(const ispc_space* s, const ispc_cand* from, int64_t trials, uint64_t seed, const char* order,
                      ispc_deadend_report* out) {
  try {
    if (!s || !from || !out || trials <= 0) return set_err(ISPC_E_ARG, "bad argument");
    std::mt19937_64 rng(seed);
    DecisionOrder ord;
    if (order) ord = parse_order(*s->ctx, order);
    int64_t dead = 0, decisions = 0;
    for (int64_t i = 0; i < trials; ++i) {
      Candidate leaf;
      WalkResult w = random_walk(*s->ctx, from->c, rng, leaf, order ? &ord : nullptr);
      decisions += w.decisions;
      if (!w.ok) ++dead;
    }
    const double n = double(trials), p = double(dead) / n, z = 1.959963984540054;
    const double den = 1 + z * z / n;
    const double centre = (p + z * z / (2 * n)) / den;
    const double half = z * std::sqrt(p * (1 - p) / n + z * z / (4 * n * n)) / den;
    out->trials = trials;
    out->dead_ends = dead;
    out->ratio = p;
    out->ci_lo = std::max(0.0, centre - half);
    out->ci_hi = std::min(1.0, centre + half);
    out->mean_decisions = double(decisions) / n;
    return ISPC_OK;
  } catch (const std::exception& e) {
    return set_err(ISPC_E_ARG, e.what());
  }
}

// A uniform partial descent of `steps` decisions (the first open instance,
// or the first in `order`): subtrees of chosen depth for the estimator and
// dead-end oracles. 1 when it meets a dead end or a leaf first.
int ispc_cand_descend(const ispc_space* s, const ispc_cand* from, const char* order, uint64_t seed, int steps,
                      ispc_cand** out) {
  try {
    if (!s || !from || !out || steps < 0) return set_err(ISPC_E_ARG, "bad argument");
    DecisionOrder ord;
    if (order) ord = parse_order(*s->ctx, order);
    SpaceTree t(*s->ctx, from->c, order ? &ord : nullptr);
    std::mt19937_64 rng(seed);
    SpaceNode cur = t.root();
    std::vector<SpaceNode> kids;
    for (int i = 0; i < steps; ++i) {
      if (!t.children(cur, kids) || kids.empty()) return 1;
      cur = std::move(kids[size_t(rng() % kids.size())]);
    }
    *out = new ispc_cand{cur.c};
    return ISPC_OK;
  } catch (const std::exception& e) {
    return set_err(ISPC_E_ARG, e.what());
  }
}

// The exact probability that a uniform random descent (random_walk: a value
// drawn uniformly from the instance's domain, dead end when propagation
// fails) ends at a dead end: p(n) = mean over the domain's values of
// [fails ? 1 : p(child)]; the oracle of ispc_deadend_rate on small trees.
int ispc_deadend_exact(const ispc_space* s, const ispc_cand* from, const char* order, int64_t node_budget,
                       double* p_dead) {
  try {
    if (!s || !from || !p_dead || node_budget <= 0) return set_err(ISPC_E_ARG, "bad argument");
    DecisionOrder ord;
    if (order) ord = parse_order(*s->ctx, order);
    const DecisionOrder* op = order ? &ord : nullptr;
    static const DecisionOrder declaration;
    const DecisionOrder& o = op ? *op : declaration;
    int64_t seen = 0;
    std::function<double(const Candidate&)> rec = [&](const Candidate& c) -> double {
      if (++seen > node_budget) throw std::range_error("node budget");
      const std::uint32_t inst = o.pick(*s->ctx, c);
      if (inst == kNoInstance) return 0.0;
      const Mask m = c.dom[inst];
      double sum = 0;
      int n = 0;
      for (int v = 0; v < kMaxDomainBits; ++v) {
        if (!mask_has(m, v)) continue;
        ++n;
        Candidate ch;
        sum += apply_decision(*s->ctx, c, inst, v, ch) != PropStatus::Ok ? 1.0 : rec(ch);
      }
      return n ? sum / n : 1.0;
    };
    try {
      *p_dead = rec(from->c);
    } catch (const std::range_error&) {
      return set_err(ISPC_E_ARG, "exact dead-end probability refused: more than " + std::to_string(node_budget) +
                                     " nodes");
    }
    return ISPC_OK;
  } catch (const std::exception& e) {
    return set_err(ISPC_E_ARG, e.what());
  }
}

// The reference's order round trip (nest_test.cpp:309-334) over every leaf
// below `from`: reconstruct -> derive_orders (loop_nest.cpp:359-385), and each
// derived pair's relation must be the single value the leaf's order(a, b)
// instance holds (oriented like the reference test).
int ispc_order_round_trip(const ispc_space* s, const ispc_cand* from, int64_t node_budget, int64_t* leaves,
                          int64_t* pairs, int64_t* mismatches) {
  try {
    if (!s || !from || !leaves || !pairs || !mismatches || node_budget <= 0) return set_err(ISPC_E_ARG, "bad argument");
    if (s->tiles) return set_err(ISPC_E_ARG, "order round trip: loop-nest spaces only");
    const SpaceContext& ctx = *s->ctx;
    const std::uint32_t order_c = ctx.table.find_choice("order");
    if (order_c == kNoInstance) return set_err(ISPC_E_ARG, "space has no order choice");
    *leaves = *pairs = *mismatches = 0;
    SpaceTree t(ctx, from->c, nullptr);
    std::vector<SpaceNode> stack{t.root()}, kids;
    int64_t seen = 0;
    while (!stack.empty()) {
      SpaceNode n = std::move(stack.back());
      stack.pop_back();
      if (++seen > node_budget) return set_err(ISPC_E_ARG, "order round trip refused: node budget exceeded");
      if (t.children(n, kids)) {
        for (auto& k : kids) stack.push_back(std::move(k));
        continue;
      }
      ++*leaves;
      LoopNest l = reconstruct(s->kernel, ctx, n.c);
      for (const auto& [pr, name] : derive_orders(l)) {
        ++*pairs;
        ObjId ids[2] = {pr.first, pr.second};
        InstanceRef ref = ctx.table.resolve(order_c, ids, 2);
        bool ok = ref.inst != kNoInstance;
        if (ok) {
          Mask m = ctx.table.oriented(order_c, n.c.dom[ref.inst], ref.swapped);
          ok = mask_single(m) && ctx.table.choices[order_c].values[mask_first(m)] == name;
        }
        if (!ok) ++*mismatches;
      }
    }
    return ISPC_OK;
  } catch (const std::exception& e) {
    return set_err(ISPC_E_ARG, e.what());
  }
}

// Paper §5.4's "ratio of nodes that the performance model can prune in the
// first levels": every node of the first `depth_cap` levels (tree in `order`)
// is bounded with the B200 model; a node is prunable when its bound >= T.
// The bound is monotone, so descendants of a prunable node are prunable too
// and are still counted at their depth (the denominator is the unpruned tree).
int ispc_prune_profile(const ispc_space* s, const ispc_cand* from, const char* order, double threshold_s,
                       int depth_cap, int64_t node_budget, int64_t* nodes_per_depth, int64_t* pruned_per_depth) {
  try {
    if (!s || !from || !nodes_per_depth || !pruned_per_depth || depth_cap <= 0 || node_budget <= 0)
      return set_err(ISPC_E_ARG, "bad argument");
    if (s->tiles) return set_err(ISPC_E_ARG, "prune profile: loop-nest spaces only");
    std::fill(nodes_per_depth, nodes_per_depth + depth_cap, int64_t(0));
    std::fill(pruned_per_depth, pruned_per_depth + depth_cap, int64_t(0));
    DecisionOrder ord;
    if (order) ord = parse_order(*s->ctx, order);
    SpaceTree t(*s->ctx, from->c, order ? &ord : nullptr);
    B200Machine m;
    BoundModel bm(s->kernel, *s->ctx, m);
    struct Item {
      SpaceNode n;
      bool pruned;
    };
    std::vector<Item> stack{{t.root(), false}};
    std::vector<SpaceNode> kids;
    int64_t seen = 0;
    while (!stack.empty()) {
      Item it = std::move(stack.back());
      stack.pop_back();
      if (++seen > node_budget)
        return set_err(ISPC_E_ARG, "prune profile refused: more than " + std::to_string(node_budget) +
                                         " nodes in the first " + std::to_string(depth_cap) + " levels");
      const bool pruned = it.pruned || !(bm.bound(it.n.c).total < threshold_s);
      ++nodes_per_depth[it.n.depth];
      if (pruned) ++pruned_per_depth[it.n.depth];
      if (it.n.depth + 1 >= depth_cap) continue;
      if (!t.children(it.n, kids)) continue;
      for (auto& k : kids) stack.push_back(Item{std::move(k), pruned});
    }
    return ISPC_OK;
  } catch (const std::exception& e) {
    return set_err(ISPC_E_ARG, e.what());
  }
}

// The lowest-bound descent: at every decision the child with the smallest
// B200 bound first (value order on ties), backtracking out of dead ends and
// infinite-bound subtrees; 1 when none is found within the node budget.
// Gives order-compare an incumbent without a GPU.
int ispc_greedy_leaf(const ispc_space* s, const ispc_cand* from, const char* order, ispc_cand** out,
                     double* bound_s) {
  try {
    if (!s || !from || !out) return set_err(ISPC_E_ARG, "bad argument");
    if (s->tiles) return set_err(ISPC_E_ARG, "greedy leaf: loop-nest spaces only");
    DecisionOrder ord;
    if (order) ord = parse_order(*s->ctx, order);
    SpaceTree t(*s->ctx, from->c, order ? &ord : nullptr);
    B200Machine m;
    BoundModel bm(s->kernel, *s->ctx, m);
    // depth-first, children in ascending bound order (finite bounds only),
    // backtracking out of dead ends within a node budget
    struct Frame {
      std::vector<std::pair<double, SpaceNode>> kids;
      size_t next = 0;
    };
    SpaceNode cur;
    double b = std::numeric_limits<double>::infinity();
    std::vector<Frame> stack;
    std::vector<SpaceNode> kids;
    auto expand = [&](const SpaceNode& n) -> int {  // 0 leaf, 1 frame pushed
      if (!t.children(n, kids)) return 0;
      Frame f;
      for (auto& k : kids) {
        const double x = bm.bound(k.c).total;
        if (std::isfinite(x)) f.kids.emplace_back(x, std::move(k));
      }
      std::stable_sort(f.kids.begin(), f.kids.end(),
                       [](const auto& a, const auto& c) { return a.first < c.first; });
      stack.push_back(std::move(f));
      return 1;
    };
    int64_t budget = 200000;
    SpaceNode root = t.root();
    bool found = false;
    if (expand(root) == 0) {
      cur = root, b = bm.bound(root.c).total, found = true;
    }
    while (!found && !stack.empty() && budget-- > 0) {
      Frame& f = stack.back();
      if (f.next >= f.kids.size()) {
        stack.pop_back();
        continue;
      }
      auto& [x, n] = f.kids[f.next++];
      const double xb = x;
      SpaceNode node = n;
      if (expand(node) == 0) {
        cur = std::move(node), b = xb, found = true;
      }
    }
    if (!found) return 1;
    *out = new ispc_cand{cur.c};
    if (bound_s) *bound_s = b;
    return ISPC_OK;
  } catch (const std::exception& e) {
    return set_err(ISPC_E_ARG, e.what());
  }
}

}  // extern "C"
