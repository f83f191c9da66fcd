// Tree walks over the reference's decision space. Each helper applies
// decisions only through the reference API (open_choices / apply_decision,
// candidate.hpp:75-95), so node and leaf counts are the reference's own.
#include <algorithm>
#include <cmath>
#include <limits>

#include "host_internal.hpp"

namespace ispc_host {

using namespace ispace;

DecisionOrder DecisionOrder::from_names(const SpaceContext& ctx, const std::vector<std::string>& names) {
  DecisionOrder o;
  o.rank.assign(ctx.table.choices.size(), std::numeric_limits<int>::max());
  for (size_t i = 0; i < names.size(); ++i) {
    std::uint32_t ch = ctx.table.find_choice(names[i]);
    if (ch != kNoInstance) o.rank[ch] = int(i);
  }
  return o;
}

std::uint32_t DecisionOrder::pick(const SpaceContext& ctx, const Candidate& c) const {
  std::uint32_t best = kNoInstance;
  int best_rank = std::numeric_limits<int>::max();
  for (std::uint32_t i = 0; i < ctx.table.instances.size(); ++i) {
    const Instance& in = ctx.table.instances[i];
    if (in.counter_slot != ~std::uint32_t{0}) continue;
    if (!instance_live(ctx, c, i)) continue;
    if (mask_single(c.dom[i])) continue;
    int r = rank.empty() ? 0 : rank[in.choice];
    if (best == kNoInstance || r < best_rank) {
      best = i;
      best_rank = r;
      if (rank.empty()) break;
    }
  }
  return best;
}

WalkResult random_walk(const SpaceContext& ctx, const Candidate& from, std::mt19937_64& rng, Candidate& leaf,
                       const DecisionOrder* order) {
  WalkResult w;
  Candidate cur = from;
  static const DecisionOrder declaration;
  const DecisionOrder& ord = order ? *order : declaration;
  for (;;) {
    std::uint32_t inst = ord.pick(ctx, cur);
    if (inst == kNoInstance) {
      leaf = std::move(cur);
      w.ok = true;
      return w;
    }
    Mask m = cur.dom[inst];
    int count = mask_count(m);
    int pick = int(rng() % std::uint64_t(count));
    int v = 0;
    for (int b = 0; b < kMaxDomainBits; ++b)
      if (mask_has(m, b) && pick-- == 0) {
        v = b;
        break;
      }
    Candidate child;
    ++w.decisions;
    if (apply_decision(ctx, cur, inst, v, child) != PropStatus::Ok) return w;
    cur = std::move(child);
  }
}

bool first_leaf(const SpaceContext& ctx, const Candidate& root, Candidate& out, int* budget) {
  std::vector<std::uint32_t> open = open_choices(ctx, root);
  if (open.empty()) {
    out = root;
    return true;
  }
  std::uint32_t inst = open.front();
  Mask m = root.dom[inst];
  for (int v = 0; v < kMaxDomainBits; ++v) {
    if (!mask_has(m, v)) continue;
    if (--*budget <= 0) return false;
    Candidate child;
    if (apply_decision(ctx, root, inst, v, child) != PropStatus::Ok) continue;
    if (first_leaf(ctx, child, out, budget)) return true;
  }
  return false;
}

void count_leaves(const SpaceContext& ctx, const Candidate& c, int64_t& n, int64_t cap) {
  if (n >= cap) return;
  std::vector<std::uint32_t> open = open_choices(ctx, c);
  if (open.empty()) {
    ++n;
    return;
  }
  std::uint32_t inst = open.front();
  Mask m = c.dom[inst];
  for (int v = 0; v < kMaxDomainBits && n < cap; ++v) {
    if (!mask_has(m, v)) continue;
    Candidate child;
    if (apply_decision(ctx, c, inst, v, child) != PropStatus::Ok) continue;
    count_leaves(ctx, child, n, cap);
  }
}

}  // namespace ispc_host
