// Internal types of libispc_host: the opaque handles of ispc_host.h and the
// tree-walk helpers shared by the C-ABI, the bound and the search.
#pragma once

#include <memory>
#include <random>
#include <string>
#include <vector>

#include "ispace/candidate.hpp"
#include "ispace/kernels.hpp"
#include "ispace/machine.hpp"
#include "ispc_host.h"
#include "tiles.hpp"

struct ispc_space {
  ispc_kernel_spec spec{};
  std::string kind;
  ispace::Kernel kernel;
  ispace::MachineParams mp;
  std::shared_ptr<const ispace::SpaceContext> ctx;
  ispace::Candidate root;
  double build_seconds = 0;
  // building-block kinds (gemv, sgemm, batched, sgemm_tc): the tiles.space
  // family; `kernel` stays empty for them
  std::unique_ptr<ispc_host::TileFamily> tiles;
};

struct ispc_cand {
  ispace::Candidate c;
};

namespace ispc_host {

using PropStatusInt = int;

int set_err(int code, const std::string& s);
const char* g_err_text();
ispace::MachineParams machine_for(int mode);
PropStatusInt decide_named(const ispace::SpaceContext& ctx, ispace::Candidate& c, const std::string& choice,
                           const std::vector<std::string>& args, const std::string& value);

// Decision order: rank per choice id (lower first); empty = declaration order.
struct DecisionOrder {
  std::vector<int> rank;  // indexed by choice id
  static DecisionOrder from_names(const ispace::SpaceContext& ctx, const std::vector<std::string>& names);
  // next instance to decide, kNoInstance when fully specified
  std::uint32_t pick(const ispace::SpaceContext& ctx, const ispace::Candidate& c) const;
};

struct WalkResult {
  bool ok = false;
  int64_t decisions = 0;
};

// Uniform random descent: the next open instance (by `order`, or the first
// open one) takes a uniformly drawn value; a dead end ends the walk.
WalkResult random_walk(const ispace::SpaceContext& ctx, const ispace::Candidate& from, std::mt19937_64& rng,
                       ispace::Candidate& leaf, const DecisionOrder* order);

bool first_leaf(const ispace::SpaceContext& ctx, const ispace::Candidate& root, ispace::Candidate& out,
                int* budget);
void count_leaves(const ispace::SpaceContext& ctx, const ispace::Candidate& c, int64_t& n, int64_t cap);

struct TreeEstimate {
  double leaves = 0, leaves_stderr = 0, nodes = 0, dead_probe_ratio = 0;
  int64_t probes = 0;
};
TreeEstimate knuth_estimate(const ispace::SpaceContext& ctx, const ispace::Candidate& from, int64_t probes,
                            std::mt19937_64& rng, const DecisionOrder* order);

}  // namespace ispc_host
