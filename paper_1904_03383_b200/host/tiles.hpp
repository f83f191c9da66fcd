// B200 building-block spaces (host side): the decision space of the kernels
// the reference's gpu.space cannot express, written in the reference's space
// language (tiles.space) and built through its public plugin point
//   build_space(BuildInput{SpaceDefinition, Backbone, Providers, pre})
// (proj/core/include/ispace/candidate.hpp:37-49, providers.hpp:19-35), the
// same way build_gpu_space() instantiates gpu.space (gpu_space.cpp:104-113).
// Candidates, propagation, digests and serialization are the reference's.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "ispace/candidate.hpp"
#include "ispc.h"

namespace ispc_host {

struct TileParam {
  std::string name;
  std::vector<std::int64_t> values;
  bool thread = false, warp = false, acc = false, cluster = false, stage = false;
  bool persist = false;  // persistent grid size (0 = one CTA per tile)
};

struct TileFamily {
  std::uint32_t kind = ISPC_TILE_GEMV;
  std::int64_t m = 0, n = 0, k = 0, batch = 1;
  std::vector<TileParam> params;
  std::vector<std::pair<std::string, std::string>> covers;  // (outer, inner)
  std::vector<ispace::PreRestriction> pre;
  std::int64_t min_threads = 1, warp_lanes = 1, max_acc = 256, max_cluster = 8;
  bool x3_only = false;  // sgemm_tc_x3

  // checking rule of this kind's outputs
  bool bit_exact() const;
  double rtol() const;
};

// Parameter sets of a kernel kind ("gemv" | "sgemm" | "batched" | "sgemm_tc").
// Throws std::invalid_argument for other kinds or empty shapes.
TileFamily make_family(const std::string& kind, std::int64_t m, std::int64_t n, std::int64_t k,
                       std::int64_t batch);

bool is_tile_kind(const std::string& kind);

// Checking rule of one configuration: bit-exact for FFMA kernels with one
// k-ascending fmaf chain per output, norm-wise (TileFamily::rtol) otherwise.
bool tile_bit_exact(const ispc_tile_config& t);

const char* tiles_space_text();

// Builds the space (null ctx + diagnostics on failure, like build_gpu_space).
ispace::BuildResult build_tile_space(const TileFamily& f);

// Reads a fully specified candidate into the flat C-ABI configuration.
// Throws std::invalid_argument while a choice is still open.
ispc_tile_config tile_config(const TileFamily& f, const ispace::SpaceContext& ctx, const ispace::Candidate& c);

// B200 lower bound of every completion of `c`, in seconds (+inf when no
// completion can run): compulsory DRAM bytes at nominal HBM3e bandwidth, the
// flops at the FFMA / tensor peak of the SMs the grid can occupy, a launch
// floor; illegal leaves (ispc_emit_tiles rejects them) are +inf.
struct TileBoundReport {
  double total = 0, dram = 0, compute = 0, launch = 0;
  double dram_bytes = 0, ctas = 0;
  bool illegal = false;
};
TileBoundReport tile_bound(const TileFamily& f, const ispace::SpaceContext& ctx, const ispace::Candidate& c);

}  // namespace ispc_host
