// Reference-side adapter: flattens the reference's Kernel backbone and a
// reconstructed LoopNest (proj/core/include/ispace/{kernels,loop_nest}.hpp)
// into the C-ABI `ispc_nest` (include/ispc.h). This is the binding a
// maintainer adds next to the reference's evaluate() call site
// (INTEGRATION.md); it owns the arrays the ispc_nest points into.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "ispace/kernels.hpp"
#include "ispace/loop_nest.hpp"
#include "ispc.h"

namespace ispc_host {

struct NestBuf {
  std::string kernel_name;
  std::vector<std::string> names;
  std::vector<const char*> name_ptrs;
  std::vector<std::string> inputs;
  std::vector<const char*> input_ptrs;
  std::vector<ispc_inst> insts;
  std::vector<ispc_region> regions;
  std::vector<ispc_dim> dims;
  std::vector<ispc_ivar> ivars;
  std::vector<ispc_addr_term> terms;
  std::vector<ispc_operand> operands;
  std::vector<ispc_comm> comms;
  std::vector<uint32_t> pool;
  std::vector<ispc_node> nodes;
  ispc_nest nest{};
};

// Builds the flat description. The LoopNest must come from reconstruct() on
// the same kernel.
std::unique_ptr<NestBuf> flatten(const ispace::Kernel& k, const ispace::LoopNest& l);

}  // namespace ispc_host
