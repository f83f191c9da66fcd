// Indexed, validated view of a flat ispc_nest (include/ispc.h). Both emitters
// (CUDA and the reference-compatible pseudo text) and the static legality
// checks read the schedule through this class.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "ispc.h"

namespace ispc {

struct NestError : std::runtime_error {
  int code;
  NestError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

class NestView {
 public:
  explicit NestView(const ispc_nest& n);

  const ispc_nest& n;

  // pool slices
  const uint32_t* pool(uint32_t begin) const { return n.pool + begin; }
  std::vector<uint32_t> slice(uint32_t begin, uint32_t count) const;

  const std::string& name(uint32_t obj) const { return names_.at(obj); }

  bool has_inst(uint32_t obj) const { return inst_.count(obj) != 0; }
  const ispc_inst& inst(uint32_t obj) const;
  const ispc_region& region(uint32_t obj) const;
  const ispc_dim& dim(uint32_t obj) const;
  bool is_dim(uint32_t obj) const { return dim_.count(obj) != 0; }
  const ispc_node& node(uint32_t idx) const { return n.nodes[idx]; }

  // Node that owns a dimension / holds an instruction (ISPC_NONE if absent).
  uint32_t node_of_dim(uint32_t dim_obj) const;
  uint32_t node_of_inst(uint32_t inst_obj) const;
  uint32_t parent(uint32_t node_idx) const { return parent_[node_idx]; }
  bool inst_present(uint32_t obj) const { return node_of_inst(obj) != ISPC_NONE; }

  // A comm is realized through memory when its copy-out store is in the tree
  // (the same test the reference emitter uses, loop_nest.cpp:396-397).
  bool comm_fired(uint32_t ci) const;

  // Dim nodes enclosing `node_idx` (innermost first).
  std::vector<uint32_t> ancestors(uint32_t node_idx) const;

  // Static extent of a dim (LoopNest::sizes).
  int64_t size_of(uint32_t dim_obj) const { return dim(dim_obj).size; }
  // base * prod(size(size_dims)) of an address term.
  int64_t term_mult(const ispc_addr_term& t) const;

  int64_t threads_per_block() const;
  int64_t blocks() const;

  // Pre-order list of node indices.
  const std::vector<uint32_t>& preorder() const { return preorder_; }

 private:
  std::vector<std::string> names_;
  std::unordered_map<uint32_t, const ispc_inst*> inst_;
  std::unordered_map<uint32_t, const ispc_region*> region_;
  std::unordered_map<uint32_t, const ispc_dim*> dim_;
  std::unordered_map<uint32_t, uint32_t> node_dim_, node_inst_;
  std::vector<uint32_t> parent_;
  std::vector<uint32_t> preorder_;
};

// Thread-local error text for device-less entry points.
void set_thread_error(const std::string& s);
const char* thread_error();

}  // namespace ispc
