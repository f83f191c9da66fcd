#include "nest_view.hpp"

#include <functional>

namespace ispc {

namespace {
thread_local std::string g_thread_error;
}

void set_thread_error(const std::string& s) { g_thread_error = s; }
const char* thread_error() { return g_thread_error.c_str(); }

NestView::NestView(const ispc_nest& nest) : n(nest) {
  if (n.abi_version != ISPC_ABI_VERSION)
    throw NestError(ISPC_E_ARG, "ispc_nest abi_version mismatch");
  names_.resize(n.num_objects);
  for (uint32_t i = 0; i < n.num_objects; ++i)
    names_[i] = n.object_names && n.object_names[i] ? n.object_names[i] : ("o" + std::to_string(i));
  for (uint32_t i = 0; i < n.num_insts; ++i) inst_[n.insts[i].obj] = &n.insts[i];
  for (uint32_t i = 0; i < n.num_regions; ++i) region_[n.regions[i].obj] = &n.regions[i];
  for (uint32_t i = 0; i < n.num_dims; ++i) dim_[n.dims[i].obj] = &n.dims[i];

  auto check_slice = [&](uint32_t b, uint32_t c, uint32_t lim, const char* what) {
    if (uint64_t(b) + c > lim) throw NestError(ISPC_E_ARG, std::string("slice out of range: ") + what);
  };
  check_slice(n.roots_begin, n.roots_count, n.num_nodes, "roots");
  parent_.assign(n.num_nodes, ISPC_NONE);
  std::vector<uint8_t> seen(n.num_nodes, 0);
  std::function<void(uint32_t, uint32_t)> walk = [&](uint32_t idx, uint32_t par) {
    if (seen[idx]) throw NestError(ISPC_E_ARG, "node visited twice: not a forest");
    seen[idx] = 1;
    parent_[idx] = par;
    preorder_.push_back(idx);
    const ispc_node& nd = n.nodes[idx];
    check_slice(nd.children_begin, nd.children_count, n.num_nodes, "children");
    if (nd.kind == ISPC_NODE_DIM) {
      check_slice(nd.dims_begin, nd.dims_count, n.pool_size, "node dims");
      for (uint32_t j = 0; j < nd.dims_count; ++j) node_dim_[n.pool[nd.dims_begin + j]] = idx;
    } else if (nd.kind == ISPC_NODE_INST) {
      if (!inst_.count(nd.inst)) throw NestError(ISPC_E_ARG, "node names an unknown instruction");
      node_inst_[nd.inst] = idx;
    }
    for (uint32_t j = 0; j < nd.children_count; ++j) walk(nd.children_begin + j, idx);
  };
  for (uint32_t r = 0; r < n.roots_count; ++r) walk(n.roots_begin + r, ISPC_NONE);
  if (n.num_thread_levels > 3 || n.num_block_levels > 3)
    throw NestError(ISPC_E_ARG, "more than 3 thread or block levels");
}

std::vector<uint32_t> NestView::slice(uint32_t begin, uint32_t count) const {
  if (uint64_t(begin) + count > n.pool_size) throw NestError(ISPC_E_ARG, "pool slice out of range");
  return std::vector<uint32_t>(n.pool + begin, n.pool + begin + count);
}

const ispc_inst& NestView::inst(uint32_t obj) const {
  auto it = inst_.find(obj);
  if (it == inst_.end()) throw NestError(ISPC_E_ARG, "unknown instruction " + std::to_string(obj));
  return *it->second;
}
const ispc_region& NestView::region(uint32_t obj) const {
  auto it = region_.find(obj);
  if (it == region_.end()) throw NestError(ISPC_E_ARG, "unknown region " + std::to_string(obj));
  return *it->second;
}
const ispc_dim& NestView::dim(uint32_t obj) const {
  auto it = dim_.find(obj);
  if (it == dim_.end()) throw NestError(ISPC_E_ARG, "unknown dimension " + std::to_string(obj));
  return *it->second;
}
uint32_t NestView::node_of_dim(uint32_t d) const {
  auto it = node_dim_.find(d);
  return it == node_dim_.end() ? ISPC_NONE : it->second;
}
uint32_t NestView::node_of_inst(uint32_t i) const {
  auto it = node_inst_.find(i);
  return it == node_inst_.end() ? ISPC_NONE : it->second;
}
bool NestView::comm_fired(uint32_t ci) const {
  if (ci >= n.num_comms) throw NestError(ISPC_E_ARG, "comm index out of range");
  return inst_present(n.comms[ci].store);
}
std::vector<uint32_t> NestView::ancestors(uint32_t idx) const {
  std::vector<uint32_t> out;
  for (uint32_t p = parent_[idx]; p != ISPC_NONE; p = parent_[p]) out.push_back(p);
  return out;
}
int64_t NestView::term_mult(const ispc_addr_term& t) const {
  int64_t m = t.base;
  for (uint32_t j = 0; j < t.size_dims_count; ++j) m *= size_of(n.pool[t.size_dims_begin + j]);
  return m;
}
int64_t NestView::threads_per_block() const {
  int64_t t = 1;
  for (uint32_t i = 0; i < n.num_thread_levels; ++i) t *= n.thread_shape[i];
  return t;
}
int64_t NestView::blocks() const {
  int64_t b = 1;
  for (uint32_t i = 0; i < n.num_block_levels; ++i) b *= n.block_shape[i];
  return b;
}

}  // namespace ispc
