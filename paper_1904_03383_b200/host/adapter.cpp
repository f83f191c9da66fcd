#include "adapter.hpp"

#include <deque>
#include <map>
#include <stdexcept>

namespace ispc_host {

using namespace ispace;

namespace {

uint32_t push_ids(std::vector<uint32_t>& pool, const std::vector<ObjId>& ids) {
  uint32_t b = uint32_t(pool.size());
  pool.insert(pool.end(), ids.begin(), ids.end());
  return b;
}

uint32_t push_pairs(std::vector<uint32_t>& pool, const std::vector<std::pair<ObjId, ObjId>>& pairs) {
  uint32_t b = uint32_t(pool.size());
  for (auto& [s, d] : pairs) {
    pool.push_back(s);
    pool.push_back(d);
  }
  return b;
}

uint32_t dim_kind_of(NestDimKind k) {
  switch (k) {
    case NestDimKind::Loop: return ISPC_LOOP;
    case NestDimKind::Block: return ISPC_BLOCK;
    case NestDimKind::Thread: return ISPC_THREAD;
    case NestDimKind::Unroll: return ISPC_UNROLL;
    case NestDimKind::Vector: return ISPC_VECTOR;
  }
  throw std::logic_error("unknown NestDimKind");
}

uint32_t cache_of(CacheKind k) {
  switch (k) {
    case CacheKind::L1: return ISPC_CACHE_L1;
    case CacheKind::L2: return ISPC_CACHE_L2;
    case CacheKind::ReadOnly: return ISPC_CACHE_READ_ONLY;
    case CacheKind::None: return ISPC_CACHE_NONE;
  }
  throw std::logic_error("unknown CacheKind");
}

}  // namespace

std::unique_ptr<NestBuf> flatten(const Kernel& k, const LoopNest& l) {
  auto b = std::make_unique<NestBuf>();
  b->kernel_name = k.name;
  for (const BackboneObject& o : k.bb.objects) b->names.push_back(o.name);

  // instructions present in the tree
  std::map<ObjId, bool> present;
  std::deque<const NestNode*> walk;
  for (const NestNode& r : l.roots) walk.push_back(&r);
  while (!walk.empty()) {
    const NestNode* n = walk.front();
    walk.pop_front();
    if (n->kind == NestNode::Kind::Inst) present[n->inst] = true;
    for (const NestNode& c : n->children) walk.push_back(&c);
  }

  // scalar inputs, in first-use order
  std::map<std::string, uint32_t> input_idx;
  for (const auto& [id, ii] : k.insts)
    for (const Operand& o : ii.operands)
      if (o.kind == Operand::Kind::Input && !input_idx.count(o.input)) {
        input_idx[o.input] = uint32_t(b->inputs.size());
        b->inputs.push_back(o.input);
      }

  for (const InductionVar& iv : k.ivars) {
    ispc_ivar fv{};
    fv.offset = iv.offset;
    fv.terms_begin = uint32_t(b->terms.size());
    fv.terms_count = uint32_t(iv.terms.size());
    for (const AddrTerm& t : iv.terms) {
      ispc_addr_term ft{};
      ft.dim = t.dim;
      ft.base = t.base;
      ft.size_dims_begin = push_ids(b->pool, t.size_dims);
      ft.size_dims_count = uint32_t(t.size_dims.size());
      b->terms.push_back(ft);
    }
    b->ivars.push_back(fv);
  }

  for (const auto& [id, ii] : k.insts) {
    ispc_inst fi{};
    fi.obj = id;
    fi.op = uint32_t(ii.op);  // same enumerator order (kernels.hpp:14)
    fi.region = ii.region == kNoObj ? ISPC_NONE : ii.region;
    fi.ivar = ii.ivar == kNoIndex ? ISPC_NONE : ii.ivar;
    fi.dims_begin = push_ids(b->pool, ii.dims);
    fi.dims_count = uint32_t(ii.dims.size());
    fi.live = present.count(id) ? 1u : 0u;
    auto c = l.cache.find(id);
    fi.cache = c == l.cache.end() ? uint32_t(ISPC_CACHE_L1) : cache_of(c->second);
    fi.operands_begin = uint32_t(b->operands.size());
    fi.operands_count = uint32_t(ii.operands.size());
    for (const Operand& o : ii.operands) {
      ispc_operand fo{};
      fo.kind = uint32_t(o.kind);  // same enumerator order (kernels.hpp:33)
      fo.value = o.value;
      fo.input = o.kind == Operand::Kind::Input ? input_idx.at(o.input) : ISPC_NONE;
      fo.ivar = o.ivar == kNoIndex ? ISPC_NONE : o.ivar;
      fo.producer = o.producer == kNoObj ? ISPC_NONE : o.producer;
      fo.init = o.init == kNoObj ? ISPC_NONE : o.init;
      fo.comm = o.comm == kNoIndex ? ISPC_NONE : o.comm;
      fo.pairs_begin = push_pairs(b->pool, o.pairs);
      fo.pairs_count = uint32_t(o.pairs.size());
      fo.reduce_begin = push_ids(b->pool, o.reduce_dims);
      fo.reduce_count = uint32_t(o.reduce_dims.size());
      b->operands.push_back(fo);
    }
    b->insts.push_back(fi);
  }

  for (const auto& [id, ri] : k.regions) {
    ispc_region fr{};
    fr.obj = id;
    fr.input = ri.input;
    fr.elems = ri.elems;
    fr.elem_bytes = ri.elem_bytes;
    auto ms = l.mem_space.find(id);
    fr.live = ms != l.mem_space.end();
    fr.mem_space = fr.live && ms->second == MemSpaceKind::Shared ? ISPC_SHARED : ISPC_GLOBAL;
    b->regions.push_back(fr);
  }

  for (const auto& [id, di] : k.dims) {
    ispc_dim fd{};
    fd.obj = id;
    fd.logical = di.logical;
    fd.is_static = di.is_static;
    auto s = l.sizes.find(id);
    fd.size = s == l.sizes.end() ? 0 : s->second;
    b->dims.push_back(fd);
  }

  for (const Comm& c : k.comms) {
    ispc_comm fc{};
    fc.producer = c.producer;
    fc.consumer = c.consumer;
    fc.region = c.region;
    fc.store = c.store;
    fc.load = c.load;
    fc.pairs_begin = push_pairs(b->pool, c.pairs);
    fc.pairs_count = uint32_t(c.pairs.size());
    fc.fired = present.count(c.store) ? 1u : 0u;
    b->comms.push_back(fc);
  }

  // Tree, breadth first so the children of a node are contiguous.
  std::vector<const NestNode*> order;
  b->nodes.resize(l.roots.size());
  for (const NestNode& r : l.roots) order.push_back(&r);
  for (size_t i = 0; i < order.size(); ++i) {
    const NestNode* n = order[i];
    ispc_node& f = b->nodes[i];
    f.kind = n->kind == NestNode::Kind::Dim ? ISPC_NODE_DIM
             : n->kind == NestNode::Kind::Inst ? ISPC_NODE_INST
                                               : ISPC_NODE_BARRIER;
    f.dim_kind = n->kind == NestNode::Kind::Dim ? dim_kind_of(n->dim_kind) : 0u;
    f.size = n->size;
    f.thread_level = n->thread_level;
    f.block_level = n->block_level;
    f.inst = n->inst == kNoObj ? ISPC_NONE : n->inst;
    f.dims_begin = push_ids(b->pool, n->dims);
    f.dims_count = uint32_t(n->dims.size());
    f.children_begin = uint32_t(order.size());
    f.children_count = uint32_t(n->children.size());
    for (const NestNode& c : n->children) order.push_back(&c);
    b->nodes.resize(order.size());
  }

  for (const std::string& s : b->names) b->name_ptrs.push_back(s.c_str());
  for (const std::string& s : b->inputs) b->input_ptrs.push_back(s.c_str());

  ispc_nest& n = b->nest;
  n.abi_version = ISPC_ABI_VERSION;
  n.kernel_name = b->kernel_name.c_str();
  n.num_objects = uint32_t(b->names.size());
  n.object_names = b->name_ptrs.data();
  n.num_insts = uint32_t(b->insts.size());
  n.insts = b->insts.data();
  n.num_regions = uint32_t(b->regions.size());
  n.regions = b->regions.data();
  n.num_dims = uint32_t(b->dims.size());
  n.dims = b->dims.data();
  n.num_ivars = uint32_t(b->ivars.size());
  n.ivars = b->ivars.data();
  n.num_terms = uint32_t(b->terms.size());
  n.terms = b->terms.data();
  n.num_operands = uint32_t(b->operands.size());
  n.operands = b->operands.data();
  n.num_comms = uint32_t(b->comms.size());
  n.comms = b->comms.data();
  n.num_inputs = uint32_t(b->inputs.size());
  n.input_names = b->input_ptrs.data();
  n.pool_size = uint32_t(b->pool.size());
  n.pool = b->pool.data();
  n.num_nodes = uint32_t(b->nodes.size());
  n.nodes = b->nodes.data();
  n.roots_begin = 0;
  n.roots_count = uint32_t(l.roots.size());
  if (l.thread_shape.size() > 3 || l.block_shape.size() > 3)
    throw std::invalid_argument("more than 3 hardware levels");
  n.num_thread_levels = uint32_t(l.thread_shape.size());
  n.num_block_levels = uint32_t(l.block_shape.size());
  for (size_t i = 0; i < l.thread_shape.size(); ++i) n.thread_shape[i] = l.thread_shape[i];
  for (size_t i = 0; i < l.block_shape.size(); ++i) n.block_shape[i] = l.block_shape[i];
  return b;
}

}  // namespace ispc_host
