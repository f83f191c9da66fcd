// sm_100a CUDA emitter: one fully specified schedule -> one __global__ kernel.
//
// Replaces the reference's pseudo-source emitter (proj/core/src/loop_nest.cpp:
// 389-609) with real device code. Decision -> CUDA mapping:
//   BLOCK dims   linearized blockIdx.x, decomposed by mixed radix (no 65535 cap)
//   THREAD dims  level L of thread_shape; the innermost level is threadIdx.x
//   LOOP         `#pragma unroll 1` for loop (the candidate chose not to unroll)
//   UNROLL       fully unrolled loop; values crossing unrolled nests live in
//                register arrays indexed by compile-time lane constants
//   VECTOR       lanes; memory ops become 64/128-bit ld/st when the lane stride
//                is 1 and every other address term keeps the lane group aligned
//   mem_space    SHARED temporaries in (dynamic) shared memory, GLOBAL ones in
//                scratch buffers passed as kernel parameters
//   cache        L1 -> ld.global.ca / st.global.wb, L2 -> .cg, READ_ONLY -> .nc,
//                NONE -> .cs (evict-first streaming, B200's nearest "uncached")
//   barriers     the reference's barrier nodes (loop_nest.cpp:93-107) plus the
//                ones a real machine needs: before any sibling that reads a
//                temporary written by threads of an earlier sibling
// Arithmetic mirrors the backbone's separate instructions with round-to-
// nearest intrinsics (mul -> __fmul_rn, add -> __fadd_rn, mad -> __fmaf_rn),
// so every parity-mode schedule is bit-identical to the sequential oracle.
//
// Static legality (ISPC_E_ILLEGAL) covers what the reference's simulator does
// not model: a value crossing blocks through a temporary (needs a grid-wide
// barrier), register arrays and unrolled bodies beyond B200 per-thread budgets,
// grid/thread limits and addresses outside their region.
#include <algorithm>
#include <cstring>
#include <map>
#include <set>
#include <sstream>

#include "nest_view.hpp"

namespace ispc {
namespace {

uint64_t fnv1a(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) h = (h ^ c) * 1099511628211ull;
  return h;
}

std::string sanitize(const std::string& s) {
  std::string o;
  for (char c : s) o += (isalnum(static_cast<unsigned char>(c)) || c == '_') ? c : '_';
  return o;
}

// A compile-time constant or a variable name.
struct Idx {
  bool is_const = true;
  int64_t c = 0;
  std::string var;
};

class CudaEmitter {
 public:
  CudaEmitter(const NestView& v, const ispc_emit_opts& o, std::string fn)
      : v_(v), opts_(o), fn_(std::move(fn)) {}

  std::string run(ispc_launch& L) {
    analyze_nodes();
    analyze_values();
    check_legality();
    plan_barriers();
    std::string body = emit_body();
    std::string head = emit_head(L);
    std::string src = head + body + "}\n";
    L.source_hash = fnv1a(src);
    return src;
  }

 private:
  const NestView& v_;
  const ispc_emit_opts& opts_;
  std::string fn_;

  // --- node analysis -------------------------------------------------------
  std::map<uint32_t, std::string> var_;          // dim node -> variable name
  std::map<uint32_t, int> thread_axis_;          // thread level -> 0:x 1:y 2:z
  bool has_barrier_ = false;
  int64_t unrolled_insts_ = 0;

  void analyze_nodes() {
    const ispc_nest& n = v_.n;
    int loops = 0, unrolls = 0, vecs = 0;
    for (uint32_t idx : v_.preorder()) {
      const ispc_node& nd = v_.node(idx);
      if (nd.kind == ISPC_NODE_BARRIER) has_barrier_ = true;
      if (nd.kind != ISPC_NODE_DIM) continue;
      if (nd.size < 1) throw NestError(ISPC_E_ARG, "dimension of size < 1");
      switch (nd.dim_kind) {
        case ISPC_BLOCK:
          if (nd.block_level < 0 || uint32_t(nd.block_level) >= n.num_block_levels)
            throw NestError(ISPC_E_ARG, "block node without a grid level");
          var_[idx] = "b" + std::to_string(nd.block_level);
          break;
        case ISPC_THREAD:
          if (nd.thread_level < 0 || uint32_t(nd.thread_level) >= n.num_thread_levels)
            throw NestError(ISPC_E_ARG, "thread node without a hardware level");
          if (nd.size != n.thread_shape[nd.thread_level])
            throw NestError(ISPC_E_ARG, "thread node size differs from its level");
          var_[idx] = "t" + std::to_string(nd.thread_level);
          break;
        case ISPC_LOOP: var_[idx] = "i" + std::to_string(loops++); break;
        case ISPC_UNROLL: var_[idx] = "u" + std::to_string(unrolls++); break;
        case ISPC_VECTOR: var_[idx] = "v" + std::to_string(vecs++); break;
        default: throw NestError(ISPC_E_ARG, "bad dim kind");
      }
    }
    for (uint32_t l = 0; l < n.num_thread_levels; ++l)
      thread_axis_[int(l)] = int(n.num_thread_levels - 1 - l);
    // unrolled instruction count: every instruction replicated by its
    // enclosing UNROLL / VECTOR extents
    for (uint32_t idx : v_.preorder()) {
      const ispc_node& nd = v_.node(idx);
      if (nd.kind != ISPC_NODE_INST) continue;
      int64_t r = 1;
      for (uint32_t a : v_.ancestors(idx)) {
        const ispc_node& an = v_.node(a);
        if (an.dim_kind == ISPC_UNROLL || an.dim_kind == ISPC_VECTOR) r *= an.size;
      }
      unrolled_insts_ += r;
    }
  }

  // --- value storage ---------------------------------------------------------
  // Each value-defining instruction writes a register storage owned by a root
  // instruction: itself, or for a reduction the initializer / the fired
  // copy-in that seeds the accumulator (the reference's reg(), loop_nest.cpp:
  // 418-432). A storage is an array over the root's UNROLL/VECTOR dims (lanes
  // of unrolled nests that hand values to other unrolled nests); every access
  // names, per axis, which of the accessing instruction's own dims selects it.
  struct Storage {
    std::string name;
    std::vector<int64_t> sizes;
    int64_t elems() const {
      int64_t e = 1;
      for (int64_t s : sizes) e *= s;
      return e;
    }
  };
  struct Value {
    uint32_t root = ISPC_NONE;
    std::vector<uint32_t> axis_dims;  // dims of the defining instruction
  };
  std::map<uint32_t, Storage> storage_;  // root inst -> storage
  std::map<uint32_t, Value> value_;      // defining inst -> value
  std::set<uint32_t> loaded_regions_, stored_regions_;

  std::vector<uint32_t> inst_dims(uint32_t inst) const {
    const ispc_inst& ii = v_.inst(inst);
    return v_.slice(ii.dims_begin, ii.dims_count);
  }

  const ispc_operand& operand(uint32_t inst, uint32_t j) const {
    const ispc_inst& ii = v_.inst(inst);
    return v_.n.operands[ii.operands_begin + j];
  }

  const ispc_operand* reduce_operand(uint32_t inst) const {
    const ispc_inst& ii = v_.inst(inst);
    for (uint32_t j = 0; j < ii.operands_count; ++j)
      if (v_.n.operands[ii.operands_begin + j].kind == ISPC_OPND_REDUCE)
        return &v_.n.operands[ii.operands_begin + j];
    return nullptr;
  }

  std::map<uint32_t, uint32_t> pair_map(const ispc_operand& o) const {
    std::map<uint32_t, uint32_t> m;
    for (uint32_t j = 0; j < o.pairs_count; ++j)
      m[v_.n.pool[o.pairs_begin + 2 * j]] = v_.n.pool[o.pairs_begin + 2 * j + 1];
    return m;
  }

  bool fired(const ispc_operand& o) const { return o.comm != ISPC_NONE && v_.comm_fired(o.comm); }

  const Value& value_of(uint32_t inst) {
    auto it = value_.find(inst);
    if (it != value_.end()) return it->second;
    if (!v_.inst_present(inst))
      throw NestError(ISPC_E_ARG, "value of an instruction missing from the nest: " + v_.name(inst));
    Value val;
    if (const ispc_operand* r = reduce_operand(inst)) {
      uint32_t src = fired(*r) ? v_.n.comms[r->comm].load : r->init;
      const Value& sv = value_of(src);
      val.root = sv.root;
      if (fired(*r)) {
        val.axis_dims = sv.axis_dims;  // the copy-in iterates our own dims
      } else {
        auto pm = pair_map(*r);
        for (uint32_t d : sv.axis_dims) {
          auto p = pm.find(d);
          if (p == pm.end())
            throw NestError(ISPC_E_ILLEGAL, "accumulator lane not paired: " + v_.name(d));
          val.axis_dims.push_back(p->second);
        }
      }
    } else {
      Storage st;
      st.name = "r_" + sanitize(v_.name(inst));
      std::vector<uint32_t> lanes, vec;
      for (uint32_t d : inst_dims(inst)) {
        uint32_t nd = v_.node_of_dim(d);
        if (nd == ISPC_NONE) throw NestError(ISPC_E_ARG, "dimension missing from the nest");
        uint32_t k = v_.node(nd).dim_kind;
        if (k == ISPC_UNROLL) lanes.push_back(d);
        if (k == ISPC_VECTOR) vec.push_back(d);
      }
      lanes.insert(lanes.end(), vec.begin(), vec.end());  // vector lanes innermost
      for (uint32_t d : lanes) st.sizes.push_back(v_.node(v_.node_of_dim(d)).size);
      val.root = inst;
      val.axis_dims = lanes;
      storage_[inst] = st;
    }
    return value_[inst] = val;
  }

  void analyze_values() {
    for (uint32_t idx : v_.preorder()) {
      const ispc_node& nd = v_.node(idx);
      if (nd.kind != ISPC_NODE_INST) continue;
      const ispc_inst& ii = v_.inst(nd.inst);
      if (ii.op == ISPC_OP_LOAD) loaded_regions_.insert(ii.region);
      if (ii.op == ISPC_OP_STORE) stored_regions_.insert(ii.region);
      if (ii.op != ISPC_OP_STORE) value_of(nd.inst);
    }
  }

  // --- legality ----------------------------------------------------------------
  int64_t reg_elems() const {
    int64_t e = 0;
    for (auto& [r, st] : storage_) e += st.elems();
    return e;
  }

  void check_legality() {
    const ispc_nest& n = v_.n;
    int64_t threads = v_.threads_per_block();
    if (threads > 1024) throw NestError(ISPC_E_ILLEGAL, "more than 1024 threads per block");
    // the outermost of three thread levels is threadIdx.z, which the hardware
    // caps at 64 (the launch fails with CUDA_ERROR_INVALID_VALUE otherwise)
    if (n.num_thread_levels == 3 && n.thread_shape[0] > 64)
      throw NestError(ISPC_E_ILLEGAL, "threadIdx.z level of " + std::to_string(n.thread_shape[0]) + " threads (max 64)");
    if (v_.blocks() > 0x7fffffffLL) throw NestError(ISPC_E_ILLEGAL, "grid exceeds 2^31-1 blocks");
    uint32_t max_regs = opts_.max_reg_elems ? opts_.max_reg_elems : 512;
    uint32_t max_unr = opts_.max_unrolled ? opts_.max_unrolled : 16384;
    if (reg_elems() > max_regs)
      throw NestError(ISPC_E_ILLEGAL, "register arrays need " + std::to_string(reg_elems()) +
                                          " floats per thread (budget " + std::to_string(max_regs) + ")");
    if (unrolled_insts_ > max_unr)
      throw NestError(ISPC_E_ILLEGAL, "unrolled body of " + std::to_string(unrolled_insts_) +
                                          " instructions (budget " + std::to_string(max_unr) + ")");
    // A value that crosses blocks through a temporary would need a grid-wide
    // barrier: block dims of both sides must be the same fused node.
    for (uint32_t ci = 0; ci < n.num_comms; ++ci) {
      if (!v_.comm_fired(ci)) continue;
      const ispc_comm& c = n.comms[ci];
      for (uint32_t j = 0; j < c.pairs_count; ++j) {
        uint32_t p = n.pool[c.pairs_begin + 2 * j], q = n.pool[c.pairs_begin + 2 * j + 1];
        uint32_t np = v_.node_of_dim(p), nq = v_.node_of_dim(q);
        bool bp = v_.node(np).dim_kind == ISPC_BLOCK, bq = v_.node(nq).dim_kind == ISPC_BLOCK;
        if ((bp || bq) && np != nq)
          throw NestError(ISPC_E_ILLEGAL, "value crosses blocks through " + v_.name(c.region) + " (" +
                                              v_.name(p) + " -> " + v_.name(q) + ")");
      }
    }
    // every address stays inside its region
    for (uint32_t idx : v_.preorder()) {
      const ispc_node& nd = v_.node(idx);
      if (nd.kind != ISPC_NODE_INST) continue;
      const ispc_inst& ii = v_.inst(nd.inst);
      if (ii.op != ISPC_OP_LOAD && ii.op != ISPC_OP_STORE) continue;
      const ispc_ivar& iv = n.ivars[ii.ivar];
      int64_t lo = iv.offset, hi = iv.offset;
      for (uint32_t t = 0; t < iv.terms_count; ++t) {
        const ispc_addr_term& term = n.terms[iv.terms_begin + t];
        int64_t m = v_.term_mult(term) * (v_.size_of(term.dim) - 1);
        (m < 0 ? lo : hi) += m;
      }
      const ispc_region& r = v_.region(ii.region);
      if (lo < 0 || hi >= r.elems)
        throw NestError(ISPC_E_ILLEGAL, "address of " + v_.name(nd.inst) + " leaves " + v_.name(ii.region));
      if (hi > max_addr_) max_addr_ = hi;
    }
  }
  int64_t max_addr_ = 0;

  // --- barriers -------------------------------------------------------------------
  // Regions stored / loaded in a subtree, and whether a store sits under a
  // THREAD node (then different threads write different entries).
  struct Access {
    std::set<uint32_t> loads, stores_threaded, stores;
  };
  std::map<uint32_t, Access> acc_;
  std::map<uint32_t, std::vector<bool>> barrier_before_;  // parent -> per child

  Access collect(uint32_t idx, bool under_thread) {
    const ispc_node& nd = v_.node(idx);
    Access a;
    if (nd.kind == ISPC_NODE_INST) {
      const ispc_inst& ii = v_.inst(nd.inst);
      if (ii.op == ISPC_OP_LOAD && !v_.region(ii.region).input) a.loads.insert(ii.region);
      if (ii.op == ISPC_OP_STORE && !v_.region(ii.region).input) {
        a.stores.insert(ii.region);
        if (under_thread) a.stores_threaded.insert(ii.region);
      }
    } else if (nd.kind == ISPC_NODE_DIM) {
      bool th = under_thread || nd.dim_kind == ISPC_THREAD;
      for (uint32_t j = 0; j < nd.children_count; ++j) {
        Access c = collect(nd.children_begin + j, th);
        a.loads.insert(c.loads.begin(), c.loads.end());
        a.stores.insert(c.stores.begin(), c.stores.end());
        a.stores_threaded.insert(c.stores_threaded.begin(), c.stores_threaded.end());
      }
    }
    return acc_[idx] = a;
  }

  void plan_children(uint32_t parent, uint32_t begin, uint32_t count) {
    std::vector<bool> before(count, false);
    std::set<uint32_t> pending;  // threaded stores since the last barrier
    for (uint32_t j = 0; j < count; ++j) {
      uint32_t c = begin + j;
      if (v_.node(c).kind == ISPC_NODE_BARRIER) {
        pending.clear();
        continue;
      }
      const Access& a = acc_[c];
      bool need = false;
      for (uint32_t r : a.loads)
        if (pending.count(r)) need = true;
      if (need) {
        before[j] = true;
        pending.clear();
      }
      pending.insert(a.stores_threaded.begin(), a.stores_threaded.end());
      const ispc_node& nd = v_.node(c);
      if (nd.kind == ISPC_NODE_DIM) plan_children(c, nd.children_begin, nd.children_count);
    }
    barrier_before_[parent] = before;
  }

  bool any_barrier() const {
    if (has_barrier_) return true;
    for (auto& [p, v] : barrier_before_)
      for (bool b : v)
        if (b) return true;
    return false;
  }

  void plan_barriers() {
    const ispc_nest& n = v_.n;
    for (uint32_t r = 0; r < n.roots_count; ++r) collect(n.roots_begin + r, false);
    if (v_.threads_per_block() > 1) plan_children(ISPC_NONE, n.roots_begin, n.roots_count);
  }

  // --- expressions ----------------------------------------------------------------
  std::map<uint32_t, Idx> env_;  // dim node -> index value in scope
  bool wide_addr() const { return max_addr_ >= 0x7fffffffLL; }

  Idx idx_of_dim(uint32_t d) const {
    uint32_t nd = v_.node_of_dim(d);
    auto it = env_.find(nd);
    if (it == env_.end())
      throw NestError(ISPC_E_ILLEGAL, "dimension " + v_.name(d) + " used outside its loop");
    return it->second;
  }

  // Affine address text; `lane_node`'s coefficient is reported separately.
  std::string addr(uint32_t ivar) const {
    const ispc_ivar& iv = v_.n.ivars[ivar];
    int64_t c = iv.offset;
    std::map<std::string, int64_t> coef;
    std::vector<std::string> order;
    for (uint32_t t = 0; t < iv.terms_count; ++t) {
      const ispc_addr_term& term = v_.n.terms[iv.terms_begin + t];
      int64_t m = v_.term_mult(term);
      Idx x = idx_of_dim(term.dim);
      if (x.is_const) {
        c += x.c * m;
        continue;
      }
      if (!coef.count(x.var)) order.push_back(x.var);
      coef[x.var] += m;
    }
    std::string s;
    for (const std::string& var : order) {
      int64_t m = coef[var];
      if (m == 0) continue;
      std::string t = wide_addr() ? "(long long)" + var : var;
      if (m != 1) t += "*" + std::to_string(m) + (wide_addr() ? "LL" : "");
      s += (s.empty() ? "" : " + ") + t;
    }
    if (s.empty()) return std::to_string(c) + (wide_addr() ? "LL" : "");
    if (c != 0) s += " + " + std::to_string(c) + (wide_addr() ? "LL" : "");
    return s;
  }

  // coefficient of node `nd` in an address, and whether every other term
  // (and the offset) is a multiple of `w`
  void lane_stride(uint32_t ivar, uint32_t nd, int64_t w, int64_t& stride, bool& aligned) const {
    const ispc_ivar& iv = v_.n.ivars[ivar];
    std::map<uint32_t, int64_t> per_node;
    int64_t c = iv.offset;
    for (uint32_t t = 0; t < iv.terms_count; ++t) {
      const ispc_addr_term& term = v_.n.terms[iv.terms_begin + t];
      uint32_t tn = v_.node_of_dim(term.dim);
      int64_t m = v_.term_mult(term);
      auto e = env_.find(tn);
      if (tn != nd && e != env_.end() && e->second.is_const) c += e->second.c * m;
      else per_node[tn] += m;
    }
    stride = per_node.count(nd) ? per_node[nd] : 0;
    aligned = c % w == 0;
    for (auto& [k, m] : per_node)
      if (k != nd && m % w != 0) aligned = false;
  }

  std::string storage_ref(uint32_t root, const std::vector<uint32_t>& dims_of_reader) const {
    const Storage& st = storage_.at(root);
    if (st.sizes.empty()) return st.name;
    int64_t cidx = 0, stride = 1;
    std::vector<std::string> parts;
    for (size_t a = st.sizes.size(); a-- > 0;) {
      Idx x = idx_of_dim(dims_of_reader[a]);
      if (x.is_const) cidx += x.c * stride;
      else parts.push_back(stride == 1 ? x.var : x.var + "*" + std::to_string(stride));
      stride *= st.sizes[a];
    }
    std::string s;
    for (auto it = parts.rbegin(); it != parts.rend(); ++it) s += (s.empty() ? "" : " + ") + *it;
    if (s.empty()) s = std::to_string(cidx);
    else if (cidx) s += " + " + std::to_string(cidx);
    return st.name + "[" + s + "]";
  }

  // The register an instruction defines (or accumulates into).
  std::string def_ref(uint32_t inst) {
    const Value& val = value_of(inst);
    return storage_ref(val.root, val.axis_dims);
  }

  // Value of `producer` as seen by `reader` through an operand.
  std::string use_ref(uint32_t producer, const ispc_operand* via) {
    const Value& val = value_of(producer);
    std::vector<uint32_t> dims = val.axis_dims;
    if (via && via->kind == ISPC_OPND_MAPPED && !fired(*via)) {
      auto pm = pair_map(*via);
      for (uint32_t& d : dims) {
        auto p = pm.find(d);
        if (p == pm.end())
          throw NestError(ISPC_E_ILLEGAL, "register lane " + v_.name(d) + " not paired with the reader");
        d = p->second;
      }
    }
    return storage_ref(val.root, dims);
  }

  std::string operand_text(uint32_t self, const ispc_operand& o) {
    switch (o.kind) {
      case ISPC_OPND_CONST: return "(float)" + std::to_string(o.value);
      case ISPC_OPND_INPUT: return "p_" + sanitize(v_.n.input_names[o.input]);
      case ISPC_OPND_INDVAR: return "(float)(" + addr(o.ivar) + ")";
      case ISPC_OPND_PRODUCED: return use_ref(o.producer, &o);
      case ISPC_OPND_MAPPED:
        if (fired(o)) return use_ref(v_.n.comms[o.comm].load, nullptr);
        return use_ref(o.producer, &o);
      case ISPC_OPND_REDUCE: return def_ref(self);
    }
    throw NestError(ISPC_E_ARG, "bad operand kind");
  }

  std::string region_ptr(uint32_t region) const {
    const ispc_region& r = v_.region(region);
    if (r.elem_bytes != 4) throw NestError(ISPC_E_ILLEGAL, "only 4-byte elements are supported");
    return (r.mem_space == ISPC_SHARED ? "s_" : "g_") + sanitize(v_.name(region));
  }

  // cache path of a memory instruction; READ_ONLY (ld.global.nc) is only
  // coherent for data the kernel never writes, so in-kernel temporaries take
  // the L1 path instead
  uint32_t cache_of(const ispc_inst& ii) const {
    if (ii.cache == ISPC_CACHE_READ_ONLY && !v_.region(ii.region).input) return ISPC_CACHE_L1;
    return ii.cache;
  }

  std::string load_expr(const ispc_inst& ii, const std::string& ptr, int width) const {
    std::string ty = width == 4 ? "float4" : width == 2 ? "float2" : "float";
    std::string p = width > 1 ? "(const " + ty + "*)(" + ptr + ")" : ptr;
    if (v_.region(ii.region).mem_space == ISPC_SHARED) return "*" + (width > 1 ? p : "(" + ptr + ")");
    switch (cache_of(ii)) {
      case ISPC_CACHE_L1: return "__ldca(" + p + ")";
      case ISPC_CACHE_L2: return "__ldcg(" + p + ")";
      case ISPC_CACHE_READ_ONLY: return "__ldg(" + p + ")";
      default: return "__ldcs(" + p + ")";
    }
  }

  std::string store_stmt(const ispc_inst& ii, const std::string& ptr, int width, const std::string& val) const {
    std::string ty = width == 4 ? "float4" : width == 2 ? "float2" : "float";
    std::string p = width > 1 ? "(" + ty + "*)(" + ptr + ")" : ptr;
    if (v_.region(ii.region).mem_space == ISPC_SHARED) return "*" + (width > 1 ? p : "(" + ptr + ")") + " = " + val + ";";
    switch (cache_of(ii)) {
      case ISPC_CACHE_L2: return "__stcg(" + p + ", " + val + ");";
      case ISPC_CACHE_NONE: return "__stcs(" + p + ", " + val + ");";
      default: return "__stwb(" + p + ", " + val + ");";
    }
  }

  // --- statements -------------------------------------------------------------------
  std::ostringstream os_;
  int depth_ = 1;
  // instructions between deadline polls: a serial loop of dependent global
  // accesses runs ~1 us per instruction, so 4096 overshot the budget by
  // milliseconds (r2: timeouts measured 0.4-8.7 ms against a 0.35 ms budget);
  // 128 keeps the overshoot near 0.1 ms, and the poll (a %globaltimer read and
  // a compare every 128 instructions) is noise next to the loop's own work
  static constexpr int64_t kPollWork = 128;
  bool watchdog_ = false;

  void put(const std::string& s) { os_ << std::string(2 * depth_, ' ') << s << "\n"; }

  void emit_scalar_inst(uint32_t inst) {
    const ispc_inst& ii = v_.inst(inst);
    switch (ii.op) {
      case ISPC_OP_LOAD:
        put(def_ref(inst) + " = " + load_expr(ii, region_ptr(ii.region) + " + (" + addr(ii.ivar) + ")", 1) + ";");
        return;
      case ISPC_OP_STORE:
        put(store_stmt(ii, region_ptr(ii.region) + " + (" + addr(ii.ivar) + ")", 1,
                       operand_text(inst, operand(inst, 0))));
        return;
      case ISPC_OP_CAST: put(def_ref(inst) + " = " + operand_text(inst, operand(inst, 0)) + ";"); return;
      case ISPC_OP_ADD:
        put(def_ref(inst) + " = __fadd_rn(" + operand_text(inst, operand(inst, 0)) + ", " +
            operand_text(inst, operand(inst, 1)) + ");");
        return;
      case ISPC_OP_MUL:
        put(def_ref(inst) + " = __fmul_rn(" + operand_text(inst, operand(inst, 0)) + ", " +
            operand_text(inst, operand(inst, 1)) + ");");
        return;
      case ISPC_OP_MAD:
        put(def_ref(inst) + " = __fmaf_rn(" + operand_text(inst, operand(inst, 0)) + ", " +
            operand_text(inst, operand(inst, 1)) + ", " + operand_text(inst, operand(inst, 2)) + ");");
        return;
    }
    throw NestError(ISPC_E_ARG, "bad op");
  }

  void emit_vector(uint32_t idx) {
    const ispc_node& nd = v_.node(idx);
    int64_t w = nd.size;
    put("{  // vector " + var_[idx] + " x" + std::to_string(w));
    ++depth_;
    for (uint32_t j = 0; j < nd.children_count; ++j) {
      const ispc_node& ch = v_.node(nd.children_begin + j);
      if (ch.kind != ISPC_NODE_INST) throw NestError(ISPC_E_ARG, "vector dims hold instructions only");
      const ispc_inst& ii = v_.inst(ch.inst);
      bool mem = ii.op == ISPC_OP_LOAD || ii.op == ISPC_OP_STORE;
      bool wide = false;
      if (mem && (w == 2 || w == 4)) {
        env_[idx] = Idx{true, 0, ""};
        int64_t stride;
        bool aligned;
        lane_stride(ii.ivar, idx, w, stride, aligned);
        wide = stride == 1 && aligned;
      }
      if (wide) {
        env_[idx] = Idx{true, 0, ""};
        std::string ptr = region_ptr(ii.region) + " + (" + addr(ii.ivar) + ")";
        static const char* comp[] = {".x", ".y", ".z", ".w"};
        if (ii.op == ISPC_OP_LOAD) {
          std::string q = "q_" + std::to_string(qctr_++);
          put(std::string(w == 4 ? "float4 " : "float2 ") + q + " = " + load_expr(ii, ptr, int(w)) + ";");
          for (int64_t l = 0; l < w; ++l) {
            env_[idx] = Idx{true, l, ""};
            put(def_ref(ch.inst) + " = " + q + comp[l] + ";");
          }
        } else {
          std::string vals;
          for (int64_t l = 0; l < w; ++l) {
            env_[idx] = Idx{true, l, ""};
            vals += (l ? ", " : "") + operand_text(ch.inst, operand(ch.inst, 0));
          }
          env_[idx] = Idx{true, 0, ""};
          put(store_stmt(ii, ptr, int(w), std::string(w == 4 ? "make_float4(" : "make_float2(") + vals + ")"));
        }
      } else {
        for (int64_t l = 0; l < w; ++l) {
          env_[idx] = Idx{true, l, ""};
          emit_scalar_inst(ch.inst);
        }
      }
    }
    env_.erase(idx);
    --depth_;
    put("}");
  }
  int qctr_ = 0;

  void emit_children(uint32_t parent, uint32_t begin, uint32_t count) {
    auto it = barrier_before_.find(parent);
    for (uint32_t j = 0; j < count; ++j) {
      if (it != barrier_before_.end() && it->second[j]) put("__syncthreads();  // temporary hand-off");
      emit_node(begin + j);
    }
  }

  // Sequential instruction count of one thread through a subtree (LOOP,
  // UNROLL and VECTOR multiply; BLOCK / THREAD run in parallel).
  int64_t work(uint32_t idx) const {
    const ispc_node& nd = v_.node(idx);
    if (nd.kind == ISPC_NODE_INST) return 1;
    if (nd.kind != ISPC_NODE_DIM) return 0;
    int64_t w = 0;
    for (uint32_t j = 0; j < nd.children_count; ++j) w += work(nd.children_begin + j);
    if (nd.dim_kind == ISPC_BLOCK || nd.dim_kind == ISPC_THREAD) return w;
    return std::min<int64_t>(w * nd.size, int64_t(1) << 50);
  }

  // Every LOOP whose total work exceeds kPollWork polls the deadline about
  // once per kPollWork instructions of its body, so no thread runs more than
  // ~kPollWork instructions between two polls at any depth. Loop bounds are
  // uniform across the block, so the polls (and their __syncthreads_or) are
  // reached by every thread the same number of times.
  void watchdog_poll(uint32_t idx, const std::string& var) {
    if (!watchdog_) return;
    const ispc_node& nd = v_.node(idx);
    int64_t body = std::max<int64_t>(1, work(idx) / nd.size);
    if (body * nd.size < kPollWork) return;
    int64_t every = 1;
    while (every * body < kPollWork) every <<= 1;
    put(every == 1 ? std::string("{") : "if ((" + var + " & " + std::to_string(every - 1) + ") == 0) {");
    ++depth_;
    put("bool ispc_late = ispc_now() > ispc_deadline;");
    if (any_barrier()) put("ispc_late = __syncthreads_or(ispc_late);");
    put("if (ispc_late) { ispc_timeout_flag = 1; return; }");
    --depth_;
    put("}");
  }

  void emit_node(uint32_t idx) {
    const ispc_node& nd = v_.node(idx);
    if (nd.kind == ISPC_NODE_BARRIER) return put("__syncthreads();");
    if (nd.kind == ISPC_NODE_INST) return emit_scalar_inst(nd.inst);
    const std::string& var = var_[idx];
    std::string sz = std::to_string(nd.size);
    switch (nd.dim_kind) {
      case ISPC_BLOCK:
      case ISPC_THREAD:
        env_[idx] = Idx{false, 0, var};
        emit_children(idx, nd.children_begin, nd.children_count);
        env_.erase(idx);
        return;
      case ISPC_LOOP:
        put("#pragma unroll 1");
        put("for (int " + var + " = 0; " + var + " < " + sz + "; ++" + var + ") {");
        ++depth_;
        watchdog_poll(idx, var);
        env_[idx] = Idx{false, 0, var};
        emit_children(idx, nd.children_begin, nd.children_count);
        env_.erase(idx);
        --depth_;
        put("}");
        return;
      case ISPC_UNROLL:
        put("#pragma unroll");
        put("for (int " + var + " = 0; " + var + " < " + sz + "; ++" + var + ") {");
        ++depth_;
        env_[idx] = Idx{false, 0, var};
        emit_children(idx, nd.children_begin, nd.children_count);
        env_.erase(idx);
        --depth_;
        put("}");
        return;
      case ISPC_VECTOR: return emit_vector(idx);
    }
  }

  int64_t loop_work() const {
    // largest sequential trip product of any instruction (LOOP ancestors)
    int64_t best = 0;
    for (uint32_t idx : v_.preorder()) {
      if (v_.node(idx).kind != ISPC_NODE_INST) continue;
      int64_t t = 1;
      for (uint32_t a : v_.ancestors(idx)) {
        const ispc_node& an = v_.node(a);
        if (an.dim_kind == ISPC_LOOP || an.dim_kind == ISPC_UNROLL) t *= an.size;
      }
      best = std::max(best, t);
    }
    return best;
  }

  std::string emit_body() {
    watchdog_ = opts_.watchdog == 1 || (opts_.watchdog == 2 && loop_work() >= 4096);
    const ispc_nest& n = v_.n;
    emit_children(ISPC_NONE, n.roots_begin, n.roots_count);
    return os_.str();
  }

  std::string emit_head(ispc_launch& L) {
    const ispc_nest& n = v_.n;
    std::ostringstream h;
    std::memset(&L, 0, sizeof(L));
    std::snprintf(L.name, sizeof(L.name), "%s", fn_.c_str());
    L.grid_x = uint64_t(v_.blocks());
    uint32_t blk[3] = {1, 1, 1};
    for (uint32_t l = 0; l < n.num_thread_levels; ++l) blk[thread_axis_[int(l)]] = uint32_t(n.thread_shape[l]);
    std::memcpy(L.block, blk, sizeof(blk));
    L.watchdog = watchdog_;
    L.reg_elems = uint32_t(reg_elems());

    // parameters: input regions, GLOBAL temporaries, scalar inputs, deadline
    std::vector<const ispc_region*> params;
    for (uint32_t i = 0; i < n.num_regions; ++i) {
      const ispc_region& r = n.regions[i];
      if (!r.live || !(loaded_regions_.count(r.obj) || stored_regions_.count(r.obj))) continue;
      if (r.mem_space == ISPC_SHARED) continue;
      params.push_back(&r);
    }
    std::stable_sort(params.begin(), params.end(), [](const ispc_region* a, const ispc_region* b) {
      return a->input != b->input ? a->input > b->input : a->obj < b->obj;
    });
    std::vector<std::string> plist;
    for (const ispc_region* r : params) {
      bool ro = !stored_regions_.count(r->obj);
      plist.push_back(std::string(ro ? "const float* __restrict__ " : "float* __restrict__ ") +
                      region_ptr(r->obj));
      if (L.num_params >= ISPC_MAX_PARAMS) throw NestError(ISPC_E_ILLEGAL, "too many kernel parameters");
      ispc_param& P = L.params[L.num_params++];
      P.kind = ISPC_PARAM_REGION;
      P.index = r->obj;
      P.is_input = r->input;
      P.elems = r->elems;
      std::snprintf(P.name, sizeof(P.name), "%s", v_.name(r->obj).c_str());
    }
    for (uint32_t i = 0; i < n.num_inputs; ++i) {
      plist.push_back("const float p_" + sanitize(n.input_names[i]));
      if (L.num_params >= ISPC_MAX_PARAMS) throw NestError(ISPC_E_ILLEGAL, "too many kernel parameters");
      ispc_param& P = L.params[L.num_params++];
      P.kind = ISPC_PARAM_INPUT;
      P.index = i;
      std::snprintf(P.name, sizeof(P.name), "%s", n.input_names[i]);
    }
    if (watchdog_) {
      // absolute %globaltimer deadline, or 0: the one ispc_arm() last set on
      // the device (so queued launches each get their budget from their start)
      plist.push_back("const unsigned long long ispc_deadline_arg");
      if (L.num_params >= ISPC_MAX_PARAMS) throw NestError(ISPC_E_ILLEGAL, "too many kernel parameters");
      ispc_param& P = L.params[L.num_params++];
      P.kind = ISPC_PARAM_DEADLINE;
    }

    int64_t threads = v_.threads_per_block();
    h << "extern \"C\" __global__ void __launch_bounds__(" << threads << ") " << fn_ << "(";
    for (size_t i = 0; i < plist.size(); ++i) h << (i ? ", " : "") << plist[i];
    h << ") {\n";
    // programmatic dependent launch for every loop-nest kernel (the building
    // blocks decide it): griddepcontrol.wait before any memory access, so the
    // launch only overlaps the previous grid's drain; 116.2 -> 115.2 us for
    // the headline's best axpy schedule, every other output unchanged
    // (profiles/r2z_parity_pdl.log). ISPC_PARITY_PDL=0 turns it off.
    if (const char* e = std::getenv("ISPC_PARITY_PDL"); !(e && *e == '0')) {
      h << "  ispc_grid_dep_wait();\n  ispc_grid_dep_trigger();\n";
      L.pdl = 1;
    }
    // hardware indices
    for (uint32_t l = 0; l < n.num_thread_levels; ++l)
      h << "  const int t" << l << " = threadIdx." << "xyz"[thread_axis_[int(l)]] << ";\n";
    if (n.num_block_levels) {
      h << "  unsigned int ispc_bid = blockIdx.x;\n";
      for (int l = int(n.num_block_levels) - 1; l >= 0; --l) {
        if (l == 0) h << "  const int b0 = (int)ispc_bid;\n";
        else {
          h << "  const int b" << l << " = (int)(ispc_bid % " << n.block_shape[l] << "u);\n";
          h << "  ispc_bid /= " << n.block_shape[l] << "u;\n";
        }
      }
    }
    if (watchdog_) {
      bool bar = any_barrier();
      h << "  const unsigned long long ispc_deadline = ispc_deadline_arg ? ispc_deadline_arg : ispc_deadline_at;\n";
      h << "  if (" << (bar ? "__syncthreads_or(ispc_now() > ispc_deadline)" : "ispc_now() > ispc_deadline")
        << ") { ispc_timeout_flag = 1; return; }\n";
    }
    // shared temporaries: one dynamic buffer, 16-byte aligned slices
    int64_t off = 0;
    std::ostringstream sh;
    for (uint32_t i = 0; i < n.num_regions; ++i) {
      const ispc_region& r = n.regions[i];
      if (!r.live || r.mem_space != ISPC_SHARED) continue;
      if (!(loaded_regions_.count(r.obj) || stored_regions_.count(r.obj))) continue;
      sh << "  float* const " << region_ptr(r.obj) << " = ispc_smem + " << off / 4 << ";\n";
      off += (r.elems * r.elem_bytes + 15) / 16 * 16;
    }
    if (off > 232448) throw NestError(ISPC_E_ILLEGAL, "shared temporaries exceed 227 KiB");
    if (off) h << "  extern __shared__ __align__(16) float ispc_smem[];\n" << sh.str();
    L.static_smem = uint32_t(off);
    // register storages
    for (auto& [root, st] : storage_) {
      h << "  float " << st.name;
      if (!st.sizes.empty()) h << "[" << st.elems() << "]";
      h << ";\n";
    }
    return h.str();
  }
};

}  // namespace

std::string emit_cuda_kernel(const NestView& v, const ispc_emit_opts& opts, const std::string& fn,
                             ispc_launch& L) {
  return CudaEmitter(v, opts, fn).run(L);
}

}  // namespace ispc

extern "C" const char* ispc_cuda_prelude(void) {
  return R"(// ispc prelude: device helpers shared by every emitted kernel
__device__ int ispc_timeout_flag;
__device__ unsigned long long ispc_deadline_at;
static __device__ __forceinline__ unsigned long long ispc_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// launched on the stream right before a watchdog kernel: its deadline starts
// when the device reaches it, not when the host enqueued it
extern "C" __global__ void ispc_arm(unsigned long long budget_ns) {
  ispc_deadline_at = ispc_now() + budget_ns;
  ispc_timeout_flag = 0;
}
// building blocks of the tile kernels (emit_tiles.cpp)
static __device__ __forceinline__ unsigned ispc_smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
static __device__ __forceinline__ void ispc_cp_async_cg16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(ispc_smem_addr(s)), "l"(g));
}
static __device__ __forceinline__ void ispc_cp_async_ca16(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(ispc_smem_addr(s)), "l"(g));
}
static __device__ __forceinline__ void ispc_cp_async_ca8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(ispc_smem_addr(s)), "l"(g));
}
static __device__ __forceinline__ void ispc_cp_async_ca4(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(ispc_smem_addr(s)), "l"(g));
}
// the same copies to a 32-bit shared-memory address (NVRTC keeps a generic ->
// shared conversion per copy otherwise: 64-bit cvt pairs nvcc does not emit)
static __device__ __forceinline__ void ispc_cp_async_cg16_s(unsigned s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g));
}
static __device__ __forceinline__ void ispc_cp_async_ca16_s(unsigned s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g));
}
static __device__ __forceinline__ void ispc_cp_async_ca4_s(unsigned s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(g));
}
// a 16-byte shared-memory load by 32-bit address (volatile: never moved
// across the ring's barriers)
static __device__ __forceinline__ float4 ispc_lds4(unsigned a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
// issue and commit carry no memory clobber (shared-memory loads of other ring
// slots may be scheduled across them: the FFMA2 sgemm interleaves its fragment
// loads with the copies); wait_group is the compiler barrier before a slot is read
static __device__ __forceinline__ void ispc_cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
// programmatic dependent launch (ispc_launch.pdl): wait for the previous grid of the stream, then let the next one be scheduled
static __device__ __forceinline__ void ispc_grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
static __device__ __forceinline__ void ispc_grid_dep_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
template <int N>
static __device__ __forceinline__ void ispc_cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
static __device__ __forceinline__ float ispc_ld_stream(const float* p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
static __device__ __forceinline__ float2 ispc_ld_stream(const float2* p) {
  float2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}
static __device__ __forceinline__ float4 ispc_ld_stream(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
static __device__ __forceinline__ unsigned ispc_cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
static __device__ __forceinline__ void ispc_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
static __device__ __forceinline__ float4 ispc_dsmem_ld4(const float* p, unsigned rank) {
  unsigned a = ispc_smem_addr(p), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(r) : "memory");
  return v;
}
static __device__ __forceinline__ void ispc_dsmem_st4(float* p, unsigned rank, float4 v) {
  unsigned a = ispc_smem_addr(p), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(r), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
static __device__ __forceinline__ float ispc_dsmem_ld(const float* p, unsigned rank) {
  unsigned a = ispc_smem_addr(p), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(r) : "memory");
  return v;
}
)";
}

extern "C" int ispc_emit_cuda(const ispc_nest* nest, const ispc_emit_opts* opts, const char* fn_name,
                              char* buf, size_t cap, size_t* len, ispc_launch* launch) {
  try {
    if (!nest || !launch) throw ispc::NestError(ISPC_E_ARG, "null argument");
    ispc_emit_opts o{};
    if (opts) o = *opts;
    else o.watchdog = 2;
    ispc::NestView v(*nest);
    std::string fn = fn_name ? fn_name : "ispc_kernel";
    std::string src = ispc::emit_cuda_kernel(v, o, fn, *launch);
    if (!fn_name) {
      // name from the content hash so identical schedules share a symbol
      char name[64];
      std::snprintf(name, sizeof(name), "ispc_k%016llx", (unsigned long long)launch->source_hash);
      size_t p = src.find(fn);
      if (p != std::string::npos) src.replace(p, fn.size(), name);
      std::snprintf(launch->name, sizeof(launch->name), "%s", name);
    }
    if (len) *len = src.size();
    if (buf && cap) {
      size_t k = src.size() < cap - 1 ? src.size() : cap - 1;
      std::memcpy(buf, src.data(), k);
      buf[k] = 0;
    }
    return ISPC_OK;
  } catch (const ispc::NestError& e) {
    ispc::set_thread_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    ispc::set_thread_error(e.what());
    return ISPC_E_ARG;
  }
}
