// Reference-compatible pseudo-source rendering driven only by the flat ABI.
//
// The text format is the one the reference's emit_source() produces
// (proj/core/src/loop_nest.cpp:389-609) and that its golden files pin
// (proj/tests/data/golden/{axpy_vector,matmul_fused,matmul_staged}.txt).
// Reproducing it byte for byte from an ispc_nest proves that the flat
// description carries the whole schedule: loop structure, hardware mapping,
// register hand-offs (Reduce / fired comms) and every affine address.
#include <cstring>
#include <map>
#include <sstream>

#include "nest_view.hpp"

namespace ispc {
namespace {

constexpr int64_t kReplicate = 8;  // unroll replication limit (loop_nest.cpp:401)

class PseudoWriter {
 public:
  explicit PseudoWriter(const NestView& v) : v_(v) {
    int loops = 0, unrolls = 0, vecs = 0;
    for (uint32_t idx : v_.preorder()) {
      const ispc_node& nd = v_.node(idx);
      if (nd.kind != ISPC_NODE_DIM) continue;
      switch (nd.dim_kind) {
        case ISPC_BLOCK: var_[idx] = "b" + std::to_string(nd.block_level); break;
        case ISPC_THREAD: var_[idx] = "t" + std::to_string(nd.thread_level); break;
        case ISPC_LOOP: var_[idx] = "i" + std::to_string(loops++); break;
        case ISPC_VECTOR: var_[idx] = "v" + std::to_string(vecs++); break;
        case ISPC_UNROLL:
          if (nd.size > kReplicate) var_[idx] = "u" + std::to_string(unrolls++);
          break;
      }
    }
  }

  std::string run() {
    const ispc_nest& n = v_.n;
    out_ << "kernel " << (n.kernel_name ? n.kernel_name : "") << "\n// grid: blocks=[";
    for (uint32_t i = 0; i < n.num_block_levels; ++i) out_ << (i ? ", " : "") << n.block_shape[i];
    out_ << "] threads=[";
    for (uint32_t i = 0; i < n.num_thread_levels; ++i) out_ << (i ? ", " : "") << n.thread_shape[i];
    out_ << "]\n";
    for (uint32_t r = 0; r < n.roots_count; ++r) node(n.roots_begin + r, 0, 1);
    return out_.str();
  }

 private:
  const NestView& v_;
  std::ostringstream out_;
  std::map<uint32_t, std::string> var_;
  std::map<uint32_t, int64_t> lane_;  // unrolled node -> replica index

  void put(int depth, const std::string& s) { out_ << std::string(2 * depth, ' ') << s << "\n"; }

  std::string reg(uint32_t inst) const {
    const ispc_inst& ii = v_.inst(inst);
    for (uint32_t j = 0; j < ii.operands_count; ++j) {
      const ispc_operand& o = v_.n.operands[ii.operands_begin + j];
      if (o.kind != ISPC_OPND_REDUCE) continue;
      uint32_t src = o.init;
      if (o.comm != ISPC_NONE && v_.comm_fired(o.comm)) src = v_.n.comms[o.comm].load;
      return reg(src);
    }
    return "r_" + v_.name(inst);
  }

  std::string addr(uint32_t ivar) const {
    const ispc_ivar& iv = v_.n.ivars[ivar];
    int64_t c = iv.offset;
    std::string s;
    for (uint32_t j = 0; j < iv.terms_count; ++j) {
      const ispc_addr_term& t = v_.n.terms[iv.terms_begin + j];
      int64_t m = v_.term_mult(t);
      uint32_t nd = v_.node_of_dim(t.dim);
      auto ln = lane_.find(nd);
      if (ln != lane_.end()) {
        c += ln->second * m;
        continue;
      }
      std::string p = var_.at(nd);
      if (m != 1) p += "*" + std::to_string(m);
      s += (s.empty() ? "" : " + ") + p;
    }
    if (s.empty()) return std::to_string(c);
    if (c != 0) s += " + " + std::to_string(c);
    return s;
  }

  std::string operand(const ispc_operand& o, uint32_t self) const {
    switch (o.kind) {
      case ISPC_OPND_CONST: return std::to_string(o.value);
      case ISPC_OPND_INPUT: return v_.n.input_names[o.input];
      case ISPC_OPND_INDVAR: return "(" + addr(o.ivar) + ")";
      case ISPC_OPND_PRODUCED: return reg(o.producer);
      case ISPC_OPND_MAPPED:
        if (o.comm != ISPC_NONE && v_.comm_fired(o.comm)) return reg(v_.n.comms[o.comm].load);
        return reg(o.producer);
      case ISPC_OPND_REDUCE: return reg(self);
    }
    return "?";
  }

  std::string note(const ispc_inst& ii) const {
    if (v_.region(ii.region).mem_space == ISPC_SHARED) return "shared";
    switch (ii.cache) {
      case ISPC_CACHE_L1: return "global via L1";
      case ISPC_CACHE_L2: return "global via L2";
      case ISPC_CACHE_READ_ONLY: return "global via read-only path";
      default: return "global uncached";
    }
  }

  std::string members(const ispc_node& nd) const {
    std::string s;
    for (uint32_t j = 0; j < nd.dims_count; ++j)
      s += (j ? " + " : "") + v_.name(v_.n.pool[nd.dims_begin + j]);
    return s;
  }

  static const char* opname(uint32_t op) {
    static const char* names[] = {"add", "mul", "mad", "cast", "load", "store"};
    return op < 6 ? names[op] : "?";
  }

  void inst(const ispc_node& nd, int depth, int64_t width) {
    const ispc_inst& ii = v_.inst(nd.inst);
    std::string sfx = width > 1 ? ".v" + std::to_string(width) : "";
    const ispc_operand* ops = v_.n.operands + ii.operands_begin;
    switch (ii.op) {
      case ISPC_OP_LOAD:
        put(depth, reg(nd.inst) + " = load" + sfx + " " + v_.name(ii.region) + "[" + addr(ii.ivar) +
                       "]  // " + note(ii));
        return;
      case ISPC_OP_STORE:
        put(depth, "store" + sfx + " " + v_.name(ii.region) + "[" + addr(ii.ivar) + "], " +
                       operand(ops[0], nd.inst) + "  // " + note(ii));
        return;
      case ISPC_OP_CAST: put(depth, reg(nd.inst) + " = " + operand(ops[0], nd.inst)); return;
      default: {
        std::string args;
        for (uint32_t j = 0; j < ii.operands_count; ++j)
          args += (j ? ", " : "") + operand(ops[j], nd.inst);
        put(depth, reg(nd.inst) + " = " + opname(ii.op) + sfx + "(" + args + ")");
      }
    }
  }

  void children(const ispc_node& nd, int depth, int64_t width) {
    for (uint32_t j = 0; j < nd.children_count; ++j) node(nd.children_begin + j, depth, width);
  }

  void node(uint32_t idx, int depth, int64_t width) {
    const ispc_node& nd = v_.node(idx);
    if (nd.kind == ISPC_NODE_BARRIER) return put(depth, "barrier");
    if (nd.kind == ISPC_NODE_INST) return inst(nd, depth, width);
    std::string range = "0.." + std::to_string(nd.size);
    switch (nd.dim_kind) {
      case ISPC_BLOCK:
        put(depth, "par " + var_.at(idx) + " in " + range + ":  // block level " +
                       std::to_string(nd.block_level) + ": " + members(nd));
        return children(nd, depth + 1, width);
      case ISPC_THREAD:
        put(depth, "par " + var_.at(idx) + " in " + range + ":  // thread level " +
                       std::to_string(nd.thread_level) + ": " + members(nd));
        return children(nd, depth + 1, width);
      case ISPC_LOOP:
        put(depth, "for " + var_.at(idx) + " in " + range + ":  // " + members(nd));
        return children(nd, depth + 1, width);
      case ISPC_VECTOR:
        put(depth, "vec " + var_.at(idx) + " in " + range + ":  // " + members(nd));
        return children(nd, depth + 1, width * nd.size);
      case ISPC_UNROLL:
        if (nd.size > kReplicate) {
          put(depth, "unroll " + var_.at(idx) + " in " + range + ":  // " + members(nd));
          return children(nd, depth + 1, width);
        }
        put(depth, "// unroll " + members(nd) + " x" + std::to_string(nd.size));
        for (int64_t i = 0; i < nd.size; ++i) {
          lane_[idx] = i;
          put(depth, "// lane " + std::to_string(i));
          children(nd, depth + 1, width);
        }
        lane_.erase(idx);
        return;
    }
  }
};

}  // namespace
}  // namespace ispc

extern "C" int ispc_emit_pseudo(const ispc_nest* nest, char* buf, size_t cap, size_t* len) {
  try {
    if (!nest) throw ispc::NestError(ISPC_E_ARG, "null nest");
    ispc::NestView v(*nest);
    std::string s = ispc::PseudoWriter(v).run();
    if (len) *len = s.size();
    if (buf && cap) {
      size_t k = s.size() < cap - 1 ? s.size() : cap - 1;
      std::memcpy(buf, s.data(), k);
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
