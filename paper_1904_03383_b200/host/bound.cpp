#include "bound.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <map>
#include <numeric>
#include <set>
#include <stdexcept>

namespace ispc_host {

using namespace ispace;

namespace {

std::uint32_t choice_id(const SpaceContext& ctx, const char* name) {
  std::uint32_t ch = ctx.table.find_choice(name);
  if (ch == kNoInstance) throw std::logic_error(std::string("space lacks choice ") + name);
  return ch;
}

int vindex(const SpaceContext& ctx, std::uint32_t ch, const char* v) {
  int i = ctx.table.value_index(ch, v);
  if (i < 0) throw std::logic_error(std::string("choice lacks value ") + v);
  return i;
}

struct UF {
  std::vector<std::size_t> p;
  explicit UF(std::size_t n) : p(n) { std::iota(p.begin(), p.end(), std::size_t{0}); }
  std::size_t find(std::size_t x) {
    while (p[x] != x) x = p[x] = p[p[x]];
    return x;
  }
  void unite(std::size_t a, std::size_t b) { p[find(a)] = find(b); }
};

}  // namespace

BoundModel::BoundModel(const Kernel& k, const SpaceContext& ctx, const B200Machine& m) : k_(k), ctx_(ctx), m_(m) {
  std::uint32_t kind_c = choice_id(ctx, "dim_kind");
  std::uint32_t size_c = choice_id(ctx, "size");
  std::uint32_t space_c = choice_id(ctx, "mem_space");
  order_c_ = choice_id(ctx, "order");
  v_loop_ = vindex(ctx, kind_c, "LOOP");
  v_block_ = vindex(ctx, kind_c, "BLOCK");
  v_thread_ = vindex(ctx, kind_c, "THREAD");
  v_unroll_ = vindex(ctx, kind_c, "UNROLL");
  v_vector_ = vindex(ctx, kind_c, "VECTOR");
  v_merged_ = vindex(ctx, order_c_, "MERGED");
  v_global_ = vindex(ctx, space_c, "GLOBAL");
  std::uint32_t cache_c = choice_id(ctx, "cache");
  v_cache_l2_ = vindex(ctx, cache_c, "L2");

  std::map<ObjId, std::size_t> dim_index;
  for (const auto& [id, di] : k.dims) {
    DimRec r;
    r.id = id;
    r.is_static = di.is_static;
    r.logical = di.logical;
    r.kind_inst = ctx.table.find(kind_c, id);
    r.size_inst = di.is_static ? ctx.table.find(size_c, id) : kNoInstance;
    dim_index[id] = dims_.size();
    dim_index_[id] = dims_.size();
    dims_.push_back(r);
  }
  pair_order_.assign(dims_.size(), std::vector<std::uint32_t>(dims_.size(), kNoInstance));
  for (std::size_t a = 0; a < dims_.size(); ++a)
    for (std::size_t b = 0; b < dims_.size(); ++b)
      if (a != b) {
        ObjId args[2] = {dims_[a].id, dims_[b].id};
        pair_order_[a][b] = ctx.table.resolve(order_c_, args, 2).inst;
      }

  for (const auto& [id, ii] : k.insts) {
    InstRec r;
    r.id = id;
    r.lowering = k.bb.obj(id).lowering;
    std::set<ObjId> logicals;
    for (ObjId d : ii.dims) {
      r.dims.push_back(dim_index.at(d));
      logicals.insert(k.dims.at(d).logical);
    }
    r.instances = 1;
    for (ObjId l : logicals) r.instances *= double(k.logicals.at(l).extent);
    r.memory = ii.op == Op::Load || ii.op == Op::Store;
    r.load = ii.op == Op::Load;
    r.region = ii.region;
    if (r.memory) r.cache_inst = ctx.table.find(cache_c, id);
    r.stride_terms.resize(ii.dims.size());
    if (r.memory && ii.ivar != kNoIndex)
      for (const AddrTerm& t : k.ivars[ii.ivar].terms)
        for (std::size_t p = 0; p < ii.dims.size(); ++p)
          if (ii.dims[p] == t.dim) {
            std::vector<std::size_t> sd;
            for (ObjId x : t.size_dims) sd.push_back(dim_index.at(x));
            r.stride_terms[p].emplace_back(double(t.base), std::move(sd));
          }
    insts_.push_back(r);
  }
  for (const auto& [id, ii] : k.insts) {
    bool reduce = false;
    for (const Operand& o : ii.operands) reduce = reduce || o.kind == Operand::Kind::Reduce;
    inst_has_storage_.push_back(ii.op != Op::Store && !reduce);
  }
  for (const Comm& cm : k.comms)
    for (auto& [src, dst] : cm.pairs) comm_pairs_.push_back({dim_index.at(src), dim_index.at(dst), cm.lowering});
  for (const auto& [id, ri] : k.regions) {
    RegionRec r;
    r.id = id;
    r.input = ri.input;
    r.bytes = double(ri.elems) * double(ri.elem_bytes);
    r.lowering = k.bb.obj(id).lowering;
    r.space_inst = ctx.table.find(space_c, id);
    regions_.push_back(r);
  }
}

Mask BoundModel::kinds(const Candidate& c, std::size_t d) const {
  std::uint32_t i = dims_[d].kind_inst;
  return i == kNoInstance ? full_mask(5) : c.dom[i];
}

void BoundModel::extents(const Candidate& c, std::size_t d, double& lo, double& hi) const {
  auto size_range = [&](std::uint32_t inst, double& mn, double& mx) {
    const auto& u = ctx_.table.universe_of(inst);
    Mask m = c.dom[inst];
    mn = 1e300;
    mx = 0;
    for (std::size_t v = 0; v < u.size(); ++v)
      if (mask_has(m, int(v))) {
        mn = std::min(mn, double(u[v]));
        mx = std::max(mx, double(u[v]));
      }
  };
  const DimRec& r = dims_[d];
  if (r.is_static) {
    size_range(r.size_inst, lo, hi);
    return;
  }
  const LogicalInfo& li = k_.logicals.at(r.logical);
  lo = hi = double(li.extent);
  for (ObjId t : li.tiles) {
    double mn, mx;
    size_range(dims_[dim_index_.at(t)].size_inst, mn, mx);
    lo /= mx;
    hi /= mn;
  }
}

BoundReport BoundModel::bound(const Candidate& c) const {
  BoundReport rep;
  const double f = m_.f_max_hz;
  const std::size_t nd = dims_.size();
  std::vector<Mask> km(nd);
  std::vector<double> lo(nd), hi(nd);
  for (std::size_t d = 0; d < nd; ++d) {
    km[d] = kinds(c, d);
    extents(c, d, lo[d], hi[d]);
  }
  auto can = [&](std::size_t d, int v) { return mask_has(km[d], v); };
  auto is = [&](std::size_t d, int v) { return km[d] == bit(v); };
  auto may_merge = [&](std::size_t a, std::size_t b) {
    std::uint32_t i = pair_order_[a][b];
    return i != kNoInstance && mask_has(c.dom[i], v_merged_);
  };
  auto fired = [&](std::uint32_t lw) { return lw == kNoLowering || ((c.fired >> lw) & 1u); };
  auto illegal = [&](Illegal why) {
    rep.illegal = why;
    rep.total = std::numeric_limits<double>::infinity();
    return rep;
  };

  // -- hardware legality: subtrees no completion of which can run correctly --
  // a value crossing blocks through a temporary needs a grid-wide barrier
  for (const PairRec& p : comm_pairs_)
    if (fired(p.lowering) && (is(p.src, v_block_) || is(p.dst, v_block_)) && !may_merge(p.src, p.dst))
      return illegal(Illegal::CrossBlock);
  // grid: dims certainly BLOCK that can never fuse multiply the block count
  double blocks_lo = 1;
  {
    UF pm(nd);
    for (std::size_t a = 0; a < nd; ++a)
      for (std::size_t b = a + 1; b < nd; ++b)
        if (is(a, v_block_) && is(b, v_block_) && may_merge(a, b)) pm.unite(a, b);
    std::map<std::size_t, double> comp;
    for (std::size_t d = 0; d < nd; ++d)
      if (is(d, v_block_)) comp[pm.find(d)] = std::max(comp[pm.find(d)], lo[d]);
    for (auto& [r, e] : comp) blocks_lo *= e;
    if (blocks_lo > 2147483647.0) return illegal(Illegal::Grid);
  }
  // threads per block every completion has at least (certainly-THREAD dims)
  double threads_lo = 1;
  {
    UF pm(nd);
    for (std::size_t a = 0; a < nd; ++a)
      for (std::size_t b = a + 1; b < nd; ++b)
        if (is(a, v_thread_) && is(b, v_thread_) && may_merge(a, b)) pm.unite(a, b);
    std::map<std::size_t, double> comp;
    for (std::size_t d = 0; d < nd; ++d)
      if (is(d, v_thread_)) comp[pm.find(d)] = std::max(comp[pm.find(d)], lo[d]);
    for (auto& [r, e] : comp) threads_lo *= e;
  }
  const double resident = std::max(1.0, std::min<double>(m_.max_blocks_per_sm,
                                                         std::floor(m_.max_threads_per_sm / std::max(threads_lo, 1.0))));
  const double waves = std::ceil(blocks_lo / (double(m_.sms) * resident));
  // per-thread register arrays and unrolled body
  {
    double regs = 0, unrolled = 0;
    for (std::size_t i = 0; i < insts_.size(); ++i) {
      const InstRec& r = insts_[i];
      if (!fired(r.lowering)) continue;
      double lanes = 1;
      for (std::size_t d : r.dims)
        if (is(d, v_unroll_) || is(d, v_vector_)) lanes *= lo[d];
      unrolled += lanes;
      if (inst_has_storage_[i]) regs += lanes;
    }
    if (regs > m_.max_reg_elems) return illegal(Illegal::Registers);
    if (unrolled > m_.max_unrolled) return illegal(Illegal::Unrolled);
  }

  // fusion classes decided so far
  UF uf(nd);
  for (std::size_t a = 0; a < nd; ++a)
    for (std::size_t b = a + 1; b < nd; ++b) {
      std::uint32_t i = pair_order_[a][b];
      if (i != kNoInstance && c.dom[i] == bit(v_merged_)) uf.unite(a, b);
    }
  std::map<std::size_t, std::vector<std::size_t>> cls;
  for (std::size_t d = 0; d < nd; ++d) cls[uf.find(d)].push_back(d);
  double blocks = 1, threads = 1;
  for (auto& [root, members] : cls) {
    bool all_block = true, all_thread = true;
    double ext = 1e300;
    for (std::size_t d : members) {
      all_block = all_block && can(d, v_block_);
      all_thread = all_thread && can(d, v_thread_);
      ext = std::min(ext, hi[d]);
    }
    if (all_block) blocks = std::min(blocks * ext, 2147483647.0);
    if (all_thread) threads = std::min(threads * ext, double(m_.max_threads_per_block));
  }
  rep.blocks_max = blocks;
  rep.threads_per_block_max = threads;
  const double sms = std::min<double>(blocks, m_.sms);
  const double lanes = std::min(32.0, threads);

  // instructions that exist in every completion
  double warp_insts = 0, mem_warp_insts = 0, thread_trips = 0, load_chain = 0;
  std::map<ObjId, double> region_touch;  // bytes each input region must move
  for (const InstRec& r : insts_) {
    if (r.lowering != kNoLowering && !((c.fired >> r.lowering) & 1u)) continue;
    bool packable = false;
    double seq = 1;
    for (std::size_t d : r.dims) {
      bool par = can(d, v_block_) || can(d, v_thread_) || can(d, v_vector_);
      if (can(d, v_unroll_) || can(d, v_vector_)) packable = true;
      if (!par) seq *= lo[d];
    }
    double pack = packable ? (r.memory ? 4.0 : 2.0) : 1.0;
    warp_insts += std::ceil(r.instances / (lanes * pack));
    if (r.memory) mem_warp_insts += std::ceil(r.instances / (lanes * pack));
    thread_trips += seq / pack;
    if (r.load) {  // trips of the dimensions certainly rolled loops around this load
      double trips = 1;
      for (std::size_t d : r.dims)
        if (is(d, v_loop_)) trips *= lo[d];
      const bool cg = r.cache_inst != kNoInstance && c.dom[r.cache_inst] == bit(v_cache_l2_);
      load_chain = std::max(load_chain, trips * (cg ? m_.l2_load_latency_cycles : m_.min_load_latency_cycles));
    }
    if (r.memory) {
      double& t = region_touch[r.region];
      t = std::max(t, r.instances * 4.0);
    }
  }
  // L1 lines of scattered warp accesses (see bound.hpp)
  double l1_lines = 0;
  for (const InstRec& r : insts_) {
    if (!r.memory || !fired(r.lowering)) continue;
    bool global_region = false;
    for (const RegionRec& g : regions_)
      if (g.id == r.region) global_region = g.input || (g.space_inst != kNoInstance && c.dom[g.space_inst] == bit(v_global_));
    if (!global_region) continue;
    bool some_thread = false, vec = false;
    double s_min = 1e300, lanes = 32;
    for (std::size_t p = 0; p < r.dims.size(); ++p) {
      const std::size_t d = r.dims[p];
      if (can(d, v_vector_)) vec = true;
      if (!can(d, v_thread_)) continue;
      if (is(d, v_thread_)) some_thread = true;
      double s = 0;
      for (const auto& [base, sd] : r.stride_terms[p]) {
        double m = base;
        for (std::size_t x : sd) m *= lo[x];
        s += m;
      }
      s_min = std::min(s_min, s);
      lanes = std::min(lanes, lo[d]);
    }
    if (!some_thread || vec || !(s_min >= 2)) continue;
    const double per_access = s_min >= 32 ? lanes : std::ceil(lanes * s_min / 32.0);
    l1_lines += r.instances / 32.0 * per_access;
  }

  double input_bytes = 0, tmp_dram = 0, tmp_lsu = 0;
  for (const RegionRec& g : regions_) {
    auto it = region_touch.find(g.id);
    if (it == region_touch.end()) continue;
    if (g.input) {
      input_bytes += it->second;
      continue;
    }
    if (g.lowering != kNoLowering && !((c.fired >> g.lowering) & 1u)) continue;
    bool global_only = g.space_inst != kNoInstance && c.dom[g.space_inst] == bit(v_global_);
    if (!global_only) continue;
    tmp_dram += 2.0 * std::max(0.0, g.bytes - m_.l2_bytes);
    tmp_lsu += g.bytes;
  }
  double dram_bytes = (m_.l2_flushed ? input_bytes : std::max(0.0, input_bytes - m_.l2_bytes)) + tmp_dram;
  rep.dram_bytes = dram_bytes;
  rep.dram = dram_bytes / m_.hbm_bytes_per_s;
  rep.sm_mem = (input_bytes + tmp_lsu) / (sms * m_.sm_bytes_per_cycle * f);
  rep.issue = warp_insts / (sms * m_.issue_per_sm_cycle * f);
  rep.thread = std::max(1.0, waves) * std::max(thread_trips, load_chain) / f;
  rep.launch = m_.launch_floor_s;
  rep.dispatch = blocks_lo * m_.block_dispatch_s;
  rep.l1 = l1_lines / (sms * m_.l1_lines_per_cycle * f);
  rep.lsu = mem_warp_insts / (sms * m_.lsu_per_cycle * f);
  rep.total = std::max({rep.dram, rep.sm_mem, rep.issue, rep.thread, rep.launch, rep.dispatch, rep.l1, rep.lsu});
  return rep;
}

}  // namespace ispc_host
