// B200 building-block spaces: parameter sets per kernel kind, the Backbone +
// Providers handed to the reference's build_space(), candidate -> flat
// ispc_tile_config, and the B200 lower bound of a (partial) candidate.
#include "tiles.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <map>
#include <stdexcept>

#include "ispace/parser.hpp"
#include "tiles_space_text.hpp"

namespace ispc_host {

using namespace ispace;

namespace {

std::vector<std::int64_t> pow2_upto(std::int64_t lo, std::int64_t hi) {
  std::vector<std::int64_t> v;
  for (std::int64_t x = lo; x <= hi; x *= 2) v.push_back(x);
  return v;
}

std::vector<std::int64_t> dividing(std::vector<std::int64_t> v, std::int64_t extent) {
  v.erase(std::remove_if(v.begin(), v.end(), [&](std::int64_t x) { return x <= 0 || extent % x != 0; }), v.end());
  return v;
}

TileParam P(const std::string& name, std::vector<std::int64_t> values) {
  TileParam p;
  p.name = name;
  p.values = std::move(values);
  if (p.values.empty()) throw std::invalid_argument("tile parameter '" + name + "' has no admissible value");
  if (p.values.size() > 32) throw std::invalid_argument("tile parameter '" + name + "' exceeds 32 values");
  return p;
}

// B200 constants the bound prices (nominal figures, above what a kernel can
// reach, so the bound stays below every measured time).
constexpr double kFmax = 1.965e9;           // max SM clock
constexpr int kSMs = 148;
constexpr double kHbm = 7.7e12;             // nominal HBM3e bytes/s (measured copy: 6.55e12)
constexpr double kFfmaPerSmClk = 128;       // fp32 lanes per SM
constexpr double kTf32Flops = 1.2e15;       // dense TF32 tensor peak, rounded up (nominal 1.1e15)
constexpr double kLaunch = 1e-6;

}  // namespace

bool is_tile_kind(const std::string& k) {
  return k == "gemv" || k == "sgemm" || k == "batched" || k == "sgemm_tc" || k == "sgemm_tc_x3" ||
         k == "axpy_stream";
}

const char* tiles_space_text() { return kTilesSpaceText; }

bool TileFamily::bit_exact() const {
  return kind == ISPC_TILE_SGEMM || kind == ISPC_TILE_BATCHED || kind == ISPC_TILE_AXPY;
}

bool tile_bit_exact(const ispc_tile_config& t) {
  // FFMA kernels that keep one k-ascending chain per output; split-K sums
  // cluster partials and is checked norm-wise
  return (t.kind == ISPC_TILE_SGEMM && t.split <= 1) || t.kind == ISPC_TILE_BATCHED || t.kind == ISPC_TILE_AXPY;
}

double TileFamily::rtol() const {
  // FFMA reorderings (gemv, split-K) and 3xTF32 are held to 1e-5 of
  // sum |a||b|; plain TF32 rounds operands to 10 mantissa bits (2^-11 each)
  return kind == ISPC_TILE_SGEMM_TC && !x3_only ? 4e-3 : 1e-5;
}

// every family carries `pdl` (programmatic dependent launch, ispc_launch.pdl),
// decided last (decided first with 90% elite-guided rollouts, the searches
// kept pdl = 0 more often and found slower kernels: profiles/r2n_bench.json
// against r2l_bench.json)
TileFamily make_family(const std::string& kind, std::int64_t m, std::int64_t n, std::int64_t k, std::int64_t batch) {
  TileFamily f;
  f.m = m, f.n = n, f.k = k, f.batch = std::max<std::int64_t>(batch, 1);
  auto pre = [&](const std::string& choice, std::vector<std::string> values) {
    f.pre.push_back(PreRestriction{choice, {"kernel"}, std::move(values)});
  };
  if (kind == "gemv") {
    if (m <= 0 || n <= 0) throw std::invalid_argument("gemv needs m, n > 0");
    f.kind = ISPC_TILE_GEMV;
    TileParam vec = P("vec", dividing({1, 2, 4}, m));
    TileParam lm = P("lanes_m", pow2_upto(1, 32)), ln = P("lanes_n", dividing(pow2_upto(1, 32), n));
    TileParam wm = P("warps_m", pow2_upto(1, 8)), wn = P("warps_n", dividing(pow2_upto(1, 32), n));
    TileParam split = P("split", dividing({1, 2, 4, 8}, n)), unroll = P("unroll", dividing({1, 2, 4, 8, 16}, n));
    TileParam bk = P("bk", {1, 8, 16, 32, 64, 128, 256}), st = P("stages", {1, 2, 3, 4, 6, 8});
    TileParam grid = P("grid", {0});  // > 0 (balanced row blocks / persistent TMA ring) measured slower: DESIGN.md 3
    grid.persist = true;
    lm.thread = ln.thread = wm.thread = wn.thread = true;
    lm.warp = ln.warp = true;
    vec.acc = unroll.acc = true;
    split.cluster = true;
    bk.stage = st.stage = true;
    f.params = {vec, lm, ln, wm, wn, split, unroll, bk, st, grid, P("pdl", {0, 1})};
    f.min_threads = 32;
    f.warp_lanes = 32;
    f.max_acc = 64;
    pre("staging", {"DIRECT", "CP_ASYNC", "TMA"});
    pre("engine", {"FFMA"});
  } else if (kind == "sgemm") {
    if (m <= 0 || n <= 0 || k <= 0) throw std::invalid_argument("sgemm needs m, n, k > 0");
    f.kind = ISPC_TILE_SGEMM;
    TileParam tx = P("thr_m", dividing(pow2_upto(1, 256), m)), ty = P("thr_n", dividing(pow2_upto(1, 256), n));
    TileParam tm = P("tm", dividing(pow2_upto(1, 16), m)), tn = P("tn", dividing(pow2_upto(1, 16), n));
    TileParam bk = P("bk", dividing({4, 8, 16, 32}, k)), st = P("stages", {1, 2, 3, 4});
    TileParam vec = P("vec", {1, 2, 4});
    TileParam split = P("split", dividing({1, 2, 4, 8}, k));
    tx.thread = ty.thread = true;
    tm.acc = tn.acc = true;
    split.cluster = true;
    f.params = {tx, ty, tm, tn, bk, st, vec, split, P("lds", {0, 1}), P("pdl", {0, 1})};
    f.min_threads = 32;
    f.max_acc = 128;
    pre("staging", {"SHARED", "CP_ASYNC"});
    pre("engine", {"FFMA"});
    pre("xreduce", {"SHUFFLE"});
  } else if (kind == "batched") {
    if (m <= 0 || n <= 0 || k <= 0 || batch <= 0) throw std::invalid_argument("batched needs m, n, k, batch > 0");
    f.kind = ISPC_TILE_BATCHED;
    TileParam pc = P("per_cta", dividing(pow2_upto(1, 32), f.batch));
    TileParam tm = P("tm", dividing(pow2_upto(1, 8), m)), tn = P("tn", dividing(pow2_upto(1, 8), n));
    TileParam bk = P("bk", dividing({4, 8, 16, 32, 64}, k)), vec = P("vec", {1, 2, 4});
    pc.thread = true;
    tm.acc = tn.acc = true;
    f.params = {pc, tm, tn, bk, vec, P("pdl", {0, 1})};
    f.min_threads = 1;
    f.max_acc = 64;
    pre("staging", {"DIRECT", "SHARED", "CP_ASYNC"});
    pre("engine", {"FFMA"});
    pre("xreduce", {"SHUFFLE"});
  } else if (kind == "sgemm_tc" || kind == "sgemm_tc_x3") {
    // sgemm_tc_x3: the same space with the engine fixed to 3xTF32 (fp32-level
    // accuracy, checked at 1e-5), reported beside cuBLAS FP32
    if (m <= 0 || n <= 0 || k <= 0) throw std::invalid_argument("sgemm_tc needs m, n, k > 0");
    f.kind = ISPC_TILE_SGEMM_TC;
    f.x3_only = kind == "sgemm_tc_x3";
    // split = CTAs sharing one UMMA (cta_group::2 pairs two SMs on M = 256)
    TileParam bn = P("bn", dividing({64, 128, 256}, n)), st = P("stages", {2, 3, 4, 5, 6, 8});
    // split = 4: two pairs on adjacent n-blocks sharing A by TMA multicast (persistent grid only)
    TileParam pair = P("split", m % 256 == 0 ? std::vector<std::int64_t>{1, 2, 4} : std::vector<std::int64_t>{1});
    TileParam grid = P("grid", {0, 128, 144, 148});  // 0: one tile per CTA (pair); else persistent CTAs (<= one per SM)
    pair.cluster = true;
    grid.persist = true;
    f.params = {bn, st, pair, grid, P("pdl", {0, 1})};
    f.min_threads = 1;
    f.max_acc = 1;
    f.max_cluster = 4;
    // A by TMA (transposed in shared memory) or through registers; B by TMA
    pre("staging", {"TMA", "SHARED"});
    if (f.x3_only) pre("engine", {"TF32X3"});
    else pre("engine", {"TF32", "TF32X3"});
    pre("xreduce", {"SHUFFLE"});
    pre("cache", {"L2"});
  } else if (kind == "axpy_stream") {
    // the elementwise streaming block for axpy (the parity space's axpy is
    // the reference's own gpu.space; this one is B200 building blocks only)
    if (n <= 0) throw std::invalid_argument("axpy_stream needs n > 0");
    f.kind = ISPC_TILE_AXPY;
    TileParam vec = P("vec", dividing({1, 2, 4}, n)), thr = P("threads", pow2_upto(32, 1024));
    TileParam unroll = P("unroll", {1, 2, 4, 8}), grid = P("grid", {0, 148, 296, 592, 1184, 2368, 4736});
    thr.thread = true;
    vec.acc = unroll.acc = true;
    f.params = {vec, thr, unroll, grid, P("pdl", {0, 1})};
    f.min_threads = 32;
    f.max_acc = 32;
    pre("staging", {"DIRECT"});
    pre("engine", {"FFMA"});
    pre("xreduce", {"SHUFFLE"});
  } else {
    throw std::invalid_argument("not a building-block kernel kind: " + kind);
  }
  // inner tiles never exceed their outer tile
  if (f.kind == ISPC_TILE_SGEMM) f.covers = {};
  return f;
}

BuildResult build_tile_space(const TileFamily& f) {
  ParseResult pr = parse_space(tiles_space_text());
  if (!pr.ok()) return {nullptr, std::move(pr.diagnostics)};
  Backbone bb;
  ObjId kern = bb.add_object("kernel");
  bb.add_to_set("Kernels", kern);
  auto values = std::make_shared<std::map<ObjId, std::vector<std::int64_t>>>();
  for (const TileParam& p : f.params) {
    ObjId o = bb.add_object(p.name);
    bb.add_to_set("Params", o);
    if (p.thread) bb.add_to_set("ThreadParams", o);
    if (p.warp) bb.add_to_set("WarpParams", o);
    if (p.acc) bb.add_to_set("AccParams", o);
    if (p.cluster) bb.add_to_set("ClusterParams", o);
    if (p.stage) bb.add_to_set("StageParams", o);
    if (p.persist) bb.add_to_set("PersistParams", o);
    (*values)[o] = p.values;
  }
  for (const auto& [outer, inner] : f.covers) {
    ObjId c = bb.add_object("cover_" + outer + "_" + inner);
    bb.add_to_set("Covers", c);
    bb.add_to_param_set("CoverOuter", c, bb.find(outer));
    bb.add_to_param_set("CoverInner", c, bb.find(inner));
  }
  for (const char* s : {"ThreadParams", "WarpParams", "AccParams", "ClusterParams", "StageParams", "PersistParams",
                        "Covers"})
    if (!bb.sets.count(s)) bb.sets[s] = {};

  Providers pv;
  pv.universe = [values](const std::string& key, const std::vector<ObjId>& args) {
    if (key != "$p.values()" || args.size() != 1)
      throw std::invalid_argument("unknown universe fragment \"" + key + "\"");
    return values->at(args[0]);
  };
  const TileFamily fam = f;
  pv.num = [fam](const std::string& key, const std::vector<ObjId>& args) -> std::int64_t {
    if (!args.empty()) throw std::invalid_argument("unknown numeric fragment \"" + key + "\"");
    if (key == "machine.max_threads") return 1024;
    if (key == "machine.min_threads") return fam.min_threads;
    if (key == "machine.warp_lanes") return fam.warp_lanes;
    if (key == "machine.max_acc_regs") return fam.max_acc;
    if (key == "machine.max_cluster") return fam.max_cluster;
    throw std::invalid_argument("unknown numeric fragment \"" + key + "\"");
  };
  pv.pred = [](const std::string& key, const std::vector<ObjId>&) -> bool {
    throw std::invalid_argument("unknown predicate fragment \"" + key + "\"");
  };
  pv.lowering = [](const std::string& cb, const std::vector<ObjId>&) -> std::uint32_t {
    throw std::invalid_argument("unknown trigger callback \"" + cb + "\"");
  };
  BuildInput in;
  in.def = std::move(pr.def);
  in.bb = std::move(bb);
  in.providers = std::move(pv);
  in.pre = f.pre;
  return build_space(std::move(in));
}

namespace {

struct Reader {
  const SpaceContext& ctx;
  const Candidate& c;
  std::uint32_t ch_tile;

  Reader(const SpaceContext& x, const Candidate& cand) : ctx(x), c(cand), ch_tile(x.table.find_choice("tile")) {}

  std::uint32_t inst_of(std::uint32_t ch, const std::string& obj) const {
    ObjId o = ctx.bb.find(obj);
    if (o == kNoObj) return kNoInstance;
    return ctx.table.resolve(ch, &o, 1).inst;
  }
  // [lo, hi] of a tile parameter's remaining values; {0,0} when absent
  std::pair<std::int64_t, std::int64_t> range(const std::string& name) const {
    std::uint32_t i = inst_of(ch_tile, name);
    if (i == kNoInstance) return {0, 0};
    const auto& u = ctx.table.universe_of(i);
    std::int64_t lo = std::numeric_limits<std::int64_t>::max(), hi = 0;
    for (size_t v = 0; v < u.size(); ++v)
      if (mask_has(c.dom[i], int(v))) lo = std::min(lo, u[v]), hi = std::max(hi, u[v]);
    return {lo, hi};
  }
  // remaining values of a tile parameter ({} when absent)
  std::vector<std::int64_t> remaining(const std::string& name) const {
    std::vector<std::int64_t> out;
    std::uint32_t i = inst_of(ch_tile, name);
    if (i == kNoInstance) return out;
    const auto& u = ctx.table.universe_of(i);
    for (size_t v = 0; v < u.size(); ++v)
      if (mask_has(c.dom[i], int(v))) out.push_back(u[v]);
    return out;
  }
  std::int64_t value(const std::string& name) const {
    std::uint32_t i = inst_of(ch_tile, name);
    if (i == kNoInstance) return 0;
    int v = decided_value(c, i);
    if (v < 0) throw std::invalid_argument("tile(" + name + ") is still open");
    return ctx.table.universe_of(i)[size_t(v)];
  }
  int enum_value(const std::string& choice) const {
    std::uint32_t ch = ctx.table.find_choice(choice);
    std::uint32_t i = inst_of(ch, "kernel");
    int v = decided_value(c, i);
    if (v < 0) throw std::invalid_argument(choice + "(kernel) is still open");
    return v;  // value index in declaration order, which is the ispc_* enum order
  }
  Mask enum_mask(const std::string& choice) const {
    std::uint32_t ch = ctx.table.find_choice(choice);
    return c.dom[inst_of(ch, "kernel")];
  }
};

}  // namespace

ispc_tile_config tile_config(const TileFamily& f, const SpaceContext& ctx, const Candidate& c) {
  Reader r(ctx, c);
  ispc_tile_config t{};
  t.kind = f.kind;
  t.m = f.m, t.n = f.n, t.k = f.k, t.batch = f.batch;
  t.staging = uint32_t(r.enum_value("staging"));
  t.engine = uint32_t(r.enum_value("engine"));
  t.xreduce = uint32_t(r.enum_value("xreduce"));
  t.cache = uint32_t(r.enum_value("cache"));
  auto v = [&](const char* name) { return int32_t(r.value(name)); };
  t.thr_m = v("thr_m"), t.thr_n = v("thr_n"), t.tm = v("tm"), t.tn = v("tn"), t.bk = v("bk"), t.bn = v("bn");
  t.stages = v("stages"), t.vec = v("vec"), t.lanes_m = v("lanes_m"), t.lanes_n = v("lanes_n");
  t.warps_m = v("warps_m"), t.warps_n = v("warps_n"), t.split = v("split"), t.unroll = v("unroll");
  t.per_cta = v("per_cta");
  t.threads = v("threads");
  t.grid = v("grid");
  t.pdl = v("pdl");
  t.lds = uint32_t(v("lds"));
  return t;
}

TileBoundReport tile_bound(const TileFamily& f, const SpaceContext& ctx, const Candidate& c) {
  Reader r(ctx, c);
  TileBoundReport b;
  const double M = double(f.m), N = double(f.n), K = double(f.k), B = double(f.batch);
  double flops = 0, per_thread = 0;  // per_thread: sequential FMA instructions of one thread (lower bound)
  auto lo = [&](const char* p) { return double(r.range(p).first); };
  auto hi = [&](const char* p) { return double(r.range(p).second); };
  switch (f.kind) {
    case ISPC_TILE_GEMV:
      b.dram_bytes = 4 * (M * N + M + N);
      flops = 2 * M * N;
      b.ctas = M / (lo("vec") * lo("lanes_m") * lo("warps_m")) * hi("split");
      if (lo("grid") > 0) b.ctas = std::min(b.ctas, hi("grid"));
      per_thread = N / (hi("split") * hi("warps_n") * hi("lanes_n")) * lo("vec");
      break;
    case ISPC_TILE_SGEMM:
    case ISPC_TILE_SGEMM_TC:
      b.dram_bytes = 4 * (M * K + K * N + M * N);
      flops = 2 * M * N * K;
      if (f.kind == ISPC_TILE_SGEMM) {
        b.ctas = M / (lo("thr_m") * lo("tm")) * (N / (lo("thr_n") * lo("tn"))) * hi("split");
        per_thread = lo("tm") * lo("tn") * K / hi("split");
      } else {
        b.ctas = M / 128 * (N / lo("bn"));
        if (lo("grid") > 0) b.ctas = std::min(b.ctas, hi("grid"));
      }
      break;
    case ISPC_TILE_AXPY:
      b.dram_bytes = 12 * N;
      flops = 2 * N;
      b.ctas = N / (lo("vec") * lo("threads") * lo("unroll"));
      break;
    case ISPC_TILE_BATCHED:
      b.dram_bytes = 4 * B * (M * K + K * N + M * N);
      flops = 2 * B * M * N * K;
      b.ctas = B / lo("per_cta");
      per_thread = lo("tm") * lo("tn") * K;
      break;
  }
  b.dram = b.dram_bytes / kHbm;
  const double sms = std::min<double>(kSMs, std::max(1.0, b.ctas));
  bool tensor = false;
  if (f.kind == ISPC_TILE_SGEMM_TC) {
    Mask eng = r.enum_mask("engine");  // TF32 = 1, TF32X3 = 2
    bool only_x3 = !mask_has(eng, ISPC_ENGINE_TF32);
    b.compute = flops * (only_x3 ? 3 : 1) / (kTf32Flops * sms / kSMs);
    tensor = true;
  } else {
    b.compute = flops / (sms * kFfmaPerSmClk * 2 * kFmax);
  }
  if (!tensor) b.compute = std::max(b.compute, per_thread / kFmax);
  if (f.kind == ISPC_TILE_SGEMM) {
    // shared-memory operand traffic: per k step a warp reads tm values for
    // each of its min(thr_m, 32) distinct rows and tn values for each of its
    // max(1, 32/thr_m) distinct columns (equal addresses broadcast), i.e.
    // (tm*min(tx,32) + tn*max(1,32/tx)) * 4 B per 32*tm*tn FMAs, at 128 B per
    // clock per SM; minimised over the values still open
    double best = std::numeric_limits<double>::infinity();
    for (std::int64_t tx : r.remaining("thr_m"))
      for (std::int64_t tm : r.remaining("tm"))
        for (std::int64_t tn : r.remaining("tn")) {
          double per_fma = (double(tm) * double(std::min<std::int64_t>(tx, 32)) +
                            double(tn) * double(std::max<std::int64_t>(1, 32 / std::max<std::int64_t>(tx, 1)))) *
                           4.0 / (32.0 * double(tm) * double(tn));
          best = std::min(best, per_fma);
        }
    if (std::isfinite(best)) b.compute = std::max(b.compute, flops / 2 * best / (sms * 128.0 * kFmax));
  }
  b.launch = kLaunch;
  b.total = std::max({b.dram, b.compute, b.launch});
  if (fully_specified(ctx, c)) {
    ispc_tile_config t = tile_config(f, ctx, c);
    ispc_launch L{};
    size_t len = 0;
    if (ispc_emit_tiles(&t, "k", nullptr, 0, &len, &L) != ISPC_OK) {
      b.illegal = true;
      b.total = std::numeric_limits<double>::infinity();
    }
  }
  return b;
}

}  // namespace ispc_host
