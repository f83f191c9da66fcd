// C-ABI of the reference-side host library (include/ispc_host.h).
#include <chrono>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>

#include "adapter.hpp"
#include "host_internal.hpp"
#include "ispace/gpu_space.hpp"
#include "ispace/simulate.hpp"
#include "ispc_host.h"

namespace ispc_host {

namespace {
thread_local std::string g_err;
}

int set_err(int code, const std::string& s) {
  g_err = s;
  return code;
}

ispace::MachineParams machine_for(int mode) {
  ispace::MachineParams mp;  // defaults: the reference's parity machine (machine.hpp:17-34)
  if (mode == ISPC_SPACE_B200) {
    mp.max_threads = 1024;
    mp.max_thread_levels = 3;
    mp.max_block_levels = 3;
    mp.shared_capacity = 232448;  // 227 KiB opt-in per block
    mp.vector_width = 4;          // 128-bit ld/st.global.v4.f32
    mp.parallel_blocks = 148 * 16;
  }
  return mp;
}

PropStatusInt decide_named(const ispace::SpaceContext& ctx, ispace::Candidate& c, const std::string& choice,
                           const std::vector<std::string>& args, const std::string& value) {
  using namespace ispace;
  std::uint32_t ch = ctx.table.find_choice(choice);
  if (ch == kNoInstance) throw std::invalid_argument("unknown choice " + choice);
  std::vector<ObjId> ids;
  for (const auto& a : args) {
    ObjId o = ctx.bb.find(a);
    if (o == kNoObj) throw std::invalid_argument("unknown object " + a);
    ids.push_back(o);
  }
  InstanceRef ref = ctx.table.resolve(ch, ids.data(), ids.size());
  if (ref.inst == kNoInstance) throw std::invalid_argument("no instance of " + choice);
  int v = -1;
  if (ctx.table.choices[ch].kind == InstKind::Integer) {
    const auto& u = ctx.table.universe_of(ref.inst);
    for (size_t i = 0; i < u.size(); ++i)
      if (std::to_string(u[i]) == value) v = int(i);
  } else {
    v = ctx.table.value_index(ch, value);
    if (v >= 0 && ref.swapped) v = ctx.table.choices[ch].swap[size_t(v)];
  }
  if (v < 0) throw std::invalid_argument("unknown value " + value + " of " + choice);
  Candidate child;
  if (apply_decision(ctx, c, ref.inst, v, child) != PropStatus::Ok) return 1;
  c = std::move(child);
  return 0;
}

}  // namespace ispc_host

using namespace ispc_host;

struct ispc_nest_buf {
  std::unique_ptr<NestBuf> b;
};

extern "C" {

const char* ispc_host_last_error(void) { return g_err_text(); }

int ispc_space_create(const ispc_kernel_spec* spec, ispc_space** out) {
  try {
    if (!spec || !out || !spec->kind) return set_err(ISPC_E_ARG, "null argument");
    auto t0 = std::chrono::steady_clock::now();
    auto s = std::make_unique<ispc_space>();
    s->spec = *spec;
    s->kind = spec->kind;
    s->spec.kind = s->kind.c_str();
    ispace::KernelSpec ks;
    ks.kind = spec->kind;
    ks.m = spec->m;
    ks.n = spec->n;
    ks.k = spec->k;
    ks.a_stride = spec->a_stride > 0 ? spec->a_stride : 1;
    if (spec->num_factors < 0 || spec->num_factors > 4) return set_err(ISPC_E_ARG, "bad factor count");
    for (int i = 0; i < spec->num_factors; ++i) {
      if (spec->factor_len[i] <= 0 || spec->factor_len[i] > 32) return set_err(ISPC_E_ARG, "bad factor list");
      ks.factors.emplace_back(spec->factors[i], spec->factors[i] + spec->factor_len[i]);
    }
    ispace::BuildResult br;
    if (is_tile_kind(s->kind)) {
      s->tiles = std::make_unique<TileFamily>(make_family(s->kind, spec->m, spec->n, spec->k, spec->batch));
      br = build_tile_space(*s->tiles);
    } else {
      s->kernel = ispace::build_kernel(ks);
      s->mp = machine_for(spec->mode);
      br = ispace::build_gpu_space(s->kernel, s->mp);
    }
    if (!br.ctx) {
      std::string msg = "space build failed";
      for (const auto& d : br.diagnostics) msg += "\n" + d.message;
      return set_err(ISPC_E_ARG, msg);
    }
    s->ctx = br.ctx;
    if (ispace::make_root(*s->ctx, s->root) != ispace::PropStatus::Ok)
      return set_err(ISPC_E_ARG, "root candidate is a dead end");
    s->build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = s.release();
    return ISPC_OK;
  } catch (const std::exception& e) {
    return set_err(ISPC_E_ARG, e.what());
  }
}

void ispc_space_free(ispc_space* s) { delete s; }

int ispc_space_stats_get(const ispc_space* s, ispc_space_stats* o) {
  if (!s || !o) return set_err(ISPC_E_ARG, "null argument");
  std::memset(o, 0, sizeof(*o));
  const auto& t = s->ctx->table;
  o->instances = t.instances.size();
  for (const auto& in : t.instances) {
    switch (t.choices[in.choice].kind) {
      case ispace::InstKind::Enum: ++o->enum_instances; break;
      case ispace::InstKind::Integer: ++o->int_instances; break;
      case ispace::InstKind::Counter: ++o->counter_instances; break;
    }
  }
  o->objects = s->ctx->bb.objects.size();
  o->lowerings = s->ctx->bb.lowerings.size();
  o->root_open = ispace::open_choices(*s->ctx, s->root).size();
  o->root_digest = ispace::digest(*s->ctx, s->root);
  o->build_seconds = s->build_seconds;
  return ISPC_OK;
}

int ispc_space_problem(const ispc_space* s, ispc_problem* p) {
  if (!s || !p) return set_err(ISPC_E_ARG, "null argument");
  std::memset(p, 0, sizeof(*p));
  const std::string& k = s->kind;
  p->seed = 0x190403383ull;
  p->alpha = 1.5f;
  p->m = s->spec.m;
  p->n = s->spec.n;
  p->k = s->spec.k;
  p->a_stride = s->spec.a_stride > 0 ? s->spec.a_stride : 1;
  p->batch = 1;
  if (k == "axpy" || k == "axpy_stream") p->kind = ISPC_PROB_AXPY;
  else if (k == "outer_product") p->kind = ISPC_PROB_OUTER;
  else if (k == "matmul" || k == "sgemm" || k == "sgemm_tc" || k == "sgemm_tc_x3") p->kind = ISPC_PROB_MATMUL;
  else if (k == "gemv") p->kind = ISPC_PROB_GEMV;
  else if (k == "batched") {
    p->kind = ISPC_PROB_BATCHED;
    p->batch = s->spec.batch;
  }
  else return set_err(ISPC_E_ARG, "no problem for kernel kind " + k);
  return ISPC_OK;
}

int ispc_cand_root(const ispc_space* s, ispc_cand** out) {
  if (!s || !out) return set_err(ISPC_E_ARG, "null argument");
  *out = new ispc_cand{s->root};
  return ISPC_OK;
}

ispc_cand* ispc_cand_clone(const ispc_cand* c) { return c ? new ispc_cand{c->c} : nullptr; }
void ispc_cand_free(ispc_cand* c) { delete c; }

int ispc_cand_decide(const ispc_space* s, ispc_cand* c, const char* choice, const char* arg0, const char* arg1,
                     const char* value) {
  try {
    if (!s || !c || !choice || !value) return set_err(ISPC_E_ARG, "null argument");
    std::vector<std::string> args;
    if (arg0) args.push_back(arg0);
    if (arg1) args.push_back(arg1);
    return decide_named(*s->ctx, c->c, choice, args, value);
  } catch (const std::exception& e) {
    return set_err(ISPC_E_ARG, e.what());
  }
}

int ispc_cand_open_count(const ispc_space* s, const ispc_cand* c) {
  return int(ispace::open_choices(*s->ctx, c->c).size());
}
int ispc_cand_fully_specified(const ispc_space* s, const ispc_cand* c) {
  return ispace::fully_specified(*s->ctx, c->c) ? 1 : 0;
}
uint64_t ispc_cand_digest(const ispc_space* s, const ispc_cand* c) { return ispace::digest(*s->ctx, c->c); }
uint64_t ispc_cand_fired(const ispc_cand* c) { return c->c.fired; }

int ispc_cand_first_leaf(const ispc_space* s, const ispc_cand* from, int budget, ispc_cand** out) {
  if (!s || !from || !out) return set_err(ISPC_E_ARG, "null argument");
  ispace::Candidate leaf;
  int b = budget;
  if (!first_leaf(*s->ctx, from->c, leaf, &b)) return 1;
  *out = new ispc_cand{leaf};
  return 0;
}

int ispc_cand_random_leaf(const ispc_space* s, const ispc_cand* from, uint64_t seed, int max_restarts,
                          ispc_cand** out, int64_t* decisions, int64_t* dead_ends) {
  return ispc_cand_random_leaf_ordered(s, from, seed, nullptr, max_restarts, out, decisions, dead_ends);
}

int ispc_cand_random_leaf_ordered(const ispc_space* s, const ispc_cand* from, uint64_t seed, const char* order,
                                  int max_restarts, ispc_cand** out, int64_t* decisions, int64_t* dead_ends) {
  if (!s || !from || !out) return set_err(ISPC_E_ARG, "null argument");
  std::mt19937_64 rng(seed);
  DecisionOrder ord;
  if (order) {
    std::vector<std::string> names;
    std::string cur;
    for (const char* p = order;; ++p) {
      if (*p == ',' || *p == 0) {
        if (!cur.empty()) names.push_back(cur);
        cur.clear();
        if (!*p) break;
      } else {
        cur += *p;
      }
    }
    ord = DecisionOrder::from_names(*s->ctx, names);
  }
  int64_t dec = 0, dead = 0;
  ispace::Candidate leaf;
  bool ok = false;
  for (int attempt = 0; attempt <= max_restarts && !ok; ++attempt) {
    WalkResult w = random_walk(*s->ctx, from->c, rng, leaf, order ? &ord : nullptr);
    dec += w.decisions;
    if (w.ok) ok = true;
    else ++dead;
  }
  if (decisions) *decisions = dec;
  if (dead_ends) *dead_ends = dead;
  if (!ok) return 1;
  *out = new ispc_cand{leaf};
  return 0;
}

int64_t ispc_count_leaves(const ispc_space* s, const ispc_cand* from, int64_t cap) {
  if (!s || !from) return set_err(ISPC_E_ARG, "null argument");
  int64_t n = 0;
  count_leaves(*s->ctx, from->c, n, cap);
  return n;
}

int ispc_estimate_tree(const ispc_space* s, const ispc_cand* from, int64_t probes, uint64_t seed, const char* order,
                       double out[5]) {
  try {
    if (!s || !from || !out || probes <= 0) return set_err(ISPC_E_ARG, "bad argument");
    std::mt19937_64 rng(seed);
    DecisionOrder ord;
    if (order) {
      std::vector<std::string> names;
      std::string cur;
      for (const char* p = order;; ++p) {
        if (*p == ',' || *p == 0) {
          if (!cur.empty()) names.push_back(cur);
          cur.clear();
          if (!*p) break;
        } else {
          cur += *p;
        }
      }
      ord = DecisionOrder::from_names(*s->ctx, names);
    }
    TreeEstimate e = knuth_estimate(*s->ctx, from->c, probes, rng, order ? &ord : nullptr);
    out[0] = e.leaves;
    out[1] = e.leaves_stderr;
    out[2] = e.nodes;
    out[3] = e.dead_probe_ratio;
    out[4] = double(e.probes);
    return ISPC_OK;
  } catch (const std::exception& e) {
    return set_err(ISPC_E_ARG, e.what());
  }
}

int ispc_cand_to_tiles(const ispc_space* s, const ispc_cand* c, ispc_tile_config* out) {
  try {
    if (!s || !c || !out) return set_err(ISPC_E_ARG, "null argument");
    if (!s->tiles) return set_err(ISPC_E_ARG, "not a building-block space (use ispc_cand_to_nest)");
    *out = tile_config(*s->tiles, *s->ctx, c->c);
    return ISPC_OK;
  } catch (const std::exception& e) {
    return set_err(ISPC_E_ARG, e.what());
  }
}

int ispc_cand_to_nest(const ispc_space* s, const ispc_cand* c, ispc_nest_buf** out) {
  try {
    if (!s || !c || !out) return set_err(ISPC_E_ARG, "null argument");
    if (s->tiles) return set_err(ISPC_E_ARG, "building-block spaces have no loop nest (use ispc_cand_to_tiles)");
    ispace::LoopNest l = ispace::reconstruct(s->kernel, *s->ctx, c->c);
    auto nb = std::make_unique<ispc_nest_buf>();
    nb->b = flatten(s->kernel, l);
    *out = nb.release();
    return ISPC_OK;
  } catch (const std::exception& e) {
    return set_err(ISPC_E_ARG, e.what());
  }
}

const ispc_nest* ispc_nest_buf_get(const ispc_nest_buf* b) { return b ? &b->b->nest : nullptr; }
void ispc_nest_buf_free(ispc_nest_buf* b) { delete b; }

static int put_text(const std::string& s, char* buf, size_t cap, size_t* len) {
  if (len) *len = s.size();
  if (buf && cap) {
    size_t k = s.size() < cap - 1 ? s.size() : cap - 1;
    std::memcpy(buf, s.data(), k);
    buf[k] = 0;
  }
  return ISPC_OK;
}

int ispc_cand_reference_source(const ispc_space* s, const ispc_cand* c, char* buf, size_t cap, size_t* len) {
  try {
    if (s->tiles) return set_err(ISPC_E_ARG, "building-block spaces have no reference pseudo-source");
    ispace::LoopNest l = ispace::reconstruct(s->kernel, *s->ctx, c->c);
    return put_text(ispace::emit_source(s->kernel, l), buf, cap, len);
  } catch (const std::exception& e) {
    return set_err(ISPC_E_ARG, e.what());
  }
}

int ispc_cand_simulate(const ispc_space* s, const ispc_cand* c, int64_t out[5]) {
  try {
    if (s->tiles) return set_err(ISPC_E_ARG, "building-block spaces have no reference simulation");
    ispace::LoopNest l = ispace::reconstruct(s->kernel, *s->ctx, c->c);
    ispace::CostReport r = ispace::evaluate(s->kernel, l, s->mp);
    out[0] = r.compute;
    out[1] = r.memory;
    out[2] = r.sync;
    out[3] = r.block_serial;
    out[4] = r.total;
    return ISPC_OK;
  } catch (const std::exception& e) {
    return set_err(ISPC_E_ARG, e.what());
  }
}

int ispc_cand_serialize(const ispc_space* s, const ispc_cand* c, char* buf, size_t cap, size_t* len) {
  try {
    return put_text(ispace::serialize_text(*s->ctx, c->c), buf, cap, len);
  } catch (const std::exception& e) {
    return set_err(ISPC_E_ARG, e.what());
  }
}

int ispc_cand_deserialize(const ispc_space* s, const char* text, ispc_cand** out) {
  if (!s || !text || !out) return set_err(ISPC_E_ARG, "null argument");
  ispace::Candidate c;
  std::string err;
  if (!ispace::deserialize_text(*s->ctx, text, c, &err)) return set_err(ISPC_E_ARG, err);
  *out = new ispc_cand{c};
  return ISPC_OK;
}

}  // extern "C"

namespace ispc_host {
const char* g_err_text() { return g_err.c_str(); }
}  // namespace ispc_host
