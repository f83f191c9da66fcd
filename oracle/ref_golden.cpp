// Golden-vector generator — TEST INFRASTRUCTURE ONLY.
//
// Executes the reference's own Kernel objects (make_axpy / make_outer_product
// / make_matmul, proj/core/src/kernels.cpp:373-488) instance by instance:
// every instruction is evaluated at every point of its iteration space, every
// address comes from the reference's eval_addr() over its InductionVars
// (kernels.cpp:30-41), sizes from a reconstructed leaf of the reference's GPU
// space. The value flow follows the Operand kinds (kernels.hpp:32-43): Mapped
// operands read the producer at the paired indices, Reduce operands accumulate
// over the reduction dims in increasing order from the initializer. Nothing
// here shares code with oracle/numeric.c; tests/test_oracle_golden.py checks
// numeric.c bit-for-bit against the vectors written here.
//
// Usage: ref_golden <out.json>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <functional>
#include <map>
#include <string>
#include <vector>

#include "ispace/candidate.hpp"
#include "ispace/gpu_space.hpp"
#include "ispace/kernels.hpp"
#include "ispace/loop_nest.hpp"

using namespace ispace;

namespace {

uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// The generator both libispc's fill kernel and numeric.c implement; restated
// here independently from its definition (24 random bits on a 2^-23 grid).
float input(uint64_t seed, uint32_t tag, uint64_t i) {
  uint64_t h = splitmix64(splitmix64(seed ^ (uint64_t(tag) << 48)) + i);
  long m = long(h >> 40) - 8388608L;
  return float(std::ldexp(double(m), -23));
}

using Point = std::map<ObjId, std::int64_t>;

struct Interp {
  const Kernel& k;
  std::map<ObjId, std::int64_t> sizes;  // every dim's extent
  uint64_t seed;
  float alpha;
  std::map<ObjId, std::vector<float>> mem;  // region -> contents
  std::map<std::pair<ObjId, Point>, float> memo;

  std::string name(ObjId o) const { return k.bb.obj(o).name; }

  std::vector<float>& region(ObjId r) {
    auto it = mem.find(r);
    if (it != mem.end()) return it->second;
    const RegionInfo& ri = k.regions.at(r);
    std::vector<float> v(size_t(ri.elems), std::nanf(""));
    if (ri.input && name(r) != "z" && name(r) != "c")
      for (std::int64_t i = 0; i < ri.elems; ++i) v[size_t(i)] = input(seed, uint32_t(name(r)[0]), uint64_t(i));
    return mem[r] = v;
  }

  // A consumer outside the reduction reads the finished accumulator: the
  // producer's unpaired (reduction) dims sit at their last index.
  Point complete(ObjId producer, Point q) {
    for (ObjId d : k.insts.at(producer).dims)
      if (!q.count(d)) q[d] = sizes.at(d) - 1;
    return q;
  }

  float value(ObjId inst, const Point& p) {
    auto key = std::make_pair(inst, p);
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
    const InstInfo& ii = k.insts.at(inst);
    auto opnd = [&](const Operand& o) -> float {
      switch (o.kind) {
        case Operand::Kind::Const: return float(o.value);
        case Operand::Kind::Input:
          if (o.input != "alpha") throw std::runtime_error("unknown input " + o.input);
          return alpha;
        case Operand::Kind::Produced: {
          Point q;
          for (ObjId d : k.insts.at(o.producer).dims) q[d] = p.at(d);
          return value(o.producer, q);
        }
        case Operand::Kind::Mapped: {
          Point q;
          for (auto& [src, dst] : o.pairs) q[src] = p.at(dst);
          return value(o.producer, complete(o.producer, q));
        }
        default: throw std::runtime_error("unexpected operand");
      }
    };
    float r = 0;
    switch (ii.op) {
      case Op::Load: r = region(ii.region).at(size_t(eval_addr(k, k.ivars[ii.ivar], p, sizes))); break;
      case Op::Cast: r = opnd(ii.operands[0]); break;
      case Op::Mul: {
        volatile float a = opnd(ii.operands[0]), b = opnd(ii.operands[1]);
        r = a * b;
        break;
      }
      case Op::Add: {
        volatile float a = opnd(ii.operands[0]), b = opnd(ii.operands[1]);
        r = a + b;
        break;
      }
      case Op::Mad: {
        const Operand* red = nullptr;
        for (const Operand& o : ii.operands)
          if (o.kind == Operand::Kind::Reduce) red = &o;
        float a = opnd(ii.operands[0]), b = opnd(ii.operands[1]);
        float acc;
        // previous reduction point in lexicographic order of reduce_dims
        Point prev = p;
        bool first = true;
        for (auto it2 = red->reduce_dims.rbegin(); it2 != red->reduce_dims.rend(); ++it2) {
          if (prev.at(*it2) > 0) {
            prev[*it2] -= 1;
            first = false;
            break;
          }
          prev[*it2] = sizes.at(*it2) - 1;
        }
        if (first) {
          Point q;
          for (auto& [src, dst] : red->pairs) q[src] = p.at(dst);
          acc = value(red->init, q);
        } else {
          acc = value(inst, prev);
        }
        r = std::fmaf(a, b, acc);
        break;
      }
      default: throw std::runtime_error("value of a store");
    }
    memo[key] = r;
    return r;
  }

  void each_point(const std::vector<ObjId>& dims, const std::function<void(const Point&)>& f) {
    Point p;
    std::function<void(size_t)> rec = [&](size_t i) {
      if (i == dims.size()) return f(p);
      for (std::int64_t x = 0; x < sizes.at(dims[i]); ++x) {
        p[dims[i]] = x;
        rec(i + 1);
      }
    };
    rec(0);
  }

  void run() {
    for (const auto& [id, ii] : k.insts) {
      if (ii.op != Op::Store || k.bb.obj(id).lowering != kNoLowering) continue;
      std::vector<float>& out = region(ii.region);
      each_point(ii.dims, [&](const Point& p) {
        out.at(size_t(eval_addr(k, k.ivars[ii.ivar], p, sizes))) = opnd_store(ii, p);
      });
    }
  }

  float opnd_store(const InstInfo& ii, const Point& p) {
    const Operand& o = ii.operands[0];
    Point q;
    if (o.kind == Operand::Kind::Mapped)
      for (auto& [src, dst] : o.pairs) q[src] = p.at(dst);
    else
      for (ObjId d : k.insts.at(o.producer).dims) q[d] = p.at(d);
    return value(o.producer, complete(o.producer, q));
  }
};

struct Case {
  std::string label;
  KernelSpec spec;
};

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s out.json\n", argv[0]);
    return 2;
  }
  const uint64_t seed = 0x190403383ull;
  const float alpha = 1.5f;
  std::vector<Case> cases;
  auto add = [&](std::string label, std::string kind, std::int64_t m, std::int64_t n, std::int64_t kk,
                 std::vector<std::vector<std::int64_t>> f, std::int64_t s) {
    KernelSpec ks;
    ks.kind = kind;
    ks.m = m;
    ks.n = n;
    ks.k = kk;
    ks.factors = f;
    ks.a_stride = s;
    cases.push_back({label, ks});
  };
  add("axpy_64", "axpy", 0, 64, 0, {{2, 4}, {2, 4, 8}}, 1);
  add("axpy_1000", "axpy", 0, 1000, 0, {{2, 5}}, 1);
  add("outer_4x3", "outer_product", 4, 3, 0, {}, 1);
  add("outer_16x8", "outer_product", 16, 8, 0, {}, 1);
  add("matmul_8x8x8", "matmul", 8, 8, 8, {{2, 4}}, 1);
  add("matmul_16x8x4", "matmul", 16, 8, 4, {{2}, {2, 4}}, 1);
  add("strided_matmul_8x4x4_s3", "matmul", 8, 4, 4, {{2}}, 3);
  add("matmul_12x6x5", "matmul", 12, 6, 5, {{3}}, 1);
  // gemv and batched have no reference builder (kernel_test.cpp:351); their
  // semantics are the reference matmul's with n = 1 (y = A x, A column-major)
  // and a sequence of independent matmuls: pinned through these cases
  add("gemv_as_matmul_32x1x24", "matmul", 32, 1, 24, {}, 1);
  add("gemv_as_matmul_64x1x100", "matmul", 64, 1, 100, {}, 1);

  FILE* f = std::fopen(argv[1], "w");
  std::fprintf(f, "{\n  \"generator\": \"oracle/ref_golden.cpp (reference Kernel interpreted via eval_addr)\",\n");
  std::fprintf(f, "  \"seed\": %llu,\n  \"alpha\": %.9g,\n  \"cases\": [\n", (unsigned long long)seed, alpha);
  for (size_t ci = 0; ci < cases.size(); ++ci) {
    const Case& c = cases[ci];
    Kernel k = build_kernel(c.spec);
    MachineParams mp;
    BuildResult br = build_gpu_space(k, mp);
    Candidate root, leaf;
    make_root(*br.ctx, root);
    // sizes from a fully specified leaf (first-open DFS, nest_test.cpp:57-75)
    std::vector<std::uint32_t> open;
    Candidate cur = root;
    while (!(open = open_choices(*br.ctx, cur)).empty()) {
      Candidate child;
      Mask m = cur.dom[open.front()];
      bool moved = false;
      for (int v = kMaxDomainBits - 1; v >= 0 && !moved; --v)  // largest tiles first
        if (mask_has(m, v) && apply_decision(*br.ctx, cur, open.front(), v, child) == PropStatus::Ok) {
          cur = child;
          moved = true;
        }
      if (!moved) return 3;
    }
    LoopNest l = reconstruct(k, *br.ctx, cur);
    Interp in{k, l.sizes, seed, alpha, {}, {}};
    in.run();
    ObjId out = kNoObj;
    for (const auto& [id, ii] : k.insts)
      if (ii.op == Op::Store && k.bb.obj(id).lowering == kNoLowering) out = ii.region;
    const std::vector<float>& v = in.mem.at(out);
    std::fprintf(f, "    {\"label\": \"%s\", \"kind\": \"%s\", \"m\": %lld, \"n\": %lld, \"k\": %lld, \"a_stride\": %lld,",
                 c.label.c_str(), c.spec.kind.c_str(), (long long)c.spec.m, (long long)c.spec.n,
                 (long long)c.spec.k, (long long)c.spec.a_stride);
    std::fprintf(f, " \"sizes\": {");
    bool firsts = true;
    for (auto& [d, s] : l.sizes) {
      std::fprintf(f, "%s\"%s\": %lld", firsts ? "" : ", ", k.bb.obj(d).name.c_str(), (long long)s);
      firsts = false;
    }
    std::fprintf(f, "}, \"output\": \"%s\", \"bits\": [", k.bb.obj(out).name.c_str());
    for (size_t i = 0; i < v.size(); ++i) {
      uint32_t b;
      std::memcpy(&b, &v[i], 4);
      std::fprintf(f, "%s%u", i ? ", " : "", b);
    }
    std::fprintf(f, "]}%s\n", ci + 1 < cases.size() ? "," : "");
  }
  std::fprintf(f, "  ]\n}\n");
  std::fclose(f);
  return 0;
}
