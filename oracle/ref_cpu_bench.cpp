// The reference's own CPU evaluation path, timed — TEST/BASELINE
// INFRASTRUCTURE ONLY (bench.py's cpu_baseline leg and `--impl reference`).
//
// Runs, on P host threads sharing one read-only SpaceContext, seeded uniform
// first-open random descents through the reference's apply_decision
// (propagate.cpp:445-448); every leaf reached goes through the reference's
// complete evaluation: reconstruct (loop_nest.cpp:111-332) + evaluate
// (simulate.cpp:131-133). Nothing of this repository's backend is involved.
//
// Usage: ref_cpu_bench <kind> <n|m> <n> <k> <seconds> <threads> <factor-list>...
//   factor list: comma separated sizes per universe, e.g. 2,4 2,4,8,...,1024
// Prints one JSON object. With REF_DUMP_WALKS=K in the environment it instead
// runs thread 0's first K walks and prints their leaf digests (0 = dead end):
// the walk ispc_walk_digests must reproduce (tests/test_spec_search.py).
#include <atomic>
#include <limits>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "ispace/candidate.hpp"
#include "ispace/gpu_space.hpp"
#include "ispace/kernels.hpp"
#include "ispace/loop_nest.hpp"
#include "ispace/simulate.hpp"

using namespace ispace;

int main(int argc, char** argv) {
  if (argc < 7) {
    std::fprintf(stderr, "usage: %s kind m n k seconds threads [factors...]\n", argv[0]);
    return 2;
  }
  KernelSpec ks;
  ks.kind = argv[1];
  ks.m = std::atoll(argv[2]);
  ks.n = std::atoll(argv[3]);
  ks.k = std::atoll(argv[4]);
  double seconds = std::atof(argv[5]);
  int threads = std::atoi(argv[6]);
  for (int i = 7; i < argc; ++i) {
    std::vector<std::int64_t> u;
    std::stringstream ss(argv[i]);
    std::string tok;
    while (std::getline(ss, tok, ',')) u.push_back(std::atoll(tok.c_str()));
    ks.factors.push_back(u);
  }
  auto t0 = std::chrono::steady_clock::now();
  Kernel k = build_kernel(ks);
  MachineParams mp;
  BuildResult br = build_gpu_space(k, mp);
  if (!br.ctx) {
    std::fprintf(stderr, "space build failed\n");
    return 1;
  }
  Candidate root;
  make_root(*br.ctx, root);
  double build_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

  if (const char* dump = std::getenv("REF_DUMP_WALKS")) {
    std::mt19937_64 rng(0x190403383ull);  // thread 0's generator
    const long long K = std::atoll(dump);
    std::printf("{\"seed\": %llu, \"digests\": [", 0x190403383ull);
    for (long long w = 0; w < K; ++w) {
      Candidate cur = root;
      bool ok = true;
      for (;;) {
        std::vector<std::uint32_t> open = open_choices(*br.ctx, cur);
        if (open.empty()) break;
        Mask m = cur.dom[open.front()];
        int pick = int(rng() % std::uint64_t(mask_count(m)));
        int v = 0;
        for (int b = 0; b < kMaxDomainBits; ++b)
          if (mask_has(m, b) && pick-- == 0) {
            v = b;
            break;
          }
        Candidate child;
        if (apply_decision(*br.ctx, cur, open.front(), v, child) != PropStatus::Ok) {
          ok = false;
          break;
        }
        cur = std::move(child);
      }
      std::printf("%s\"%llu\"", w ? ", " : "", ok ? (unsigned long long)digest(*br.ctx, cur) : 0ull);
    }
    std::printf("]}\n");
    return 0;
  }
  std::atomic<long long> walks{0}, leaves{0}, decisions{0}, dead{0};
  std::atomic<long long> best{std::numeric_limits<long long>::max()};
  auto deadline = std::chrono::steady_clock::now() + std::chrono::duration<double>(seconds);
  auto worker = [&](int tid) {
    std::mt19937_64 rng(0x190403383ull + 7919ull * tid);
    while (std::chrono::steady_clock::now() < deadline) {
      Candidate cur = root;
      bool ok = true;
      for (;;) {
        std::vector<std::uint32_t> open = open_choices(*br.ctx, cur);
        if (open.empty()) break;
        Mask m = cur.dom[open.front()];
        int pick = int(rng() % std::uint64_t(mask_count(m)));
        int v = 0;
        for (int b = 0; b < kMaxDomainBits; ++b)
          if (mask_has(m, b) && pick-- == 0) {
            v = b;
            break;
          }
        Candidate child;
        decisions.fetch_add(1);
        if (apply_decision(*br.ctx, cur, open.front(), v, child) != PropStatus::Ok) {
          ok = false;
          break;
        }
        cur = std::move(child);
      }
      walks.fetch_add(1);
      if (!ok) {
        dead.fetch_add(1);
        continue;
      }
      LoopNest l = reconstruct(k, *br.ctx, cur);
      CostReport r = evaluate(k, l, mp);
      leaves.fetch_add(1);
      long long prev = best.load();
      while (r.total < prev && !best.compare_exchange_weak(prev, r.total)) {
      }
    }
  };
  auto t1 = std::chrono::steady_clock::now();
  std::vector<std::thread> ts;
  for (int i = 0; i < threads; ++i) ts.emplace_back(worker, i);
  for (auto& t : ts) t.join();
  double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
  std::printf(
      "{\"kind\": \"%s\", \"threads\": %d, \"seconds\": %.3f, \"build_seconds\": %.3f, \"walks\": %lld, "
      "\"leaves\": %lld, \"decisions\": %lld, \"dead_ends\": %lld, \"leaves_per_s\": %.3f, "
      "\"walks_per_s\": %.3f, \"best_simulated_cycles\": %lld}\n",
      ks.kind.c_str(), threads, el, build_s, walks.load(), leaves.load(), decisions.load(), dead.load(),
      leaves.load() / el, walks.load() / el, best.load());
  return 0;
}
