// B200 lower-bound performance model, in seconds.
//
// The reference's bound.cpp is a stub (proj/core/src/bound.cpp:1); its
// contract is SPEC.md:416-457: per-instruction independent minimisation over
// the remaining domains, admissible (never above the time of any completion)
// and monotone (a child's bound is never below its parent's). This model
// keeps that construction but prices a B200 instead of the reference's
// Kepler-like cycle table (machine.hpp:17-34), so pruning against MEASURED
// times stays sound. Each term is a resource every completion must consume:
//
//   dram    compulsory DRAM bytes (every input element read, every output
//           element written, plus the spill of any GLOBAL temporary larger than
//           L2) / nominal HBM3e bandwidth (7.7 TB/s, above the measured
//           6.55 TB/s copy peak so the bound stays below any achievable time)
//   sm_mem  the same global traffic / (active SMs x 256 B/cycle x f_max);
//           active SMs <= min(148, upper bound on the block count)
//   issue   warp instructions (instances / (min(32, threads/block) x vector
//           lanes)) / (active SMs x 4 schedulers x f_max)
//   thread  the sequential trips of one thread: every dim that cannot become
//           BLOCK/THREAD/VECTOR multiplies by its smallest possible extent;
//           one instruction per cycle at f_max, and each trip of the LOOPs
//           around a load waits for it (29 cycles, 234 for ld.global.cg);
//           times the waves the grid needs (blocks / (148 x resident blocks
//           per SM, <= 32 and <= 2048 / threads per block))
//   launch  1 us launch floor
//   dispatch  the blocks every completion launches x 0.5 ns: the B200's block
//           dispatch rate, measured with empty blocks (0.517 ns/block for
//           <= 128 threads, 1.02 ns for 1024; profiles/r2_block_dispatch.log)
//   l1      cache lines a warp access must touch: when every dim of a global
//           access that can be the warp's lane (innermost THREAD) dim walks
//           the address with stride s >= 2 elements, each warp access touches
//           ceil(lanes x min(s, 32) / 32) 128-byte lines; lines / (active SMs
//           x 2 lines/cycle x f_max) (the reference's coalescing rule,
//           simulate.cpp:46-60, priced as L1 wavefronts)
//   lsu     memory warp-instructions (instances / (active lanes x vector
//           lanes), as in `issue`) / (active SMs x 1 per cycle x f_max): the
//           load/store unit's issue floor (measured 1.82 cycles per LDG)
// bound = max of the terms. All domain reads take the most optimistic value
// still possible, so narrowing a domain can only raise a term (monotone), and
// a leaf's bound is below its measured time (admissible; checked on every
// evaluation by the search).
#pragma once

#include <cstdint>
#include <map>
#include <vector>

#include "ispace/candidate.hpp"
#include "ispace/kernels.hpp"

namespace ispc_host {

struct B200Machine {
  double f_max_hz = 1.965e9;
  int sms = 148;
  double hbm_bytes_per_s = 7.7e12;
  double sm_bytes_per_cycle = 256;
  double l2_bytes = 126.5e6;
  int issue_per_sm_cycle = 4;
  double launch_floor_s = 1e-6;
  int max_threads_per_block = 1024;
  bool l2_flushed = false;  // inputs start outside L2 (timed with an L2 flush)
  // per-thread budgets of the emitter (ispc_emit_opts); exceeding them makes
  // every completion unrunnable, i.e. an infinite bound
  // the search's emit budgets (ispc_search_config.max_unrolled default, the
  // register-array cap it passes to ispc_emit_cuda): one source of truth, so
  // ispc_bound reports +inf for exactly the leaves the search cannot run
  static constexpr int kDefaultMaxUnrolled = 512;
  static constexpr int kMaxRegElems = 160;
  double max_reg_elems = kMaxRegElems;
  double max_unrolled = kDefaultMaxUnrolled;
  // a loaded value is consumed in the iteration that loads it, and the
  // emitter keeps LOOP dimensions rolled (#pragma unroll 1): each trip of the
  // LOOP dimensions around a load waits at least the fastest load latency
  // (LDS 29 cycles, L1 hit 31.8; B300_MICROARCH.md)
  double min_load_latency_cycles = 29;
  // an ld.global.cg (cache = L2) bypasses L1: at least an L2 hit (234 cycles
  // near-die, B300_MICROARCH.md)
  double l2_load_latency_cycles = 234;
  // residency: at most 32 blocks and 2048 threads per SM, so a grid runs in
  // waves of 148 x that many blocks, each wave at least one block's
  // sequential time
  int max_blocks_per_sm = 32;
  int max_threads_per_sm = 2048;
  double block_dispatch_s = 0.5e-9;  // per block, whatever the block does
  // memory warp-instructions (global or shared, any width, any number of
  // active lanes) an SM's load/store unit accepts per cycle: measured LDG
  // issue floor 1.82 cycles per instruction (B300_MICROARCH.md "LDG"), 1 keeps
  // the term admissible; a warp of a 1-thread block moves one vector per
  // instruction, so tiny blocks pay it per element
  double lsu_per_cycle = 1;
  double l1_lines_per_cycle = 2;     // per SM (the L1 serves ~1 wavefront/clk; 2 keeps a margin)
};

// Why a subtree can never run correctly on the device (bound = +inf).
enum class Illegal : int { None = 0, Grid, CrossBlock, Registers, Unrolled };

struct BoundReport {
  Illegal illegal = Illegal::None;
  double total = 0, dram = 0, sm_mem = 0, issue = 0, thread = 0, launch = 0, dispatch = 0, l1 = 0, lsu = 0;
  double dram_bytes = 0;
  double blocks_max = 0, threads_per_block_max = 0;
};

class BoundModel {
 public:
  BoundModel(const ispace::Kernel& k, const ispace::SpaceContext& ctx, const B200Machine& m);
  BoundReport bound(const ispace::Candidate& c) const;
  const B200Machine& machine() const { return m_; }

 private:
  struct DimRec {
    ispace::ObjId id;
    bool is_static;
    ispace::ObjId logical;
    std::uint32_t kind_inst;  // dim_kind(d)
    std::uint32_t size_inst;  // size(d), static dims
  };
  struct InstRec {
    ispace::ObjId id;
    std::uint32_t lowering;
    std::vector<std::size_t> dims;  // indices into dims_
    double instances;               // product of logical extents
    bool memory;
    bool load;
    ispace::ObjId region;
    std::uint32_t cache_inst = ~0u;  // cache(inst), memory instructions
    // per position of `dims`: the address terms of that dim, (base, indices
    // of the dims whose sizes multiply it) - its element stride
    std::vector<std::vector<std::pair<double, std::vector<std::size_t>>>> stride_terms;
  };
  struct PairRec {
    std::size_t src, dst;  // dim indices
    std::uint32_t lowering;
  };
  std::vector<PairRec> comm_pairs_;
  std::vector<bool> inst_has_storage_;  // value-defining and not a reduction
  struct RegionRec {
    ispace::ObjId id;
    bool input;
    double bytes;
    std::uint32_t lowering;
    std::uint32_t space_inst;  // mem_space(r), kNoInstance for inputs
  };
  const ispace::Kernel& k_;
  const ispace::SpaceContext& ctx_;
  B200Machine m_;
  std::vector<DimRec> dims_;
  std::map<ispace::ObjId, std::size_t> dim_index_;
  std::vector<InstRec> insts_;
  std::vector<RegionRec> regions_;
  std::vector<std::vector<std::uint32_t>> pair_order_;  // order(a,b) instance per dim pair
  int v_loop_ = 0, v_block_ = 1, v_thread_ = 2, v_unroll_ = 3, v_vector_ = 4;
  int v_merged_ = 4, v_global_ = 0, v_cache_l2_ = 1;
  std::uint32_t order_c_ = 0;

  ispace::Mask kinds(const ispace::Candidate& c, std::size_t d) const;
  void extents(const ispace::Candidate& c, std::size_t d, double& lo, double& hi) const;
};

}  // namespace ispc_host
