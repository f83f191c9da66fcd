// CPU emulation of the CUDA subset the ispc emitter produces — TEST
// INFRASTRUCTURE ONLY. Every CUDA thread of a block runs as a user-space fiber
// (ucontext) on one OS thread; __syncthreads() parks the fiber until every
// fiber of the block arrived, so barrier placement decides which values a
// fiber can observe exactly as on the device. Fibers run in a fixed order
// between barriers (deterministic). Blocks run one after another.
#pragma once
#include <ucontext.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <vector>

struct emu_dim3 {
  unsigned x = 1, y = 1, z = 1;
};
inline emu_dim3 threadIdx, blockIdx, blockDim, gridDim;

struct float2 {
  float x, y;
};
struct float4 {
  float x, y, z, w;
};
inline float2 make_float2(float a, float b) { return {a, b}; }
inline float4 make_float4(float a, float b, float c, float d) { return {a, b, c, d}; }

struct EmuSched {
  ucontext_t main;
  std::vector<ucontext_t> ctx;
  std::vector<char*> stacks;
  std::vector<int> state;  // 0 runnable, 1 at barrier, 2 done
  int cur = -1;
  int or_accum = 0, or_result = 0;
  std::function<void()> kernel;
};
inline EmuSched* emu_s = nullptr;

inline void emu_yield_barrier() {
  EmuSched& s = *emu_s;
  s.state[size_t(s.cur)] = 1;
  swapcontext(&s.ctx[size_t(s.cur)], &s.main);
}
inline void __syncthreads() { emu_yield_barrier(); }
inline int __syncthreads_or(int p) {
  if (p) emu_s->or_accum = 1;
  emu_yield_barrier();
  return emu_s->or_result;
}

template <class T>
inline T emu_ld(const T* p) {
  T v;
  std::memcpy(&v, p, sizeof(T));
  return v;
}
template <class T>
inline void emu_st(T* p, T v) {
  std::memcpy(p, &v, sizeof(T));
}
#define __ldca(p) emu_ld(p)
#define __ldcg(p) emu_ld(p)
#define __ldcs(p) emu_ld(p)
#define __ldg(p) emu_ld(p)
#define ispc_ld_stream(p) emu_ld(p)
#define __stwb(p, v) emu_st(p, v)
#define __stcg(p, v) emu_st(p, v)
#define __stcs(p, v) emu_st(p, v)

inline float __fmul_rn(float a, float b) {
  volatile float r = a * b;
  return r;
}
inline float __fadd_rn(float a, float b) {
  volatile float r = a + b;
  return r;
}
inline float __fmaf_rn(float a, float b, float c) { return std::fmaf(a, b, c); }
inline float2 __ffma2_rn(float2 a, float2 b, float2 c) { return {std::fmaf(a.x, b.x, c.x), std::fmaf(a.y, b.y, c.y)}; }

#define __global__
#define __device__
#define __forceinline__
#define __shared__
#define __launch_bounds__(x)
#define __align__(x)
#define __restrict__ __restrict

// warp-level exchange and the tile kernels' building blocks. The emulated
// kernels call these uniformly across the block, so a block-wide phase
// boundary stands in for the warp-wide one.
inline float emu_xchg[1024];
inline unsigned emu_tid() { return threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z); }
inline float __shfl_xor_sync(unsigned, float v, int off) {
  const unsigned t = emu_tid();
  emu_xchg[t] = v;
  emu_yield_barrier();
  float r = emu_xchg[t ^ unsigned(off)];
  emu_yield_barrier();
  return r;
}
inline void __syncwarp() { emu_yield_barrier(); }
inline void ispc_cp_async_cg16(void* s, const void* g) { std::memcpy(s, g, 16); }
inline void ispc_cp_async_ca16(void* s, const void* g) { std::memcpy(s, g, 16); }
inline void ispc_cp_async_ca8(void* s, const void* g) { std::memcpy(s, g, 8); }
inline void ispc_cp_async_ca4(void* s, const void* g) { std::memcpy(s, g, 4); }
inline void ispc_cp_async_commit() {}
inline void ispc_grid_dep_wait() {}
inline void ispc_grid_dep_trigger() {}
template <int N>
inline void ispc_cp_async_wait() {}
inline unsigned ispc_cluster_rank() { return 0; }  // clusters of one CTA only
inline void ispc_cluster_sync() { emu_yield_barrier(); }
inline float ispc_dsmem_ld(const float* p, unsigned) { return *p; }
inline float4 ispc_dsmem_ld4(const float* p, unsigned) { return emu_ld(reinterpret_cast<const float4*>(p)); }
inline void ispc_dsmem_st4(float* p, unsigned, float4 v) { emu_st(reinterpret_cast<float4*>(p), v); }

inline int ispc_timeout_flag = 0;
inline unsigned long long ispc_deadline_at = ~0ull;  // the emulator never times out
inline unsigned long long ispc_now() { return 0; }
alignas(16) inline float ispc_smem[1 << 16];
inline unsigned ispc_smem_addr(const void* p) {
  return unsigned(static_cast<const char*>(p) - reinterpret_cast<const char*>(ispc_smem));
}
inline float4 ispc_lds4(unsigned a) {
  return emu_ld(reinterpret_cast<const float4*>(reinterpret_cast<const char*>(ispc_smem) + a));
}
inline void ispc_cp_async_cg16_s(unsigned s, const void* g) { std::memcpy(reinterpret_cast<char*>(ispc_smem) + s, g, 16); }
inline void ispc_cp_async_ca16_s(unsigned s, const void* g) { std::memcpy(reinterpret_cast<char*>(ispc_smem) + s, g, 16); }
inline void ispc_cp_async_ca4_s(unsigned s, const void* g) { std::memcpy(reinterpret_cast<char*>(ispc_smem) + s, g, 4); }

inline void emu_fiber_entry() {
  emu_s->kernel();
  emu_s->state[size_t(emu_s->cur)] = 2;
  swapcontext(&emu_s->ctx[size_t(emu_s->cur)], &emu_s->main);
}

// Returns 0 on success, 1 when fibers deadlock (some finished while others
// wait at a barrier), 2 when the kernel exceeds `max_phases` barrier phases
// (too long to emulate).
template <class F>
int emu_launch(unsigned grid, unsigned bx, unsigned by, unsigned bz, F&& kernel, long max_phases = 20000) {
  blockDim = {bx, by, bz};
  gridDim = {grid, 1, 1};
  const unsigned nt = bx * by * bz;
  const size_t stack = 256 * 1024;
  EmuSched s;
  emu_s = &s;
  s.kernel = kernel;
  s.ctx.resize(nt);
  s.state.assign(nt, 0);
  for (unsigned t = 0; t < nt; ++t) s.stacks.push_back(static_cast<char*>(std::malloc(stack)));
  int rc = 0;
  for (unsigned b = 0; b < grid && !rc; ++b) {
    blockIdx = {b, 0, 0};
    for (unsigned t = 0; t < nt; ++t) {
      getcontext(&s.ctx[t]);
      s.ctx[t].uc_stack.ss_sp = s.stacks[t];
      s.ctx[t].uc_stack.ss_size = stack;
      s.ctx[t].uc_link = nullptr;
      makecontext(&s.ctx[t], emu_fiber_entry, 0);
      s.state[t] = 0;
    }
    for (;;) {
      for (unsigned t = 0; t < nt; ++t) {
        if (s.state[t] != 0) continue;
        s.cur = int(t);
        threadIdx = {t % bx, (t / bx) % by, t / (bx * by)};
        swapcontext(&s.main, &s.ctx[t]);
      }
      unsigned done = 0, waiting = 0;
      for (unsigned t = 0; t < nt; ++t) {
        done += s.state[t] == 2;
        waiting += s.state[t] == 1;
      }
      if (done == nt) break;
      if (done && waiting) {
        rc = 1;
        break;
      }
      if (--max_phases < 0) {
        rc = 2;
        break;
      }
      s.or_result = s.or_accum;
      s.or_accum = 0;
      for (unsigned t = 0; t < nt; ++t)
        if (s.state[t] == 1) s.state[t] = 0;
    }
  }
  for (char* p : s.stacks) std::free(p);
  emu_s = nullptr;
  return rc;
}
