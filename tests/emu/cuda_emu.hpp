// CPU emulation of the CUDA subset the ispc emitter produces — TEST
// INFRASTRUCTURE ONLY. Every CUDA thread of a block runs as a std::thread;
// __syncthreads() is a std::barrier, so barrier placement bugs show up as
// data races exactly like on the device. Blocks run one after another.
#pragma once
#include <atomic>
#include <barrier>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

struct emu_dim3 {
  unsigned x = 1, y = 1, z = 1;
};
inline thread_local emu_dim3 threadIdx, blockIdx;
inline emu_dim3 blockDim, gridDim;

struct float2 {
  float x, y;
};
struct float4 {
  float x, y, z, w;
};
inline float2 make_float2(float a, float b) { return {a, b}; }
inline float4 make_float4(float a, float b, float c, float d) { return {a, b, c, d}; }

inline std::barrier<>* emu_bar = nullptr;
inline std::atomic<int> emu_or{0};
inline void __syncthreads() { emu_bar->arrive_and_wait(); }
inline int __syncthreads_or(int p) {
  emu_bar->arrive_and_wait();
  if (p) emu_or.store(1);
  emu_bar->arrive_and_wait();
  int r = emu_or.load();
  emu_bar->arrive_and_wait();
  emu_or.store(0);  // every thread resets; all read r before this phase
  emu_bar->arrive_and_wait();
  return r;
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

#define __global__
#define __device__
#define __forceinline__
#define __shared__
#define __launch_bounds__(x)
#define __align__(x)
#define __restrict__ __restrict

inline int ispc_timeout_flag = 0;
inline unsigned long long ispc_now() { return 0; }
alignas(16) inline float ispc_smem[1 << 16];

template <class F>
void emu_launch(unsigned grid, unsigned bx, unsigned by, unsigned bz, F&& kernel) {
  blockDim = {bx, by, bz};
  gridDim = {grid, 1, 1};
  unsigned nt = bx * by * bz;
  for (unsigned b = 0; b < grid; ++b) {
    std::barrier<> bar(nt);
    emu_bar = &bar;
    std::vector<std::thread> ts;
    for (unsigned t = 0; t < nt; ++t)
      ts.emplace_back([&, t] {
        blockIdx = {b, 0, 0};
        threadIdx = {t % bx, (t / bx) % by, t / (bx * by)};
        kernel();
      });
    for (auto& th : ts) th.join();
  }
}
