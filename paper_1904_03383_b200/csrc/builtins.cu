// Fixed device kernels of the runtime (compiled ahead of time for sm_100a):
//   * seeded input generation (bit-identical to oracle/numeric.c's generator)
//   * golden kernels: the expected outputs of each problem, written as plain
//     sequential-order loops over the backbone semantics (kernels.cpp:373-488)
//     so every parity-mode schedule must match them bit for bit
//   * on-device output comparison
//   * globaltimer probe for the watchdog's host<->device clock offset
#include <cstdint>
#include <cuda_runtime.h>

#include "builtins.hpp"

namespace ispc {

__host__ __device__ inline uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Uniform in [-1, 1) on a 2^-23 grid: exactly representable, so the CPU
// oracle reproduces every bit.
__device__ inline float input_value(uint64_t seed, uint32_t tag, uint64_t i) {
  uint64_t h = splitmix64(splitmix64(seed ^ (uint64_t(tag) << 48)) + i);
  int32_t m = int32_t(h >> 40);  // 24 bits
  return float(m - 8388608) * 1.1920928955078125e-07f;
}

__global__ void fill_kernel(float* p, int64_t n, uint64_t seed, uint32_t tag) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    p[i] = input_value(seed, tag, i);
}

__global__ void axpy_golden(const float* x, const float* y, float* z, int64_t n, float alpha) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    z[i] = __fadd_rn(__fmul_rn(alpha, x[i]), y[i]);
}

__global__ void outer_golden(const float* a, const float* b, float* c, int64_t m, int64_t n) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < m * n; t += int64_t(gridDim.x) * blockDim.x)
    c[t] = __fmul_rn(a[t / n], b[t % n]);
}

// C[i + j*m] = sum_k A[i*s + k*m*s] * B[k + j*kk], k ascending from a 0 init.
// A tile of B columns is staged in shared memory; the per-element operation
// order is the sequential one regardless of staging.
__global__ void matmul_golden(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ c,
                              int64_t m, int64_t n, int64_t kk, int64_t s, int64_t batch_stride_a,
                              int64_t batch_stride_b, int64_t batch_stride_c, float* __restrict__ scale) {
  const int64_t bz = blockIdx.z;
  a += bz * batch_stride_a;
  b += bz * batch_stride_b;
  c += bz * batch_stride_c;
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  int64_t j = blockIdx.y;
  if (j >= n) return;
  __shared__ float bs[1024];
  float acc = 0.0f, sabs = 0.0f;
  for (int64_t k0 = 0; k0 < kk; k0 += 1024) {
    int64_t kn = kk - k0 < 1024 ? kk - k0 : 1024;
    __syncthreads();
    for (int64_t t = threadIdx.x; t < kn; t += blockDim.x) bs[t] = b[k0 + t + j * kk];
    __syncthreads();
    if (i < m)
      for (int64_t k = 0; k < kn; ++k) {
        float av = a[i * s + (k0 + k) * m * s];
        acc = __fmaf_rn(av, bs[k], acc);
        if (scale) sabs = __fmaf_rn(fabsf(av), fabsf(bs[k]), sabs);
      }
  }
  if (i < m) {
    c[i + j * m] = acc;
    if (scale) scale[bz * batch_stride_c + i + j * m] = sabs;
  }
}

// y[i] = sum_j A[i + j*m] * x[j], j ascending (gemv backbone order).
__global__ void gemv_golden(const float* __restrict__ a, const float* __restrict__ x, float* __restrict__ y,
                            int64_t m, int64_t n, float* __restrict__ scale) {
  int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= m) return;
  float acc = 0.0f, sabs = 0.0f;
  for (int64_t j = 0; j < n; ++j) {
    acc = __fmaf_rn(a[i + j * m], x[j], acc);
    sabs = __fmaf_rn(fabsf(a[i + j * m]), fabsf(x[j]), sabs);
  }
  y[i] = acc;
  if (scale) scale[i] = sabs;
}

struct CmpOut {
  unsigned long long mismatches;
  unsigned int max_err_bits;  // float bits of the max relative error (>= 0)
  unsigned int timeout;
};

__global__ void compare_kernel(const float* out, const float* exp, const float* scale, int64_t n, int bit_exact,
                               float rtol, CmpOut* res) {
  unsigned long long bad = 0;
  float worst = 0.0f;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    float o = out[i], e = exp[i];
    float den = scale ? scale[i] : fabsf(e);
    den = den > 1e-30f ? den : 1e-30f;
    float err = fabsf(o - e) / den;
    if (o != o) err = __int_as_float(0x7f800000);  // NaN output (unwritten) -> inf
    bool diff = bit_exact ? (__float_as_uint(o) != __float_as_uint(e)) : !(err <= rtol);
    bad += diff;
    worst = fmaxf(worst, err);
  }
  for (int off = 16; off; off >>= 1) {
    bad += __shfl_xor_sync(0xffffffffu, bad, off);
    worst = fmaxf(worst, __shfl_xor_sync(0xffffffffu, worst, off));
  }
  if ((threadIdx.x & 31) == 0) {
    if (bad) atomicAdd(&res->mismatches, bad);
    atomicMax(&res->max_err_bits, __float_as_uint(worst));
  }
}

// The same comparison behind the watchdog flag of the kernel just launched
// (float4 loads when the element count allows; the arithmetic per element is
// compare_kernel's).
__device__ __forceinline__ void cmp_one(float o, float e, float den, int bit_exact, float rtol,
                                        unsigned long long& bad, float& worst) {
  den = den > 1e-30f ? den : 1e-30f;
  float err = fabsf(o - e) / den;
  if (o != o) err = __int_as_float(0x7f800000);
  bool diff = bit_exact ? (__float_as_uint(o) != __float_as_uint(e)) : !(err <= rtol);
  bad += diff;
  worst = fmaxf(worst, err);
}

__global__ void check_kernel(const float* out, const float* exp, const float* scale, int64_t n, int bit_exact,
                             float rtol, const int* timeout_flag, CmpOut* res) {
  if (timeout_flag && *(volatile const int*)timeout_flag) {
    if (blockIdx.x == 0 && threadIdx.x == 0) res->timeout = 1;
    return;
  }
  unsigned long long bad = 0;
  float worst = 0.0f;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t t0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if ((n & 3) == 0 && ((reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(exp) |
                        reinterpret_cast<uintptr_t>(scale)) & 15) == 0) {
    const float4* o4 = reinterpret_cast<const float4*>(out);
    const float4* e4 = reinterpret_cast<const float4*>(exp);
    const float4* s4 = reinterpret_cast<const float4*>(scale);
    for (int64_t i = t0; i < n / 4; i += stride) {
      float4 o = __ldcs(o4 + i), e = __ldcs(e4 + i);
      float4 d = scale ? __ldcs(s4 + i) : make_float4(fabsf(e.x), fabsf(e.y), fabsf(e.z), fabsf(e.w));
      cmp_one(o.x, e.x, d.x, bit_exact, rtol, bad, worst);
      cmp_one(o.y, e.y, d.y, bit_exact, rtol, bad, worst);
      cmp_one(o.z, e.z, d.z, bit_exact, rtol, bad, worst);
      cmp_one(o.w, e.w, d.w, bit_exact, rtol, bad, worst);
    }
  } else {
    for (int64_t i = t0; i < n; i += stride) cmp_one(out[i], exp[i], scale ? scale[i] : fabsf(exp[i]), bit_exact, rtol, bad, worst);
  }
  for (int off = 16; off; off >>= 1) {
    bad += __shfl_xor_sync(0xffffffffu, bad, off);
    worst = fmaxf(worst, __shfl_xor_sync(0xffffffffu, worst, off));
  }
  if ((threadIdx.x & 31) == 0) {
    if (bad) atomicAdd(&res->mismatches, bad);
    atomicMax(&res->max_err_bits, __float_as_uint(worst));
  }
}

__global__ void collect_kernel(const int* timeout_flag, CmpOut* res) {
  if (*(volatile const int*)timeout_flag) res->timeout = 1;
}

// Reads the flush buffer after it was written: the written (dirty) lines are
// written back here, so the timed kernel starts on a clean L2 that holds none
// of its inputs.
__global__ void flush_read_kernel(const uint4* __restrict__ p, int64_t n, unsigned* sink) {
  unsigned acc = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    uint4 v = __ldcg(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x9e3779b9u) *sink = acc;  // practically never: keeps the loads alive
}

__global__ void fault_kernel(float* bad) { bad[threadIdx.x] = 1.0f; }

__global__ void timer_kernel(unsigned long long* out) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *out = t;
}

namespace {
int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return int(g < 1 ? 1 : g);
}
}  // namespace

cudaError_t launch_fill(float* p, int64_t n, uint64_t seed, uint32_t tag, cudaStream_t s) {
  fill_kernel<<<grid_for(n), 256, 0, s>>>(p, n, seed, tag);
  return cudaGetLastError();
}

cudaError_t launch_axpy_golden(const float* x, const float* y, float* z, int64_t n, float alpha,
                               cudaStream_t s) {
  axpy_golden<<<grid_for(n), 256, 0, s>>>(x, y, z, n, alpha);
  return cudaGetLastError();
}

cudaError_t launch_outer_golden(const float* a, const float* b, float* c, int64_t m, int64_t n,
                                cudaStream_t s) {
  outer_golden<<<grid_for(m * n), 256, 0, s>>>(a, b, c, m, n);
  return cudaGetLastError();
}

cudaError_t launch_matmul_golden(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k,
                                 int64_t a_stride, int64_t batch, float* scale, cudaStream_t s) {
  dim3 grid(unsigned((m + 127) / 128), unsigned(n), unsigned(batch));
  matmul_golden<<<grid, 128, 0, s>>>(a, b, c, m, n, k, a_stride, m * k * a_stride, k * n, m * n, scale);
  return cudaGetLastError();
}

cudaError_t launch_gemv_golden(const float* a, const float* x, float* y, int64_t m, int64_t n, float* scale,
                               cudaStream_t s) {
  gemv_golden<<<unsigned((m + 127) / 128), 128, 0, s>>>(a, x, y, m, n, scale);
  return cudaGetLastError();
}

cudaError_t launch_compare(const float* out, const float* exp, const float* scale, int64_t n, int bit_exact,
                           float rtol, void* dev_res, cudaStream_t s) {
  compare_kernel<<<grid_for(n), 256, 0, s>>>(out, exp, scale, n, bit_exact, rtol, static_cast<CmpOut*>(dev_res));
  return cudaGetLastError();
}

cudaError_t launch_check(const float* out, const float* exp, const float* scale, int64_t n, int bit_exact,
                         float rtol, const int* timeout_flag, void* slot, cudaStream_t s) {
  int64_t g = (n / 4 + 255) / 256;
  g = g < 1 ? 1 : g > 148 * 8 ? 148 * 8 : g;
  check_kernel<<<unsigned(g), 256, 0, s>>>(out, exp, scale, n, bit_exact, rtol, timeout_flag, static_cast<CmpOut*>(slot));
  return cudaGetLastError();
}

cudaError_t launch_collect(const int* timeout_flag, void* slot, cudaStream_t s) {
  collect_kernel<<<1, 1, 0, s>>>(timeout_flag, static_cast<CmpOut*>(slot));
  return cudaGetLastError();
}

cudaError_t launch_flush_read(const void* p, size_t bytes, void* sink, cudaStream_t s) {
  flush_read_kernel<<<148 * 8, 512, 0, s>>>(static_cast<const uint4*>(p), int64_t(bytes / 16),
                                            static_cast<unsigned*>(sink));
  return cudaGetLastError();
}

cudaError_t launch_timer(unsigned long long* out, cudaStream_t s) {
  timer_kernel<<<1, 1, 0, s>>>(out);
  return cudaGetLastError();
}

cudaError_t launch_fault(cudaStream_t s) {
  fault_kernel<<<1, 32, 0, s>>>(reinterpret_cast<float*>(uintptr_t(8)));
  return cudaGetLastError();
}

}  // namespace ispc
