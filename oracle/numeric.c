/*
 * CPU numeric oracle — TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker. The product path (libispc,
 * libispc_host) never links or calls it.
 *
 * What it restates: the values the reference's kernel backbones define
 * (proj/core/src/kernels.cpp). The reference never executes a kernel, so
 * there are no numeric golden vectors upstream; these functions are pinned
 * instead by tests/golden/*.json, outputs of an interpreter that executes the
 * reference's own Kernel objects instance by instance through the reference's
 * eval_addr/dim_extent (oracle/ref_golden.cpp, built from /root/reference by
 * oracle/Makefile; tests/test_oracle_golden.py checks these functions against it).
 *
 *   axpy    kernels.cpp:373-408  z[i] = add(mul(alpha, x[i]), y[i]) — two
 *           separately rounded fp32 operations
 *   outer   kernels.cpp:410-433  c[i*n + j] = mul(a[i], b[j])
 *   matmul  kernels.cpp:435-488  c[i + j*m] = mad over k ascending from a
 *           Cast-0 initializer; A[i*s + k*m*s], B[k + j*K] (column major, A
 *           element stride s)
 *   gemv    B200 extension (no reference builder, kernel_test.cpp:351):
 *           y[i] = mad over j ascending of A[i + j*m] * x[j]
 *   batched B200 extension: batch of independent column-major matmuls
 *
 * Inputs come from the same seeded generator the device uses
 * (paper_1904_03383_b200/csrc/builtins.cu input_value), so both sides see the
 * same bits.
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

static uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

float oracle_input_value(uint64_t seed, uint32_t tag, uint64_t i) {
  uint64_t h = splitmix64(splitmix64(seed ^ ((uint64_t)tag << 48)) + i);
  int32_t m = (int32_t)(h >> 40);
  return (float)((double)(m - 8388608) / 8388608.0);
}

void oracle_fill(float* p, int64_t n, uint64_t seed, uint32_t tag) {
  for (int64_t i = 0; i < n; ++i) p[i] = oracle_input_value(seed, tag, (uint64_t)i);
}

/* volatile-free but strictly IEEE: compiled with -ffp-contract=off so the
 * mul and add stay two roundings, and fmaf() is the single-rounding mad. */
void oracle_axpy(const float* x, const float* y, float* z, int64_t n, float alpha) {
  for (int64_t i = 0; i < n; ++i) {
    float t = alpha * x[i];
    z[i] = t + y[i];
  }
}

void oracle_outer(const float* a, const float* b, float* c, int64_t m, int64_t n) {
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) c[i * n + j] = a[i] * b[j];
}

void oracle_matmul(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k, int64_t s) {
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) {
      float acc = 0.0f;
      for (int64_t kk = 0; kk < k; ++kk) acc = fmaf(a[i * s + kk * m * s], b[kk + j * k], acc);
      c[i + j * m] = acc;
    }
}

void oracle_gemv(const float* a, const float* x, float* y, int64_t m, int64_t n) {
  for (int64_t i = 0; i < m; ++i) {
    float acc = 0.0f;
    for (int64_t j = 0; j < n; ++j) acc = fmaf(a[i + j * m], x[j], acc);
    y[i] = acc;
  }
}

/* fp64 reference with the |a||x| scale, for tolerance checks of reordered
 * (warp-shuffle / split-k) reductions. */
void oracle_gemv_f64(const float* a, const float* x, double* y, double* scale, int64_t m, int64_t n) {
  for (int64_t i = 0; i < m; ++i) {
    double acc = 0.0, sc = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      acc += (double)a[i + j * m] * (double)x[j];
      sc += fabs((double)a[i + j * m] * (double)x[j]);
    }
    y[i] = acc;
    scale[i] = sc;
  }
}

void oracle_batched(const float* a, const float* b, float* c, int64_t batch, int64_t m, int64_t n, int64_t k) {
  for (int64_t q = 0; q < batch; ++q)
    oracle_matmul(a + q * m * k, b + q * k * n, c + q * m * n, m, n, k, 1);
}
