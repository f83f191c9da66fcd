#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ispc {

// Per-evaluation result slot on the device: the compare kernel's verdict and
// the watchdog flag of the kernel it checked (copied out of the module).
struct CmpResult {
  unsigned long long mismatches;
  unsigned int max_err_bits;
  unsigned int timeout;
};

cudaError_t launch_fill(float* p, int64_t n, uint64_t seed, uint32_t tag, cudaStream_t s);
cudaError_t launch_axpy_golden(const float* x, const float* y, float* z, int64_t n, float alpha,
                               cudaStream_t s);
cudaError_t launch_outer_golden(const float* a, const float* b, float* c, int64_t m, int64_t n,
                                cudaStream_t s);
cudaError_t launch_matmul_golden(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k,
                                 int64_t a_stride, int64_t batch, float* scale, cudaStream_t s);
cudaError_t launch_gemv_golden(const float* a, const float* x, float* y, int64_t m, int64_t n, float* scale,
                               cudaStream_t s);
cudaError_t launch_compare(const float* out, const float* exp, const float* scale, int64_t n, int bit_exact,
                           float rtol, void* dev_res, cudaStream_t s);
// Compare that first reads the module's watchdog flag: a timed-out kernel's
// output is partial, so only the flag is recorded (slot->timeout = 1).
cudaError_t launch_check(const float* out, const float* exp, const float* scale, int64_t n, int bit_exact,
                         float rtol, const int* timeout_flag, void* slot, cudaStream_t s);
// slot->timeout |= *timeout_flag (timed launches that are not checked)
cudaError_t launch_collect(const int* timeout_flag, void* slot, cudaStream_t s);
cudaError_t launch_timer(unsigned long long* out, cudaStream_t s);
cudaError_t launch_flush_read(const void* p, size_t bytes, void* sink, cudaStream_t s);
// Fault injection (tests of the context-respawn path): a store through an
// invalid address, i.e. a context-killing illegal-address fault.
cudaError_t launch_fault(cudaStream_t s);

}  // namespace ispc
