// Development probe (not product): what one launch can stream from HBM at the
// gemv 4096^2 size (64 MiB), and gemv structures that approach it, timed like
// the bench (back-to-back launches over rotating copies larger than L2).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/gemv_lab tools/gemv_lab.cu -lcublas -lcuda
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      std::exit(1);                                                                  \
    }                                                                                \
  } while (0)

constexpr int M = 4096, N = 4096, NCOPY = 6, R = 48;

__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

// pure read: grid-stride over n4 float4s, U loads in flight per thread
template <int U>
__global__ void read_k(const float4* __restrict__ a, long long n4, float* out) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // no-ops unless launched with PDL
  asm volatile("griddepcontrol.launch_dependents;");
  float s = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld_stream(a + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  for (; i < n4; i += stride) {
    float4 v = ld_stream(a + i);
    s += v.x + v.y + v.z + v.w;
  }
  if (s == 12345.678f) out[0] = s;
}

// pure read, contiguous chunk per CTA (each CTA walks its own 64 MiB / grid)
template <int U>
__global__ void read_chunk_k(const float4* __restrict__ a, long long n4, float* out) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const long long per = n4 / gridDim.x;
  const float4* p = a + per * blockIdx.x;
  float s = 0;
  long long i = threadIdx.x;
  for (; i + (long long)(U - 1) * blockDim.x < per; i += (long long)U * blockDim.x) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld_stream(p + i + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  for (; i < per; i += blockDim.x) {
    float4 v = ld_stream(p + i);
    s += v.x + v.y + v.z + v.w;
  }
  if (s == 12345.678f) out[0] = s;
}

// gemv, column blocks: CTA c owns columns [c*CPB, (c+1)*CPB) for all M rows;
// thread t owns rows 4t..4t+3 of each column of its slice (blockDim = M/4/RS
// threads per row-slice... here: blockDim.x threads cover M rows as float4,
// RS = M / (4 * blockDim.x) row groups per thread), U columns in flight.
// Partial y of each CTA -> atomicAdd (norm-wise checked).
template <int T, int U>
__global__ void __launch_bounds__(T) gemv_cols_k(const float* __restrict__ A, const float* __restrict__ x,
                                                 float* __restrict__ y, int cpb) {
  constexpr int RG = M / 4 / T;  // float4 row groups per thread
  float4 acc[RG];
#pragma unroll
  for (int r = 0; r < RG; ++r) acc[r] = make_float4(0, 0, 0, 0);
  const int j0 = blockIdx.x * cpb;
  for (int j = j0; j < j0 + cpb; j += U) {
    float xs[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xs[u] = __ldg(x + j + u);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float4* col = (const float4*)(A + (long long)(j + u) * M);
#pragma unroll
      for (int r = 0; r < RG; ++r) {
        float4 v = ld_stream(col + threadIdx.x + r * T);
        acc[r].x = fmaf(v.x, xs[u], acc[r].x);
        acc[r].y = fmaf(v.y, xs[u], acc[r].y);
        acc[r].z = fmaf(v.z, xs[u], acc[r].z);
        acc[r].w = fmaf(v.w, xs[u], acc[r].w);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < RG; ++r) {
    float* py = y + 4 * (threadIdx.x + r * T);
    atomicAdd(py + 0, acc[r].x);
    atomicAdd(py + 1, acc[r].y);
    atomicAdd(py + 2, acc[r].z);
    atomicAdd(py + 3, acc[r].w);
  }
}

// pure read through a cp.async.bulk (TMA 1-D) ring: one elected thread per
// CTA streams CH-byte chunks of the CTA's contiguous slice into S stages; all
// threads consume each landed chunk
template <int CH, int S>
__global__ void __launch_bounds__(256) read_bulk_k(const float* __restrict__ a, long long n, float* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) unsigned long long full[S], empty[S];
  // chunks b, b + G, b + 2G, ... of the whole array
  const long long total = n * 4 / CH;
  const int nch = int((total - blockIdx.x + gridDim.x - 1) / gridDim.x);
  const float* p = a;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      unsigned fa = (unsigned)__cvta_generic_to_shared(&full[s]), ea = (unsigned)__cvta_generic_to_shared(&empty[s]);
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(fa));
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(ea), "r"((int)blockDim.x));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](int c) {
    const int s = c % S;
    unsigned fa = (unsigned)__cvta_generic_to_shared(&full[s]);
    unsigned dst = (unsigned)__cvta_generic_to_shared(smem + s * CH);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(fa), "r"(CH));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(p + ((long long)c * gridDim.x + blockIdx.x) * (CH / 4)), "r"(CH), "r"(fa)
                 : "memory");
  };
  if (threadIdx.x == 0)
    for (int c = 0; c < S && c < nch; ++c) issue(c);
  float sum = 0;
  for (int c = 0; c < nch; ++c) {
    const int s = c % S;
    const unsigned ph = (c / S) & 1;
    unsigned fa = (unsigned)__cvta_generic_to_shared(&full[s]);
    asm volatile(
        "{ .reg .pred P; W: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra W; }" ::"r"(fa), "r"(ph));
    const float4* q = (const float4*)(smem + s * CH);
    for (int i = threadIdx.x; i < CH / 16; i += blockDim.x) {
      float4 v = q[i];
      sum += v.x + v.y + v.z + v.w;
    }
    unsigned ea = (unsigned)__cvta_generic_to_shared(&empty[s]);
    asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(ea));
    if (threadIdx.x == 0 && c + S < nch) {
      asm volatile(
          "{ .reg .pred P; W2: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra W2; }" ::"r"(ea), "r"(ph));
      issue(c + S);
    }
  }
  if (sum == 12345.678f) out[0] = sum;
}


// gemv "chunk" layout: CTA (rb, cb) reads rows [rb*R, rb*R+R) of columns
// [cb*C, cb*C+C) (C segments of R*4 bytes); thread t owns rows 4t..4t+3 and
// keeps one float4 per column in flight. Clusters of CL CTAs along columns
// sum their partials through DSMEM; each cluster's partial goes to a
// workspace; the last cluster of a row block (atomic counter) sums the
// workspace column and writes y, then resets the counter.
template <int R, int C, int CL>
__global__ void __launch_bounds__(R / 4) gemv_chunk_k(const float* __restrict__ A, const float* __restrict__ x,
                                                    float* __restrict__ y, float* __restrict__ ws,
                                                    unsigned* __restrict__ counters) {
  constexpr int T = R / 4, NCB = N / C, NCL = NCB / CL;  // column blocks, clusters per row block
  __shared__ __align__(16) float4 part[T];
  __shared__ bool last;
  const int rb = blockIdx.x / NCB, cb = blockIdx.x % NCB;
  const int t = threadIdx.x;
  const float4* col = (const float4*)(A + (long long)cb * C * M + rb * R) + t;
  float4 v[C];
#pragma unroll
  for (int c = 0; c < C; ++c) v[c] = ld_stream(col + (long long)c * (M / 4));
  float4 acc = make_float4(0, 0, 0, 0);
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const float xc = __ldg(x + cb * C + c);
    acc.x = fmaf(v[c].x, xc, acc.x); acc.y = fmaf(v[c].y, xc, acc.y);
    acc.z = fmaf(v[c].z, xc, acc.z); acc.w = fmaf(v[c].w, xc, acc.w);
  }
  part[t] = acc;
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (rank == 0) {
    float4 s = acc;
    const unsigned a = (unsigned)__cvta_generic_to_shared(&part[t]);
#pragma unroll
    for (unsigned q = 1; q < CL; ++q) {
      unsigned r;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(q));
      float4 o;
      asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(o.x), "=f"(o.y), "=f"(o.z), "=f"(o.w) : "r"(r));
      s.x += o.x; s.y += o.y; s.z += o.z; s.w += o.w;
    }
    const int cl = cb / CL;
    ((float4*)(ws + ((long long)rb * NCL + cl) * R))[t] = s;
    __threadfence();
    __syncthreads();
    if (t == 0) last = atomicAdd(counters + rb, 1u) == NCL - 1;
    __syncthreads();
    if (last) {
      __threadfence();
      float4 tot = make_float4(0, 0, 0, 0);
      for (int q = 0; q < NCL; ++q) {
        const float4 o = __ldcg((const float4*)(ws + ((long long)rb * NCL + q) * R) + t);
        tot.x += o.x; tot.y += o.y; tot.z += o.z; tot.w += o.w;
      }
      ((float4*)(y + rb * R))[t] = tot;
      if (t == 0) counters[rb] = 0;
    }
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void zero_k(float* y, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = 0;
}

template <class F>
float timeit(F launch, cudaStream_t st) {
  for (int w = 0; w < 3; ++w) launch(w % NCOPY);
  CK(cudaStreamSynchronize(st));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<float> ts;
  for (int t = 0; t < 7; ++t) {
    cudaEventRecord(e0, st);
    for (int r = 0; r < R; ++r) launch(r % NCOPY);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ts.push_back(ms * 1e3f / R);
  }
  CK(cudaGetLastError());
  std::sort(ts.begin(), ts.end());
  return ts[3];
}

template <class K>
void launch_pdl(K kern, int g, int t, cudaStream_t st, const float4* a, long long n4, float* out) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g), cfg.blockDim = dim3(t), cfg.dynamicSmemBytes = 0, cfg.stream = st;
  cfg.attrs = at, cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, kern, a, n4, out));
}

int main() {
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  const long long nA = (long long)M * N;
  std::vector<float*> A(NCOPY), X(NCOPY), Y(NCOPY);
  std::vector<float> h(nA);
  srand(3);
  for (auto& v : h) v = float(rand() % 2001 - 1000) / 1024.f;
  for (int c = 0; c < NCOPY; ++c) {
    CK(cudaMalloc(&A[c], nA * 4));
    CK(cudaMalloc(&X[c], N * 4));
    CK(cudaMalloc(&Y[c], M * 4));
    CK(cudaMemcpy(A[c], h.data(), nA * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(X[c], h.data(), N * 4, cudaMemcpyHostToDevice));
  }
  float* out;
  CK(cudaMalloc(&out, 64));
  const double bytes_read = nA * 4.0, bytes_gemv = 4.0 * (nA + M + N);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  std::printf("SMs %d\n", sms);
#define READ(U, G, T)                                                                                    \
  {                                                                                                      \
    float us = timeit([&](int c) { read_k<U><<<G, T, 0, st>>>((const float4*)A[c], nA / 4, out); }, st); \
    std::printf("read grid-stride U%-2d grid %5d x %4d: %7.2f us  %7.1f GB/s\n", U, G, T, us, bytes_read / us / 1e3); \
  }
#define READP(U, G, T)                                                                                   \
  {                                                                                                      \
    float us = timeit([&](int c) { launch_pdl(read_k<U>, G, T, st, (const float4*)A[c], nA / 4, out); }, st); \
    std::printf("read grid-stride U%-2d grid %5d x %4d PDL: %7.2f us  %7.1f GB/s\n", U, G, T, us, bytes_read / us / 1e3); \
  }
#define CHUNKP(U, G, T)                                                                                   \
  {                                                                                                      \
    float us = timeit([&](int c) { launch_pdl(read_chunk_k<U>, G, T, st, (const float4*)A[c], nA / 4, out); }, st); \
    std::printf("read chunked    U%-2d grid %5d x %4d PDL: %7.2f us  %7.1f GB/s\n", U, G, T, us, bytes_read / us / 1e3); \
  }
  READP(8, 16 * sms, 128);
  READP(8, 8 * sms, 256);
  READP(4, 8 * sms, 256);
  READP(16, 4 * sms, 256);
  READP(8, 2 * sms, 512);
  CHUNKP(4, 2048, 256);
  CHUNKP(4, 4096, 256);
  CHUNKP(8, 2048, 256);
  CHUNKP(8, 1184, 256);
  CHUNKP(4, 1024, 512);
  READ(8, 16 * sms, 128);
  READ(4, sms, 1024);
  READ(8, sms, 1024);
  READ(4, 2 * sms, 1024);
  READ(8, 2 * sms, 512);
  READ(16, 2 * sms, 512);
  READ(8, 4 * sms, 512);
  READ(4, 8 * sms, 256);
  READ(8, 8 * sms, 256);
  READ(16, 4 * sms, 256);
  READ(8, 16 * sms, 128);
  READ(16, 8 * sms, 128);
#define CHUNK(U, G, T)                                                                                        \
  {                                                                                                           \
    float us = timeit([&](int c) { read_chunk_k<U><<<G, T, 0, st>>>((const float4*)A[c], nA / 4, out); }, st); \
    std::printf("read chunked    U%-2d grid %5d x %4d: %7.2f us  %7.1f GB/s\n", U, G, T, us, bytes_read / us / 1e3); \
  }
  CHUNK(8, 2 * sms, 512);
  CHUNK(8, 4 * sms, 256);
  CHUNK(4, 1024, 256);
  CHUNK(8, 512, 512);
  CHUNK(4, 2048, 256);
  CHUNK(8, 8 * sms, 256);
  CHUNK(16, 8 * sms, 128);
  CHUNK(4, 4096, 256);
  CHUNK(2, 4096, 256);
  CHUNK(4, 2048, 512);
  CHUNK(2, 8192, 256);
  CHUNK(4, 1024, 1024);
  CHUNK(1, 16384, 256);
#define BULK(CH, S, G)                                                                                      \
  {                                                                                                         \
    auto k = read_bulk_k<CH, S>;                                                                            \
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * S));                       \
    float us = timeit([&](int c) { k<<<G, 256, CH * S, st>>>(A[c], nA, out); }, st);                        \
    std::printf("read bulk  CH %6d S %d grid %4d: %7.2f us  %7.1f GB/s\n", CH, S, G, us, bytes_read / us / 1e3); \
  }
  BULK(16384, 8, 148);
  BULK(32768, 6, 148);
  BULK(16384, 6, 256);
  BULK(16384, 4, 296);
  BULK(8192, 8, 296);
  BULK(32768, 3, 296);
  BULK(16384, 12, 148);
  // cuBLAS sgemv
  {
    cublasHandle_t hb;
    cublasCreate(&hb);
    cublasSetStream(hb, st);
    const float one = 1, zero = 0;
    float us = timeit([&](int c) { cublasSgemv(hb, CUBLAS_OP_N, M, N, &one, A[c], M, X[c], 1, &zero, Y[c], 1); }, st);
    std::printf("cublas sgemv: %7.2f us  %7.1f GB/s\n", us, bytes_gemv / us / 1e3);
  }
#define COLS(T, U, G)                                                                                  \
  {                                                                                                    \
    const int cpb = N / G;                                                                             \
    float us = timeit(                                                                                 \
        [&](int c) {                                                                                   \
          zero_k<<<M / 256, 256, 0, st>>>(Y[c], M);                                                    \
          gemv_cols_k<T, U><<<G, T, 0, st>>>(A[c], X[c], Y[c], cpb);                                   \
        },                                                                                             \
        st);                                                                                           \
    std::printf("gemv cols T%-4d U%-2d grid %4d (+zero kernel): %7.2f us  %7.1f GB/s\n", T, U, G, us, \
                bytes_gemv / us / 1e3);                                                                \
  }
#define CHUNKG(R, C, CL)                                                                                  \
  {                                                                                                        \
    float* ws;                                                                                             \
    unsigned* cnt;                                                                                         \
    CK(cudaMalloc(&ws, sizeof(float) * M * (N / C / CL)));                                                 \
    CK(cudaMalloc(&cnt, 4096));                                                                            \
    CK(cudaMemset(cnt, 0, 4096));                                                                          \
    cudaLaunchConfig_t cfg = {};                                                                           \
    cfg.gridDim = dim3((M / R) * (N / C));                                                                 \
    cfg.blockDim = dim3(R / 4);                                                                            \
    cfg.stream = st;                                                                                       \
    cudaLaunchAttribute at[1];                                                                             \
    at[0].id = cudaLaunchAttributeClusterDimension;                                                        \
    at[0].val.clusterDim.x = CL, at[0].val.clusterDim.y = 1, at[0].val.clusterDim.z = 1;                  \
    cfg.attrs = at, cfg.numAttrs = 1;                                                                      \
    auto k = gemv_chunk_k<R, C, CL>;                                                                       \
    float us = timeit([&](int c) { CK(cudaLaunchKernelEx(&cfg, k, (const float*)A[c], (const float*)X[c], Y[c], ws, cnt)); }, st); \
    std::vector<float> hy(M), hx(N);                                                                       \
    CK(cudaMemcpy(hy.data(), Y[0], M * 4, cudaMemcpyDeviceToHost));                                        \
    double maxerr = 0;                                                                                     \
    for (int i = 0; i < M; i += 97) {                                                                      \
      double s = 0, sa = 0;                                                                                \
      for (int j = 0; j < N; ++j) { s += double(h[i + (long long)j * M]) * h[j]; sa += std::fabs(double(h[i + (long long)j * M]) * h[j]); } \
      maxerr = std::max(maxerr, std::fabs(s - hy[i]) / sa);                                                \
    }                                                                                                      \
    std::printf("gemv chunk R%-4d C%-3d CL%d grid %5d: %7.2f us  %7.1f GB/s  maxerr %.2e\n", R, C, CL, (M / R) * (N / C), us, bytes_gemv / us / 1e3, maxerr); \
    cudaFree(ws); cudaFree(cnt);                                                                           \
  }
  CHUNKG(1024, 8, 8);
  CHUNKG(1024, 4, 8);
  CHUNKG(1024, 16, 8);
  CHUNKG(512, 8, 8);
  CHUNKG(512, 16, 8);
  CHUNKG(2048, 8, 8);
  CHUNKG(1024, 8, 4);
  CHUNKG(512, 4, 8);
  COLS(1024, 2, 256);
  COLS(1024, 4, 256);
  COLS(512, 2, 256);
  COLS(512, 4, 512);
  COLS(1024, 2, 512);
  COLS(256, 4, 1024);
  return 0;
}
