// tcgen05 probe (development tool, run on a B200): isolates the pieces of
// the TF32 tensor-core sgemm.
//   P1  TMEM round trip: tcgen05.st then tcgen05.ld
//   P2  one MMA (M128 N64 K8), A and B K-major, no swizzle, filled by threads
//   P3  same with A MN-major (no swizzle)
//   P4  four MMAs over a 32-deep k block, A MN-major and B K-major with the
//       128-byte swizzle, filled by threads with the swizzle function the
//       emitter assumes TMA produces
//   P5  P4 with the operands landed by TMA (cuTensorMapEncodeTiled), plus a
//       byte-compare of the landed tiles against P4's layout
//   P6  A and B both K-major with the 128-byte swizzle (the layout the kernel
//       builds by transposing A in shared memory)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_probe tc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      std::exit(1);                                                                \
    }                                                                              \
  } while (0)

__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned b, unsigned ph) {
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(b),
               "r"(ph) : "memory");
}
__device__ __forceinline__ unsigned long long desc(unsigned addr, unsigned lbo, unsigned sbo, unsigned layout) {
  return (unsigned long long)((addr >> 4) & 0x3FFF) | ((unsigned long long)((lbo >> 4) & 0x3FFF) << 16) |
         ((unsigned long long)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((unsigned long long)layout << 61);
}
__device__ __forceinline__ void mma(unsigned tmem, unsigned long long da, unsigned long long db, unsigned idesc,
                                    unsigned acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
               "l"(da), "l"(db), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit(unsigned b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b) : "memory");
}
#define LD32(taddr, r)                                                                                           \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17," \
               "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                               \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), \
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),        \
                 "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),      \
                 "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),      \
                 "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                                         \
               : "r"(taddr))
#define ST32(taddr, r)                                                                                            \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17," \
               "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),                       \
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),  \
               "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),        \
               "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),       \
               "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])                    \
               : "memory")

struct __align__(64) TMap { unsigned long long v[16]; };

// A: M x K (m contiguous, column-major), B: K x N (k contiguous), D row m col n -> out[m + n*M]
// mode: 1 = TMEM round trip, 2 = K-major both no swizzle, 3 = A MN-major no swizzle,
//       4 = SW128 by threads, 5 = SW128 by TMA (dump = landed bytes)
__global__ void __launch_bounds__(128, 1) probe(int mode, const float* A, const float* B, float* out, int M, int N,
                                                int K, const __grid_constant__ TMap tma, const __grid_constant__ TMap tmb,
                                                const __grid_constant__ TMap tma32,
                                                unsigned* dump) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned base = (saddr(raw) + 1023u) & ~1023u;
  unsigned char* gen = raw + (base - saddr(raw));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned* slot = (unsigned*)(gen + 65536);
  const unsigned bar = base + 65536 + 64, fullb = bar + 8;
  float* sA = (float*)gen;            // 16 KiB
  float* sB = (float*)(gen + 16384);  // 32 KiB max
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(fullb, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(saddr(slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = *(volatile unsigned*)slot;
  if (tid == 0) dump[4096] = tmem;
  const int Kb = (mode >= 4) ? 32 : 8;
  if (mode == 1) {
    unsigned r[32];
    for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(float(1000 * (warp * 32 + lane) + j));
    ST32(tmem + ((unsigned)(warp * 32) << 16), r);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  } else {
    if (mode == 5 || mode == 10) {
      if (tid == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fullb), "r"(16384u + 64u * 128u)
                     : "memory");
        for (int i = 0; i < 4; ++i)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                  base + i * 4096u),
              "l"(mode == 10 ? &tma32 : &tma), "r"(i * 32), "r"(0), "r"(fullb)
              : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                base + 16384u),
            "l"(&tmb), "r"(0), "r"(0), "r"(fullb)
            : "memory");
      }
      mbar_wait(fullb, 0);
      for (int i = tid; i < (16384 + 64 * 128) / 4; i += 128) dump[8192 + i] = ((unsigned*)gen)[i];
    } else {
      for (int m = tid; m < 128; m += 128)
        for (int k = 0; k < Kb; ++k) {
          float v = A[m + k * M];
          unsigned off;
          if (mode == 2) off = (m / 8) * 256 + (k / 4) * 128 + (m % 8) * 16 + (k % 4) * 4;
          else if (mode == 3) off = (m / 4) * 128 + (k % 8) * 16 + (m % 4) * 4;
          else if (mode == 6 || mode == 7 || mode == 9) off = (m / 8) * 1024 + (m % 8) * 128 + ((((k % 32) / 4) ^ (m % 8)) * 16) + (k % 4) * 4;
          else if (mode == 8)  // MN-major, 128-B swizzle with 32-B atoms: 4-row groups of 128-B rows
            off = (m / 32) * 4096 + (k / 4) * 512 + (k % 4) * 128 + ((((m % 32) / 8) ^ (k % 4)) * 32) + (m % 8) * 4;
          else off = (m / 32) * 4096 + (k / 8) * 1024 + (k % 8) * 128 + ((((m % 32) / 4) ^ (k % 8)) * 16) + (m % 4) * 4;
          *(float*)(gen + off) = v;
        }
      for (int n = tid; n < 64; n += 128)
        for (int k = 0; k < Kb; ++k) {
          float v = B[k + n * K];
          unsigned off;
          if (mode == 2 || mode == 3) off = (n / 8) * 256 + (k / 4) * 128 + (n % 8) * 16 + (k % 4) * 4;
          else if (mode == 7) off = (n / 32) * 4096 + (k / 8) * 1024 + (k % 8) * 128 + ((((n % 32) / 4) ^ (k % 8)) * 16) + (n % 4) * 4;
          else if (mode == 9) off = (n / 32) * 4096 + (k / 4) * 512 + (k % 4) * 128 + ((((n % 32) / 8) ^ (k % 4)) * 32) + (n % 8) * 4;
          else off = (n / 8) * 1024 + (n % 8) * 128 + ((((k % 32) / 4) ^ (n % 8)) * 16) + (k % 4) * 4;
          *(float*)(gen + 16384 + off) = v;
        }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
    }
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const unsigned amaj = (mode == 3 || mode == 4 || mode == 5 || mode == 8 || mode == 10) ? 1u : 0u;
      const unsigned bmaj = (mode == 7 || mode == 9) ? 1u : 0u;
      const unsigned idesc = (1u << 4) | (2u << 7) | (2u << 10) | (amaj << 15) | (bmaj << 16) | ((64u >> 3) << 17) |
                             ((128u >> 4) << 24);
      if (mode == 2) {
        mma(tmem, desc(base, 128, 256, 0), desc(base + 16384, 128, 256, 0), idesc, 0);
      } else if (mode == 3) {
        // MN-major, no swizzle: SBO = stride between 4-element MN core matrices, LBO = next 8 k
        mma(tmem, desc(base, 1024, 128, 0), desc(base + 16384, 128, 256, 0), idesc, 0);
      } else if (mode == 6) {
        for (int kk = 0; kk < 4; ++kk)
          mma(tmem, desc(base + kk * 32u, 16, 1024, 2), desc(base + 16384 + kk * 32u, 16, 1024, 2), idesc, kk != 0);
      } else if (mode == 8 || mode == 10) {  // A MN-major, SWIZZLE_128B_BASE32B (layout 1): LBO 4 KiB per 32 m, SBO 512 B per 4 k
        for (int kk = 0; kk < 4; ++kk)
          mma(tmem, desc(base + kk * 1024u, 4096, 512, 1), desc(base + 16384 + kk * 32u, 16, 1024, 2), idesc, kk != 0);
      } else if (mode == 9) {  // B MN-major, SWIZZLE_128B_BASE32B
        for (int kk = 0; kk < 4; ++kk)
          mma(tmem, desc(base + kk * 32u, 16, 1024, 2), desc(base + 16384 + kk * 1024u, 4096, 512, 1), idesc, kk != 0);
      } else if (mode == 7) {  // A K-major (as P6), B MN-major: LBO 4 KiB between 32-n groups, SBO 1 KiB per 8 k
        for (int kk = 0; kk < 4; ++kk)
          mma(tmem, desc(base + kk * 32u, 16, 1024, 2), desc(base + 16384 + kk * 1024u, 4096, 1024, 2), idesc, kk != 0);
      } else {
        for (int kk = 0; kk < 4; ++kk)
          mma(tmem, desc(base + kk * 1024u, 4096, 1024, 2), desc(base + 16384 + kk * 32u, 16, 1024, 2), idesc,
              kk != 0);
      }
      commit(bar);
    }
    __syncwarp();
    mbar_wait(bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  for (int c0 = 0; c0 < 64; c0 += 32) {
    unsigned r[32];
    LD32(tmem + ((unsigned)(warp * 32) << 16) + c0, r);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 32; ++j) out[(warp * 32 + lane) + (c0 + j) * 128] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem) : "memory");
}

int main() {
  const int M = 128, N = 64, K = 32;
  std::vector<float> hA(M * K), hB(K * N);
  srand(7);
  for (auto& v : hA) v = float(rand() % 17 - 8) / 8.0f;  // exact in tf32
  for (auto& v : hB) v = float(rand() % 17 - 8) / 8.0f;
  float *dA, *dB, *dO;
  unsigned* dD;
  CK(cudaMalloc(&dA, hA.size() * 4));
  CK(cudaMalloc(&dB, hB.size() * 4));
  CK(cudaMalloc(&dO, M * N * 4));
  CK(cudaMalloc(&dD, 65536 * 4));
  CK(cudaMemcpy(dA, hA.data(), hA.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), hB.size() * 4, cudaMemcpyHostToDevice));
  TMap ta{}, tb{}, ta32{};
  {
    cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)K}, str[1] = {(cuuint64_t)M * 4};
    cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled((CUtensorMap*)&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dA, dims, str, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    std::printf("encode A: %d\n", int(r));
    r = cuTensorMapEncodeTiled((CUtensorMap*)&ta32, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dA, dims, str, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    std::printf("encode A (128B, 32B atoms): %d\n", int(r));
    cuuint64_t dims2[2] = {(cuuint64_t)K, (cuuint64_t)N}, str2[1] = {(cuuint64_t)K * 4};
    cuuint32_t box2[2] = {32, 64};
    r = cuTensorMapEncodeTiled((CUtensorMap*)&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dB, dims2, str2, box2, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    std::printf("encode B: %d\n", int(r));
  }
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000));
  std::vector<unsigned> land4(16384 / 4 + 64 * 32);
  for (int mode = 1; mode <= 10; ++mode) {
    CK(cudaMemset(dO, 0xff, M * N * 4));
    CK(cudaMemset(dD, 0, 65536 * 4));
    probe<<<1, 128, 70000>>>(mode, dA, dB, dO, M, N, K, ta, tb, ta32, dD);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> o(M * N);
    std::vector<unsigned> dd(65536);
    CK(cudaMemcpy(o.data(), dO, M * N * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(dd.data(), dD, 65536 * 4, cudaMemcpyDeviceToHost));
    int Kb = mode >= 4 ? 32 : 8;
    double maxerr = 0;
    int bad = 0, zeros = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        if (mode == 1) ref = 1000.0 * m + (n % 32) + (n >= 32 ? 0 : 0);
        else
          for (int k = 0; k < Kb; ++k) ref += double(hA[m + k * M]) * hB[k + n * K];
        if (mode == 1 && n >= 32) ref = 1000.0 * m + (n - 32);  // second ld chunk reads cols 32.. (unwritten by st)
        double g = o[m + n * M];
        if (g == 0) ++zeros;
        double err = std::fabs(g - ref);
        if (!(err <= 1e-3)) ++bad;
        if (err > maxerr || std::isnan(g)) maxerr = std::isnan(g) ? 1e30 : err;
      }
    std::printf("P%d: err=%s max_err=%g bad=%d/%d zeros=%d tmem=0x%08x sample=%g,%g,%g\n", mode, cudaGetErrorString(e),
                maxerr, bad, M * N, zeros, dd[4096], o[0], o[1], o[M]);
    if (mode == 4) {
      // expected landed layout (what P4 wrote), for P5's comparison
      for (int m = 0; m < 128; ++m)
        for (int k = 0; k < 32; ++k) {
          unsigned off = (m / 32) * 4096 + (k / 8) * 1024 + (k % 8) * 128 + ((((m % 32) / 4) ^ (k % 8)) * 16) + (m % 4) * 4;
          float v = hA[m + k * M];
          std::memcpy(&land4[off / 4], &v, 4);
        }
      for (int n = 0; n < 64; ++n)
        for (int k = 0; k < 32; ++k) {
          unsigned off = (n / 8) * 1024 + (n % 8) * 128 + ((((k % 32) / 4) ^ (n % 8)) * 16) + (k % 4) * 4;
          float v = hB[k + n * K];
          std::memcpy(&land4[(16384 + off) / 4], &v, 4);
        }
    }
    if (mode == 10) {
      int diffA = 0;
      for (int m = 0; m < 128; ++m)
        for (int k = 0; k < 32; ++k) {
          unsigned off = (m / 32) * 4096 + (k / 4) * 512 + (k % 4) * 128 + ((((m % 32) / 8) ^ (k % 4)) * 32) + (m % 8) * 4;
          float v = hA[m + k * M];
          unsigned u;
          std::memcpy(&u, &v, 4);
          diffA += dd[8192 + off / 4] != u;
        }
      std::printf("P10 landed A (TMA 128B_ATOM_32B) vs the BASE32B layout: %d/4096 words differ\n", diffA);
    }
    if (mode == 5) {
      int diffA = 0, diffB = 0;
      for (int i = 0; i < 4096; ++i) diffA += dd[8192 + i] != land4[i];
      for (int i = 0; i < 2048; ++i) diffB += dd[8192 + 4096 + i] != land4[4096 + i];
      std::printf("P5 landed bytes vs assumed swizzle: A words differ %d/4096, B words differ %d/2048\n", diffA, diffB);
      for (int i = 0; i < 8; ++i) std::printf("  A[%d] landed=%08x assumed=%08x\n", i, dd[8192 + i], land4[i]);
    }
    if (e != cudaSuccess) break;
  }
  return 0;
}
