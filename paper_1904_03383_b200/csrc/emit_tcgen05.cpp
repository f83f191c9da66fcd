// tcgen05 / TMEM sgemm building block: the tensor-core tile decision of the
// matmul contraction (BASELINE.json config 5), C = A B with fp32 column-major
// operands on the TF32 tensor pipe, fp32 accumulation in tensor memory.
//
// One CTA computes a 128 x BN tile of C with 128 threads:
//   warp 0 lane 0  TMA producer: per k block (32 deep) one 3-D box of A and
//                  one 2-D box of B into stage s of a `stages`-deep ring,
//                  completion counted on full[s] (mbarrier expect_tx)
//   warp 1         allocates BN TMEM columns; lane 0 issues 4 x
//                  tcgen05.mma.cta_group::1.kind::tf32 (M=128, N=BN, K=8)
//                  per k block and tcgen05.commit's empty[s] back to the
//                  producer, then the accumulator barrier
//   warps 0-3      epilogue: tcgen05.ld 32x32b.x32 (warp w owns TMEM lanes
//                  32w..32w+31 = rows), coalesced column-major stores
// Shared-memory operand layouts (UMMA canonical forms, 128-byte swizzle):
//   A  MN-major (m contiguous, as in memory): atoms of 32 m x 8 k (1 KiB);
//      four TMA boxes {32 m, 32 k} land k rows of 128 B per 32 m, so
//      SBO (next 8 k) = 1 KiB and LBO (next 32 m) = 4 KiB
//   B  K-major (k contiguous, as in memory): row n = 32 k (128 B), 8-row
//      atoms, SBO = 1 KiB; the k step inside the 128-B row advances the
//      descriptor start by 32 B
// TF32X3 (engine value): 256 threads; warps 4-7 split every landed stage in
// place, x -> big = cvt.rna.tf32(x) (exactly representable) and, in a second
// buffer of the same swizzled layout, small = x - big; they fence the writes
// to the async proxy and arrive on conv[s]. The MMA lane then issues
// big*big + big*small + small*big per k step (fp32-level accuracy from the
// TF32 pipe). The epilogue splits the columns between warps w and w+4.
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>

#include "ispc.h"
#include "nest_view.hpp"

namespace ispc {

namespace {
[[noreturn]] void illegal(const std::string& why) { throw NestError(ISPC_E_ILLEGAL, why); }
}  // namespace

const char* tcgen05_prelude() {
  return R"(
#ifndef ISPC_TCGEN05_PRELUDE
#define ISPC_TCGEN05_PRELUDE
struct __align__(64) ispc_tmap_t { unsigned long long v[16]; };
static __device__ __forceinline__ void ispc_mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
static __device__ __forceinline__ void ispc_mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n ISPC_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra ISPC_WAIT_%=;\n}\n" ::"r"(bar), "r"(parity) : "memory");
}
static __device__ __forceinline__ void ispc_mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
static __device__ __forceinline__ void ispc_tma_2d(unsigned dst, const ispc_tmap_t* map, int c0, int c1,
                                                   unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(bar) : "memory");
}
static __device__ __forceinline__ unsigned long long ispc_umma_desc(unsigned addr, unsigned lbo, unsigned sbo) {
  return (unsigned long long)((addr >> 4) & 0x3FFF) | ((unsigned long long)((lbo >> 4) & 0x3FFF) << 16) |
         ((unsigned long long)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
static __device__ __forceinline__ void ispc_mma_tf32(unsigned tmem, unsigned long long da, unsigned long long db,
                                                     unsigned idesc, unsigned accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(da), "l"(db), "r"(idesc),
      "r"(accumulate) : "memory");
}
static __device__ __forceinline__ void ispc_mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
static __device__ __forceinline__ float ispc_tf32_rna(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
static __device__ __forceinline__ void ispc_mma_commit(unsigned bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
#define ISPC_TMEM_LD32(taddr, r)                                                                              \
  asm volatile(                                                                                              \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17," \
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                     \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),       \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), \
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),           \
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),           \
        "=r"(r[30]), "=r"(r[31])                                                                             \
      : "r"(taddr))
#endif
)";
}

std::string emit_tcgen05_kernel(const ispc_tile_config& c, const std::string& fn, ispc_launch& L) {
  const int64_t M = c.m, N = c.n, K = c.k;
  const int BN = c.bn, S = c.stages;
  if (c.staging != ISPC_STAGE_TMA) illegal("the tensor-core tile reads TMA-staged operands");
  if (c.engine != ISPC_ENGINE_TF32 && c.engine != ISPC_ENGINE_TF32X3) illegal("tcgen05 kernel needs a tensor engine");
  const bool X3 = c.engine == ISPC_ENGINE_TF32X3;
  const int T = 256;
  if (!(BN == 64 || BN == 128 || BN == 256)) illegal("UMMA N must be 64, 128 or 256");
  if (S < 2 || S > 8) illegal("TMA ring depth must be 2..8");
  if (M % 128 || N % BN || K % 32) illegal("shape not divisible by the 128 x BN x 32 tile");
  if (M > (int64_t(1) << 31) || K > (int64_t(1) << 31)) illegal("shape too large for the tensor maps");
  // TMA ring stage: [A as landed, m contiguous][B, k contiguous]([B small])
  // transposed-A ring, 2 slots: [A k contiguous]([A small]); 1 KiB aligned parts
  const int64_t a_bytes = 128 * 32 * 4, b_bytes = int64_t(BN) * 32 * 4, tma_bytes = a_bytes + b_bytes;
  const int64_t off_b = a_bytes, off_bs = a_bytes + b_bytes;
  const int64_t stage = tma_bytes + (X3 ? b_bytes : 0);
  const int64_t slot = a_bytes * (X3 ? 2 : 1);
  const int64_t ak_off = S * stage, bar_off = ak_off + 2 * slot;
  const int nbar = 2 * S + 4 + 1;  // full[S], empty[S], conv[2], akfree[2], acc
  const int64_t smem = bar_off + (nbar + 1) * 8 + 1024;  // + slack to 1 KiB-align the base
  if (smem > 232448) illegal("TMA ring exceeds 227 KiB of shared memory");
  // kind::tf32, fp32 accumulate, A and B K-major, N = BN, M = 128
  const unsigned idesc = (1u << 4) | (2u << 7) | (2u << 10) | (unsigned(BN >> 3) << 17) | (unsigned(128 >> 4) << 24);
  const int64_t KB = K / 32, MB = M / 128;
  const unsigned FULL = 0, EMPTY = 8u * S, CONV = 16u * S, AKFREE = 16u * S + 16, ACC = 16u * S + 32;

  std::ostringstream o;
  o << tcgen05_prelude();
  o << "extern \"C\" __global__ void __launch_bounds__(" << T << ", 1) " << fn
    << "(const __grid_constant__ ispc_tmap_t tm_a, const __grid_constant__ ispc_tmap_t tm_b, float* __restrict__ g_c) {\n";
  o << "  extern __shared__ __align__(1024) unsigned char ispc_smem_raw[];\n";
  o << "  const unsigned raw = ispc_smem_addr(ispc_smem_raw);\n";
  o << "  const unsigned base = (raw + 1023u) & ~1023u;\n";
  o << "  const unsigned bars = base + " << bar_off << "u;  // full[S], empty[S], conv[2], akfree[2], acc, tmem slot\n";
  o << "  const unsigned ak = base + " << ak_off << "u;     // transposed-A slots\n";
  o << "  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;\n";
  o << "  const int m_blk = blockIdx.x % " << MB << ", n_blk = blockIdx.x / " << MB << ";\n";
  o << "  unsigned char* gen = ispc_smem_raw + (base - raw);\n";
  o << "  unsigned* tmem_slot = (unsigned*)(gen + " << bar_off + nbar * 8 << ");\n";
  o << "  if (threadIdx.x == 0) {\n";
  o << "    for (int s = 0; s < " << nbar << "; ++s)\n";
  o << "      ispc_mbar_init(bars + 8u * s, (s >= " << 2 * S << " && s < " << 2 * S + 2 << ") ? 128u : 1u);\n";
  o << "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n";
  o << "    asm volatile(\"prefetch.tensormap [%0];\" ::\"l\"(&tm_a) : \"memory\");\n";
  o << "    asm volatile(\"prefetch.tensormap [%0];\" ::\"l\"(&tm_b) : \"memory\");\n";
  o << "  }\n";
  o << "  if (warp == 1) {\n";
  o << "    asm volatile(\"tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], " << BN
    << ";\" ::\"r\"(ispc_smem_addr(tmem_slot)) : \"memory\");\n";
  o << "    asm volatile(\"tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\" ::: \"memory\");\n";
  o << "  }\n";
  o << "  asm volatile(\"tcgen05.fence::before_thread_sync;\" ::: \"memory\");\n";
  o << "  __syncthreads();\n";
  o << "  asm volatile(\"tcgen05.fence::after_thread_sync;\" ::: \"memory\");\n";
  o << "  const unsigned tmem = *(volatile unsigned*)tmem_slot;\n";
  // producer: TMA ring of S stages
  o << "  if (warp == 0 && lane == 0) {\n";
  o << "    for (int kb = 0; kb < " << KB << "; ++kb) {\n";
  o << "      const int s = kb % " << S << ";\n";
  o << "      if (kb >= " << S << ") ispc_mbar_wait(bars + " << EMPTY << "u + 8u * s, ((kb / " << S << ") + 1) & 1);\n";
  o << "      const unsigned full = bars + " << FULL << "u + 8u * s;\n";
  o << "      const unsigned sa = base + s * " << stage << "u;\n";
  o << "      ispc_mbar_expect_tx(full, " << tma_bytes << "u);\n";
  o << "      #pragma unroll\n";
  o << "      for (int i = 0; i < 4; ++i) ispc_tma_2d(sa + i * 4096u, &tm_a, m_blk * 128 + i * 32, kb * 32, full);\n";
  o << "      ispc_tma_2d(sa + " << off_b << "u, &tm_b, kb * 32, n_blk * " << BN << ", full);\n";
  o << "    }\n";
  o << "  } else if (warp == 1 && lane == 0) {\n";
  // MMA issuer: A (transposed slot) and B (TMA stage), both K-major 128-B swizzle
  o << "    for (int kb = 0; kb < " << KB << "; ++kb) {\n";
  o << "      const int s = kb % " << S << ", a2 = kb & 1;\n";
  o << "      ispc_mbar_wait(bars + " << CONV << "u + 8u * a2, (kb >> 1) & 1);\n";
  o << "      asm volatile(\"tcgen05.fence::after_thread_sync;\" ::: \"memory\");\n";
  o << "      const unsigned sb = base + s * " << stage << "u + " << off_b << "u;\n";
  o << "      const unsigned sk = ak + a2 * " << slot << "u;\n";
  o << "      #pragma unroll\n";
  o << "      for (int kk = 0; kk < 4; ++kk) {\n";
  o << "        const unsigned long long da = ispc_umma_desc(sk + kk * 32u, 16u, 1024u);\n";
  o << "        const unsigned long long db = ispc_umma_desc(sb + kk * 32u, 16u, 1024u);\n";
  if (X3) {
    o << "        const unsigned long long das = ispc_umma_desc(sk + " << a_bytes << "u + kk * 32u, 16u, 1024u);\n";
    o << "        const unsigned long long dbs = ispc_umma_desc(sb + " << b_bytes << "u + kk * 32u, 16u, 1024u);\n";
    o << "        ispc_mma_tf32(tmem, das, db, " << idesc << "u, (kb | kk) != 0);\n";
    o << "        ispc_mma_tf32(tmem, da, dbs, " << idesc << "u, 1u);\n";
    o << "        ispc_mma_tf32(tmem, da, db, " << idesc << "u, 1u);\n";
  } else {
    o << "        ispc_mma_tf32(tmem, da, db, " << idesc << "u, (kb | kk) != 0);\n";
  }
  o << "      }\n";
  o << "      ispc_mma_commit(bars + " << EMPTY << "u + 8u * s);   // TMA stage free\n";
  o << "      ispc_mma_commit(bars + " << AKFREE << "u + 8u * a2);  // transposed slot free\n";
  o << "    }\n";
  o << "    ispc_mma_commit(bars + " << ACC << "u);\n";
  o << "  } else if (warp >= 4) {\n";
  // converters: the tf32 tensor path reads K-major operands only (MN-major
  // descriptors read zeros on sm_100a, tools/tc_probe.cu), so every landed A
  // tile is transposed into a 2-slot K-major ring, row m = thread
  o << "    const int m = threadIdx.x - 128;\n";
  o << "    for (int kb = 0; kb < " << KB << "; ++kb) {\n";
  o << "      const int s = kb % " << S << ", a2 = kb & 1;\n";
  o << "      ispc_mbar_wait(bars + " << FULL << "u + 8u * s, (kb / " << S << ") & 1);\n";
  o << "      if (kb >= 2) ispc_mbar_wait(bars + " << AKFREE << "u + 8u * a2, ((kb >> 1) + 1) & 1);\n";
  o << "      unsigned char* st = gen + s * " << stage << ";\n";
  o << "      unsigned char* sk = gen + " << ak_off << " + a2 * " << slot << ";\n";
  o << "      const unsigned src_row = (m >> 5) * 4096u + (m & 3) * 4u;\n";
  o << "      const unsigned dst_row = (m >> 3) * 1024u + (m & 7) * 128u;\n";
  o << "      #pragma unroll\n";
  o << "      for (int kq = 0; kq < 8; ++kq) {\n";
  o << "        float v[4];\n";
  o << "        #pragma unroll\n";
  o << "        for (int i = 0; i < 4; ++i) {\n";
  o << "          const int k = kq * 4 + i;\n";
  o << "          v[i] = *(const float*)(st + src_row + (k >> 3) * 1024u + (k & 7) * 128u + ((((m & 31) >> 2) ^ (k & 7)) << 4));\n";
  o << "        }\n";
  o << "        const unsigned dst = dst_row + ((kq ^ (m & 7)) << 4);\n";
  if (X3) {
    o << "        float4 hi, lo;\n";
    o << "        hi.x = ispc_tf32_rna(v[0]); hi.y = ispc_tf32_rna(v[1]); hi.z = ispc_tf32_rna(v[2]); hi.w = ispc_tf32_rna(v[3]);\n";
    o << "        lo.x = v[0] - hi.x; lo.y = v[1] - hi.y; lo.z = v[2] - hi.z; lo.w = v[3] - hi.w;\n";
    o << "        *(float4*)(sk + dst) = hi;\n";
    o << "        *(float4*)(sk + " << a_bytes << " + dst) = lo;\n";
  } else {
    o << "        *(float4*)(sk + dst) = make_float4(v[0], v[1], v[2], v[3]);\n";
  }
  o << "      }\n";
  if (X3) {  // B split in place (big) + small part beside it in the TMA stage
    o << "      #pragma unroll 4\n";
    o << "      for (int i = m; i < " << b_bytes / 16 << "; i += 128) {\n";
    o << "        float4* pb = (float4*)(st + " << off_b << ") + i;\n";
    o << "        const float4 x = *pb;\n";
    o << "        float4 hi, lo;\n";
    o << "        hi.x = ispc_tf32_rna(x.x); hi.y = ispc_tf32_rna(x.y); hi.z = ispc_tf32_rna(x.z); hi.w = ispc_tf32_rna(x.w);\n";
    o << "        lo.x = x.x - hi.x; lo.y = x.y - hi.y; lo.z = x.z - hi.z; lo.w = x.w - hi.w;\n";
    o << "        *pb = hi;\n";
    o << "        *((float4*)(st + " << off_bs << ") + i) = lo;\n";
    o << "      }\n";
  }
  o << "      asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n";
  o << "      ispc_mbar_arrive(bars + " << CONV << "u + 8u * a2);\n";
  o << "    }\n";
  o << "  }\n";
  o << "  __syncwarp();\n";
  // epilogue: TMEM lane group = warp % 4, column half = warp / 4
  const int cols = BN / 2;
  o << "  ispc_mbar_wait(bars + " << ACC << "u, 0);\n";
  o << "  asm volatile(\"tcgen05.fence::after_thread_sync;\" ::: \"memory\");\n";
  o << "  const int lg = warp & 3, c_begin = (warp >> 2) * " << cols << ";\n";
  o << "  const long long row = (long long)m_blk * 128 + lg * 32 + lane;\n";
  o << "  float* pc = g_c + row + (long long)n_blk * " << BN << " * " << M << "LL;\n";
  o << "  #pragma unroll 1\n";
  o << "  for (int c0 = c_begin; c0 < c_begin + " << cols << "; c0 += 32) {\n";
  o << "    unsigned r[32];\n";
  o << "    ISPC_TMEM_LD32(tmem + ((unsigned)(lg * 32) << 16) + c0, r);\n";
  o << "    asm volatile(\"tcgen05.wait::ld.sync.aligned;\" ::: \"memory\");\n";
  o << "    #pragma unroll\n";
  o << "    for (int j = 0; j < 32; ++j) pc[(long long)(c0 + j) * " << M << "LL] = __uint_as_float(r[j]);\n";
  o << "  }\n";
  o << "  asm volatile(\"tcgen05.fence::before_thread_sync;\" ::: \"memory\");\n";
  o << "  __syncthreads();\n";
  o << "  if (warp == 1) {\n";
  o << "    asm volatile(\"tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, " << BN << ";\" ::\"r\"(tmem) : \"memory\");\n";
  o << "  }\n";
  o << "}\n";

  L.grid_x = uint64_t(MB * (N / BN));
  L.block[0] = uint32_t(T);
  L.block[1] = L.block[2] = 1;
  L.static_smem = uint32_t(smem);
  // parameters: tensor maps over a and b, region c
  L.num_params = 3;
  for (int i = 0; i < 2; ++i) {
    ispc_param& P = L.params[i];
    P.kind = ISPC_PARAM_TMAP;
    P.is_input = 1;
    std::snprintf(P.name, sizeof(P.name), "%s", i == 0 ? "a" : "b");
  }
  ispc_param& Pc = L.params[2];
  Pc.kind = ISPC_PARAM_REGION;
  Pc.is_input = 1;
  Pc.elems = M * N;
  std::snprintf(Pc.name, sizeof(Pc.name), "c");
  L.num_tmaps = 2;
  ispc_tmap& ta = L.tmaps[0];
  ta.param = 0;
  ta.rank = 2;
  ta.swizzle = 3;
  std::snprintf(ta.region, sizeof(ta.region), "a");
  ta.dims[0] = uint64_t(M), ta.dims[1] = uint64_t(K);
  ta.strides[0] = uint64_t(M) * 4;
  ta.box[0] = 32, ta.box[1] = 32;
  ispc_tmap& tb = L.tmaps[1];
  tb.param = 1;
  tb.rank = 2;
  tb.swizzle = 3;
  std::snprintf(tb.region, sizeof(tb.region), "b");
  tb.dims[0] = uint64_t(K), tb.dims[1] = uint64_t(N);
  tb.strides[0] = uint64_t(K) * 4;
  tb.box[0] = 32, tb.box[1] = uint32_t(BN);
  L.reg_elems = 32;
  return o.str();
}

}  // namespace ispc
