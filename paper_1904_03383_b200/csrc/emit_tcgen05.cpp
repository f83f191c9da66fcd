// tcgen05 / TMEM sgemm building block: the tensor-core tile decision of the
// matmul contraction (BASELINE.json config 5), C = A B with fp32 column-major
// operands on the TF32 tensor pipe, fp32 accumulation in tensor memory.
//
// One CTA (split = 1) or a cluster pair (split = 2, cta_group::2, UMMA M = 256
// over two SMs) computes a UMMA_M x BN tile of C with 256 threads per CTA:
//   warp 0 lane 0  producer: per k block (32 deep) TMA boxes of this CTA's
//                  B rows (BN / split of them) and, for staging TMA, its 128
//                  A rows into stage s of a `stages`-deep ring; full[s]
//                  counts the bytes (mbarrier expect_tx)
//   warps 4-7      converters, row m = thread: tf32 UMMA reads K-major
//                  operands only (MN-major reads zeros on sm_100a,
//                  tools/tc_probe.cu) and A is m-contiguous, so each k block
//                  of A is written K-major (128-B swizzle) into the stage:
//                  staging TMA transposes the landed box, staging SHARED
//                  loads A from global memory one k block ahead in
//                  registers. TF32X3 also splits x -> big = cvt.rna.tf32(x),
//                  small = x - big for A and (in place) B. They fence to the
//                  async proxy and arrive on conv[s] (the leader's, remotely,
//                  for a pair)
//   warp 1         allocates BN TMEM columns; lane 0 of the (leader) CTA
//                  issues 4 (x3 for TF32X3) tcgen05.mma per k block and
//                  commits empty[s] (multicast to both CTAs of a pair), then
//                  the accumulator barrier
//   warps 0-7      epilogue: tcgen05.ld 32x32b.x32 (lane group = warp % 4,
//                  column half = warp / 4), coalesced column-major stores
// Operand descriptors: K-major, 128-B swizzle, rows of 32 tf32 (128 B),
// 8-row atoms, SBO = 1 KiB; the k step inside the row advances the start
// address by 32 B.
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
static __device__ __forceinline__ void ispc_mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
static __device__ __forceinline__ void ispc_mbar_arrive_rank(unsigned bar, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(bar), "r"(rank));
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(r) : "memory");
}
static __device__ __forceinline__ void ispc_mma_commit_pair(unsigned bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"((unsigned short)3) : "memory");
}
static __device__ __forceinline__ void ispc_mma_tf32_ts(unsigned tmem, unsigned ta, unsigned long long db,
                                                        unsigned idesc, unsigned accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem), "r"(ta), "l"(db), "r"(idesc),
      "r"(accumulate) : "memory");
}
static __device__ __forceinline__ void ispc_mma_tf32_ts_pair(unsigned tmem, unsigned ta, unsigned long long db,
                                                             unsigned idesc, unsigned accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem), "r"(ta), "l"(db), "r"(idesc),
      "r"(accumulate) : "memory");
}
#define ISPC_TMEM_ST32(taddr, v)                                                                              \
  asm volatile(                                                                                              \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16," \
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"                                    \
      ::"r"(taddr), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),   \
        "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]),         \
        "f"(v[16]), "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]),       \
        "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])        \
      : "memory")
#define ISPC_TMEM_ST16(taddr, v)                                                                              \
  asm volatile(                                                                                              \
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" \
      ::"r"(taddr), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),   \
        "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])          \
      : "memory")
static __device__ __forceinline__ void ispc_mma_commit_mask(unsigned bar, unsigned short mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"(mask) : "memory");
}
static __device__ __forceinline__ void ispc_tma_2d_mc(unsigned dst, const ispc_tmap_t* map, int c0, int c1, unsigned bar,
                                                      unsigned short mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(bar), "h"(mask) : "memory");
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

void tc_params(ispc_launch& L, int64_t M, int64_t N, int64_t K, int BNL) {
  // parameters: tensor maps over a and b, region a (register-staged A), region c
  L.num_params = 4;
  for (int i = 0; i < 2; ++i) {
    ispc_param& P = L.params[i];
    P.kind = ISPC_PARAM_TMAP;
    P.is_input = 1;
    std::snprintf(P.name, sizeof(P.name), "%s", i == 0 ? "a" : "b");
  }
  ispc_param& Pa = L.params[2];
  Pa.kind = ISPC_PARAM_REGION;
  Pa.is_input = 1;
  Pa.elems = M * K;
  std::snprintf(Pa.name, sizeof(Pa.name), "a");
  ispc_param& Pc = L.params[3];
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
  tb.box[0] = 32, tb.box[1] = uint32_t(BNL);
}

std::string emit_tcgen05_persistent(const ispc_tile_config& c, const std::string& fn, ispc_launch& L);

std::string emit_tcgen05_kernel(const ispc_tile_config& c, const std::string& fn, ispc_launch& L) {
  const int64_t M = c.m, N = c.n, K = c.k;
  if (c.grid > 0) return emit_tcgen05_persistent(c, fn, L);
  const int BN = c.bn, S = c.stages, PAIR = c.split > 1 ? c.split : 1;
  if (c.staging != ISPC_STAGE_TMA && c.staging != ISPC_STAGE_SHARED)
    illegal("the tensor-core tile stages A by TMA or through registers, B by TMA");
  if (c.engine != ISPC_ENGINE_TF32 && c.engine != ISPC_ENGINE_TF32X3) illegal("tcgen05 kernel needs a tensor engine");
  const bool X3 = c.engine == ISPC_ENGINE_TF32X3, A_TMA = c.staging == ISPC_STAGE_TMA;
  const int T = 256;
  if (!(BN == 64 || BN == 128 || BN == 256)) illegal("UMMA N must be 64, 128 or 256");
  if (PAIR != 1 && PAIR != 2) illegal("tcgen05 pairs at most two CTAs (cta_group::2)");
  if (S < 2 || S > 8) illegal("TMA ring depth must be 2..8");
  const int UM = 128 * PAIR, BNL = BN / PAIR;  // MMA M; B rows each CTA of the pair lands
  if (M % UM || N % BN || K % 32) illegal("shape not divisible by the UMMA_M x BN x 32 tile");
  if (M > (int64_t(1) << 31) || K > (int64_t(1) << 31) || N > (int64_t(1) << 31))
    illegal("shape too large for the tensor maps");
  // tensor memory: accumulator in columns [0, BN), then one A slot per ring
  // stage (32 columns = 32 k of this CTA's 128 rows; 64 with A small)
  const int a_cols = X3 ? 64 : 32;
  const int need_cols = BN + S * a_cols;
  if (need_cols > 512) illegal("accumulator + A slots exceed 512 TMEM columns");
  int tcols = 32;
  while (tcols < need_cols) tcols *= 2;
  // smem ring stage (1 KiB aligned parts): ([A as landed, m contiguous]) [B rows, k contiguous] ([B small])
  const int64_t a_bytes = 128 * 32 * 4, b_bytes = int64_t(BNL) * 32 * 4;
  const int64_t off_b = A_TMA ? a_bytes : 0, off_bs = off_b + b_bytes;
  const int64_t tma_bytes = off_b + b_bytes;
  const int64_t stage = tma_bytes + (X3 ? b_bytes : 0);
  const int64_t bar_off = S * stage;
  const int nbar = 3 * S + 1;  // full[S], empty[S], conv[S], acc
  const int64_t smem = bar_off + (nbar + 1) * 8 + 1024;  // + slack to 1 KiB-align the base
  if (smem > 232448) illegal("TMA ring exceeds 227 KiB of shared memory");
  // kind::tf32, fp32 accumulate, K-major operands, N = BN, M = UMMA_M
  const unsigned idesc = (1u << 4) | (2u << 7) | (2u << 10) | (unsigned(BN >> 3) << 17) | (unsigned(UM >> 4) << 24);
  const int64_t KB = K / 32, MB = M / UM;
  const unsigned FULL = 0, EMPTY = 8u * S, CONV = 16u * S, ACC = 24u * S;
  const char* cg = PAIR == 2 ? "2" : "1";

  std::ostringstream o;
  o << tcgen05_prelude();
  o << "extern \"C\" __global__ void __launch_bounds__(" << T << ", 1) " << fn
    << "(const __grid_constant__ ispc_tmap_t tm_a, const __grid_constant__ ispc_tmap_t tm_b, "
       "const float* __restrict__ g_a, float* __restrict__ g_c) {\n";
  o << "  extern __shared__ __align__(1024) unsigned char ispc_smem_raw[];\n";
  o << "  const unsigned raw = ispc_smem_addr(ispc_smem_raw);\n";
  o << "  const unsigned base = (raw + 1023u) & ~1023u;\n";
  o << "  const unsigned bars = base + " << bar_off << "u;  // full[S], empty[S], conv[S], acc, tmem slot\n";
  o << "  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;\n";
  if (PAIR == 2) {
    o << "  unsigned rank;\n";
    o << "  asm volatile(\"mov.u32 %0, %%cluster_ctarank;\" : \"=r\"(rank));\n";
    o << "  const int pair = blockIdx.x >> 1;\n";
  } else {
    o << "  const unsigned rank = 0;\n";
    o << "  const int pair = blockIdx.x;\n";
  }
  o << "  const int m_blk = pair % " << MB << ", n_blk = pair / " << MB << ";\n";
  o << "  const int m_base = m_blk * " << UM << " + rank * 128;\n";
  o << "  unsigned char* gen = ispc_smem_raw + (base - raw);\n";
  o << "  unsigned* tmem_slot = (unsigned*)(gen + " << bar_off + nbar * 8 << ");\n";
  o << "  if (threadIdx.x == 0) {\n";
  o << "    for (int s = 0; s < " << nbar << "; ++s)\n";
  o << "      ispc_mbar_init(bars + 8u * s, (s >= " << 2 * S << " && s < " << 3 * S << ") ? " << PAIR << "u : 1u);\n";
  o << "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n";
  if (A_TMA) o << "    asm volatile(\"prefetch.tensormap [%0];\" ::\"l\"(&tm_a) : \"memory\");\n";
  o << "    asm volatile(\"prefetch.tensormap [%0];\" ::\"l\"(&tm_b) : \"memory\");\n";
  o << "  }\n";
  o << "  if (warp == 1) {\n";
  o << "    asm volatile(\"tcgen05.alloc.cta_group::" << cg << ".sync.aligned.shared::cta.b32 [%0], " << tcols
    << ";\" ::\"r\"(ispc_smem_addr(tmem_slot)) : \"memory\");\n";
  o << "    asm volatile(\"tcgen05.relinquish_alloc_permit.cta_group::" << cg << ".sync.aligned;\" ::: \"memory\");\n";
  o << "  }\n";
  o << "  asm volatile(\"tcgen05.fence::before_thread_sync;\" ::: \"memory\");\n";
  if (PAIR == 2) {  // barriers of both CTAs initialised before any remote arrive / multicast commit
    o << "  asm volatile(\"barrier.cluster.arrive.release.aligned;\\n barrier.cluster.wait.acquire.aligned;\" ::: "
         "\"memory\");\n";
  } else {
    o << "  __syncthreads();\n";
  }
  o << "  asm volatile(\"tcgen05.fence::after_thread_sync;\" ::: \"memory\");\n";
  o << "  const unsigned tmem = *(volatile unsigned*)tmem_slot;\n";
  // producer: TMA ring of S stages (this CTA's own A rows and B rows)
  o << "  if (warp == 0 && lane == 0) {\n";
  o << "    for (int kb = 0; kb < " << KB << "; ++kb) {\n";
  o << "      const int s = kb % " << S << ";\n";
  o << "      if (kb >= " << S << ") ispc_mbar_wait(bars + " << EMPTY << "u + 8u * s, ((kb / " << S << ") + 1) & 1);\n";
  o << "      const unsigned full = bars + " << FULL << "u + 8u * s;\n";
  o << "      const unsigned sa = base + s * " << stage << "u;\n";
  o << "      ispc_mbar_expect_tx(full, " << tma_bytes << "u);\n";
  if (A_TMA) {
    o << "      #pragma unroll\n";
    o << "      for (int i = 0; i < 4; ++i) ispc_tma_2d(sa + i * 4096u, &tm_a, m_base + i * 32, kb * 32, full);\n";
  }
  o << "      ispc_tma_2d(sa + " << off_b << "u, &tm_b, kb * 32, n_blk * " << BN << " + rank * " << BNL
    << ", full);\n";
  o << "    }\n";
  o << "  } else if (warp == 1 && lane == 0 && rank == 0) {\n";
  // MMA issuer (the pair's leader): A from tensor memory (slot s), B from the
  // smem stage (K-major, 128-B swizzle); with cta_group::2 the same TMEM and
  // smem addresses in the peer CTA supply rows 128..255 and the second half of B
  const char* mma = PAIR == 2 ? "ispc_mma_tf32_ts_pair" : "ispc_mma_tf32_ts";
  const char* commit = PAIR == 2 ? "ispc_mma_commit_pair" : "ispc_mma_commit";
  o << "    for (int kb = 0; kb < " << KB << "; ++kb) {\n";
  o << "      const int s = kb % " << S << ";\n";
  o << "      ispc_mbar_wait(bars + " << CONV << "u + 8u * s, (kb / " << S << ") & 1);\n";
  o << "      asm volatile(\"tcgen05.fence::after_thread_sync;\" ::: \"memory\");\n";
  o << "      const unsigned sb = base + s * " << stage << "u + " << off_b << "u;\n";
  o << "      const unsigned ta = tmem + " << BN << "u + s * " << a_cols << "u;\n";
  o << "      #pragma unroll\n";
  o << "      for (int kk = 0; kk < 4; ++kk) {\n";
  o << "        const unsigned long long db = ispc_umma_desc(sb + kk * 32u, 16u, 1024u);\n";
  if (X3) {
    o << "        const unsigned long long dbs = ispc_umma_desc(sb + " << off_bs - off_b << "u + kk * 32u, 16u, 1024u);\n";
    o << "        " << mma << "(tmem, ta + 32u + kk * 8u, db, " << idesc << "u, (kb | kk) != 0);\n";
    o << "        " << mma << "(tmem, ta + kk * 8u, dbs, " << idesc << "u, 1u);\n";
    o << "        " << mma << "(tmem, ta + kk * 8u, db, " << idesc << "u, 1u);\n";
  } else {
    o << "        " << mma << "(tmem, ta + kk * 8u, db, " << idesc << "u, (kb | kk) != 0);\n";
  }
  o << "      }\n";
  o << "      " << commit << "(bars + " << EMPTY << "u + 8u * s);   // stage + A slot free (both CTAs of a pair)\n";
  o << "    }\n";
  o << "    " << commit << "(bars + " << ACC << "u);\n";
  o << "  } else if (warp >= 4) {\n";
  // converters, row m = thread = TMEM lane: A is m-contiguous, so each thread
  // holds its row's 32 k values of a k block in registers (a transposed read
  // of the landed TMA box, or straight from global memory one k block ahead)
  // and tcgen05.st's them into the stage's A slot (TF32X3: big and small)
  o << "    const int m = threadIdx.x - 128;\n";
  o << "    const unsigned trow = (unsigned)((warp & 3) * 32) << 16;\n";
  o << "    float v[32];\n";
  if (!A_TMA) {
    o << "    const float* pa = g_a + m_base + m;\n";
    o << "    #pragma unroll\n";
    o << "    for (int k = 0; k < 32; ++k) v[k] = __ldg(pa + (long long)k * " << M << "LL);\n";
  }
  o << "    for (int kb = 0; kb < " << KB << "; ++kb) {\n";
  o << "      const int s = kb % " << S << ";\n";
  o << "      ispc_mbar_wait(bars + " << FULL << "u + 8u * s, (kb / " << S << ") & 1);\n";
  o << "      unsigned char* st = gen + s * " << stage << ";\n";
  if (A_TMA) {
    o << "      const unsigned src_row = (m >> 5) * 4096u + (m & 3) * 4u;\n";
    o << "      #pragma unroll\n";
    o << "      for (int k = 0; k < 32; ++k)\n";
    o << "        v[k] = *(const float*)(st + src_row + (k >> 3) * 1024u + (k & 7) * 128u + ((((m & 31) >> 2) ^ (k & 7)) << 4));\n";
  }
  o << "      const unsigned ta = tmem + trow + " << BN << "u + s * " << a_cols << "u;\n";
  if (X3) {
    o << "      float lo[32];\n";
    o << "      #pragma unroll\n";
    o << "      for (int k = 0; k < 32; ++k) { const float h = ispc_tf32_rna(v[k]); lo[k] = v[k] - h; v[k] = h; }\n";
    o << "      ISPC_TMEM_ST32(ta, v);\n";
    o << "      ISPC_TMEM_ST32(ta + 32u, lo);\n";
    // B split in place (big) + small part beside it in the TMA stage
    o << "      #pragma unroll 4\n";
    o << "      for (int i = m; i < " << b_bytes / 16 << "; i += 128) {\n";
    o << "        float4* pb = (float4*)(st + " << off_b << ") + i;\n";
    o << "        const float4 x = *pb;\n";
    o << "        float4 hi, l4;\n";
    o << "        hi.x = ispc_tf32_rna(x.x); hi.y = ispc_tf32_rna(x.y); hi.z = ispc_tf32_rna(x.z); hi.w = ispc_tf32_rna(x.w);\n";
    o << "        l4.x = x.x - hi.x; l4.y = x.y - hi.y; l4.z = x.z - hi.z; l4.w = x.w - hi.w;\n";
    o << "        *pb = hi;\n";
    o << "        *((float4*)(st + " << off_bs << ") + i) = l4;\n";
    o << "      }\n";
    o << "      asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n";
  } else {
    o << "      ISPC_TMEM_ST32(ta, v);\n";
  }
  o << "      asm volatile(\"tcgen05.wait::st.sync.aligned;\" ::: \"memory\");\n";
  o << "      asm volatile(\"tcgen05.fence::before_thread_sync;\" ::: \"memory\");\n";
  // one arrive per CTA after the converter warps meet on named barrier 1
  o << "      asm volatile(\"bar.sync 1, 128;\" ::: \"memory\");\n";
  if (PAIR == 2)  // the leader's conv barrier counts both CTAs
    o << "      if (m == 0) ispc_mbar_arrive_rank(bars + " << CONV << "u + 8u * s, 0u);\n";
  else
    o << "      if (m == 0) ispc_mbar_arrive(bars + " << CONV << "u + 8u * s);\n";
  if (!A_TMA) {  // next k block's A, issued after the arrive so its release does not wait on the loads
    o << "      if (kb + 1 < " << KB << ") {\n";
    o << "        const float* pn = pa + (long long)(kb + 1) * 32 * " << M << "LL;\n";
    o << "        #pragma unroll\n";
    o << "        for (int k = 0; k < 32; ++k) v[k] = __ldg(pn + (long long)k * " << M << "LL);\n";
    o << "      }\n";
  }
  o << "    }\n";
  o << "  }\n";
  o << "  __syncwarp();\n";
  // epilogue: TMEM lane group = warp % 4, column half = warp / 4
  const int cols = BN / 2;
  o << "  ispc_mbar_wait(bars + " << ACC << "u, 0);\n";
  o << "  asm volatile(\"tcgen05.fence::after_thread_sync;\" ::: \"memory\");\n";
  o << "  const int lg = warp & 3, c_begin = (warp >> 2) * " << cols << ";\n";
  o << "  const long long row = (long long)m_base + lg * 32 + lane;\n";
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
  if (PAIR == 2)  // neither CTA frees TMEM or exits while its peer may still touch it
    o << "  asm volatile(\"barrier.cluster.arrive.release.aligned;\\n barrier.cluster.wait.acquire.aligned;\" ::: "
         "\"memory\");\n";
  else
    o << "  __syncthreads();\n";
  o << "  if (warp == 1) {\n";
  o << "    asm volatile(\"tcgen05.dealloc.cta_group::" << cg << ".sync.aligned.b32 %0, " << tcols
    << ";\" ::\"r\"(tmem) : \"memory\");\n";
  o << "  }\n";
  o << "}\n";

  L.grid_x = uint64_t(MB * (N / BN) * PAIR);
  L.block[0] = uint32_t(T);
  L.block[1] = L.block[2] = 1;
  L.static_smem = uint32_t(smem);
  if (PAIR == 2) {
    L.cluster[0] = 2;
    L.cluster[1] = L.cluster[2] = 1;
  }
  tc_params(L, M, N, K, BNL);
  L.reg_elems = 32;
  return o.str();
}

// Persistent variant (grid > 0): `grid` CTAs (grid / split clusters) walk the
// UMMA_M x BN output tiles t = cluster, cluster + clusters, ... (m fastest);
// every role keeps one running k-block counter across tiles, so the TMA ring
// and the converters run ahead into the next tile, and the accumulator is
// double-buffered in tensor memory: four dedicated epilogue warps (8-11)
// drain tile i's buffer while the MMA lane fills the other with tile i+1.
// Barriers: full[S], empty[S], conv[S] as in the one-tile kernel, plus
// accfull[2] (MMA commit -> epilogue) and accempty[2] (epilogue -> the
// leader's MMA lane; one arrive per CTA after the epilogue warps meet).
// The 1 x 4 wave tail of a one-tile-per-CTA grid (512 tiles over 148 SMs =
// 3.46 waves at 4096^3, BN 256) becomes 7 rounds of 74 pair tiles at BN 128.
std::string emit_tcgen05_persistent(const ispc_tile_config& c, const std::string& fn, ispc_launch& L) {
  const int64_t M = c.m, N = c.n, K = c.k;
  // split: 1 = one CTA per tile, 2 = a cta_group::2 pair, 4 = two pairs in a
  // cluster of 4 on adjacent n-blocks of one m-block, each A box landed once
  // per pair member rank and multicast to both pairs (TMA .multicast::cluster)
  const int CL = c.split > 1 ? c.split : 1, BN = c.bn, S = c.stages, PAIR = CL >= 2 ? 2 : 1;
  const bool QUAD = CL == 4;
  if (c.staging != ISPC_STAGE_TMA && c.staging != ISPC_STAGE_SHARED)
    illegal("the tensor-core tile stages A by TMA or through registers, B by TMA");
  if (c.engine != ISPC_ENGINE_TF32 && c.engine != ISPC_ENGINE_TF32X3) illegal("tcgen05 kernel needs a tensor engine");
  const bool X3 = c.engine == ISPC_ENGINE_TF32X3, A_TMA = c.staging == ISPC_STAGE_TMA;
  const int T = 512;  // + warps 12-15: a second converter group (k 16..31 of each block)
  if (!(BN == 64 || BN == 128 || BN == 256)) illegal("UMMA N must be 64, 128 or 256");
  if (CL != 1 && CL != 2 && CL != 4) illegal("tcgen05 clusters are 1, a pair, or two pairs");
  if (QUAD && c.staging != ISPC_STAGE_TMA) illegal("A multicast needs the TMA-staged A");
  if (S < 2 || S > 8) illegal("TMA ring depth must be 2..8");
  if (c.grid % CL) illegal("persistent grid is not a whole number of clusters");
  const int UM = 128 * PAIR, BNL = BN / PAIR;
  if (M % UM || N % (BN * (QUAD ? 2 : 1)) || K % 32) illegal("shape not divisible by the UMMA_M x BN x 32 tile");
  if (M > (int64_t(1) << 31) || K > (int64_t(1) << 31) || N > (int64_t(1) << 31))
    illegal("shape too large for the tensor maps");
  const int a_cols = X3 ? 64 : 32;
  // two accumulator buffers when they fit beside the A slots, else one (the
  // MMA of tile i + 1 then waits for the epilogue of tile i)
  const int NB = 2 * BN + S * a_cols <= 512 ? 2 : 1;
  const int need_cols = NB * BN + S * a_cols;
  if (need_cols > 512) illegal("accumulator + A slots exceed 512 TMEM columns");
  int tcols = 32;
  while (tcols < need_cols) tcols *= 2;
  const int64_t a_bytes = 128 * 32 * 4, b_bytes = int64_t(BNL) * 32 * 4;
  const int64_t off_b = A_TMA ? a_bytes : 0, off_bs = off_b + b_bytes;
  const int64_t tma_bytes = off_b + b_bytes;
  const int64_t stage = tma_bytes + (X3 ? b_bytes : 0);
  const int64_t bar_off = S * stage;
  const int nbar = 3 * S + 4;  // full[S], empty[S], conv[S], accfull[2], accempty[2]
  const int64_t smem = bar_off + (nbar + 1) * 8 + 1024;
  if (smem > 232448) illegal("TMA ring exceeds 227 KiB of shared memory");
  const unsigned idesc = (1u << 4) | (2u << 7) | (2u << 10) | (unsigned(BN >> 3) << 17) | (unsigned(UM >> 4) << 24);
  const int64_t KB = K / 32, MB = M / UM, TILES = MB * (N / BN / (QUAD ? 2 : 1));  // QUAD: tile pairs
  // tail split: when the last round of full tiles would leave most clusters
  // idle, its tiles are cut in half along n (UMMA N = BN / 2) and spread over
  // twice as many clusters
  const int64_t NCL = c.grid / CL, RFULL = TILES / NCL, REM = TILES - RFULL * NCL;
  const bool TS = !QUAD && BN == 256 && REM > 0 && 2 * REM <= NCL;
  const unsigned idesc_half =
      (1u << 4) | (2u << 7) | (2u << 10) | (unsigned((BN / 2) >> 3) << 17) | (unsigned(UM >> 4) << 24);
  const unsigned FULL = 0, EMPTY = 8u * S, CONV = 16u * S, AFULL = 24u * S, AEMPTY = 24u * S + 16;
  const char* cg = PAIR == 2 ? "2" : "1";
  const char* mma = PAIR == 2 ? "ispc_mma_tf32_ts_pair" : "ispc_mma_tf32_ts";
  const char* commit = PAIR == 2 ? "ispc_mma_commit_pair" : "ispc_mma_commit";
  auto commit_to = [&](const std::string& bar, const char* mask) {  // both pairs (QUAD) or the own pair
    if (QUAD) return std::string("ispc_mma_commit_mask(") + bar + ", " + mask + ")";
    return std::string(commit) + "(" + bar + ")";
  };

  std::ostringstream o;
  o << tcgen05_prelude();
  o << "extern \"C\" __global__ void __launch_bounds__(" << T << ", 1) " << fn
    << "(const __grid_constant__ ispc_tmap_t tm_a, const __grid_constant__ ispc_tmap_t tm_b, "
       "const float* __restrict__ g_a, float* __restrict__ g_c) {\n";
  o << "  extern __shared__ __align__(1024) unsigned char ispc_smem_raw[];\n";
  o << "  const unsigned raw = ispc_smem_addr(ispc_smem_raw);\n";
  o << "  const unsigned base = (raw + 1023u) & ~1023u;\n";
  o << "  const unsigned bars = base + " << bar_off << "u;\n";
  o << "  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;\n";
  if (PAIR == 2) {
    o << "  unsigned rank;\n";
    o << "  asm volatile(\"mov.u32 %0, %%cluster_ctarank;\" : \"=r\"(rank));\n";
  } else {
    o << "  const unsigned rank = 0;\n";
  }
  o << "  const int cl = blockIdx.x / " << CL << ", ncl = gridDim.x / " << CL << ";\n";
  o << "  const unsigned prank = rank & 1u, lead = rank & ~1u, sub = rank >> 1;  // rank in the pair, its leader, the pair\n";
  o << "  const unsigned short pair_mask = (unsigned short)(3u << (2u * sub));\n";
  if (TS) {
    o << "  const int my_tiles = " << RFULL << " + (cl < " << 2 * REM << " ? 1 : 0);\n";
  } else {
    o << "  const int my_tiles = cl < " << TILES << " ? (" << TILES - 1 << " - cl) / ncl + 1 : 0;\n";
  }
  // tile i of this cluster -> (m block, first column, width)
  o << "  auto tile_of = [&](int i, int& m_blk, int& n_off, int& width) {\n";
  if (TS) {
    o << "    if (i >= " << RFULL << ") {\n";
    o << "      const int t = " << RFULL * NCL << " + cl / 2;\n";
    o << "      m_blk = t % " << MB << ";\n";
    o << "      n_off = (t / " << MB << ") * " << BN << " + (cl & 1) * " << BN / 2 << ";\n";
    o << "      width = " << BN / 2 << ";\n";
    o << "      return;\n";
    o << "    }\n";
  }
  o << "    const int t = cl + i * ncl;\n";
  o << "    m_blk = t % " << MB << ";\n";
  o << "    n_off = " << (QUAD ? "((t / " + std::to_string(MB) + ") * 2 + sub)" : "(t / " + std::to_string(MB) + ")") << " * "
    << BN << ";\n";
  o << "    width = " << BN << ";\n";
  o << "  };\n";
  o << "  unsigned char* gen = ispc_smem_raw + (base - raw);\n";
  o << "  unsigned* tmem_slot = (unsigned*)(gen + " << bar_off + nbar * 8 << ");\n";
  o << "  if (threadIdx.x == 0) {\n";
  o << "    for (int s = 0; s < " << nbar << "; ++s) {\n";
  o << "      const bool per_cta = (s >= " << 2 * S << " && s < " << 3 * S << ") || s >= " << 3 * S + 2 << ";\n";
  o << "      const bool empty = s >= " << S << " && s < " << 2 * S << ";\n";
  o << "      ispc_mbar_init(bars + 8u * s, per_cta ? " << PAIR << "u : empty ? " << (QUAD ? 2 : 1) << "u : 1u);\n";
  o << "    }\n";
  o << "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n";
  if (A_TMA) o << "    asm volatile(\"prefetch.tensormap [%0];\" ::\"l\"(&tm_a) : \"memory\");\n";
  o << "    asm volatile(\"prefetch.tensormap [%0];\" ::\"l\"(&tm_b) : \"memory\");\n";
  o << "  }\n";
  o << "  if (warp == 1) {\n";
  o << "    asm volatile(\"tcgen05.alloc.cta_group::" << cg << ".sync.aligned.shared::cta.b32 [%0], " << tcols
    << ";\" ::\"r\"(ispc_smem_addr(tmem_slot)) : \"memory\");\n";
  o << "    asm volatile(\"tcgen05.relinquish_alloc_permit.cta_group::" << cg << ".sync.aligned;\" ::: \"memory\");\n";
  o << "  }\n";
  o << "  asm volatile(\"tcgen05.fence::before_thread_sync;\" ::: \"memory\");\n";
  if (PAIR == 2)
    o << "  asm volatile(\"barrier.cluster.arrive.release.aligned;\\n barrier.cluster.wait.acquire.aligned;\" ::: "
         "\"memory\");\n";
  else
    o << "  __syncthreads();\n";
  o << "  asm volatile(\"tcgen05.fence::after_thread_sync;\" ::: \"memory\");\n";
  o << "  const unsigned tmem = *(volatile unsigned*)tmem_slot;\n";
  // producer
  o << "  if (warp == 0 && lane == 0) {\n";
  o << "    int g = 0;\n";
  o << "    for (int i = 0; i < my_tiles; ++i) {\n";
  o << "      int m_blk, n_off, width;\n";
  o << "      tile_of(i, m_blk, n_off, width);\n";
  o << "      const int m_base = m_blk * " << UM << " + prank * 128;\n";
  o << "      for (int kb = 0; kb < " << KB << "; ++kb, ++g) {\n";
  o << "        const int s = g % " << S << ";\n";
  o << "        if (g >= " << S << ") ispc_mbar_wait(bars + " << EMPTY << "u + 8u * s, ((g / " << S << ") + 1) & 1);\n";
  o << "        const unsigned full = bars + " << FULL << "u + 8u * s;\n";
  o << "        const unsigned sa = base + s * " << stage << "u;\n";
  o << "        ispc_mbar_expect_tx(full, " << tma_bytes << "u);\n";
  if (A_TMA && QUAD) {  // this CTA lands boxes 2 sub, 2 sub + 1 in itself and in the other pair's same-rank CTA
    o << "        const unsigned short amask = (unsigned short)((1u << rank) | (1u << (rank ^ 2u)));\n";
    o << "        #pragma unroll\n";
    o << "        for (int q = 2 * sub; q < 2 * sub + 2; ++q)\n";
    o << "          ispc_tma_2d_mc(sa + q * 4096u, &tm_a, m_base + q * 32, kb * 32, full, amask);\n";
  } else if (A_TMA) {
    o << "        #pragma unroll\n";
    o << "        for (int q = 0; q < 4; ++q) ispc_tma_2d(sa + q * 4096u, &tm_a, m_base + q * 32, kb * 32, full);\n";
  }
  // the box always holds BN / PAIR rows; a half-width tile uses its first half
  o << "        ispc_tma_2d(sa + " << off_b << "u, &tm_b, kb * 32, n_off + prank * (width / " << PAIR
    << "), full);\n";
  o << "      }\n    }\n";
  o << "  } else if (warp == 1 && lane == 0 && prank == 0) {\n";
  // MMA issuer
  o << "    int g = 0;\n";
  o << "    for (int i = 0; i < my_tiles; ++i) {\n";
  o << "      const int ab = i % " << NB << ";\n";
  o << "      int m_blk, n_off, width;\n";
  o << "      tile_of(i, m_blk, n_off, width);\n";
  o << "      const unsigned idesc = width == " << BN << " ? " << idesc << "u : " << idesc_half << "u;\n";
  o << "      if (i >= " << NB << ") ispc_mbar_wait(bars + " << AEMPTY << "u + 8u * ab, ((i / " << NB
    << ") + 1) & 1);\n";
  o << "      asm volatile(\"tcgen05.fence::after_thread_sync;\" ::: \"memory\");\n";
  o << "      const unsigned acc = tmem + ab * " << BN << "u;\n";
  o << "      for (int kb = 0; kb < " << KB << "; ++kb, ++g) {\n";
  o << "        const int s = g % " << S << ";\n";
  o << "        ispc_mbar_wait(bars + " << CONV << "u + 8u * s, (g / " << S << ") & 1);\n";
  o << "        asm volatile(\"tcgen05.fence::after_thread_sync;\" ::: \"memory\");\n";
  o << "        const unsigned sb = base + s * " << stage << "u + " << off_b << "u;\n";
  o << "        const unsigned ta = tmem + " << NB * BN << "u + s * " << a_cols << "u;\n";
  o << "        #pragma unroll\n";
  o << "        for (int kk = 0; kk < 4; ++kk) {\n";
  o << "          const unsigned long long db = ispc_umma_desc(sb + kk * 32u, 16u, 1024u);\n";
  if (X3) {
    o << "          const unsigned long long dbs = ispc_umma_desc(sb + " << off_bs - off_b
      << "u + kk * 32u, 16u, 1024u);\n";
    o << "          " << mma << "(acc, ta + 32u + kk * 8u, db, " << idesc << "u, (kb | kk) != 0);\n";
    o << "          " << mma << "(acc, ta + kk * 8u, dbs, " << idesc << "u, 1u);\n";
    o << "          " << mma << "(acc, ta + kk * 8u, db, " << idesc << "u, 1u);\n";
  } else {
    o << "          " << mma << "(acc, ta + kk * 8u, db, " << idesc << "u, (kb | kk) != 0);\n";
  }
  o << "        }\n";
  o << "        " << commit_to("bars + " + std::to_string(EMPTY) + "u + 8u * s", "(unsigned short)15") << ";\n";
  o << "      }\n";
  o << "      " << commit_to("bars + " + std::to_string(AFULL) + "u + 8u * ab", "pair_mask")
    << ";  // tile done: epilogue may drain\n";
  o << "    }\n";
  o << "  } else if ((warp >= 4 && warp < 8) || warp >= 12) {\n";
  // converters: two groups of 4 warps, group kh owns k = 16 kh .. 16 kh + 15
  // of every k block (row m = TMEM lane of warp % 4)
  o << "    const int m = threadIdx.x & 127, kh = warp >= 12 ? 1 : 0, ct = kh * 128 + m;\n";
  o << "    const unsigned trow = (unsigned)((warp & 3) * 32) << 16;\n";
  o << "    float v[16];\n";
  o << "    int g = 0;\n";
  o << "    for (int i = 0; i < my_tiles; ++i) {\n";
  o << "      int m_blk, n_off, width;\n";
  o << "      tile_of(i, m_blk, n_off, width);\n";
  o << "      const int m_base = m_blk * " << UM << " + prank * 128;\n";
  if (!A_TMA) {
    o << "      const float* pa = g_a + m_base + m + (long long)kh * 16 * " << M << "LL;\n";
    o << "      #pragma unroll\n";
    o << "      for (int k = 0; k < 16; ++k) v[k] = __ldg(pa + (long long)k * " << M << "LL);\n";
  }
  o << "      for (int kb = 0; kb < " << KB << "; ++kb, ++g) {\n";
  o << "        const int s = g % " << S << ";\n";
  o << "        ispc_mbar_wait(bars + " << FULL << "u + 8u * s, (g / " << S << ") & 1);\n";
  o << "        unsigned char* st = gen + s * " << stage << ";\n";
  if (A_TMA) {
    o << "        const unsigned src_row = (m >> 5) * 4096u + (m & 3) * 4u;\n";
    o << "        #pragma unroll\n";
    o << "        for (int q = 0; q < 16; ++q) {\n";
    o << "          const int k = kh * 16 + q;\n";
    o << "          v[q] = *(const float*)(st + src_row + (k >> 3) * 1024u + (k & 7) * 128u + ((((m & 31) >> 2) ^ (k & 7)) << 4));\n";
    o << "        }\n";
  }
  o << "        const unsigned ta = tmem + trow + " << NB * BN << "u + s * " << a_cols << "u + kh * 16u;\n";
  if (X3) {
    o << "        float lo[16];\n";
    o << "        #pragma unroll\n";
    o << "        for (int k = 0; k < 16; ++k) { const float h = ispc_tf32_rna(v[k]); lo[k] = v[k] - h; v[k] = h; }\n";
    o << "        ISPC_TMEM_ST16(ta, v);\n";
    o << "        ISPC_TMEM_ST16(ta + 32u, lo);\n";
    o << "        #pragma unroll 4\n";
    o << "        for (int q = ct; q < " << b_bytes / 16 << "; q += 256) {\n";
    o << "          float4* pb = (float4*)(st + " << off_b << ") + q;\n";
    o << "          const float4 x = *pb;\n";
    o << "          float4 hi, l4;\n";
    o << "          hi.x = ispc_tf32_rna(x.x); hi.y = ispc_tf32_rna(x.y); hi.z = ispc_tf32_rna(x.z); hi.w = ispc_tf32_rna(x.w);\n";
    o << "          l4.x = x.x - hi.x; l4.y = x.y - hi.y; l4.z = x.z - hi.z; l4.w = x.w - hi.w;\n";
    o << "          *pb = hi;\n";
    o << "          *((float4*)(st + " << off_bs << ") + q) = l4;\n";
    o << "        }\n";
    o << "        asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n";
  } else {
    o << "        ISPC_TMEM_ST16(ta, v);\n";
  }
  o << "        asm volatile(\"tcgen05.wait::st.sync.aligned;\" ::: \"memory\");\n";
  o << "        asm volatile(\"tcgen05.fence::before_thread_sync;\" ::: \"memory\");\n";
  o << "        asm volatile(\"bar.sync 1, 256;\" ::: \"memory\");\n";
  if (PAIR == 2)
    o << "        if (ct == 0) ispc_mbar_arrive_rank(bars + " << CONV << "u + 8u * s, lead);\n";
  else
    o << "        if (ct == 0) ispc_mbar_arrive(bars + " << CONV << "u + 8u * s);\n";
  if (!A_TMA) {
    o << "        if (kb + 1 < " << KB << ") {\n";
    o << "          const float* pn = pa + (long long)(kb + 1) * 32 * " << M << "LL;\n";
    o << "          #pragma unroll\n";
    o << "          for (int k = 0; k < 16; ++k) v[k] = __ldg(pn + (long long)k * " << M << "LL);\n";
    o << "        }\n";
  }
  o << "      }\n    }\n";
  o << "  } else if (warp >= 8 && warp < 12) {\n";
  // epilogue warps: lane group = warp % 4
  o << "    const int lg = warp & 3;\n";
  o << "    for (int i = 0; i < my_tiles; ++i) {\n";
  o << "      int m_blk, n_off, width;\n";
  o << "      tile_of(i, m_blk, n_off, width);\n";
  o << "      const int ab = i % " << NB << ";\n";
  o << "      ispc_mbar_wait(bars + " << AFULL << "u + 8u * ab, (i / " << NB << ") & 1);\n";
  o << "      asm volatile(\"tcgen05.fence::after_thread_sync;\" ::: \"memory\");\n";
  o << "      const long long row = (long long)m_blk * " << UM << " + prank * 128 + lg * 32 + lane;\n";
  o << "      float* pc = g_c + row + (long long)n_off * " << M << "LL;\n";
  o << "      #pragma unroll 1\n";
  o << "      for (int c0 = 0; c0 < width; c0 += 32) {\n";
  o << "        unsigned r[32];\n";
  o << "        ISPC_TMEM_LD32(tmem + ((unsigned)(lg * 32) << 16) + ab * " << BN << "u + c0, r);\n";
  o << "        asm volatile(\"tcgen05.wait::ld.sync.aligned;\" ::: \"memory\");\n";
  o << "        #pragma unroll\n";
  o << "        for (int j = 0; j < 32; ++j) pc[(long long)(c0 + j) * " << M << "LL] = __uint_as_float(r[j]);\n";
  o << "      }\n";
  o << "      asm volatile(\"tcgen05.fence::before_thread_sync;\" ::: \"memory\");\n";
  o << "      asm volatile(\"bar.sync 2, 128;\" ::: \"memory\");\n";
  if (PAIR == 2)
    o << "      if (warp == 8 && lane == 0) ispc_mbar_arrive_rank(bars + " << AEMPTY << "u + 8u * ab, lead);\n";
  else
    o << "      if (warp == 8 && lane == 0) ispc_mbar_arrive(bars + " << AEMPTY << "u + 8u * ab);\n";
  o << "    }\n";
  o << "  }\n";
  o << "  __syncwarp();\n";
  o << "  asm volatile(\"tcgen05.fence::before_thread_sync;\" ::: \"memory\");\n";
  if (PAIR == 2)
    o << "  asm volatile(\"barrier.cluster.arrive.release.aligned;\\n barrier.cluster.wait.acquire.aligned;\" ::: "
         "\"memory\");\n";
  else
    o << "  __syncthreads();\n";
  o << "  if (warp == 1) {\n";
  o << "    asm volatile(\"tcgen05.dealloc.cta_group::" << cg << ".sync.aligned.b32 %0, " << tcols
    << ";\" ::\"r\"(tmem) : \"memory\");\n";
  o << "  }\n";
  o << "}\n";

  L.grid_x = uint64_t(c.grid);
  L.block[0] = uint32_t(T);
  L.block[1] = L.block[2] = 1;
  L.static_smem = uint32_t(smem);
  if (CL > 1) {
    L.cluster[0] = uint32_t(CL);
    L.cluster[1] = L.cluster[2] = 1;
  }
  tc_params(L, M, N, K, BNL);
  L.reg_elems = 32;
  return o.str();
}

}  // namespace ispc
