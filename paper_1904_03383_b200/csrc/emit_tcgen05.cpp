// tcgen05 / TMEM sgemm building block: the tensor-core tile decision of the
// matmul contraction (BASELINE.json config 5), C = A B with fp32 column-major
// operands on the TF32 tensor pipe, fp32 accumulation in tensor memory.
//
// Both operands reach the UMMA straight from shared memory (kind::tf32, SS):
//   A  column-major, so m-contiguous = MN-major. The TF32 UMMA reads an
//      MN-major operand only in the 128-B swizzle with 32-B atoms
//      (descriptor layout SWIZZLE_128B_BASE32B; with the plain 128-B swizzle it
//      reads zeros), and TMA lands exactly that layout with
//      CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B (tools/tc_probe.cu P8-P10): a
//      {32 m x 32 k} box is 32 rows of 128 B (one per k), 32-B chunks XOR'd
//      with k % 4; four boxes hold a CTA's 128 rows, LBO = 4 KiB between them,
//      SBO = 512 B between groups of 4 k rows, +1 KiB per K = 8 MMA step.
//   B  column-major K x N, so k-contiguous = K-major: one {32 k x BN/split n}
//      box in the plain 128-B swizzle (SBO 1 KiB, +32 B per K = 8 step).
// No thread touches the operands on the TF32 path: the MMA waits for the TMA
// bytes. Converter warps run only where values must change or move:
// TF32X3 splits A and B in place (big = cvt.rna.tf32(x), small = x - big
// beside it, same layout), and staging SHARED brings A from global memory
// through registers (one k block ahead) into the same MN-major layout.
//
// One-tile kernel (grid = 0): one CTA (split = 1) or a cluster pair
// (split = 2, cta_group::2, UMMA M = 256 over two SMs, each CTA landing its
// own 128 rows of A and half of B's BN rows) per UMMA_M x BN tile, 256 threads:
//   warp 0 lane 0  producer: TMA ring of `stages` stages (full[s] expect_tx)
//   warp 1         TMEM allocation (BN columns); lane 0 of the leader issues
//                  4 (x3 for TF32X3) tcgen05.mma per k block and commits
//                  empty[s] (multicast to both CTAs of a pair), then acc
//   warps 4-7      converters (TF32X3 / staging SHARED only): conv[s]
//   warps 0-7      epilogue: tcgen05.ld 32x32b.x32, coalesced column stores
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <sstream>
#include <string>

#include "ispc.h"
#include "nest_view.hpp"

namespace ispc {

namespace {
[[noreturn]] void illegal(const std::string& why) { throw NestError(ISPC_E_ILLEGAL, why); }
// a pair's peer CTA signals the leader's full barrier with its own TMA
// (cta_group::2) instead of through a relay lane: the same results and 0-1.6
// us faster at 4096^3 (profiles/r2n_tc_pair_probe.log); ISPC_TC_PAIR_TMA=relay
// restores the relay for comparison
bool tc_pair_direct() {
  const char* e = std::getenv("ISPC_TC_PAIR_TMA");
  return !(e && std::string(e) == "relay");
}
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
// a pair's peer CTA lands its box in its own shared memory and signals the
// leader's mbarrier (cta_group::2: the barrier may live in the peer CTA)
static __device__ __forceinline__ void ispc_tma_2d_cg2(unsigned dst, const ispc_tmap_t* map, int c0, int c1,
                                                       unsigned bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(bar_cluster) : "memory");
}
static __device__ __forceinline__ unsigned ispc_mapa(unsigned addr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
static __device__ __forceinline__ unsigned long long ispc_umma_desc(unsigned addr, unsigned lbo, unsigned sbo) {
  return (unsigned long long)((addr >> 4) & 0x3FFF) | ((unsigned long long)((lbo >> 4) & 0x3FFF) << 16) |
         ((unsigned long long)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
// MN-major operand, 128-B swizzle with 32-B atoms (layout type 1)
static __device__ __forceinline__ unsigned long long ispc_umma_desc_mn32(unsigned addr, unsigned lbo, unsigned sbo) {
  return (unsigned long long)((addr >> 4) & 0x3FFF) | ((unsigned long long)((lbo >> 4) & 0x3FFF) << 16) |
         ((unsigned long long)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (1ull << 61);
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
static __device__ __forceinline__ void ispc_mma_tf32_ss(unsigned tmem, unsigned long long da, unsigned long long db,
                                                        unsigned idesc, unsigned accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(da), "l"(db), "r"(idesc),
      "r"(accumulate) : "memory");
}
static __device__ __forceinline__ void ispc_mma_tf32_ss_pair(unsigned tmem, unsigned long long da,
                                                             unsigned long long db, unsigned idesc,
                                                             unsigned accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(da), "l"(db), "r"(idesc),
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
  ta.swizzle = 4;  // 128-B swizzle, 32-B atoms: the MN-major TF32 operand layout
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

// Stage layout and the pieces both kernels emit.
struct TcStage {
  int64_t a_bytes = 128 * 32 * 4, b_bytes = 0;
  int64_t off_a = 0, off_b = 0, off_as = 0, off_bs = 0, stage = 0, tma_bytes = 0;
};

TcStage tc_stage(int BNL, bool X3, bool A_TMA) {
  TcStage t;
  t.b_bytes = int64_t(BNL) * 32 * 4;
  t.off_a = 0;
  t.off_b = t.a_bytes;
  t.off_as = t.off_b + t.b_bytes;
  t.off_bs = t.off_as + t.a_bytes;
  t.stage = X3 ? t.off_bs + t.b_bytes : t.off_as;
  t.tma_bytes = (A_TMA ? t.a_bytes : 0) + t.b_bytes;
  return t;
}

// kind::tf32, fp32 accumulate, A MN-major, B K-major, N, M
unsigned tc_idesc(int n, int um) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (unsigned(n >> 3) << 17) | (unsigned(um >> 4) << 24);
}

// The 4 (x3) MMAs of one k block from stage base `sa` into accumulator `acc`.
void tc_emit_mmas(std::ostringstream& o, const TcStage& t, bool X3, const char* mma, const std::string& acc,
                  const std::string& idesc, const std::string& first, const char* ind) {
  o << ind << "#pragma unroll\n";
  o << ind << "for (int kk = 0; kk < 4; ++kk) {\n";
  o << ind << "  const unsigned long long da = ispc_umma_desc_mn32(sa + " << t.off_a << "u + kk * 1024u, 4096u, 512u);\n";
  o << ind << "  const unsigned long long db = ispc_umma_desc(sa + " << t.off_b << "u + kk * 32u, 16u, 1024u);\n";
  if (X3) {
    o << ind << "  const unsigned long long das = ispc_umma_desc_mn32(sa + " << t.off_as
      << "u + kk * 1024u, 4096u, 512u);\n";
    o << ind << "  const unsigned long long dbs = ispc_umma_desc(sa + " << t.off_bs << "u + kk * 32u, 16u, 1024u);\n";
    o << ind << "  " << mma << "(" << acc << ", das, db, " << idesc << ", (" << first << ") != 0);\n";
    o << ind << "  " << mma << "(" << acc << ", da, dbs, " << idesc << ", 1u);\n";
    o << ind << "  " << mma << "(" << acc << ", da, db, " << idesc << ", 1u);\n";
  } else {
    o << ind << "  " << mma << "(" << acc << ", da, db, " << idesc << ", (" << first << ") != 0);\n";
  }
  o << ind << "}\n";
}

// Converter work on stage `st` (generic pointer) of k block kb: thread `ct`
// of `nct` converter threads. Staging SHARED: row m = ct % 128 stores its k
// values v[] (16 or 32 of them, k0 = first k) into the MN-major layout.
// TF32X3: every converter thread splits its share of the A and B float4s.
void tc_emit_convert(std::ostringstream& o, const TcStage& t, bool X3, bool A_TMA, int nct, int kper,
                     const char* ind) {
  if (!A_TMA) {
    // element (m, k) of the stage: (m / 32) 4 KiB + (k / 4) 512 B + (k % 4) 128 B + ((m % 32 / 8) ^ (k % 4)) 32 B + (m % 8) 4 B
    o << ind << "#pragma unroll\n";
    o << ind << "for (int q = 0; q < " << kper << "; ++q) {\n";
    o << ind << "  const int k = k0 + q;\n";
    o << ind << "  const unsigned off = (unsigned)(m >> 5) * 4096u + (unsigned)(k >> 2) * 512u + (unsigned)(k & 3) * 128u + "
         "((((unsigned)(m & 31) >> 3) ^ (unsigned)(k & 3)) << 5) + (unsigned)(m & 7) * 4u;\n";
    if (X3) {
      o << ind << "  const float h = ispc_tf32_rna(v[q]);\n";
      o << ind << "  *(float*)(st + " << t.off_a << " + off) = h;\n";
      o << ind << "  *(float*)(st + " << t.off_as << " + off) = v[q] - h;\n";
    } else {
      o << ind << "  *(float*)(st + " << t.off_a << " + off) = v[q];\n";
    }
    o << ind << "}\n";
  }
  if (X3) {
    auto split = [&](int64_t off, int64_t off_small, int64_t bytes) {
      o << ind << "#pragma unroll 4\n";
      o << ind << "for (int q = ct; q < " << bytes / 16 << "; q += " << nct << ") {\n";
      o << ind << "  float4* px = (float4*)(st + " << off << ") + q;\n";
      o << ind << "  const float4 x = *px;\n";
      o << ind << "  float4 hi, lo;\n";
      o << ind << "  hi.x = ispc_tf32_rna(x.x); hi.y = ispc_tf32_rna(x.y); hi.z = ispc_tf32_rna(x.z); hi.w = ispc_tf32_rna(x.w);\n";
      o << ind << "  lo.x = x.x - hi.x; lo.y = x.y - hi.y; lo.z = x.z - hi.z; lo.w = x.w - hi.w;\n";
      o << ind << "  *px = hi;\n";
      o << ind << "  *((float4*)(st + " << off_small << ") + q) = lo;\n";
      o << ind << "}\n";
    };
    if (A_TMA) split(t.off_a, t.off_as, t.a_bytes);
    split(t.off_b, t.off_bs, t.b_bytes);
  }
  o << ind << "asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");  // the UMMA reads through the async proxy\n";
}

// Tile rasterisation: tile t -> (m block, n tile). Groups of G m-blocks walk
// the n tiles together, so the tiles in flight at once share A panels and B
// panels (G = 1: m fastest over the whole column of m-blocks). ISPC_TC_GROUP
// overrides the default (development knob).
int tc_group(int64_t MB) {
  int G = 8;
  if (const char* e = std::getenv("ISPC_TC_GROUP")) G = std::max(1, std::atoi(e));
  while (G > 1 && MB % G) G /= 2;
  return int(std::min<int64_t>(G, MB));
}

std::string tc_tile_map(const std::string& t, const std::string& m, const std::string& nt, int64_t MB, int64_t NT,
                        int G) {
  std::ostringstream o;
  if (G <= 1) {
    o << m << " = " << t << " % " << MB << "; " << nt << " = " << t << " / " << MB << ";";
  } else {
    o << "{ const int g_ = " << t << " / " << G * NT << ", r_ = " << t << " % " << G * NT << "; " << m << " = g_ * " << G
      << " + r_ % " << G << "; " << nt << " = r_ / " << G << "; }";
  }
  return o.str();
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
  const bool CONV = X3 || !A_TMA;
  const int T = 256;
  const int PAIR0 = c.split > 1 ? c.split : 1;
  // a pair's MMA (issued by the leader) reads both CTAs' stages: without
  // converters, warp 2 lane 0 of each CTA relays its stage's TMA completion
  // to the leader's conv barrier, which counts both CTAs
  const bool RELAY0 = !CONV && PAIR0 == 2;
  // direct pair TMA (default): the peer's TMA signals the leader's full
  // barrier itself (cta_group::2), the leader expects both CTAs' bytes, and
  // no relay lane runs
  const bool DIRECT = RELAY0 && tc_pair_direct();
  const bool RELAY = RELAY0 && !DIRECT;
  if (!(BN == 64 || BN == 128 || BN == 256)) illegal("UMMA N must be 64, 128 or 256");
  if (PAIR != 1 && PAIR != 2) illegal("tcgen05 pairs at most two CTAs (cta_group::2)");
  if (S < 2 || S > 8) illegal("TMA ring depth must be 2..8");
  const int UM = 128 * PAIR, BNL = BN / PAIR;  // MMA M; B rows each CTA of the pair lands
  if (M % UM || N % BN || K % 32) illegal("shape not divisible by the UMMA_M x BN x 32 tile");
  if (M > (int64_t(1) << 31) || K > (int64_t(1) << 31) || N > (int64_t(1) << 31))
    illegal("shape too large for the tensor maps");
  int tcols = 32;
  while (tcols < BN) tcols *= 2;
  const TcStage t = tc_stage(BNL, X3, A_TMA);
  const int64_t bar_off = S * t.stage;
  const int nbar = 3 * S + 1;  // full[S], empty[S], conv[S], acc
  const int64_t smem = bar_off + (nbar + 1) * 8 + 1024;  // + slack to 1 KiB-align the base
  if (smem > 232448) illegal("TMA ring exceeds 227 KiB of shared memory");
  const unsigned idesc = tc_idesc(BN, UM);
  const int64_t KB = K / 32, MB = M / UM;
  const unsigned FULL = 0, EMPTY = 8u * S, CONV_B = 16u * S, ACC = 24u * S;
  const char* cg = PAIR == 2 ? "2" : "1";
  const char* mma = PAIR == 2 ? "ispc_mma_tf32_ss_pair" : "ispc_mma_tf32_ss";
  const char* commit = PAIR == 2 ? "ispc_mma_commit_pair" : "ispc_mma_commit";

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
  o << "  int m_blk, n_blk;\n  " << tc_tile_map("pair", "m_blk", "n_blk", MB, N / BN, tc_group(MB)) << "\n";
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
  o << "      const unsigned sa = base + s * " << t.stage << "u;\n";
  if (DIRECT) {
    o << "      const unsigned lfull = rank == 0 ? full : ispc_mapa(full, 0u);\n";
    o << "      if (rank == 0) ispc_mbar_expect_tx(full, " << 2 * t.tma_bytes << "u);\n";
    o << "      #pragma unroll\n";
    o << "      for (int i = 0; i < 4; ++i) ispc_tma_2d_cg2(sa + " << t.off_a << "u + i * 4096u, &tm_a, m_base + i * 32, kb * 32, lfull);\n";
    o << "      ispc_tma_2d_cg2(sa + " << t.off_b << "u, &tm_b, kb * 32, n_blk * " << BN << " + rank * " << BNL << ", lfull);\n";
  } else {
  o << "      ispc_mbar_expect_tx(full, " << t.tma_bytes << "u);\n";
  if (A_TMA) {
    o << "      #pragma unroll\n";
    o << "      for (int i = 0; i < 4; ++i) ispc_tma_2d(sa + " << t.off_a << "u + i * 4096u, &tm_a, m_base + i * 32, kb * 32, full);\n";
  }
  o << "      ispc_tma_2d(sa + " << t.off_b << "u, &tm_b, kb * 32, n_blk * " << BN << " + rank * " << BNL << ", full);\n";
  }
  o << "    }\n";
  o << "  } else if (warp == 1 && lane == 0 && rank == 0) {\n";
  // MMA issuer (the pair's leader): with cta_group::2 the same smem offsets in
  // the peer CTA supply rows 128..255 of A and the second half of B
  o << "    for (int kb = 0; kb < " << KB << "; ++kb) {\n";
  o << "      const int s = kb % " << S << ";\n";
  o << "      ispc_mbar_wait(bars + " << (CONV || RELAY ? CONV_B : FULL) << "u + 8u * s, (kb / " << S << ") & 1);\n";
  o << "      asm volatile(\"tcgen05.fence::after_thread_sync;\" ::: \"memory\");\n";
  o << "      const unsigned sa = base + s * " << t.stage << "u;\n";
  tc_emit_mmas(o, t, X3, mma, "tmem", std::to_string(idesc) + "u", "kb | kk", "      ");
  o << "      " << commit << "(bars + " << EMPTY << "u + 8u * s);   // the stage is free (both CTAs of a pair)\n";
  o << "    }\n";
  o << "    " << commit << "(bars + " << ACC << "u);\n";
  if (RELAY) {
    o << "  } else if (warp == 2 && lane == 0) {\n";
    o << "    for (int kb = 0; kb < " << KB << "; ++kb) {\n";
    o << "      const int s = kb % " << S << ";\n";
    o << "      ispc_mbar_wait(bars + " << FULL << "u + 8u * s, (kb / " << S << ") & 1);\n";
    o << "      ispc_mbar_arrive_rank(bars + " << CONV_B << "u + 8u * s, 0u);\n";
    o << "    }\n";
  }
  if (CONV) {
    o << "  } else if (warp >= 4) {\n";
    o << "    const int m = threadIdx.x - 128, ct = m;\n";
    if (!A_TMA) {
      o << "    float v[32];\n";
      o << "    const int k0 = 0;\n";
      o << "    const float* pa = g_a + m_base + m;\n";
      o << "    #pragma unroll\n";
      o << "    for (int k = 0; k < 32; ++k) v[k] = __ldg(pa + (long long)k * " << M << "LL);\n";
    }
    o << "    for (int kb = 0; kb < " << KB << "; ++kb) {\n";
    o << "      const int s = kb % " << S << ";\n";
    o << "      ispc_mbar_wait(bars + " << FULL << "u + 8u * s, (kb / " << S << ") & 1);\n";
    o << "      unsigned char* st = gen + s * " << t.stage << ";\n";
    tc_emit_convert(o, t, X3, A_TMA, 128, 32, "      ");
    o << "      asm volatile(\"bar.sync 1, 128;\" ::: \"memory\");\n";
    if (PAIR == 2)  // the leader's conv barrier counts both CTAs
      o << "      if (m == 0) ispc_mbar_arrive_rank(bars + " << CONV_B << "u + 8u * s, 0u);\n";
    else
      o << "      if (m == 0) ispc_mbar_arrive(bars + " << CONV_B << "u + 8u * s);\n";
    if (!A_TMA) {  // next k block's A, issued after the arrive
      o << "      if (kb + 1 < " << KB << ") {\n";
      o << "        const float* pn = pa + (long long)(kb + 1) * 32 * " << M << "LL;\n";
      o << "        #pragma unroll\n";
      o << "        for (int k = 0; k < 32; ++k) v[k] = __ldg(pn + (long long)k * " << M << "LL);\n";
      o << "      }\n";
    }
    o << "    }\n";
  }
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
  const bool CONV = X3 || !A_TMA;
  const bool DIRECT = !CONV && PAIR == 2 && !QUAD && tc_pair_direct();  // as in the one-tile kernel
  const bool RELAY = !CONV && PAIR == 2 && !DIRECT;
  // tensor memory holds only the accumulators, double buffered (2 x BN <= 512
  // columns), so the epilogue of tile i overlaps the MMAs of tile i + 1
  const int NB = 2;
  int tcols = 32;
  while (tcols < NB * BN) tcols *= 2;
  const TcStage t = tc_stage(BNL, X3, A_TMA);
  const int64_t stage = t.stage;
  const int64_t bar_off = S * stage;
  const int nbar = 3 * S + 4;  // full[S], empty[S], conv[S], accfull[2], accempty[2]
  const int64_t smem = bar_off + (nbar + 1) * 8 + 1024;
  if (smem > 232448) illegal("TMA ring exceeds 227 KiB of shared memory");
  const unsigned idesc = tc_idesc(BN, UM);
  const int64_t KB = K / 32, MB = M / UM, TILES = MB * (N / BN / (QUAD ? 2 : 1));  // QUAD: tile pairs
  // tail split: when the last round of full tiles would leave most clusters
  // idle, its tiles are cut in half along n (UMMA N = BN / 2) and spread over
  // twice as many clusters
  const int64_t NCL = c.grid / CL, RFULL = TILES / NCL, REM = TILES - RFULL * NCL;
  const bool TS = !QUAD && BN == 256 && REM > 0 && 2 * REM <= NCL;
  const unsigned idesc_half = tc_idesc(BN / 2, UM);
  const unsigned FULL = 0, EMPTY = 8u * S, CONV_B = 16u * S, AFULL = 24u * S, AEMPTY = 24u * S + 16;
  const char* cg = PAIR == 2 ? "2" : "1";
  const char* mma = PAIR == 2 ? "ispc_mma_tf32_ss_pair" : "ispc_mma_tf32_ss";
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
    o << "      int nt;\n      " << tc_tile_map("t", "m_blk", "nt", MB, N / BN, tc_group(MB)) << "\n";
    o << "      n_off = nt * " << BN << " + (cl & 1) * " << BN / 2 << ";\n";
    o << "      width = " << BN / 2 << ";\n";
    o << "      return;\n";
    o << "    }\n";
  }
  o << "    const int t = cl + i * ncl;\n";
  o << "    int nt;\n    " << tc_tile_map("t", "m_blk", "nt", MB, N / BN / (QUAD ? 2 : 1), tc_group(MB)) << "\n";
  o << "    n_off = " << (QUAD ? "(nt * 2 + sub)" : "nt") << " * "
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
  if (DIRECT) {
    o << "        const unsigned lfull = prank == 0 ? full : ispc_mapa(full, lead);\n";
    o << "        if (prank == 0) ispc_mbar_expect_tx(full, " << 2 * t.tma_bytes << "u);\n";
    o << "        #pragma unroll\n";
    o << "        for (int q = 0; q < 4; ++q) ispc_tma_2d_cg2(sa + " << t.off_a << "u + q * 4096u, &tm_a, m_base + q * 32, kb * 32, lfull);\n";
    o << "        ispc_tma_2d_cg2(sa + " << t.off_b << "u, &tm_b, kb * 32, n_off + prank * (width / " << PAIR << "), lfull);\n";
    o << "      }\n    }\n";
  } else {
  o << "        ispc_mbar_expect_tx(full, " << t.tma_bytes << "u);\n";
  if (A_TMA && QUAD) {  // this CTA lands boxes 2 sub, 2 sub + 1 in itself and in the other pair's same-rank CTA
    o << "        const unsigned short amask = (unsigned short)((1u << rank) | (1u << (rank ^ 2u)));\n";
    o << "        #pragma unroll\n";
    o << "        for (int q = 2 * sub; q < 2 * sub + 2; ++q)\n";
    o << "          ispc_tma_2d_mc(sa + " << t.off_a << "u + q * 4096u, &tm_a, m_base + q * 32, kb * 32, full, amask);\n";
  } else if (A_TMA) {
    o << "        #pragma unroll\n";
    o << "        for (int q = 0; q < 4; ++q) ispc_tma_2d(sa + " << t.off_a << "u + q * 4096u, &tm_a, m_base + q * 32, kb * 32, full);\n";
  }
  // the box always holds BN / PAIR rows; a half-width tile uses its first half
  o << "        ispc_tma_2d(sa + " << t.off_b << "u, &tm_b, kb * 32, n_off + prank * (width / " << PAIR
    << "), full);\n";
  o << "      }\n    }\n";
  }
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
  o << "        ispc_mbar_wait(bars + " << (CONV || RELAY ? CONV_B : FULL) << "u + 8u * s, (g / " << S << ") & 1);\n";
  o << "        asm volatile(\"tcgen05.fence::after_thread_sync;\" ::: \"memory\");\n";
  o << "        const unsigned sa = base + s * " << stage << "u;\n";
  tc_emit_mmas(o, t, X3, mma, "acc", "idesc", "kb | kk", "        ");
  o << "        " << commit_to("bars + " + std::to_string(EMPTY) + "u + 8u * s", "(unsigned short)15") << ";\n";
  o << "      }\n";
  o << "      " << commit_to("bars + " + std::to_string(AFULL) + "u + 8u * ab", "pair_mask")
    << ";  // tile done: epilogue may drain\n";
  o << "    }\n";
  if (RELAY) {
    o << "  } else if (warp == 2 && lane == 0) {\n";
    o << "    int g = 0;\n";
    o << "    for (int i = 0; i < my_tiles; ++i)\n";
    o << "      for (int kb = 0; kb < " << KB << "; ++kb, ++g) {\n";
    o << "        const int s = g % " << S << ";\n";
    o << "        ispc_mbar_wait(bars + " << FULL << "u + 8u * s, (g / " << S << ") & 1);\n";
    o << "        ispc_mbar_arrive_rank(bars + " << CONV_B << "u + 8u * s, lead);\n";
    o << "      }\n";
  }
  if (CONV) {
    // converters: two groups of 4 warps; staging SHARED: group kh brings k =
    // 16 kh .. 16 kh + 15 of every k block of row m = thread; TF32X3: all 256
    // threads split the landed A and B
    o << "  } else if ((warp >= 4 && warp < 8) || warp >= 12) {\n";
    o << "    const int m = threadIdx.x & 127, kh = warp >= 12 ? 1 : 0, ct = kh * 128 + m;\n";
    if (!A_TMA) o << "    float v[16];\n    const int k0 = kh * 16;\n";
    o << "    int g = 0;\n";
    o << "    for (int i = 0; i < my_tiles; ++i) {\n";
    o << "      int m_blk, n_off, width;\n";
    o << "      tile_of(i, m_blk, n_off, width);\n";
    o << "      const int m_base = m_blk * " << UM << " + prank * 128;\n";
    if (!A_TMA) {
      o << "      const float* pa = g_a + m_base + m + (long long)k0 * " << M << "LL;\n";
      o << "      #pragma unroll\n";
      o << "      for (int k = 0; k < 16; ++k) v[k] = __ldg(pa + (long long)k * " << M << "LL);\n";
    }
    o << "      for (int kb = 0; kb < " << KB << "; ++kb, ++g) {\n";
    o << "        const int s = g % " << S << ";\n";
    o << "        ispc_mbar_wait(bars + " << FULL << "u + 8u * s, (g / " << S << ") & 1);\n";
    o << "        unsigned char* st = gen + s * " << stage << ";\n";
    tc_emit_convert(o, t, X3, A_TMA, 256, 16, "        ");
    o << "        asm volatile(\"bar.sync 1, 256;\" ::: \"memory\");\n";
    if (PAIR == 2)
      o << "        if (ct == 0) ispc_mbar_arrive_rank(bars + " << CONV_B << "u + 8u * s, lead);\n";
    else
      o << "        if (ct == 0) ispc_mbar_arrive(bars + " << CONV_B << "u + 8u * s);\n";
    if (!A_TMA) {
      o << "        if (kb + 1 < " << KB << ") {\n";
      o << "          const float* pn = pa + (long long)(kb + 1) * 32 * " << M << "LL;\n";
      o << "          #pragma unroll\n";
      o << "          for (int k = 0; k < 16; ++k) v[k] = __ldg(pn + (long long)k * " << M << "LL);\n";
      o << "        }\n";
    }
    o << "      }\n    }\n";
  }
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
