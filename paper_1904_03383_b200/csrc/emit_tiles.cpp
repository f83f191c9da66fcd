// sm_100a building-block emitter: one fully specified candidate of the tile
// space (host/tiles.space, decided through the reference's engine) -> one
// __global__ kernel. This is the half of the code generator the reference's
// gpu.space cannot reach: gemv with warp-shuffle and
// cluster (DSMEM) reductions, shared-memory / cp.async multi-stage sgemm,
// batched sgemm, and the tcgen05/TMEM sgemm (emit_tcgen05.cpp).
//
// Blocks (each a decision of the candidate):
//   vec      ld.global.v2/v4 (float2/float4) operand loads
//   cache    L1 -> ld.global.ca, L2 -> .cg, READ_ONLY -> .nc, NONE -> .cs,
//            STREAM -> ld.global.nc.L1::no_allocate.L2::256B
//   xreduce  SHUFFLE: __shfl_xor_sync butterfly; SHARED: through shared memory
//   split    thread-block cluster of `split` CTAs splitting the reduction axis,
//            partial sums combined through distributed shared memory
//   staging  SHARED: ld.global -> st.shared (stages 2: register prefetch of
//            the next k tile); CP_ASYNC: cp.async ring of `stages` tiles;
//            TMA (gemv): cp.async.bulk.tensor ring with full/empty mbarriers
//   grid     0: one tile per CTA; > 0: gemv balanced row blocks (DIRECT) or a
//            persistent TMA ring, tcgen05 persistent grids (emit_tcgen05.cpp);
//            axpy_stream: grid-stride CTAs
// The FFMA sgemm / batched kernels keep every output's k order ascending
// (one fmaf chain per output), so they are bit-identical to the sequential
// golden kernel; gemv reorders its sum and is checked norm-wise.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>

#include "ispc.h"
#include "nest_view.hpp"

namespace ispc {

std::string emit_tcgen05_kernel(const ispc_tile_config& c, const std::string& fn, ispc_launch& L);
const char* tcgen05_prelude();

namespace {

uint64_t fnv1a(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char ch : s) h = (h ^ ch) * 1099511628211ull;
  return h;
}

[[noreturn]] void illegal(const std::string& why) { throw NestError(ISPC_E_ILLEGAL, why); }

bool pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

std::string ld(uint32_t cache, int width, const std::string& ptr) {
  std::string ty = width == 4 ? "float4" : width == 2 ? "float2" : "float";
  std::string p = width > 1 ? "(const " + ty + "*)(" + ptr + ")" : "(" + ptr + ")";
  switch (cache) {
    case ISPC_CACHE_L1: return "__ldca(" + p + ")";
    case ISPC_CACHE_L2: return "__ldcg(" + p + ")";
    case ISPC_CACHE_READ_ONLY: return "__ldg(" + p + ")";
    case ISPC_CACHE_STREAM: return "ispc_ld_stream(" + p + ")";
    default: return "__ldcs(" + p + ")";
  }
}

const char* comp(int i) {
  static const char* c[] = {".x", ".y", ".z", ".w"};
  return c[i];
}

void add_region(ispc_launch& L, const char* name, int64_t elems) {
  ispc_param& P = L.params[L.num_params++];
  P.kind = ISPC_PARAM_REGION;
  P.is_input = 1;
  P.elems = elems;
  std::snprintf(P.name, sizeof(P.name), "%s", name);
}

// ---------------------------------------------------------------- gemv
// y[i] = sum_j A[i + j*m] x[j]. Lane (lm, ln) of warp (wm, wn) in cluster CTA
// `rank` owns rows row0 .. row0+vec-1 and walks columns
//   j = rank*n/split + (wn*lanes_n + ln) + t * warps_n*lanes_n,   t ascending.
// Persistent TMA gemv (grid > 0): `grid` CTAs (grid / split clusters) walk
// the row blocks rb = rb0, rb0 + clusters, ... of R rows; thread 0 streams the
// CTA's {R rows x bk columns} boxes of every row block it owns through one
// continuous ring (the TMA for the next row block is in flight while this
// one is reduced), so the grid is sized to the 148 SMs instead of to the
// matrix and no SM idles in a partial last wave.
std::string gemv_tma_persistent(const ispc_tile_config& c, const std::string& fn, ispc_launch& L) {
  const int64_t m = c.m, n = c.n;
  const int V = c.vec, LM = c.lanes_m, LN = c.lanes_n, WM = c.warps_m, WN = c.warps_n, S = c.split;
  const int T = 32 * WM * WN;
  const int64_t R = int64_t(V) * LM * WM, G = int64_t(WN) * LN, NRB = m / R;
  const int64_t CB = c.bk, ST = c.stages, KT = n / S / CB, box_bytes = R * CB * 4;
  if (c.grid % S) illegal("persistent grid is not a whole number of clusters");
  const bool xr_shared = LN > 1 && c.xreduce == ISPC_XRED_SHARED;
  const int64_t part_off = 0, cl_off = WN * R, xr_off = WN * R + R;
  const int64_t ring_off = (xr_off + (xr_shared ? int64_t(T) * V : 0) + 31) / 32 * 32;
  const int64_t smem = 4 * (ring_off + ST * R * CB) + 16 * ST;
  if (smem > 232448) illegal("shared memory exceeds 227 KiB");
  const std::string ty = V == 4 ? "float4" : V == 2 ? "float2" : "float";
  std::ostringstream o;
  o << tcgen05_prelude();
  o << "extern \"C\" __global__ void __launch_bounds__(" << T << ") " << fn
    << "(const float* __restrict__ g_a, const float* __restrict__ g_x, float* __restrict__ g_y, "
       "const __grid_constant__ ispc_tmap_t tm_a) {\n";
  o << "  extern __shared__ __align__(128) float ispc_smem[];\n";
  o << "  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;\n";
  o << "  const int lm = lane % " << LM << ", ln = lane / " << LM << ";\n";
  o << "  const int wm = warp % " << WM << ", wn = warp / " << WM << ";\n";
  o << "  const int rank = " << (S > 1 ? "(int)ispc_cluster_rank()" : "0") << ";\n";
  o << "  const int cl = wn * " << LN << " + ln, rl = (wm * " << LM << " + lm) * " << V << ";\n";
  o << "  const int col_c = rank * " << n / S << ";\n";
  o << "  const float* px_cta = g_x + col_c;\n";
  o << "  const int stride = gridDim.x / " << S << ", rb0 = blockIdx.x / " << S << ";\n";
  o << "  const int my_it = rb0 < " << NRB << " ? (" << NRB - 1 << " - rb0) / stride + 1 : 0;\n";
  o << "  const int total = my_it * " << KT << ";\n";
  o << "  float* ring = ispc_smem + " << ring_off << ";\n";
  o << "  const unsigned ring_s = ispc_smem_addr(ring);\n";
  o << "  const unsigned bars = ring_s + " << ST * box_bytes << "u;  // full[ST], empty[ST]\n";
  o << "  if (tid == 0) {\n";
  o << "    for (int s = 0; s < " << ST << "; ++s) { ispc_mbar_init(bars + 8u * s, 1u); ispc_mbar_init(bars + 8u * ("
    << ST << " + s), " << T / 32 << "u); }\n";
  o << "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n";
  o << "    asm volatile(\"prefetch.tensormap [%0];\" ::\"l\"(&tm_a) : \"memory\");\n";
  o << "    for (int g = 0; g < " << ST - 1 << " && g < total; ++g) {\n";
  o << "      ispc_mbar_expect_tx(bars + 8u * g, " << box_bytes << "u);\n";
  o << "      ispc_tma_2d(ring_s + g * " << box_bytes << "u, &tm_a, (rb0 + (g / " << KT << ") * stride) * " << R
    << ", col_c + (g % " << KT << ") * " << CB << ", bars + 8u * g);\n";
  o << "    }\n  }\n  __syncthreads();\n";
  o << "  float acc[" << V << "];\n";
  o << "  #pragma unroll 1\n  for (int g = 0; g < total; ++g) {\n";
  o << "    const int kt = g % " << KT << ";\n";
  o << "    if (kt == 0) {\n      #pragma unroll\n      for (int v = 0; v < " << V << "; ++v) acc[v] = 0.0f;\n    }\n";
  o << "    if (tid == 0) {\n";
  o << "      const int ng = g + " << ST - 1 << ";\n";
  o << "      if (ng < total) {\n";
  o << "        const int slot = ng % " << ST << ";\n";
  o << "        if (g >= 1) ispc_mbar_wait(bars + 8u * (" << ST << " + slot), ((g - 1) / " << ST << ") & 1);\n";
  o << "        ispc_mbar_expect_tx(bars + 8u * slot, " << box_bytes << "u);\n";
  o << "        ispc_tma_2d(ring_s + slot * " << box_bytes << "u, &tm_a, (rb0 + (ng / " << KT << ") * stride) * " << R
    << ", col_c + (ng % " << KT << ") * " << CB << ", bars + 8u * slot);\n";
  o << "      }\n    }\n";
  o << "    ispc_mbar_wait(bars + 8u * (g % " << ST << "), (g / " << ST << ") & 1);\n";
  o << "    const float* st = ring + (g % " << ST << ") * " << R * CB << ";\n";
  o << "    #pragma unroll\n    for (int t = 0; t < " << CB / G << "; ++t) {\n";
  o << "      const int cc = cl + t * " << G << ";\n";
  o << "      const float xv = __ldg(px_cta + kt * " << CB << " + cc);\n";
  o << "      const " << ty << " av = *(const " << ty << "*)(st + cc * " << R << " + rl);\n";
  if (V == 1) o << "      acc[0] = __fmaf_rn(av, xv, acc[0]);\n";
  else
    for (int v = 0; v < V; ++v) o << "      acc[" << v << "] = __fmaf_rn(av" << comp(v) << ", xv, acc[" << v << "]);\n";
  o << "    }\n";
  o << "    asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n";
  o << "    __syncwarp();\n";
  o << "    if (lane == 0) ispc_mbar_arrive(bars + 8u * (" << ST << " + g % " << ST << "));  // one arrive per warp\n";
  o << "    if (kt != " << KT - 1 << ") continue;\n";
  o << "    const long long rblk = rb0 + (long long)(g / " << KT << ") * stride;\n";
  // (1) lanes sharing rows, (2) warps sharing rows, (3) the cluster's CTAs
  o << "    float r_acc[" << V << "];\n";
  o << "    #pragma unroll\n    for (int v = 0; v < " << V << "; ++v) r_acc[v] = acc[v];\n";
  if (LN > 1) {
    if (c.xreduce == ISPC_XRED_SHUFFLE) {
      o << "    #pragma unroll\n    for (int off = " << LM << "; off < 32; off <<= 1) {\n";
      o << "      #pragma unroll\n      for (int v = 0; v < " << V
        << "; ++v) r_acc[v] += __shfl_xor_sync(0xffffffffu, r_acc[v], off);\n";
      o << "    }\n";
    } else {
      o << "    {\n      float* xr = ispc_smem + " << xr_off << ";\n";
      o << "      #pragma unroll\n      for (int v = 0; v < " << V << "; ++v) xr[tid * " << V << " + v] = r_acc[v];\n";
      o << "      __syncwarp();\n";
      o << "      if (ln == 0) {\n";
      o << "        for (int q = 1; q < " << LN << "; ++q)\n";
      o << "          #pragma unroll\n          for (int v = 0; v < " << V << "; ++v) r_acc[v] += xr[(tid + q * " << LM
        << ") * " << V << " + v];\n";
      o << "      }\n      __syncwarp();\n    }\n";
    }
  }
  o << "    float* part = ispc_smem + " << part_off << ";\n";
  o << "    if (ln == 0) {\n";
  o << "      #pragma unroll\n      for (int v = 0; v < " << V << "; ++v) part[wn * " << R << " + (wm * " << LM
    << " + lm) * " << V << " + v] = r_acc[v];\n    }\n";
  o << "    __syncthreads();\n";
  o << "    float* csum = ispc_smem + " << cl_off << ";\n";
  o << "    for (int r = tid; r < " << R << "; r += " << T << ") {\n";
  o << "      float s = part[r];\n";
  o << "      for (int w = 1; w < " << WN << "; ++w) s += part[w * " << R << " + r];\n";
  if (S == 1) o << "      g_y[rblk * " << R << "LL + r] = s;\n";
  else o << "      csum[r] = s;\n";
  o << "    }\n";
  if (S > 1) {
    o << "    ispc_cluster_sync();\n";
    o << "    for (int r = tid; r < " << R << "; r += " << T << ") {\n";
    o << "      if (r % " << S << " != rank) continue;\n";
    o << "      float s = 0.0f;\n";
    o << "      #pragma unroll\n      for (int q = 0; q < " << S << "; ++q) s += ispc_dsmem_ld(csum + r, q);\n";
    o << "      g_y[rblk * " << R << "LL + r] = s;\n";
    o << "    }\n";
    o << "    ispc_cluster_sync();\n";
    L.cluster[0] = uint32_t(S);
    L.cluster[1] = L.cluster[2] = 1;
  } else {
    o << "    __syncthreads();\n";
  }
  o << "  }\n}\n";
  L.static_smem = uint32_t(smem);
  L.grid_x = uint64_t(c.grid);
  L.block[0] = uint32_t(T);
  L.block[1] = L.block[2] = 1;
  add_region(L, "a", m * n);
  add_region(L, "x", n);
  add_region(L, "y", m);
  L.params[2].is_input = 1;
  ispc_param& P = L.params[L.num_params++];
  P.kind = ISPC_PARAM_TMAP;
  P.is_input = 1;
  std::snprintf(P.name, sizeof(P.name), "a");
  ispc_tmap& tm = L.tmaps[L.num_tmaps++];
  tm.param = 3;
  tm.rank = 2;
  tm.swizzle = 0;
  std::snprintf(tm.region, sizeof(tm.region), "a");
  tm.dims[0] = uint64_t(m), tm.dims[1] = uint64_t(n);
  tm.strides[0] = uint64_t(m) * 4;
  tm.box[0] = uint32_t(R), tm.box[1] = uint32_t(CB);
  L.reg_elems = uint32_t(2 * V + 2);
  return o.str();
}

// Balanced gemv (staging DIRECT, grid > 0): grid / split clusters, cluster c
// owns the rows [c RB, (c + 1) RB) with RB = ceil(m / clusters) rounded up to
// 16, so the 2 x 148 SM slots get equal work although 4096 rows do not split
// into 148 equal power-of-two blocks (the last cluster holds the remainder).
// Warp lanes cover 32 x vec consecutive rows of one column (128-512 B per
// load instruction, lanes past the cluster's last row idle); warps split the
// CTA's column slice, CTAs of a cluster split the columns; partial sums meet
// in shared memory, then across the cluster through DSMEM (rank-strided rows).
std::string gemv_balanced(const ispc_tile_config& c, const std::string& fn, ispc_launch& L) {
  const int64_t m = c.m, n = c.n;
  const int V = c.vec, WM = c.warps_m, WN = c.warps_n, S = c.split, U = c.unroll;
  if (!(V == 1 || V == 2 || V == 4)) illegal("vector width must be 1, 2 or 4");
  if (c.lanes_m != 32 || c.lanes_n != 1) illegal("balanced gemv puts all 32 lanes on rows");
  if (WM < 1 || WN < 1 || S < 1 || U < 1) illegal("non-positive tile parameter");
  const int T = 32 * WM * WN;
  if (T > 1024) illegal("more than 1024 threads per CTA");
  if (S > 8) illegal("cluster larger than 8 CTAs");
  if (c.grid % S) illegal("grid is not a whole number of clusters");
  const int64_t NC = c.grid / S;
  const int64_t RB = ((m + NC - 1) / NC + 15) / 16 * 16;  // rows per cluster
  const int64_t CAP = int64_t(32) * V * WM;                // rows a CTA's lanes cover
  if (RB > CAP) illegal("the CTA's lanes do not cover the cluster's rows");
  if (CAP > 2 * RB) illegal("more than half of the lanes would idle");
  if (RB % V || m % V) illegal("vector width does not divide the row blocks");
  if (n % (int64_t(S) * WN * U)) illegal("column split does not divide n");
  const int64_t iters = n / (int64_t(S) * WN);
  const int64_t smem = 4 * (int64_t(WN) * CAP + CAP);
  if (smem > 232448) illegal("shared memory exceeds 227 KiB");
  const std::string ty = V == 4 ? "float4" : V == 2 ? "float2" : "float";
  std::ostringstream o;
  o << "extern \"C\" __global__ void __launch_bounds__(" << T << ") " << fn
    << "(const float* __restrict__ g_a, const float* __restrict__ g_x, float* __restrict__ g_y) {\n";
  o << "  extern __shared__ __align__(16) float ispc_smem[];\n";
  o << "  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;\n";
  o << "  const int wm = warp % " << WM << ", wn = warp / " << WM << ";\n";
  o << "  const int rank = " << (S > 1 ? "(int)ispc_cluster_rank()" : "0") << ";\n";
  o << "  const long long row_begin = (long long)(blockIdx.x / " << S << ") * " << RB << "LL;\n";
  o << "  const long long row_end = row_begin + " << RB << "LL < " << m << "LL ? row_begin + " << RB << "LL : " << m
    << "LL;\n";
  o << "  const int rl = (wm * 32 + lane) * " << V << ";\n";
  o << "  const long long row0 = row_begin + rl;\n";
  o << "  const long long col0 = (long long)rank * " << n / S << "LL + wn;\n";
  o << "  float acc[" << V << "];\n";
  o << "  #pragma unroll\n  for (int v = 0; v < " << V << "; ++v) acc[v] = 0.0f;\n";
  o << "  if (row0 < row_end) {\n";
  o << "    const float* pa = g_a + row0 + col0 * " << m << "LL;\n";
  o << "    const float* px = g_x + col0;\n";
  o << "    #pragma unroll 1\n    for (long long t = 0; t < " << iters << "LL; t += " << U << ") {\n";
  o << "      " << ty << " av[" << U << "];\n      float xv[" << U << "];\n";
  o << "      #pragma unroll\n      for (int u = 0; u < " << U << "; ++u) {\n";
  o << "        av[u] = " << ld(c.cache, V, "pa + (t + u) * " + std::to_string(int64_t(WN) * m) + "LL") << ";\n";
  o << "        xv[u] = __ldg(px + (t + u) * " << WN << "LL);\n";
  o << "      }\n";
  o << "      #pragma unroll\n      for (int u = 0; u < " << U << "; ++u) {\n";
  if (V == 1) o << "        acc[0] = __fmaf_rn(av[u], xv[u], acc[0]);\n";
  else
    for (int v = 0; v < V; ++v)
      o << "        acc[" << v << "] = __fmaf_rn(av[u]" << comp(v) << ", xv[u], acc[" << v << "]);\n";
  o << "      }\n    }\n  }\n";
  o << "  float* part = ispc_smem;                  // [WN][CAP] warp partials\n";
  o << "  float* csum = ispc_smem + " << int64_t(WN) * CAP << ";  // [CAP] CTA partials\n";
  o << "  #pragma unroll\n  for (int v = 0; v < " << V << "; ++v) part[wn * " << CAP << " + rl + v] = acc[v];\n";
  o << "  __syncthreads();\n";
  o << "  for (int r = tid; r < " << CAP << "; r += " << T << ") {\n";
  o << "    float s = part[r];\n";
  o << "    for (int w = 1; w < " << WN << "; ++w) s += part[w * " << CAP << " + r];\n";
  if (S == 1) o << "    if (row_begin + r < row_end) g_y[row_begin + r] = s;\n";
  else o << "    csum[r] = s;\n";
  o << "  }\n";
  if (S > 1) {
    o << "  ispc_cluster_sync();\n";
    o << "  for (int r = tid; r < " << CAP << "; r += " << T << ") {\n";
    o << "    if (r % " << S << " != rank || row_begin + r >= row_end) continue;\n";
    o << "    float s = 0.0f;\n";
    o << "    #pragma unroll\n    for (int q = 0; q < " << S << "; ++q) s += ispc_dsmem_ld(csum + r, q);\n";
    o << "    g_y[row_begin + r] = s;\n";
    o << "  }\n";
    o << "  ispc_cluster_sync();\n";
    L.cluster[0] = uint32_t(S);
    L.cluster[1] = L.cluster[2] = 1;
  }
  o << "}\n";
  L.static_smem = uint32_t(smem);
  L.grid_x = uint64_t(c.grid);
  L.block[0] = uint32_t(T);
  L.block[1] = L.block[2] = 1;
  add_region(L, "a", m * n);
  add_region(L, "x", n);
  add_region(L, "y", m);
  L.params[2].is_input = 1;
  L.reg_elems = uint32_t(V * (U + 1) + U);
  return o.str();
}

std::string gemv(const ispc_tile_config& c, const std::string& fn, ispc_launch& L) {
  const int64_t m = c.m, n = c.n;
  const int V = c.vec, LM = c.lanes_m, LN = c.lanes_n, WM = c.warps_m, WN = c.warps_n, S = c.split,
            U = c.unroll;
  if (!(V == 1 || V == 2 || V == 4)) illegal("vector width must be 1, 2 or 4");
  if (LM * LN != 32 || !pow2(LM)) illegal("warp lanes must split 32 in powers of two");
  if (WM < 1 || WN < 1 || S < 1 || U < 1) illegal("non-positive tile parameter");
  const int T = 32 * WM * WN;
  if (T > 1024) illegal("more than 1024 threads per CTA");
  if (S > 8) illegal("cluster larger than 8 CTAs");
  const int64_t R = int64_t(V) * LM * WM;  // rows per CTA
  if (m % R) illegal("rows per CTA do not divide m");
  const int64_t G = int64_t(WN) * LN;      // column lanes per CTA
  if (n % (S * G * U)) illegal("column split does not divide n");
  const int64_t iters = n / (S * G);       // columns per thread
  const bool direct = WN == 1 && S == 1;  // lane sums go straight to y
  const bool xr_shared = LN > 1 && c.xreduce == ISPC_XRED_SHARED;
  const int64_t part_off = 0;                                // [WN][R] warp partials
  const int64_t cl_off = direct ? 0 : WN * R;                // [R] CTA partials (cluster)
  const int64_t xr_off = direct ? 0 : WN * R + R;            // [T][V] lane partials
  // CP_ASYNC staging: a ring of `stages` tiles of R rows x bk columns (column
  // segments of R contiguous floats) filled by 16-byte cp.async copies
  const bool tma = c.staging == ISPC_STAGE_TMA;
  const bool staged = c.staging == ISPC_STAGE_CP_ASYNC || tma;
  if (!staged && c.staging != ISPC_STAGE_DIRECT) illegal("gemv reads A directly or through a cp.async / TMA ring");
  const int64_t CB = staged ? c.bk : 0, ST = staged ? c.stages : 0;
  if (staged) {
    if (ST < 2 || CB < 1) illegal("the staging ring needs >= 2 stages of >= 1 column");
    if (R % 4) illegal("staged column segments need rows per CTA divisible by 4");
    if (CB % G || (n / S) % CB) illegal("stage columns do not split across column lanes / the CTA slice");
    if (tma && (R > 256 || CB > 256)) illegal("TMA boxes hold at most 256 elements per dimension");
  }
  if (c.grid > 0) {  // the balanced (DIRECT) or persistent (TMA) variants
    if (tma) return gemv_tma_persistent(c, fn, L);
    if (staged) illegal("the cp.async ring does not take a grid size");
    return gemv_balanced(c, fn, L);
  }
  // ring 128-byte aligned (TMA destination), then full[ST] / empty[ST] mbarriers
  const int64_t ring_off = (xr_off + (xr_shared ? int64_t(T) * V : 0) + 31) / 32 * 32;
  const int64_t smem = 4 * (staged ? ring_off + ST * R * CB : ring_off) + (tma ? 16 * ST : 0);
  if (smem > 232448) illegal("shared memory exceeds 227 KiB");

  std::ostringstream o;
  const std::string ty = V == 4 ? "float4" : V == 2 ? "float2" : "float";
  if (tma) o << tcgen05_prelude();
  o << "extern \"C\" __global__ void __launch_bounds__(" << T << ") " << fn
    << "(const float* __restrict__ g_a, const float* __restrict__ g_x, float* __restrict__ g_y"
    << (tma ? ", const __grid_constant__ ispc_tmap_t tm_a" : "") << ") {\n";
  o << "  extern __shared__ __align__(16) float ispc_smem[];\n";
  o << "  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;\n";
  o << "  const int lm = lane % " << LM << ", ln = lane / " << LM << ";\n";
  o << "  const int wm = warp % " << WM << ", wn = warp / " << WM << ";\n";
  o << "  const int rank = " << (S > 1 ? "(int)ispc_cluster_rank()" : "0") << ";\n";
  o << "  const long long rblk = blockIdx.x / " << S << ";\n";
  o << "  const long long row0 = rblk * " << R << "LL + (long long)(wm * " << LM << " + lm) * " << V << ";\n";
  o << "  const long long col0 = (long long)rank * " << n / S << "LL + wn * " << LN << " + ln;\n";
  o << "  const float* pa = g_a + row0 + col0 * " << m << "LL;\n";
  o << "  const float* px = g_x + col0;\n";
  o << "  float acc[" << V << "];\n";
  o << "  #pragma unroll\n  for (int v = 0; v < " << V << "; ++v) acc[v] = 0.0f;\n";
  if (!staged) {
    o << "  #pragma unroll 1\n  for (long long t = 0; t < " << iters << "LL; t += " << U << ") {\n";
    o << "    " << ty << " av[" << U << "];\n    float xv[" << U << "];\n";
    o << "    #pragma unroll\n    for (int u = 0; u < " << U << "; ++u) {\n";
    o << "      av[u] = " << ld(c.cache, V, "pa + (t + u) * " + std::to_string(G * m) + "LL") << ";\n";
    o << "      xv[u] = __ldg(px + (t + u) * " << G << "LL);\n";
    o << "    }\n";
    o << "    #pragma unroll\n    for (int u = 0; u < " << U << "; ++u) {\n";
    if (V == 1) o << "      acc[0] = __fmaf_rn(av[u], xv[u], acc[0]);\n";
    else
      for (int v = 0; v < V; ++v)
        o << "      acc[" << v << "] = __fmaf_rn(av[u]" << comp(v) << ", xv[u], acc[" << v << "]);\n";
    o << "    }\n  }\n";
  } else if (tma) {
    // TMA ring: thread 0 lands one {R rows x CB columns} box per stage
    // (mbarrier expect-tx); every thread releases the stage through empty[s]
    const int64_t KT = n / S / CB, box_bytes = R * CB * 4;
    o << "  float* ring = ispc_smem + " << ring_off << ";\n";
    o << "  const unsigned ring_s = ispc_smem_addr(ring);\n";
    o << "  const unsigned bars = ring_s + " << ST * box_bytes << "u;  // full[ST], empty[ST]\n";
    o << "  const int row_c = (int)(rblk * " << R << "), col_c = rank * " << n / S << ";\n";
    o << "  const float* px_cta = g_x + col_c;\n";
    o << "  const int cl = wn * " << LN << " + ln, rl = (wm * " << LM << " + lm) * " << V << ";\n";
    o << "  if (tid == 0) {\n";
    o << "    for (int s = 0; s < " << ST << "; ++s) { ispc_mbar_init(bars + 8u * s, 1u); ispc_mbar_init(bars + 8u * ("
      << ST << " + s), " << T << "u); }\n";
    o << "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n";
    o << "  }\n  __syncthreads();\n";
    o << "  if (tid == 0) {\n";
    o << "    for (int s = 0; s < " << ST - 1 << " && s < " << KT << "; ++s) {\n";
    o << "      ispc_mbar_expect_tx(bars + 8u * s, " << box_bytes << "u);\n";
    o << "      ispc_tma_2d(ring_s + s * " << box_bytes << "u, &tm_a, row_c, col_c + s * " << CB << ", bars + 8u * s);\n";
    o << "    }\n  }\n";
    o << "  #pragma unroll 1\n  for (int kt = 0; kt < " << KT << "; ++kt) {\n";
    o << "    if (tid == 0) {\n";
    o << "      const int nk = kt + " << ST - 1 << ";\n";
    o << "      if (nk < " << KT << ") {\n";
    o << "        const int slot = nk % " << ST << ";\n";
    o << "        if (kt >= 1) ispc_mbar_wait(bars + 8u * (" << ST << " + slot), ((kt - 1) / " << ST << ") & 1);\n";
    o << "        ispc_mbar_expect_tx(bars + 8u * slot, " << box_bytes << "u);\n";
    o << "        ispc_tma_2d(ring_s + slot * " << box_bytes << "u, &tm_a, row_c, col_c + nk * " << CB
      << ", bars + 8u * slot);\n";
    o << "      }\n    }\n";
    o << "    ispc_mbar_wait(bars + 8u * (kt % " << ST << "), (kt / " << ST << ") & 1);\n";
    o << "    const float* st = ring + (kt % " << ST << ") * " << R * CB << ";\n";
    o << "    #pragma unroll\n    for (int t = 0; t < " << CB / G << "; ++t) {\n";
    o << "      const int cc = cl + t * " << G << ";\n";
    o << "      const float xv = __ldg(px_cta + kt * " << CB << " + cc);\n";
    o << "      const " << ty << " av = *(const " << ty << "*)(st + cc * " << R << " + rl);\n";
    if (V == 1) o << "      acc[0] = __fmaf_rn(av, xv, acc[0]);\n";
    else
      for (int v = 0; v < V; ++v)
        o << "      acc[" << v << "] = __fmaf_rn(av" << comp(v) << ", xv, acc[" << v << "]);\n";
    o << "    }\n";
    // order this thread's generic-proxy reads of the slot before the TMA
    // (async proxy) that will overwrite it once every thread arrived
    o << "    asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n";
    o << "    ispc_mbar_arrive(bars + 8u * (" << ST << " + kt % " << ST << "));\n";
    o << "  }\n";
  } else {
    const int64_t KT = n / S / CB, chunks = R * CB / 4;
    const std::string cp = c.cache == ISPC_CACHE_L1 ? "ispc_cp_async_ca16" : "ispc_cp_async_cg16";
    o << "  float* ring = ispc_smem + " << ring_off << ";\n";
    o << "  const float* pa_cta = g_a + rblk * " << R << "LL + (long long)rank * " << n / S << "LL * " << m << "LL;\n";
    o << "  const float* px_cta = g_x + (long long)rank * " << n / S << "LL;\n";
    o << "  const int cl = wn * " << LN << " + ln, rl = (wm * " << LM << " + lm) * " << V << ";\n";
    auto issue = [&](const std::string& kt, const std::string& slot, const std::string& ind) {
      o << ind << "for (int ch = threadIdx.x; ch < " << chunks << "; ch += " << T << ") {\n";
      o << ind << "  const int cc = ch / " << R / 4 << ", rr = (ch % " << R / 4 << ") * 4;\n";
      o << ind << "  " << cp << "(ring + (" << slot << ") * " << R * CB << " + cc * " << R << " + rr, pa_cta + rr + ((long long)("
        << kt << ") * " << CB << " + cc) * " << m << "LL);\n";
      o << ind << "}\n";
    };
    o << "  #pragma unroll\n  for (int s = 0; s < " << ST - 1 << "; ++s) {\n";
    o << "    if (s < " << KT << ") {\n";
    issue("s", "s", "      ");
    o << "    }\n    ispc_cp_async_commit();\n  }\n";
    o << "  #pragma unroll 1\n  for (int kt = 0; kt < " << KT << "; ++kt) {\n";
    o << "    ispc_cp_async_wait<" << ST - 2 << ">();\n    __syncthreads();\n";
    o << "    {\n      const int nk = kt + " << ST - 1 << ";\n      if (nk < " << KT << ") {\n";
    issue("nk", "nk % " + std::to_string(ST), "        ");
    o << "      }\n      ispc_cp_async_commit();\n    }\n";
    o << "    const float* st = ring + (kt % " << ST << ") * " << R * CB << ";\n";
    o << "    #pragma unroll\n    for (int t = 0; t < " << CB / G << "; ++t) {\n";
    o << "      const int cc = cl + t * " << G << ";\n";
    o << "      const float xv = __ldg(px_cta + kt * " << CB << " + cc);\n";
    o << "      const " << ty << " av = *(const " << ty << "*)(st + cc * " << R << " + rl);\n";
    if (V == 1) o << "      acc[0] = __fmaf_rn(av, xv, acc[0]);\n";
    else
      for (int v = 0; v < V; ++v)
        o << "      acc[" << v << "] = __fmaf_rn(av" << comp(v) << ", xv, acc[" << v << "]);\n";
    o << "    }\n  }\n";
    o << "  ispc_cp_async_wait<0>();\n";
  }
  // (1) lanes sharing rows (ln) -> lane ln == 0
  if (LN > 1) {
    if (c.xreduce == ISPC_XRED_SHUFFLE) {
      o << "  #pragma unroll\n  for (int off = " << LM << "; off < 32; off <<= 1) {\n";
      o << "    #pragma unroll\n    for (int v = 0; v < " << V << "; ++v) acc[v] += __shfl_xor_sync(0xffffffffu, acc[v], off);\n";
      o << "  }\n";
    } else {
      o << "  {\n    float* xr = ispc_smem + " << xr_off << ";\n";
      o << "    #pragma unroll\n    for (int v = 0; v < " << V << "; ++v) xr[tid * " << V << " + v] = acc[v];\n";
      o << "    __syncwarp();\n";
      o << "    if (ln == 0) {\n";
      o << "      for (int q = 1; q < " << LN << "; ++q)\n";
      o << "        #pragma unroll\n        for (int v = 0; v < " << V << "; ++v) acc[v] += xr[(tid + q * " << LM << ") * " << V << " + v];\n";
      o << "    }\n  }\n";
    }
  }
  L.static_smem = uint32_t(smem);
  if (direct) {
    o << "  if (ln == 0) {\n";
    if (V == 1) o << "    g_y[row0] = acc[0];\n";
    else {
      o << "    *(" << ty << "*)(g_y + row0) = make_" << ty << "(";
      for (int v = 0; v < V; ++v) o << (v ? ", " : "") << "acc[" << v << "]";
      o << ");\n";
    }
    o << "  }\n}\n";
  } else {
    // (2) warps sharing rows (wn), ascending wn
    o << "  float* part = ispc_smem + " << part_off << ";\n";
    o << "  if (ln == 0) {\n";
    o << "    #pragma unroll\n    for (int v = 0; v < " << V << "; ++v) part[wn * " << R << " + (wm * " << LM
      << " + lm) * " << V << " + v] = acc[v];\n  }\n";
    o << "  __syncthreads();\n";
    o << "  float* csum = ispc_smem + " << cl_off << ";\n";
    o << "  for (int r = tid; r < " << R << "; r += " << T << ") {\n";
    o << "    float s = part[r];\n";
    o << "    for (int w = 1; w < " << WN << "; ++w) s += part[w * " << R << " + r];\n";
    if (S == 1) o << "    g_y[rblk * " << R << "LL + r] = s;\n";
    else o << "    csum[r] = s;\n";
    o << "  }\n";
    if (S > 1) {
      // (3) CTAs of the cluster, ascending rank, through distributed shared memory
      o << "  ispc_cluster_sync();\n";
      o << "  for (int r = tid; r < " << R << "; r += " << T << ") {\n";
      o << "    if (r % " << S << " != rank) continue;\n";
      o << "    float s = 0.0f;\n";
      o << "    #pragma unroll\n    for (int q = 0; q < " << S << "; ++q) s += ispc_dsmem_ld(csum + r, q);\n";
      o << "    g_y[rblk * " << R << "LL + r] = s;\n";
      o << "  }\n";
      o << "  ispc_cluster_sync();\n";
      L.cluster[0] = uint32_t(S);
      L.cluster[1] = L.cluster[2] = 1;
    }
    o << "}\n";
  }
  L.grid_x = uint64_t(m / R * S);
  L.block[0] = uint32_t(T);
  L.block[1] = L.block[2] = 1;
  add_region(L, "a", m * n);
  add_region(L, "x", n);
  add_region(L, "y", m);
  L.params[2].is_input = 1;
  if (tma) {
    ispc_param& P = L.params[L.num_params++];
    P.kind = ISPC_PARAM_TMAP;
    P.is_input = 1;
    std::snprintf(P.name, sizeof(P.name), "a");
    ispc_tmap& tm = L.tmaps[L.num_tmaps++];
    tm.param = 3;
    tm.rank = 2;
    tm.swizzle = 0;
    std::snprintf(tm.region, sizeof(tm.region), "a");
    tm.dims[0] = uint64_t(m), tm.dims[1] = uint64_t(n);
    tm.strides[0] = uint64_t(m) * 4;
    tm.box[0] = uint32_t(R), tm.box[1] = uint32_t(CB);
  }
  L.reg_elems = uint32_t(V * (U + 1) + U);
  return o.str();
}

// ---------------------------------------------------------------- sgemm (FFMA)
// C = A B, column-major: A[i + k*M], B[k + j*K], C[i + j*M]. CTA tile
// BM x BN = (thr_m*tm) x (thr_n*tn); thread (tx, ty) owns the rows
// bm*BM + (i/v)*thr_m*v + tx*v + i%v, i < tm, v = the vector width that
// divides tm (groups of v contiguous rows, interleaved across threads: a
// warp's float4 smem reads are contiguous, C stores stay vectorised) and the
// columns bn*BN + ty + j*thr_n, j < tn (interleaved, so the Bs rows a warp
// reads fall in distinct banks). Shared tiles per
// stage: As[bk][BM] (m contiguous) and Bs[BN][bk+4] (k contiguous), both
// filled with contiguous global chunks (no transposes), read as float4
// along m (A) and along k (B: four k steps at once).
struct GemmShape {
  int TX, TY, TM, TN, BK, S, V, T;
  int64_t BM, BN, ldb;  // ldb: Bs row pitch
  int64_t a_tile, b_tile, stage_floats;
};

GemmShape gemm_shape(const ispc_tile_config& c, int64_t M, int64_t N, int64_t K) {
  GemmShape g{};
  g.TX = c.thr_m, g.TY = c.thr_n, g.TM = c.tm, g.TN = c.tn, g.BK = c.bk, g.V = c.vec;
  g.S = std::max(1, c.stages);
  if (g.TX < 1 || g.TY < 1 || g.TM < 1 || g.TN < 1 || g.BK < 1) illegal("non-positive tile parameter");
  if (!(g.V == 1 || g.V == 2 || g.V == 4)) illegal("vector width must be 1, 2 or 4");
  g.T = g.TX * g.TY;
  if (g.T > 1024) illegal("more than 1024 threads per CTA");
  g.BM = int64_t(g.TX) * g.TM;
  g.BN = int64_t(g.TY) * g.TN;
  if (M % g.BM || N % g.BN) illegal("CTA tile does not divide the output");
  if (K % g.BK) illegal("k depth does not divide K");
  if (g.BK % 4 && g.BK != 1 && g.BK != 2) illegal("k depth must be 1, 2 or a multiple of 4");
  if (g.BM % g.V || g.BK % g.V) illegal("vector width does not divide the staged tiles");
  if (int64_t(g.TM) * g.TN > 256) illegal("more than 256 accumulators per thread");
  g.ldb = g.BK + (g.BK >= 4 ? 4 : 0);
  g.a_tile = int64_t(g.BK) * g.BM;
  g.b_tile = g.BN * g.ldb;
  g.stage_floats = g.a_tile + g.b_tile;
  if (g.stage_floats * g.S * 4 > 232448) illegal("shared-memory ring exceeds 227 KiB");
  return g;
}

// Per-thread compute on one staged k tile: As (m contiguous), Bs (k contiguous).
void gemm_compute(std::ostringstream& o, const GemmShape& g, const std::string& As, const std::string& Bs,
                  const std::string& indent) {
  const int KG = g.BK >= 4 ? 4 : g.BK;  // k steps read at once from Bs
  const int AV = g.TM % 4 == 0 ? 4 : g.TM % 2 == 0 ? 2 : 1;
  o << indent << "#pragma unroll\n" << indent << "for (int kq = 0; kq < " << g.BK << "; kq += " << KG << ") {\n";
  o << indent << "  float ra[" << KG << "][" << g.TM << "], rb[" << g.TN << "][" << KG << "];\n";
  o << indent << "  #pragma unroll\n" << indent << "  for (int q = 0; q < " << KG << "; ++q) {\n";
  o << indent << "    #pragma unroll\n" << indent << "    for (int i = 0; i < " << g.TM << "; i += " << AV << ") {\n";
  if (AV == 4)
    o << indent << "      float4 t = *(const float4*)(" << As << " + (kq + q) * " << g.BM << " + (i / 4) * " << g.TX * 4
      << " + tx * 4);\n"
      << indent << "      ra[q][i] = t.x; ra[q][i + 1] = t.y; ra[q][i + 2] = t.z; ra[q][i + 3] = t.w;\n";
  else if (AV == 2)
    o << indent << "      float2 t = *(const float2*)(" << As << " + (kq + q) * " << g.BM << " + (i / 2) * " << g.TX * 2
      << " + tx * 2);\n"
      << indent << "      ra[q][i] = t.x; ra[q][i + 1] = t.y;\n";
  else
    o << indent << "      ra[q][i] = " << As << "[(kq + q) * " << g.BM << " + i * " << g.TX << " + tx];\n";
  o << indent << "    }\n" << indent << "  }\n";
  o << indent << "  #pragma unroll\n" << indent << "  for (int j = 0; j < " << g.TN << "; ++j) {\n";
  if (KG == 4)
    o << indent << "    float4 t = *(const float4*)(" << Bs << " + (ty + j * " << g.TY << ") * " << g.ldb
      << " + kq);\n"
      << indent << "    rb[j][0] = t.x; rb[j][1] = t.y; rb[j][2] = t.z; rb[j][3] = t.w;\n";
  else
    o << indent << "    #pragma unroll\n" << indent << "    for (int q = 0; q < " << KG << "; ++q) rb[j][q] = "
      << Bs << "[(ty + j * " << g.TY << ") * " << g.ldb << " + kq + q];\n";
  o << indent << "  }\n";
  o << indent << "  #pragma unroll\n" << indent << "  for (int q = 0; q < " << KG << "; ++q)\n";
  o << indent << "    #pragma unroll\n" << indent << "    for (int j = 0; j < " << g.TN << "; ++j)\n";
  o << indent << "      #pragma unroll\n" << indent << "      for (int i = 0; i < " << g.TM << "; ++i)\n";
  o << indent << "        acc[j][i] = __fmaf_rn(ra[q][i], rb[j][q], acc[j][i]);\n";
  o << indent << "}\n";
}

// Issues the copies of k tile `kt` into stage buffer `buf` (cp.async) or
// loads it into registers / stores it (SHARED).
void gemm_copy_cp_async(std::ostringstream& o, const GemmShape& g, const ispc_tile_config& c, int64_t M, int64_t K,
                        const std::string& pa, const std::string& pb, const std::string& kt, const std::string& buf,
                        const std::string& indent) {
  const int V = g.V;
  const std::string cp = V == 4 ? (c.cache == ISPC_CACHE_L1 ? "ispc_cp_async_ca16" : "ispc_cp_async_cg16")
                                : V == 2 ? "ispc_cp_async_ca8" : "ispc_cp_async_ca4";
  const int64_t a_chunks = g.a_tile / V, b_chunks = int64_t(g.BN) * g.BK / V;
  o << indent << "{\n";
  o << indent << "  float* sA = ispc_smem + (" << buf << ") * " << g.stage_floats << ";\n";
  o << indent << "  float* sB = sA + " << g.a_tile << ";\n";
  o << indent << "  const long long k0 = (long long)(" << kt << ") * " << g.BK << ";\n";
  o << indent << "  #pragma unroll\n" << indent << "  for (int ch = tid; ch < " << a_chunks << "; ch += " << g.T << ") {\n";
  o << indent << "    const int kk = ch / " << g.BM / V << ", mm = (ch % " << g.BM / V << ") * " << V << ";\n";
  o << indent << "    " << cp << "(sA + kk * " << g.BM << " + mm, " << pa << " + mm + (k0 + kk) * " << M << "LL);\n";
  o << indent << "  }\n";
  o << indent << "  #pragma unroll\n" << indent << "  for (int ch = tid; ch < " << b_chunks << "; ch += " << g.T << ") {\n";
  o << indent << "    const int nn = ch / " << g.BK / V << ", kk = (ch % " << g.BK / V << ") * " << V << ";\n";
  o << indent << "    " << cp << "(sB + nn * " << g.ldb << " + kk, " << pb << " + k0 + kk + (long long)nn * " << K
    << "LL);\n";
  o << indent << "  }\n";
  o << indent << "}\n";
}

// Warp-tiled FFMA2 sgemm (CP_ASYNC staging, vec 4, tm and tn multiples of 4,
// whole warps). The thr_m x thr_n threads form warps of LX x LY lanes
// (LX = min(thr_m, 8)); a lane owns tm x tn outputs as (tm/4) x (tn/4)
// blocks of 4 x 4, rows wm*LX*tm + (i/4)*LX*4 + lx*4 + i%4 and columns
// wn*LY*tn + (j/4)*LY*4 + ly*4 + j%4, so a warp's fragment reads are LX (A)
// and LY (B) distinct float4s: one shared-memory wavefront each. Both operands
// are k-major in shared memory: As[bk][BM] by 16-byte cp.async, Bs[bk][BN+4]
// by 4-byte cp.async (B transposed on the way in, lanes walking k, which is
// contiguous in global). The per-k fragments are double buffered in
// registers (the loads of step k+1 are issued before the FFMA2s of step k;
// the last step of a tile loads the next tile's first fragment after the
// tile barrier). FFMA2 (__ffma2_rn: two IEEE fmas per lane, the B value
// broadcast) keeps each output one fmaf chain in ascending k: bit-identical
// to the sequential oracle. B200 measurements behind this structure:
// tools/sgemm_lab.cu (profiles/r2_sgemm_lab.md).
bool sgemm_warp_tiled_ok(const ispc_tile_config& c) {
  const int T = c.thr_m * c.thr_n;
  return c.staging == ISPC_STAGE_CP_ASYNC && c.vec == 4 && c.tm % 4 == 0 && c.tn % 4 == 0 && c.tm <= 8 &&
         c.tn <= 8 && T % 32 == 0 && c.stages >= 2 && c.bk >= 4 && c.thr_m >= 4 && 32 % std::min(c.thr_m, 8) == 0 &&
         c.thr_n % (32 / std::min(c.thr_m, 8)) == 0;
}

std::string sgemm_warp_tiled(const ispc_tile_config& c, const std::string& fn, ispc_launch& L) {
  const int64_t M = c.m, N = c.n, K = c.k;
  const int LX = std::min(c.thr_m, 8), LY = 32 / LX;
  const int WX = c.thr_m / LX;
  const int TM = c.tm, TN = c.tn, BK = c.bk, S = c.stages, T = c.thr_m * c.thr_n;
  const int64_t BM = int64_t(c.thr_m) * TM, BN = int64_t(c.thr_n) * TN, LDB = BN + 4;
  if (M % BM || N % BN) illegal("CTA tile does not divide the output");
  const int SP = std::max(1, c.split);
  if (SP > 8) illegal("cluster larger than 8 CTAs");
  if (K % (int64_t(SP) * BK)) illegal("split-K slices do not divide K");
  if ((BM * BN) % (4 * SP)) illegal("partial tile does not split across the cluster");
  const int64_t KT = K / (int64_t(SP) * BK);
  const int64_t a_tile = BK * BM, b_tile = BK * LDB, stage = a_tile + b_tile;
  if (stage * S * 4 > 232448) illegal("shared-memory ring exceeds 227 KiB");
  if (int64_t(TM) * TN > 64) illegal("more than 64 accumulators per thread");
  std::ostringstream o;
  o << "extern \"C\" __global__ void __launch_bounds__(" << T << ") " << fn
    << "(const float* __restrict__ g_a, const float* __restrict__ g_b, float* __restrict__ g_c) {\n";
  o << "  extern __shared__ __align__(16) float ispc_smem[];\n";
  // the k-tile count reaches the compiler as an opaque value: with the literal
  // trip count nvcc/NVRTC reshape the pipelined loop and the kernel runs 8%
  // slower (53.3 vs 49.3 us at 1024^3, profiles/r2k_sgemm_lab11.log)
  o << "  int ispc_kt = " << KT << ";\n  asm(\"\" : \"+r\"(ispc_kt));\n";
  o << "  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;\n";
  o << "  const int wm = warp % " << WX << ", wn = warp / " << WX << ", lx = lane % " << LX << ", ly = lane / " << LX
    << ";\n";
  o << "  const long long tile = blockIdx.x / " << SP << ";\n";
  o << "  const int rank = " << (SP > 1 ? "(int)ispc_cluster_rank()" : "0") << ";\n";
  o << "  const long long bm = tile % " << M / BM << ", bn = tile / " << M / BM << ";\n";
  o << "  const long long kbase = (long long)rank * " << K / SP << "LL;\n";
  o << "  const float* pa = g_a + bm * " << BM << "LL + kbase * " << M << "LL;\n";
  o << "  const float* pb = g_b + bn * " << BN << "LL * " << K << "LL + kbase;\n";
  o << "  const int arow = wm * " << LX * TM << " + lx * 4, bcol = wn * " << LY * TN << " + ly * 4;\n";
  o << "  float acc[" << TN << "][" << TM << "];\n";
  o << "  #pragma unroll\n  for (int j = 0; j < " << TN << "; ++j)\n    #pragma unroll\n    for (int i = 0; i < " << TM
    << "; ++i) acc[j][i] = 0.0f;\n";
  o << "  float fa[2][" << TM << "], fb[2][" << TN << "];\n";
  // copies of k tile kt into ring slot `slot`
  // copies address shared memory as 32-bit offsets from one converted base
  o << "  const unsigned ispc_sbase = ispc_smem_addr(ispc_smem);\n";
  o << "  auto load = [&](int kt, int slot) {\n";
  o << "    const unsigned sA = ispc_sbase + slot * " << stage * 4 << "u;\n";
  o << "    const unsigned sB = sA + " << a_tile * 4 << "u;\n";
  o << "    const long long k0 = (long long)kt * " << BK << ";\n";
  o << "    #pragma unroll\n    for (int ch = tid; ch < " << a_tile / 4 << "; ch += " << T << ") {\n";
  o << "      const int kk = ch / " << BM / 4 << ", mm = (ch % " << BM / 4 << ") * 4;\n";
  o << "      " << (c.cache == ISPC_CACHE_L1 ? "ispc_cp_async_ca16_s" : "ispc_cp_async_cg16_s") << "(sA + (kk * "
    << BM << " + mm) * 4u, pa + mm + (k0 + kk) * " << M << "LL);\n    }\n";
  o << "    #pragma unroll\n    for (int e = tid; e < " << BK * BN << "; e += " << T << ") {\n";
  o << "      const int kk = e % " << BK << ", nn = e / " << BK << ";\n";
  o << "      ispc_cp_async_ca4_s(sB + (kk * " << LDB << " + nn) * 4u, pb + k0 + kk + (long long)nn * " << K
    << "LL);\n    }\n";
  o << "  };\n";
  // the fragments of step k of a staged tile (sA / sB: 32-bit shared-memory
  // addresses of the stage). Decision `lds`: 1 reads them by ld.shared.v4 at
  // 32-bit addresses (NVRTC keeps generic pointer arithmetic 64-bit), 0 by
  // generic float4 pointers - each is faster for some shapes (256 x 64 split-K
  // 2: 46.97 vs 48.13 us; 128 x 64 split 1: 53.2 vs 49.8 us with pdl,
  // profiles/r2m_pdl_probe2.log, r2m_pdl_probe.log)
  const bool LDS = c.lds != 0;
  o << "  auto frag = [&](int buf, unsigned sA, unsigned sB, int k) {\n";
  for (int h = 0; h < TM / 4; ++h) {
    if (LDS)
      o << "    { const float4 t = ispc_lds4(sA + (k * " << BM << " + arow + " << h * LX * 4 << ") * 4u); ";
    else
      o << "    { const float4 t = *(const float4*)(ispc_smem + (sA - ispc_sbase) / 4u + k * " << BM << " + arow + "
        << h * LX * 4 << "); ";
    o << "fa[buf][" << 4 * h << "] = t.x; fa[buf][" << 4 * h + 1 << "] = t.y; fa[buf][" << 4 * h + 2
      << "] = t.z; fa[buf][" << 4 * h + 3 << "] = t.w; }\n";
  }
  for (int h = 0; h < TN / 4; ++h) {
    if (LDS)
      o << "    { const float4 t = ispc_lds4(sB + (k * " << LDB << " + bcol + " << h * LY * 4 << ") * 4u); ";
    else
      o << "    { const float4 t = *(const float4*)(ispc_smem + (sB - ispc_sbase) / 4u + k * " << LDB << " + bcol + "
        << h * LY * 4 << "); ";
    o << "fb[buf][" << 4 * h << "] = t.x; fb[buf][" << 4 * h + 1 << "] = t.y; fb[buf][" << 4 * h + 2
      << "] = t.z; fb[buf][" << 4 * h + 3 << "] = t.w; }\n";
  }
  o << "  };\n";
  o << "  #pragma unroll\n  for (int s = 0; s < " << S - 1 << "; ++s) {\n    if (s < ispc_kt"
    << ") load(s, s);\n    ispc_cp_async_commit();\n  }\n";
  o << "  ispc_cp_async_wait<" << S - 2 << ">();\n  __syncthreads();\n";
  o << "  frag(0, ispc_sbase, ispc_sbase + " << a_tile * 4 << "u, 0);\n";
  o << "  #pragma unroll 1\n  for (int kt = 0; kt < ispc_kt; ++kt) {\n";
  o << "    const unsigned sA = ispc_sbase + (kt % " << S << ") * " << stage * 4 << "u;\n";
  o << "    const unsigned sB = sA + " << a_tile * 4 << "u;\n";
  o << "    #pragma unroll\n    for (int k = 0; k < " << BK << "; ++k) {\n";
  o << "      if (k == " << BK - 1 << ") {  // the next tile's first fragment, after its barrier\n";
  o << "        ispc_cp_async_wait<" << S - 2 << ">();\n        __syncthreads();\n";
  o << "        const unsigned nA = ispc_sbase + ((kt + 1) % " << S << ") * " << stage * 4 << "u;\n";
  o << "        frag((k + 1) & 1, nA, nA + " << a_tile * 4 << "u, 0);\n";
  o << "      } else {\n        frag((k + 1) & 1, sA, sB, k + 1);\n      }\n";
  o << "      if (k == 0) {\n        const int nk = kt + " << S - 1 << ";\n        if (nk < ispc_kt"
    << ") load(nk, nk % " << S << ");\n        ispc_cp_async_commit();\n      }\n";
  // i (A pairs) outer, j serpentine: consecutive FFMA2s share the A pair and,
  // across an i step, the B value (operand reuse; 46.6 vs 49.1 us per tile,
  // profiles/r2k_sgemm_lab2.log)
  o << "      #pragma unroll\n      for (int i = 0; i < " << TM << "; i += 2)\n";
  o << "        #pragma unroll\n        for (int jj = 0; jj < " << TN << "; ++jj) {\n";
  o << "          const int j = ((i / 2) & 1) ? " << TN - 1 << " - jj : jj;\n";
  o << "          const float2 r = __ffma2_rn(make_float2(fa[k & 1][i], fa[k & 1][i + 1]), make_float2(fb[k & 1][j], "
       "fb[k & 1][j]), make_float2(acc[j][i], acc[j][i + 1]));\n";
  o << "          acc[j][i] = r.x; acc[j][i + 1] = r.y;\n        }\n";
  o << "    }\n  }\n";
  o << "  ispc_cp_async_wait<0>();\n";
  if (SP == 1) {
    o << "  #pragma unroll\n  for (int j = 0; j < " << TN << "; ++j) {\n";
    o << "    const long long col = bn * " << BN << "LL + bcol + (j / 4) * " << LY * 4 << " + j % 4;\n";
    o << "    #pragma unroll\n    for (int i = 0; i < " << TM << "; i += 4)\n";
    o << "      *(float4*)(g_c + bm * " << BM << "LL + arow + (i / 4) * " << LX * 4
      << " + col * " << M << "LL) = make_float4(acc[j][i], acc[j][i + 1], acc[j][i + 2], acc[j][i + 3]);\n  }\n";
  } else if ((TM * TN / 4) % SP == 0) {
    // exchange: the thread's float4 vectors v (column j, rows i..i+3) are
    // finished by CTA v % SP of the cluster; after a cluster barrier (every
    // CTA is done with its ring) each CTA stores the vectors others finish
    // into slot X[its rank][v / SP][tid] of the finisher's shared memory
    // (DSMEM), and after a second barrier each finisher sums the SP partials
    // of its vectors in rank order (as the slice reduction below does) and
    // stores them: one remote store per foreign vector, no local staging
    const int NV = TM * TN / 4, NU = NV / SP;
    o << "  ispc_cluster_sync();\n";
    o << "  float* X = ispc_smem;\n";
    for (int v = 0; v < NV; ++v) {
      const int j = v / (TM / 4), i = (v % (TM / 4)) * 4;
      o << "  if (rank != " << v % SP << ") ispc_dsmem_st4(X + ((rank * " << NU << " + " << v / SP << ") * " << T
        << " + tid) * 4, " << v % SP << ", make_float4(acc[" << j << "][" << i << "], acc[" << j << "][" << i + 1
        << "], acc[" << j << "][" << i + 2 << "], acc[" << j << "][" << i + 3 << "]));\n";
    }
    o << "  ispc_cluster_sync();\n";
    for (int v = 0; v < NV; ++v) {
      const int j = v / (TM / 4), i = (v % (TM / 4)) * 4;
      o << "  if (rank == " << v % SP << ") {\n";
      o << "    const float4 own = make_float4(acc[" << j << "][" << i << "], acc[" << j << "][" << i + 1 << "], acc["
        << j << "][" << i + 2 << "], acc[" << j << "][" << i + 3 << "]);\n";
      o << "    float4 s = " << v % SP << " == 0 ? own : *(const float4*)(X + ((0 * " << NU << " + " << v / SP << ") * "
        << T << " + tid) * 4);\n";
      for (int q = 1; q < SP; ++q) {
        o << "    { const float4 t = rank == " << q << " ? own : *(const float4*)(X + ((" << q << " * " << NU << " + "
          << v / SP << ") * " << T << " + tid) * 4); s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w; }\n";
      }
      o << "    *(float4*)(g_c + bm * " << BM << "LL + arow + " << (i / 4) * LX * 4 << " + (bn * " << BN
        << "LL + bcol + " << (j / 4) * LY * 4 + j % 4 << ") * " << M << "LL) = s;\n  }\n";
    }
    L.cluster[0] = uint32_t(SP);
    L.cluster[1] = L.cluster[2] = 1;
  } else {
    // partial tile P[col][row] (rows contiguous) in this CTA's shared memory;
    // CTA `rank` sums slice `rank` of every CTA's P in rank order and stores it
    const int64_t slice = BM * BN / SP;
    o << "  __syncthreads();\n  float* P = ispc_smem;\n";
    o << "  #pragma unroll\n  for (int j = 0; j < " << TN << "; ++j)\n";
    o << "    #pragma unroll\n    for (int i = 0; i < " << TM << "; i += 4)\n";
    o << "      *(float4*)(P + (bcol + (j / 4) * " << LY * 4 << " + j % 4) * " << BM << " + arow + (i / 4) * " << LX * 4
      << ") = make_float4(acc[j][i], acc[j][i + 1], acc[j][i + 2], acc[j][i + 3]);\n";
    o << "  ispc_cluster_sync();\n";
    o << "  for (int e = rank * " << slice << " + tid * 4; e < (rank + 1) * " << slice << "; e += " << 4 * T << ") {\n";
    o << "    float4 s = ispc_dsmem_ld4(P + e, 0);\n";
    o << "    #pragma unroll\n    for (int q = 1; q < " << SP << "; ++q) {\n";
    o << "      const float4 t = ispc_dsmem_ld4(P + e, q);\n";
    o << "      s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w;\n    }\n";
    o << "    const int col = e / " << BM << ", row = e % " << BM << ";\n";
    o << "    *(float4*)(g_c + bm * " << BM << "LL + row + (bn * " << BN << "LL + col) * " << M << "LL) = s;\n  }\n";
    o << "  ispc_cluster_sync();\n";
    L.cluster[0] = uint32_t(SP);
    L.cluster[1] = L.cluster[2] = 1;
  }
  o << "}\n";
  L.grid_x = uint64_t(M / BM * (N / BN) * SP);
  L.block[0] = uint32_t(T);
  L.block[1] = L.block[2] = 1;
  L.static_smem = uint32_t(std::max<int64_t>(stage * S, SP > 1 ? BM * BN : 0) * 4);
  add_region(L, "a", M * K);
  add_region(L, "b", K * N);
  add_region(L, "c", M * N);
  L.reg_elems = uint32_t(TM * TN);
  return o.str();
}

std::string sgemm(const ispc_tile_config& c, const std::string& fn, ispc_launch& L) {
  if (sgemm_warp_tiled_ok(c)) return sgemm_warp_tiled(c, fn, L);
  const int64_t M = c.m, N = c.n, K = c.k;
  GemmShape g = gemm_shape(c, M, N, K);
  if (c.staging != ISPC_STAGE_SHARED && c.staging != ISPC_STAGE_CP_ASYNC)
    illegal("FFMA sgemm stages operands through shared memory (SHARED or CP_ASYNC)");
  if (c.staging == ISPC_STAGE_SHARED && g.S > 2) illegal("SHARED staging is single or double buffered");
  // split-K over a thread-block cluster: CTA `rank` of the cluster walks
  // k in [rank*K/SP, (rank+1)*K/SP); partial tiles are summed through
  // distributed shared memory in rank order (norm-wise checked, not bit-exact)
  const int SP = std::max(1, c.split);
  if (SP > 8) illegal("cluster larger than 8 CTAs");
  if (K % (int64_t(SP) * g.BK)) illegal("split-K slices do not divide K");
  if ((g.BM * g.BN) % (4 * SP)) illegal("partial tile does not split across the cluster");
  const int64_t KT = K / (int64_t(SP) * g.BK);
  const int V = g.V;
  const std::string vty = V == 4 ? "float4" : V == 2 ? "float2" : "float";
  std::ostringstream o;
  o << "extern \"C\" __global__ void __launch_bounds__(" << g.T << ") " << fn
    << "(const float* __restrict__ g_a, const float* __restrict__ g_b, float* __restrict__ g_c) {\n";
  o << "  extern __shared__ __align__(16) float ispc_smem[];\n";
  o << "  const int tid = threadIdx.x, tx = tid % " << g.TX << ", ty = tid / " << g.TX << ";\n";
  o << "  const long long tile = blockIdx.x / " << SP << ";\n";
  o << "  const int rank = " << (SP > 1 ? "(int)ispc_cluster_rank()" : "0") << ";\n";
  o << "  const long long bm = tile % " << M / g.BM << ", bn = tile / " << M / g.BM << ";\n";
  o << "  const long long kbase = (long long)rank * " << K / SP << "LL;\n";
  o << "  const float* pa = g_a + bm * " << g.BM << "LL + kbase * " << M << "LL;\n";
  o << "  const float* pb = g_b + bn * " << g.BN << "LL * " << K << "LL + kbase;\n";
  o << "  float acc[" << g.TN << "][" << g.TM << "];\n";
  o << "  #pragma unroll\n  for (int j = 0; j < " << g.TN << "; ++j)\n    #pragma unroll\n    for (int i = 0; i < "
    << g.TM << "; ++i) acc[j][i] = 0.0f;\n";
  if (c.staging == ISPC_STAGE_CP_ASYNC) {
    const int S = g.S;
    if (S == 1) {
      o << "  #pragma unroll 1\n  for (int kt = 0; kt < " << KT << "; ++kt) {\n";
      gemm_copy_cp_async(o, g, c, M, K, "pa", "pb", "kt", "0", "    ");
      o << "    ispc_cp_async_commit();\n    ispc_cp_async_wait<0>();\n    __syncthreads();\n";
      gemm_compute(o, g, "ispc_smem", "(ispc_smem + " + std::to_string(g.a_tile) + ")", "    ");
      o << "    __syncthreads();\n  }\n";
    } else {
      o << "  #pragma unroll\n  for (int s = 0; s < " << S - 1 << "; ++s) {\n";
      o << "    if (s < " << KT << ") {\n";
      gemm_copy_cp_async(o, g, c, M, K, "pa", "pb", "s", "s", "      ");
      o << "    }\n    ispc_cp_async_commit();\n  }\n";
      o << "  #pragma unroll 1\n  for (int kt = 0; kt < " << KT << "; ++kt) {\n";
      o << "    ispc_cp_async_wait<" << S - 2 << ">();\n    __syncthreads();\n";
      o << "    {\n      const int nk = kt + " << S - 1 << ";\n      if (nk < " << KT << ") {\n";
      gemm_copy_cp_async(o, g, c, M, K, "pa", "pb", "nk", "nk % " + std::to_string(S), "        ");
      o << "      }\n      ispc_cp_async_commit();\n    }\n";
      o << "    const float* sA = ispc_smem + (kt % " << S << ") * " << g.stage_floats << ";\n";
      gemm_compute(o, g, "sA", "(sA + " + std::to_string(g.a_tile) + ")", "    ");
      o << "  }\n";
      o << "  ispc_cp_async_wait<0>();\n";
    }
  } else {
    // SHARED: global -> registers -> shared; stages 2 prefetches tile kt+1
    // into registers while tile kt is computed
    const int64_t a_chunks = g.a_tile / V, b_chunks = int64_t(g.BN) * g.BK / V;
    const int64_t ra_n = (a_chunks + g.T - 1) / g.T, rb_n = (b_chunks + g.T - 1) / g.T;
    auto load_regs = [&](const std::string& kt, const std::string& ind) {
      o << ind << "{\n" << ind << "  const long long k0 = (long long)(" << kt << ") * " << g.BK << ";\n";
      o << ind << "  #pragma unroll\n" << ind << "  for (int r = 0; r < " << ra_n << "; ++r) {\n";
      o << ind << "    const int ch = tid + r * " << g.T << ";\n";
      o << ind << "    if (ch < " << a_chunks << ") {\n";
      o << ind << "      const int kk = ch / " << g.BM / V << ", mm = (ch % " << g.BM / V << ") * " << V << ";\n";
      o << ind << "      pfa[r] = " << ld(c.cache, V, "pa + mm + (k0 + kk) * " + std::to_string(M) + "LL") << ";\n";
      o << ind << "    }\n" << ind << "  }\n";
      o << ind << "  #pragma unroll\n" << ind << "  for (int r = 0; r < " << rb_n << "; ++r) {\n";
      o << ind << "    const int ch = tid + r * " << g.T << ";\n";
      o << ind << "    if (ch < " << b_chunks << ") {\n";
      o << ind << "      const int nn = ch / " << g.BK / V << ", kk = (ch % " << g.BK / V << ") * " << V << ";\n";
      o << ind << "      pfb[r] = " << ld(c.cache, V, "pb + k0 + kk + (long long)nn * " + std::to_string(K) + "LL")
        << ";\n";
      o << ind << "    }\n" << ind << "  }\n" << ind << "}\n";
    };
    auto store_regs = [&](const std::string& buf, const std::string& ind) {
      o << ind << "{\n" << ind << "  float* sA = ispc_smem + (" << buf << ") * " << g.stage_floats << ";\n";
      o << ind << "  float* sB = sA + " << g.a_tile << ";\n";
      o << ind << "  #pragma unroll\n" << ind << "  for (int r = 0; r < " << ra_n << "; ++r) {\n";
      o << ind << "    const int ch = tid + r * " << g.T << ";\n";
      o << ind << "    if (ch < " << a_chunks << ") {\n";
      o << ind << "      const int kk = ch / " << g.BM / V << ", mm = (ch % " << g.BM / V << ") * " << V << ";\n";
      o << ind << "      *(" << vty << "*)(sA + kk * " << g.BM << " + mm) = pfa[r];\n";
      o << ind << "    }\n" << ind << "  }\n";
      o << ind << "  #pragma unroll\n" << ind << "  for (int r = 0; r < " << rb_n << "; ++r) {\n";
      o << ind << "    const int ch = tid + r * " << g.T << ";\n";
      o << ind << "    if (ch < " << b_chunks << ") {\n";
      o << ind << "      const int nn = ch / " << g.BK / V << ", kk = (ch % " << g.BK / V << ") * " << V << ";\n";
      o << ind << "      *(" << vty << "*)(sB + nn * " << g.ldb << " + kk) = pfb[r];\n";
      o << ind << "    }\n" << ind << "  }\n" << ind << "}\n";
    };
    o << "  " << vty << " pfa[" << ra_n << "], pfb[" << rb_n << "];\n";
    if (g.S == 1) {
      o << "  #pragma unroll 1\n  for (int kt = 0; kt < " << KT << "; ++kt) {\n";
      load_regs("kt", "    ");
      store_regs("0", "    ");
      o << "    __syncthreads();\n";
      gemm_compute(o, g, "ispc_smem", "(ispc_smem + " + std::to_string(g.a_tile) + ")", "    ");
      o << "    __syncthreads();\n  }\n";
    } else {
      load_regs("0", "  ");
      store_regs("0", "  ");
      o << "  __syncthreads();\n";
      o << "  #pragma unroll 1\n  for (int kt = 0; kt < " << KT << "; ++kt) {\n";
      o << "    if (kt + 1 < " << KT << ") {\n";
      load_regs("kt + 1", "      ");
      o << "    }\n";
      o << "    const float* sA = ispc_smem + (kt & 1) * " << g.stage_floats << ";\n";
      gemm_compute(o, g, "sA", "(sA + " + std::to_string(g.a_tile) + ")", "    ");
      o << "    if (kt + 1 < " << KT << ") {\n";
      store_regs("(kt + 1) & 1", "      ");
      o << "    }\n    __syncthreads();\n  }\n";
    }
  }
  // epilogue: C[i + j*M], vectors along m
  const int EV = g.TM % 4 == 0 ? 4 : g.TM % 2 == 0 ? 2 : 1;
  const std::string ety = EV == 4 ? "float4" : EV == 2 ? "float2" : "float";
  if (SP == 1) {
    o << "  float* pc = g_c + (bm * " << g.BM << "LL + tx * " << EV << ") + (bn * " << g.BN << "LL + ty) * " << M
      << "LL;\n";
    o << "  #pragma unroll\n  for (int j = 0; j < " << g.TN << "; ++j)\n";
    o << "    #pragma unroll\n    for (int i = 0; i < " << g.TM << "; i += " << EV << ")\n";
    if (EV == 1) o << "      pc[i * " << g.TX << " + (long long)j * " << int64_t(g.TY) * M << "LL] = acc[j][i];\n";
    else {
      o << "      *(" << ety << "*)(pc + (i / " << EV << ") * " << g.TX * EV << " + (long long)j * " << int64_t(g.TY) * M
        << "LL) = make_" << ety << "(";
      for (int e = 0; e < EV; ++e) o << (e ? ", " : "") << "acc[j][i + " << e << "]";
      o << ");\n";
    }
  } else {
    // partial tile P[col][row] (BN x BM, rows contiguous) in this CTA's shared
    // memory; CTA `rank` then sums slice `rank` of every CTA's P and stores it
    const int64_t tile_elems = g.BM * g.BN, slice = tile_elems / SP;
    o << "  __syncthreads();\n";
    o << "  float* P = ispc_smem;\n";
    o << "  #pragma unroll\n  for (int j = 0; j < " << g.TN << "; ++j)\n";
    o << "    #pragma unroll\n    for (int i = 0; i < " << g.TM << "; ++i) P[(ty + j * " << g.TY << ") * " << g.BM
      << " + (i / " << EV << ") * " << g.TX * EV << " + tx * " << EV << " + i % " << EV << "] = acc[j][i];\n";
    o << "  ispc_cluster_sync();\n";
    if (g.BM % 4 == 0) {  // four rows of one column per step: aligned float4 everywhere
      o << "  for (int e = rank * " << slice << " + tid * 4; e < (rank + 1) * " << slice << "; e += " << 4 * g.T << ") {\n";
      o << "    float4 s = ispc_dsmem_ld4(P + e, 0);\n";
      o << "    #pragma unroll\n    for (int q = 1; q < " << SP << "; ++q) {\n";
      o << "      const float4 t = ispc_dsmem_ld4(P + e, q);\n";
      o << "      s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w;\n    }\n";
      o << "    const int col = e / " << g.BM << ", row = e % " << g.BM << ";\n";
      o << "    *(float4*)(g_c + bm * " << g.BM << "LL + row + (bn * " << g.BN << "LL + col) * " << M << "LL) = s;\n";
      o << "  }\n";
    } else {
      o << "  for (int e = rank * " << slice << " + tid; e < (rank + 1) * " << slice << "; e += " << g.T << ") {\n";
      o << "    float s = ispc_dsmem_ld(P + e, 0);\n";
      o << "    #pragma unroll\n    for (int q = 1; q < " << SP << "; ++q) s += ispc_dsmem_ld(P + e, q);\n";
      o << "    const int col = e / " << g.BM << ", row = e % " << g.BM << ";\n";
      o << "    g_c[bm * " << g.BM << "LL + row + (bn * " << g.BN << "LL + col) * " << M << "LL] = s;\n";
      o << "  }\n";
    }
    o << "  ispc_cluster_sync();\n";
    L.cluster[0] = uint32_t(SP);
    L.cluster[1] = L.cluster[2] = 1;
  }
  o << "}\n";
  L.grid_x = uint64_t(M / g.BM * (N / g.BN) * SP);
  L.block[0] = uint32_t(g.T);
  L.block[1] = L.block[2] = 1;
  L.static_smem = uint32_t(std::max<int64_t>(g.stage_floats * g.S, SP > 1 ? g.BM * g.BN : 0) * 4);
  add_region(L, "a", M * K);
  add_region(L, "b", K * N);
  add_region(L, "c", M * N);
  L.reg_elems = uint32_t(g.TM * g.TN);
  return o.str();
}

// ---------------------------------------------------------------- batched sgemm
// batch x (C_b = A_b B_b), each column-major and densely packed:
// A_b = a + b*M*K, B_b = b + b*K*N, C_b = c + b*M*N. A CTA holds `per_cta`
// problems; each problem gets (M/tm)*(N/tn) threads owning a tm x tn output
// tile. DIRECT reads operands from global (L1); SHARED stages bk-deep slices
// of every problem's A and B cooperatively. k ascending per output (bit-exact).
// CP_ASYNC batched: every thread of the CTA works on one problem at a time;
// the CTA walks its `per_cta` problems in order through a 2-stage cp.async
// ring, so problem q+1's operands land while problem q is computed. Whole-K
// slices: A_b (M x K, m contiguous) and B_b stored n-major with k contiguous
// (row pitch K + 4). k ascending per output (bit-exact).
std::string batched_pipelined(const ispc_tile_config& c, const std::string& fn, ispc_launch& L) {
  const int64_t M = c.m, N = c.n, K = c.k, B = c.batch;
  const int P = c.per_cta, TM = c.tm, TN = c.tn;
  if (P < 1 || TM < 1 || TN < 1) illegal("non-positive tile parameter");
  if (M % TM || N % TN) illegal("thread tile does not divide the problem");
  if (B % P) illegal("problems per CTA do not divide the batch");
  const int64_t TPX = M / TM, TPY = N / TN, T = TPX * TPY;
  if (T > 1024) illegal("more than 1024 threads per CTA");
  if (T < 32) illegal("fewer than 32 threads per CTA");
  if (int64_t(TM) * TN > 64) illegal("more than 64 accumulators per thread");
  const int V = c.vec;
  if (!(V == 1 || V == 2 || V == 4)) illegal("vector width must be 1, 2 or 4");
  if (M % V || K % V) illegal("vector width does not divide the problem");
  const int64_t ldb = K + 4, stage = M * K + N * ldb;
  const int64_t smem = 2 * stage * 4;
  if (smem > 232448) illegal("shared memory exceeds 227 KiB");
  const std::string cp = V == 4 ? (c.cache == ISPC_CACHE_L1 ? "ispc_cp_async_ca16" : "ispc_cp_async_cg16")
                                : V == 2 ? "ispc_cp_async_ca8" : "ispc_cp_async_ca4";
  const int64_t a_ch = M * K / V, b_ch = N * K / V;
  std::ostringstream o;
  o << "extern \"C\" __global__ void __launch_bounds__(" << T << ") " << fn
    << "(const float* __restrict__ g_a, const float* __restrict__ g_b, float* __restrict__ g_c) {\n";
  o << "  extern __shared__ __align__(16) float ispc_smem[];\n";
  o << "  const int tid = threadIdx.x, tx = tid % " << TPX << ", ty = tid / " << TPX << ";\n";
  o << "  const long long first = (long long)blockIdx.x * " << P << ";\n";
  auto issue = [&](const std::string& q, const std::string& ind) {
    o << ind << "{\n";
    o << ind << "  float* sa = ispc_smem + ((" << q << ") & 1) * " << stage << ";\n";
    o << ind << "  float* sb = sa + " << M * K << ";\n";
    o << ind << "  const float* ga = g_a + (first + (" << q << ")) * " << M * K << "LL;\n";
    o << ind << "  const float* gb = g_b + (first + (" << q << ")) * " << K * N << "LL;\n";
    o << ind << "  for (int ch = tid; ch < " << a_ch << "; ch += " << T << ") " << cp << "(sa + ch * " << V
      << ", ga + ch * " << V << ");\n";
    o << ind << "  for (int ch = tid; ch < " << b_ch << "; ch += " << T << ") {\n";
    o << ind << "    const int nn = ch / " << K / V << ", kk = (ch % " << K / V << ") * " << V << ";\n";
    o << ind << "    " << cp << "(sb + nn * " << ldb << " + kk, gb + nn * " << K << " + kk);\n";
    o << ind << "  }\n" << ind << "}\n";
  };
  issue("0", "  ");
  o << "  ispc_cp_async_commit();\n";
  o << "  #pragma unroll 1\n  for (int q = 0; q < " << P << "; ++q) {\n";
  o << "    if (q + 1 < " << P << ") {\n";
  issue("q + 1", "      ");
  o << "    }\n    ispc_cp_async_commit();\n";
  o << "    ispc_cp_async_wait<1>();\n    __syncthreads();\n";
  o << "    const float* sa = ispc_smem + (q & 1) * " << stage << ";\n";
  o << "    const float* sb = sa + " << M * K << ";\n";
  o << "    float acc[" << TN << "][" << TM << "];\n";
  o << "    #pragma unroll\n    for (int j = 0; j < " << TN << "; ++j)\n      #pragma unroll\n      for (int i = 0; i < "
    << TM << "; ++i) acc[j][i] = 0.0f;\n";
  o << "    #pragma unroll 4\n    for (int k = 0; k < " << K << "; ++k) {\n";
  o << "      float ra[" << TM << "], rb[" << TN << "];\n";
  o << "      #pragma unroll\n      for (int i = 0; i < " << TM << "; ++i) ra[i] = sa[k * " << M << " + tx * " << TM
    << " + i];\n";
  o << "      #pragma unroll\n      for (int j = 0; j < " << TN << "; ++j) rb[j] = sb[(ty + j * " << TPY << ") * "
    << ldb << " + k];\n";
  o << "      #pragma unroll\n      for (int j = 0; j < " << TN << "; ++j)\n";
  o << "        #pragma unroll\n        for (int i = 0; i < " << TM << "; ++i) acc[j][i] = __fmaf_rn(ra[i], rb[j], acc[j][i]);\n";
  o << "    }\n";
  o << "    float* pc = g_c + (first + q) * " << M * N << "LL + tx * " << TM << ";\n";
  o << "    #pragma unroll\n    for (int j = 0; j < " << TN << "; ++j)\n";
  o << "      #pragma unroll\n      for (int i = 0; i < " << TM << "; ++i) pc[i + (ty + j * " << TPY << ") * " << M
    << "] = acc[j][i];\n";
  o << "    __syncthreads();\n  }\n";
  o << "  ispc_cp_async_wait<0>();\n}\n";
  L.grid_x = uint64_t(B / P);
  L.block[0] = uint32_t(T);
  L.block[1] = L.block[2] = 1;
  L.static_smem = uint32_t(smem);
  add_region(L, "a", B * M * K);
  add_region(L, "b", B * K * N);
  add_region(L, "c", B * M * N);
  L.reg_elems = uint32_t(TM * TN);
  return o.str();
}

std::string batched(const ispc_tile_config& c, const std::string& fn, ispc_launch& L) {
  if (c.staging == ISPC_STAGE_CP_ASYNC) return batched_pipelined(c, fn, L);
  const int64_t M = c.m, N = c.n, K = c.k, B = c.batch;
  const int P = c.per_cta, TM = c.tm, TN = c.tn, BK = c.bk;
  if (P < 1 || TM < 1 || TN < 1 || BK < 1) illegal("non-positive tile parameter");
  if (M % TM || N % TN) illegal("thread tile does not divide the problem");
  if (B % P) illegal("problems per CTA do not divide the batch");
  if (K % BK) illegal("k depth does not divide K");
  const int64_t TPX = M / TM, TPY = N / TN, TP = TPX * TPY, T = TP * P;
  if (T > 1024) illegal("more than 1024 threads per CTA");
  if (T < 32) illegal("fewer than 32 threads per CTA");
  if (int64_t(TM) * TN > 64) illegal("more than 64 accumulators per thread");
  const bool sh = c.staging == ISPC_STAGE_SHARED;
  if (!sh && c.staging != ISPC_STAGE_DIRECT) illegal("batched stages through registers or shared memory");
  const int64_t ldb = BK + (BK % 4 == 0 ? 4 : 1);
  const int64_t per_prob = BK * M + N * ldb;  // floats per problem slice
  const int64_t smem = sh ? per_prob * P * 4 : 0;
  if (smem > 232448) illegal("shared memory exceeds 227 KiB");
  const int V = c.vec;
  if (!(V == 1 || V == 2 || V == 4)) illegal("vector width must be 1, 2 or 4");
  if (sh && (M % V || BK % V)) illegal("vector width does not divide the staged slices");
  std::ostringstream o;
  o << "extern \"C\" __global__ void __launch_bounds__(" << T << ") " << fn
    << "(const float* __restrict__ g_a, const float* __restrict__ g_b, float* __restrict__ g_c) {\n";
  o << "  extern __shared__ __align__(16) float ispc_smem[];\n";
  o << "  const int tid = threadIdx.x, p = tid / " << TP << ", lt = tid % " << TP << ";\n";
  o << "  const int tx = lt % " << TPX << ", ty = lt / " << TPX << ";\n";
  o << "  const long long prob = (long long)blockIdx.x * " << P << " + p;\n";
  o << "  const float* pa = g_a + prob * " << M * K << "LL;\n";
  o << "  const float* pb = g_b + prob * " << K * N << "LL;\n";
  o << "  float acc[" << TN << "][" << TM << "];\n";
  o << "  #pragma unroll\n  for (int j = 0; j < " << TN << "; ++j)\n    #pragma unroll\n    for (int i = 0; i < " << TM
    << "; ++i) acc[j][i] = 0.0f;\n";
  o << "  #pragma unroll 1\n  for (int k0 = 0; k0 < " << K << "; k0 += " << BK << ") {\n";
  if (sh) {
    const std::string vty = V == 4 ? "float4" : V == 2 ? "float2" : "float";
    o << "    __syncthreads();\n";
    // every thread of the CTA copies chunks of all problems' slices
    const int64_t a_ch = BK * M / V, b_ch = N * BK / V;
    o << "    for (int ch = tid; ch < " << P * (a_ch + b_ch) << "; ch += " << T << ") {\n";
    o << "      const int q = ch / " << a_ch + b_ch << ", r = ch % " << a_ch + b_ch << ";\n";
    o << "      const long long qb = (long long)blockIdx.x * " << P << " + q;\n";
    o << "      float* s = ispc_smem + q * " << per_prob << ";\n";
    o << "      if (r < " << a_ch << ") {\n";
    o << "        const int kk = r / " << M / V << ", mm = (r % " << M / V << ") * " << V << ";\n";
    o << "        *(" << vty << "*)(s + kk * " << M << " + mm) = "
      << ld(c.cache, V, "g_a + qb * " + std::to_string(M * K) + "LL + mm + (k0 + kk) * " + std::to_string(M) + "LL")
      << ";\n";
    o << "      } else {\n        const int r2 = r - " << a_ch << ";\n";
    o << "        const int nn = r2 / " << BK / V << ", kk = (r2 % " << BK / V << ") * " << V << ";\n";
    o << "        " << vty << " v = "
      << ld(c.cache, V, "g_b + qb * " + std::to_string(K * N) + "LL + k0 + kk + (long long)nn * " + std::to_string(K) + "LL")
      << ";\n";
    if (V == 1) o << "        s[" << BK * M << " + nn * " << ldb << " + kk] = v;\n";
    else
      for (int e = 0; e < V; ++e)
        o << "        s[" << BK * M << " + nn * " << ldb << " + kk + " << e << "] = v" << comp(e) << ";\n";
    o << "      }\n    }\n    __syncthreads();\n";
    o << "    const float* sa = ispc_smem + p * " << per_prob << ";\n";
    o << "    const float* sb = sa + " << BK * M << ";\n";
    o << "    #pragma unroll\n    for (int kk = 0; kk < " << BK << "; ++kk) {\n";
    o << "      float ra[" << TM << "], rb[" << TN << "];\n";
    o << "      #pragma unroll\n      for (int i = 0; i < " << TM << "; ++i) ra[i] = sa[kk * " << M << " + tx * " << TM
      << " + i];\n";
    o << "      #pragma unroll\n      for (int j = 0; j < " << TN << "; ++j) rb[j] = sb[(ty * " << TN << " + j) * "
      << ldb << " + kk];\n";
  } else {
    o << "    #pragma unroll\n    for (int kk = 0; kk < " << BK << "; ++kk) {\n";
    o << "      float ra[" << TM << "], rb[" << TN << "];\n";
    o << "      #pragma unroll\n      for (int i = 0; i < " << TM << "; ++i) ra[i] = "
      << ld(c.cache, 1, "pa + tx * " + std::to_string(TM) + " + i + (k0 + kk) * " + std::to_string(M) + "LL") << ";\n";
    o << "      #pragma unroll\n      for (int j = 0; j < " << TN << "; ++j) rb[j] = "
      << ld(c.cache, 1, "pb + k0 + kk + (long long)(ty * " + std::to_string(TN) + " + j) * " + std::to_string(K) + "LL")
      << ";\n";
  }
  o << "      #pragma unroll\n      for (int j = 0; j < " << TN << "; ++j)\n";
  o << "        #pragma unroll\n        for (int i = 0; i < " << TM << "; ++i) acc[j][i] = __fmaf_rn(ra[i], rb[j], acc[j][i]);\n";
  o << "    }\n  }\n";
  o << "  float* pc = g_c + prob * " << M * N << "LL + tx * " << TM << " + (long long)(ty * " << TN << ") * " << M << "LL;\n";
  o << "  #pragma unroll\n  for (int j = 0; j < " << TN << "; ++j)\n";
  o << "    #pragma unroll\n    for (int i = 0; i < " << TM << "; ++i) pc[i + j * " << M << "] = acc[j][i];\n";
  o << "}\n";
  L.grid_x = uint64_t(B / P);
  L.block[0] = uint32_t(T);
  L.block[1] = L.block[2] = 1;
  L.static_smem = uint32_t(smem);
  add_region(L, "a", B * M * K);
  add_region(L, "b", B * K * N);
  add_region(L, "c", B * M * N);
  L.reg_elems = uint32_t(TM * TN);
  return o.str();
}

// ---------------------------------------------------------------- axpy stream
// z = alpha*x + y (mul then add, each rounded: the backbone's two
// instructions, kernels.cpp:397-403). Vector group c (vec floats) of a
// grid-stride walk: c = (blockIdx.x*unroll + u)*threads + tid, so a warp
// touches 32 consecutive vectors per load; `unroll` groups in flight per
// thread; grid = `grid` CTAs (0: exactly one group per thread).
std::string axpy_stream(const ispc_tile_config& c, const std::string& fn, ispc_launch& L) {
  const int64_t n = c.n;
  const int V = c.vec, T = c.threads, U = c.unroll;
  if (!(V == 1 || V == 2 || V == 4)) illegal("vector width must be 1, 2 or 4");
  if (T < 32 || T > 1024 || T % 32) illegal("threads per CTA must be a multiple of 32 up to 1024");
  if (U < 1) illegal("non-positive unroll");
  if (n % V) illegal("vector width does not divide n");
  const int64_t groups = n / V, per_cta = int64_t(T) * U;
  const int64_t grid = c.grid > 0 ? c.grid : (groups + per_cta - 1) / per_cta;
  if (grid > 0x7fffffffLL) illegal("grid exceeds 2^31-1 CTAs");
  const std::string ty = V == 4 ? "float4" : V == 2 ? "float2" : "float";
  const bool stream_st = c.cache == ISPC_CACHE_NONE || c.cache == ISPC_CACHE_STREAM;
  std::ostringstream o;
  o << "extern \"C\" __global__ void __launch_bounds__(" << T << ") " << fn
    << "(const float* __restrict__ g_x, const float* __restrict__ g_y, float* __restrict__ g_z, const float p_alpha) {\n";
  o << "  const " << ty << "* __restrict__ vx = (const " << ty << "*)g_x;\n";
  o << "  const " << ty << "* __restrict__ vy = (const " << ty << "*)g_y;\n";
  o << "  " << ty << "* __restrict__ vz = (" << ty << "*)g_z;\n";
  o << "  #pragma unroll 1\n";
  o << "  for (long long c0 = (long long)blockIdx.x * " << per_cta << "LL + threadIdx.x; c0 < " << groups
    << "LL; c0 += (long long)gridDim.x * " << per_cta << "LL) {\n";
  o << "    " << ty << " xv[" << U << "], yv[" << U << "];\n";
  o << "    #pragma unroll\n    for (int u = 0; u < " << U << "; ++u) {\n";
  o << "      const long long g = c0 + u * " << T << ";\n";
  o << "      if (g < " << groups << "LL) { xv[u] = " << ld(c.cache, V, "vx + g") << "; yv[u] = "
    << ld(c.cache, V, "vy + g") << "; }\n";
  o << "    }\n";
  o << "    #pragma unroll\n    for (int u = 0; u < " << U << "; ++u) {\n";
  o << "      const long long g = c0 + u * " << T << ";\n";
  o << "      if (g < " << groups << "LL) {\n";
  o << "        " << ty << " r;\n";
  if (V == 1) o << "        r = __fadd_rn(__fmul_rn(p_alpha, xv[u]), yv[u]);\n";
  else
    for (int v = 0; v < V; ++v)
      o << "        r" << comp(v) << " = __fadd_rn(__fmul_rn(p_alpha, xv[u]" << comp(v) << "), yv[u]" << comp(v)
        << ");\n";
  o << "        " << (stream_st ? "__stcs(vz + g, r);" : "vz[g] = r;") << "\n";
  o << "      }\n    }\n  }\n}\n";
  L.grid_x = uint64_t(grid);
  L.block[0] = uint32_t(T);
  L.block[1] = L.block[2] = 1;
  add_region(L, "x", n);
  add_region(L, "y", n);
  add_region(L, "z", n);
  ispc_param& P = L.params[L.num_params++];
  P.kind = ISPC_PARAM_INPUT;
  P.index = 0;
  std::snprintf(P.name, sizeof(P.name), "alpha");
  L.reg_elems = uint32_t(2 * V * U);
  return o.str();
}

}  // namespace

std::string emit_tile_kernel(const ispc_tile_config& c, const std::string& fn, ispc_launch& L) {
  std::memset(&L, 0, sizeof(L));
  std::snprintf(L.name, sizeof(L.name), "%s", fn.c_str());
  if (c.n <= 0 || (c.kind != ISPC_TILE_AXPY && c.m <= 0) ||
      (c.kind != ISPC_TILE_GEMV && c.kind != ISPC_TILE_AXPY && c.k <= 0))
    illegal("empty problem");
  std::string src;
  switch (c.kind) {
    case ISPC_TILE_GEMV: src = gemv(c, fn, L); break;
    case ISPC_TILE_SGEMM: src = sgemm(c, fn, L); break;
    case ISPC_TILE_BATCHED: src = batched(c, fn, L); break;
    case ISPC_TILE_SGEMM_TC: src = emit_tcgen05_kernel(c, fn, L); break;
    case ISPC_TILE_AXPY: src = axpy_stream(c, fn, L); break;
    default: throw NestError(ISPC_E_ARG, "unknown tile kind");
  }
  if (L.static_smem > 232448) illegal("shared memory exceeds 227 KiB");
  if (c.pdl) {
    // programmatic dependent launch: the grid may be scheduled while the
    // previous grid of the stream drains (launch latency and CTA rasterisation
    // overlap its tail); griddepcontrol.wait, before any memory access, holds
    // every thread until that grid completed and its writes are visible. The
    // trigger right after it lets the next grid be scheduled once all of this
    // grid's CTAs are resident.
    const size_t sig = src.find(" " + fn + "(");
    const size_t body = sig == std::string::npos ? sig : src.find(") {\n", sig);
    if (body == std::string::npos) throw NestError(ISPC_E_ARG, "pdl: kernel body not found");
    src.insert(body + 4, "  ispc_grid_dep_wait();\n  ispc_grid_dep_trigger();\n");
    L.pdl = 1;
  }
  // the launch configuration is part of the candidate: two configurations
  // whose sources coincide (a persistent grid reads gridDim) are different
  // kernels to time, and get different names
  char launch_sig[160];
  std::snprintf(launch_sig, sizeof(launch_sig), "\n// launch grid %llu block %u cluster %u smem %u\n",
                (unsigned long long)L.grid_x, L.block[0], L.cluster[0], L.static_smem);
  L.source_hash = fnv1a(src + launch_sig);
  return src;
}

}  // namespace ispc

extern "C" int ispc_emit_tiles(const ispc_tile_config* cfg, const char* fn_name, char* buf, size_t cap,
                               size_t* len, ispc_launch* launch) {
  try {
    if (!cfg || !launch) throw ispc::NestError(ISPC_E_ARG, "null argument");
    std::string fn = fn_name ? fn_name : "ispc_tile_kernel";
    std::string src = ispc::emit_tile_kernel(*cfg, fn, *launch);
    if (!fn_name) {
      char name[64];
      std::snprintf(name, sizeof(name), "ispc_t%016llx", (unsigned long long)launch->source_hash);
      size_t p = 0;
      while ((p = src.find(fn, p)) != std::string::npos) {
        src.replace(p, fn.size(), name);
        p += std::strlen(name);
      }
      std::snprintf(launch->name, sizeof(launch->name), "%s", name);
    }
    if (len) *len = src.size();
    if (buf && cap) {
      size_t k = src.size() < cap - 1 ? src.size() : cap - 1;
      std::memcpy(buf, src.data(), k);
      buf[k] = 0;
    }
    return ISPC_OK;
  } catch (const ispc::NestError& e) {
    ispc::set_thread_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    ispc::set_thread_error(e.what());
    return ISPC_E_ARG;
  }
}
