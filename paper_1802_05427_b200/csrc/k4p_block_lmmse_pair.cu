// K4 pair variant (k4_bf16x3_pair) -- K4's fused LS + block-LMMSE contraction (k4_block_lmmse_bf16x3.cu: tcgen05
// kind::f16 on BF16 operands, error-compensated "BF16x3": D = A_hi B_hi + A_hi B_lo + A_lo B_hi, FP32 accumulation in
// TMEM; reading B1) on CTA PAIRS: tcgen05 cta_group::2, M = 256.  The pipeline, roles and epilogue are
// K4's (the description below is K4's own); what the pair changes is in the "Pair mode" paragraph at its end.  The
// file is K4's source with PAIR fixed to true: the single-CTA kernel keeps a translation unit of its own because the
// same source compiled for both (a template over PAIR) ran config 3 9 % slower than K4 (9.89 -> 10.81 us, same box).
//
// Same operation as K2/K3 (Eq. 12 per block, LS of Eq. 9 fused into the load) and
// the same complex -> real embedding as K3 (A = interleaved LS row, D = interleaved output row,
// B_r^T rows 2i / 2i+1 = (Re W_ij, -Im W_ij) / (Im W_ij, Re W_ij)).
//
// Work unit: a tile = (instance t, window w, 128-column block ct); one CTA per SM walks its tiles.
//
// Pipeline (persistent, one CTA per SM, 480 threads):
//   warp 12   : raw producer -- 2D TMA of the raw y box [128 rows x 16 complex] and the pilot box
//               [K rows x 16 complex] of each K chunk into a 4-deep raw ring (3-deep when the staged
//               epilogue below takes 16 KB); decodes its first tile while the other warps set up
//   warps 0-7 : transform -- y and x of 4 rows x 2 tones per thread into registers, LS = y conj(x)/|x|^2,
//               release the raw slot, bf16 hi/lo -> SWIZZLE_64B K-major A tiles of the 3-deep A/B ring;
//               fence.proxy.async; arrive a_full
//   warp 14   : B producer -- cp.async.bulk of this CTA's rows of the bf16 hi/lo bank chunk
//               (pre-swizzled SW64 image)
//   warp 13   : TMEM allocator + MMA issuer: 2 K-steps x 3 MMAs per chunk, commit -> st_empty;
//               per tile commit -> tmem_full[acc] (two 256-column accumulators)
//   warps 8-11: epilogue (epi_block) -- tcgen05.ld 16x256b (4 threads hold 4 consecutive outputs of a
//               row) per 32-float column block; interior blocks go through SWIZZLE_128B staging and one TMA
//               store of [32 rows x 128 B] (per-warp staging when CTAs walk several tiles, the idle A/B
//               ring on a CTA's last tile); window edges / odd starts / ragged tiles use direct 8-byte
//               stores (8 rows x 32 contiguous bytes per warp instruction)
// The window table rides in the kernel parameters (no dependent global load before the first TMA), and
// the kernel is launched with programmatic stream serialization (PDL): its launch overlaps the previous
// kernel's tail; griddepcontrol.wait precedes every access to caller data.
//
// Pair mode (k4_bf16x3_pair; launches bf16x3_pair_wanted() selects -- config-5-like): a cluster of two CTAs on one TPC works
// on two adjacent 128-row tiles of the same (instance, window) as ONE tcgen05 cta_group::2 MMA of M = 256.  Each
// CTA transforms its own rows into its own A stage and fetches HALF of the filter chunk's rows (the pair's MMA
// reads both halves in place), so the filter-bank stream per SM and the B bytes each MMA reads from shared memory
// halve; A and B keep rings of their own (4 A stages of 16 KB, 4 B stages of 16 KB, 4 raw stages).  The leader (rank 0)
// issues every MMA; its a_full / tmem_empty barriers count the warps of both CTAs (one arrive per warp, the peer's
// through mapa + mbarrier.arrive on the leader's barrier), the peer's MMA warp forwards "my half of the chunk has
// landed" (bulk copies can only signal a barrier of their own CTA), and the commits are multicast to both CTAs.
// The cross-CTA arrives keep the default CTA-scope release: the data they guard stays in the arriving CTA's own
// shared memory, and a CLUSTER-scope release cost 1-2 us per arrive (the arrive returned only after the SM's
// outstanding loads had drained -- the pair ran 1.7x slower than two single CTAs with it).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>

#include "ce_internal.h"
#include "tc_ptx.cuh"
#include "tmap.cuh"

namespace ce {
namespace {

// Optional per-CTA event trace (tools/k4_trace.cu builds with -DCE_K4_TRACE; the product build has none).
// Timing ablations (results wrong by construction; tools/k4_trace.sh <tag> -D...): K4_ABL_NOSTORE,
// K4_ABL_NOMMA, K4_ABL_NOTRANSFORM, K4_ABL_NOB (no filter-chunk copies).
#ifdef CE_K4_TRACE
__device__ unsigned long long *g_k4_trace;
#define K4TR(slot)                                                                \
  do {                                                                            \
    const unsigned long long c_ = clock64(); /* read before the pointer load */  \
    if (g_k4_trace) g_k4_trace[size_t(blockIdx.x) * 256 + (slot)] = c_;           \
  } while (0)
#else
#define K4TR(slot) \
  do {             \
  } while (0)
#endif

constexpr bool PAIR = true;                // this file is K4's pair variant; K4 proper is k4_block_lmmse_bf16x3.cu
constexpr int K4_THREADS = 480;            // 15 warps: 8 transform, 4 epilogue, 3 single-thread roles
constexpr int NTR = 256;                   // transform threads
constexpr int CK = 16;                     // complex per K chunk = 32 bf16 = 64-byte rows
constexpr int TM = 128;                    // A rows (columns c) per CTA
constexpr int NMAXW = 256;                 // MMA N max (2*kept + row alignment)
constexpr int KMAX = 32;                   // pilot rows per raw stage (K <= 32)
constexpr int S_RAW_MAX = 4;               // raw y/x stages: 4, or 3 when the TMA-store staging is in use
constexpr int A_PLANE = TM * 64;           // 8 KB
constexpr int RAWY = TM * CK * 8;          // 16 KB
constexpr int RAWX = KMAX * CK * 8;        // 4 KB
constexpr int RAW_STAGE = RAWY + RAWX;     // 20 KB
constexpr int EPI_WARP = 4096;             // TMA-store staging per epilogue warp: [32 rows][128 B], SWIZZLE_128B
#ifndef K4_EPI_DB
#define K4_EPI_DB 0          // experiments: 1 = two staging boxes per epilogue warp (two stores in flight), 2 raw stages
#endif
constexpr int EPI_NB = K4_EPI_DB ? 2 : 1;
constexpr int EPI_BYTES = 4 * EPI_NB * EPI_WARP;
constexpr int BAR_BYTES = 384;
constexpr int MAXW_PARAM = 32;             // windows carried in the kernel parameters

#ifndef K4_S_AB
#define K4_S_AB 3
#endif
constexpr int S_AB = K4_S_AB;              // A/B stages (measured: 4 y + 3 A/B beats 5 + 2, 6 + 2)
constexpr int B_PLANE = NMAXW * 64;        // 16 KB
constexpr int AB_STAGE = 2 * A_PLANE + 2 * B_PLANE;      // 48 KB
// with staging: 3 A/B + 3 raw stages + staging; without: 3 A/B + 4 raw stages
constexpr int K4_SMEM_ST = S_AB * AB_STAGE + (S_RAW_MAX - 1 - K4_EPI_DB) * RAW_STAGE + EPI_BYTES + BAR_BYTES + 1024;
constexpr int K4_SMEM_NOST = S_AB * AB_STAGE + S_RAW_MAX * RAW_STAGE + BAR_BYTES + 1024;
constexpr int K4_SMEM = K4_SMEM_ST > K4_SMEM_NOST ? K4_SMEM_ST : K4_SMEM_NOST;
static_assert(K4_SMEM <= 232448, "K4 shared memory");
// Pair mode (a cluster of two CTAs = tcgen05 cta_group::2, M = 256): each CTA keeps its own 128 A rows and HALF of
// the filter chunk's rows (the pair's MMA reads both halves); the raw ring gets what the 227 KB leave.
constexpr int S_RAW_BARS = 6;              // raw-ring barrier slots (>= every ring depth used)
constexpr int B_PLANE_P = B_PLANE / 2;     // 8 KB
// pair mode keeps the filter chunks in a ring of their own, deeper than the A ring: a chunk does not depend on
// the data, so its copy can be issued S_B_P chunks ahead (its L2 latency, ~1 us, otherwise has to hide behind the
// MMAs of S_AB - 1 chunks)
constexpr int A_STAGE_P = 2 * A_PLANE;     // 16 KB: A_hi | A_lo
constexpr int B_STAGE_P = 2 * B_PLANE_P;   // 16 KB: this CTA's half of B_hi | B_lo
#ifndef K4_S_AB_P
#define K4_S_AB_P 4          // A stages in pair mode (4 + 4: config 5 1395-1399 us; 3 + 5: 1406-1427; 2 + 6: 1402)
#endif
#ifndef K4_S_B_P
#define K4_S_B_P 4           // filter-chunk stages in pair mode
#endif
#ifndef K4_EPI_DB_P
#define K4_EPI_DB_P 0        // experiments: 1 = two staging boxes per epilogue warp in pair mode
#endif
constexpr int S_AB_P = K4_S_AB_P;          // A stages in pair mode
constexpr int S_B_P = K4_S_B_P;            // B stages in pair mode
constexpr int S_B_MAX = 6;                 // B barrier slots
constexpr int AB_BYTES_P = S_AB_P * A_STAGE_P + S_B_P * B_STAGE_P;
constexpr int EPI_NB_P = K4_EPI_DB_P ? 2 : 1;
constexpr int EPI_BYTES_P = 4 * EPI_NB_P * EPI_WARP;
// raw stages: whatever the 227 KB leave (at most S_RAW_BARS)
constexpr int raw_fit(int rest) { return rest / RAW_STAGE > 6 ? 6 : rest / RAW_STAGE; }
constexpr int S_RAW_P_ST = raw_fit(232448 - 1024 - BAR_BYTES - AB_BYTES_P - EPI_BYTES_P);
constexpr int S_RAW_P_NOST = raw_fit(232448 - 1024 - BAR_BYTES - AB_BYTES_P);
constexpr int K4P_SMEM_ST = AB_BYTES_P + S_RAW_P_ST * RAW_STAGE + EPI_BYTES_P + BAR_BYTES + 1024;
constexpr int K4P_SMEM_NOST = AB_BYTES_P + S_RAW_P_NOST * RAW_STAGE + BAR_BYTES + 1024;
static_assert(S_RAW_P_ST >= 2 && S_AB_P <= 4 && S_B_P <= S_B_MAX && S_AB <= S_B_MAX, "K4 pair ring depths");
constexpr int K4P_SMEM = K4P_SMEM_ST > K4P_SMEM_NOST ? K4P_SMEM_ST : K4P_SMEM_NOST;
static_assert(K4P_SMEM <= 232448, "K4 pair shared memory");
static_assert(S_RAW_MAX <= S_RAW_BARS && S_RAW_P_NOST <= S_RAW_BARS, "raw-ring barrier slots");

struct K4Params {
  float2 *h;
  const uint16_t *bank_hi;   // bf16 [n_sets][nkc][NR][32] swizzled SW64 rows
  const uint16_t *bank_lo;
  const Window *geo;         // device window table (read only when n_win > MAXW_PARAM)
  const int32_t *soi;
  int T, K, N, b, n_win, n_sets, nkc, NR, cols, n_ct;   // n_ct: 128-row column tiles (pair mode: 256-row pair tiles)
  int n_tiles;               // T * n_win * n_ct
  int pair;                  // 1: k4_bf16x3_pair; CTA rank r of a pair takes the 128-row tile 2 * (g % n_ct) + r
  int tma_store;             // 1: interior 32-float column blocks leave through SW128 staging + TMA stores
  int tma_last;              // 1: the same for each CTA's last tile, staged in the then idle A/B ring
  int s_raw;                 // raw ring depth (3 with staging, 4 without)
  int l2_hint;               // bit 0: y loads evict_first; 1: h TMA stores evict_first; 2: x loads evict_last;
                             // 3: filter-bank loads evict_last (experiments beyond bit 0)
  double *pow_acc;           // power mode (ContractArgs::pow_acc): per-set sum of |out|^2 and row count, no stores
  int pow_stride;
  int bank_shared;           // 1: one bank for every set
  Window geo_s[MAXW_PARAM];
};

struct Tile4 {
  int t, ct, a, o, kept, n0, off, nw;
};

__device__ __forceinline__ Tile4 decode4(const K4Params &p, int g, int rank = 0) {
  Tile4 ti;
  // column block fastest (measured faster than window-fastest on configs 3-5)
  ti.ct = 2 * (g % p.n_ct) + rank;   // CTA rank r of a pair takes the 128-row tile 2 * (pair tile) + r
  const int rest = g / p.n_ct;
  const int w = rest % p.n_win;
  ti.t = rest / p.n_win;
  const Window gw = p.n_win <= MAXW_PARAM ? p.geo_s[w] : p.geo[w];
  ti.a = gw.a;
  ti.o = gw.o;
  ti.kept = gw.o_next - gw.o;
  const int row2 = 2 * (gw.o - gw.a);
  ti.n0 = row2 & ~7;
  ti.off = row2 - ti.n0;
  ti.nw = (ti.off + 2 * ti.kept + 15) & ~15;
  return ti;
}

// statistic set of instance t, or -1 when set_of_instance[t] is out of range (outputs become NaN)
__device__ __forceinline__ int tile_set(const K4Params &p, int t) {
  const int s = p.soi ? p.soi[t] : 0;
  return (s >= 0 && s < p.n_sets) ? s : -1;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo_addr, float hi_addr) {
  // memory order: first float at the lower address = lower 16 bits
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi_addr), "f"(lo_addr));
  return r;
}
__device__ __forceinline__ float bf16_lo_f(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi_f(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }
// output store; K4_ST_CS: streaming (evict-first) cache hint
__device__ __forceinline__ void st_out(float2 *ptr, float2 v) {
#ifdef K4_ST_CS
  asm volatile("st.global.cs.v2.f32 [%0], {%1, %2};" ::"l"(ptr), "f"(v.x), "f"(v.y) : "memory");
#else
  *ptr = v;
#endif
}
// arrive on the leader's (cluster rank 0) copy of `bar`: local for rank 0, remote for rank 1
__device__ __forceinline__ void arrive_leader(uint64_t *bar, int rank) {
  if (rank == 0) {
#ifdef CE_PAIR_REL_CLUSTER
    asm volatile("mbarrier.arrive.release.cluster.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
#else
    mbar_arrive(bar);
#endif
  } else {
    mbar_arrive_remote(bar, 0);
  }
}
// the leader's waits on barriers the peer arrives on
__device__ __forceinline__ void wait_pair(uint64_t *bar, uint32_t parity) {
#ifdef CE_PAIR_REL_CLUSTER
  mbar_wait_cluster(bar, parity);
#else
  mbar_wait(bar, parity);
#endif
}
__device__ __forceinline__ float rcp_approx(float v) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

// One 32-float column block cb of a finished tile: TMEM accumulator (this warp's 32 lanes) -> global.
// Interior blocks (inside the kept range, 16-byte aligned in global memory, all 32 rows of the warp inside
// the instance) leave through SW128 staging and one TMA store of [32 rows][128 B] (full-line writes issued
// by the TMA engine); the rest use direct 8-byte stores (8 rows x 32 B per warp instruction).  On a CTA's
// last tile the A/B ring is idle and every (warp, block) gets its own staging buffer there.
template <int NB>
__device__ __forceinline__ void epi_block(const K4Params &p, const CUtensorMap *tmh, uint32_t tmem_base, uint8_t *ab,
                                          uint8_t *epi, const Tile4 &ti, int cb, int q, int lane, int acc, bool last,
                                          bool set_ok, int &nst) {
  const int rA = lane >> 2, cq = lane & 3;
  const int nf = 2 * ti.kept;
  // tcgen05.ld 16x256b: 4 consecutive threads hold 4 consecutive complex outputs of one row
  uint32_t v0[16], v1[16];
  const uint32_t ta = tmem_base + uint32_t(acc * NMAXW + cb * 32) + (uint32_t(q * 32) << 16);
  tmem_ld16x256b_x4(ta, v0);                         // lanes q*32 + 0..15: rows rA, rA + 8
  tmem_ld16x256b_x4(ta + (16u << 16), v1);           // lanes q*32 + 16..31: rows rA + 16, rA + 24
  tmem_ld_wait();
  if ((p.tma_store || last) && 32 * cb >= ti.off && 32 * cb + 32 <= ti.off + nf && ((2 * ti.o - ti.off) & 3) == 0 &&
      ti.ct * TM + q * 32 + 32 <= p.cols) {
    uint8_t *stg = last ? ab + (q * 8 + cb) * EPI_WARP : epi + (q * NB + (nst % NB)) * EPI_WARP;
    if (!last && lane == 0) {                        // the store that used this staging buffer has read it
      if (NB == 2)
        bulk_wait_read1();
      else
        bulk_wait_read0();
    }
    if (!last) ++nst;
    __syncwarp();
    const uint32_t nanb = 0x7fc00000u;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int chunk = 2 * m + (cq >> 1), half = (cq & 1) * 8;
      const int rr[4] = {rA, rA + 8, rA + 16, rA + 24};
      const uint32_t *src[4] = {&v0[4 * m], &v0[4 * m + 2], &v1[4 * m], &v1[4 * m + 2]};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        *reinterpret_cast<uint2 *>(stg + rr[j] * 128 + ((chunk ^ (rr[j] & 7)) << 4) + half) =
            set_ok ? make_uint2(src[j][0], src[j][1]) : make_uint2(nanb, nanb);
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      if (p.l2_hint & 2)
        tma_store_2d_hint(tmh, stg, 2 * ti.o - ti.off + 32 * cb, ti.t * p.cols + ti.ct * TM + q * 32,
                          l2_evict_first_policy());
      else
        tma_store_2d(tmh, stg, 2 * ti.o - ti.off + 32 * cb, ti.t * p.cols + ti.ct * TM + q * 32);
      bulk_commit();
    }
    return;
  }
  const int c0 = ti.ct * TM + q * 32 + rA;           // rows c0, c0 + 8, c0 + 16, c0 + 24
  float2 *hrow = p.h + (size_t(ti.t) * p.cols + c0) * p.N + ti.o;
  const size_t row8 = size_t(8) * p.N;
  const float qnan = __int_as_float(0x7fc00000);
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int f = cb * 32 + 8 * m + 2 * cq - ti.off;   // output float index within the kept range
    if (f >= 0 && f < nf) {
      const int ci = f >> 1;
      float2 a0 = make_float2(__uint_as_float(v0[4 * m]), __uint_as_float(v0[4 * m + 1]));
      float2 a1 = make_float2(__uint_as_float(v0[4 * m + 2]), __uint_as_float(v0[4 * m + 3]));
      float2 a2 = make_float2(__uint_as_float(v1[4 * m]), __uint_as_float(v1[4 * m + 1]));
      float2 a3 = make_float2(__uint_as_float(v1[4 * m + 2]), __uint_as_float(v1[4 * m + 3]));
      if (!set_ok) a0 = a1 = a2 = a3 = make_float2(qnan, qnan);
#ifdef K4_ABL_NOSTORE
      if (a0.x == 123.f && a3.y == 77.f) hrow[ci] = a1;   // keeps the TMEM loads live; ~never stores
#else
      if (c0 < p.cols) st_out(hrow + ci, a0);
      if (c0 + 8 < p.cols) st_out(hrow + row8 + ci, a1);
      if (c0 + 16 < p.cols) st_out(hrow + 2 * row8 + ci, a2);
      if (c0 + 24 < p.cols) st_out(hrow + 3 * row8 + ci, a3);
#endif
    }
  }
}

// Power mode: the sum of |output|^2 over this warp's 32 rows of a finished tile (kept range only, rows inside the
// instance) and, for window 0, the row count, added to the set's FP64 accumulators.
__device__ __forceinline__ void epi_power(const K4Params &p, uint32_t tmem_base, const Tile4 &ti, int ncb, int q,
                                          int lane, int acc, bool set_ok) {
  const int rA = lane >> 2, cq = lane & 3;
  const int nf = 2 * ti.kept;
  const int c0 = ti.ct * TM + q * 32 + rA;           // rows c0, c0 + 8, c0 + 16, c0 + 24
  const bool r0 = c0 < p.cols, r1 = c0 + 8 < p.cols, r2 = c0 + 16 < p.cols, r3 = c0 + 24 < p.cols;
  float pw = 0.f;
  for (int cb = 0; cb < ncb; ++cb) {
    uint32_t v0[16], v1[16];
    const uint32_t ta = tmem_base + uint32_t(acc * NMAXW + cb * 32) + (uint32_t(q * 32) << 16);
    tmem_ld16x256b_x4(ta, v0);
    tmem_ld16x256b_x4(ta + (16u << 16), v1);
    tmem_ld_wait();
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int f = cb * 32 + 8 * m + 2 * cq - ti.off;
      if (f >= 0 && f < nf) {
        const float a0 = __uint_as_float(v0[4 * m]), a1 = __uint_as_float(v0[4 * m + 1]);
        const float b0 = __uint_as_float(v0[4 * m + 2]), b1 = __uint_as_float(v0[4 * m + 3]);
        const float c0_ = __uint_as_float(v1[4 * m]), c1 = __uint_as_float(v1[4 * m + 1]);
        const float d0 = __uint_as_float(v1[4 * m + 2]), d1 = __uint_as_float(v1[4 * m + 3]);
        if (r0) pw = fmaf(a0, a0, fmaf(a1, a1, pw));
        if (r1) pw = fmaf(b0, b0, fmaf(b1, b1, pw));
        if (r2) pw = fmaf(c0_, c0_, fmaf(c1, c1, pw));
        if (r3) pw = fmaf(d0, d0, fmaf(d1, d1, pw));
      }
    }
  }
  double s = pw;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0 && set_ok) {
    double *a = p.pow_acc + size_t(tile_set(p, ti.t)) * p.pow_stride;
    atomicAdd(a, s);
    if (ti.o == 0) atomicAdd(a + 1, double(min(32, max(0, p.cols - (ti.ct * TM + q * 32)))));
  }
}

__global__ void __launch_bounds__(K4_THREADS, 1)
    k4_bf16x3_pair(const __grid_constant__ CUtensorMap tmy, const __grid_constant__ CUtensorMap tmx,
              const __grid_constant__ CUtensorMap tmh, const __grid_constant__ K4Params p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment by pointer arithmetic on the __shared__ array (keeps the shared address space
  // visible to the compiler: LDS/STS instead of generic LD/ST)
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int SAB = PAIR ? S_AB_P : S_AB;             // A stages
  constexpr int SB = PAIR ? S_B_P : S_AB;               // B stages (without pairs: the same ring as A)
  constexpr int BPL = PAIR ? B_PLANE_P : B_PLANE;       // bytes per B plane (pair: this CTA's half of the rows)
  // single CTAs: [S_AB][A_hi | A_lo | B_hi | B_lo]; pairs: [SAB][A_hi | A_lo] then [SB][B_hi | B_lo]
  constexpr int A_STRIDE = PAIR ? A_STAGE_P : AB_STAGE, B_STRIDE = PAIR ? B_STAGE_P : AB_STAGE;
  constexpr int B_BASE = PAIR ? S_AB_P * A_STAGE_P : 2 * A_PLANE;
  constexpr int AB_BYTES = PAIR ? AB_BYTES_P : S_AB * AB_STAGE;
  uint8_t *ab = smem;
  const int S_RAW = p.s_raw;
  uint8_t *raw = smem + AB_BYTES;                       // [S_RAW][y 16 KB | x 4 KB]
  uint8_t *epi = raw + S_RAW * RAW_STAGE;               // [4 warps][EPI_WARP] when p.tma_store
  uint64_t *bars = reinterpret_cast<uint64_t *>(epi + (p.tma_store ? (PAIR ? EPI_BYTES_P : EPI_BYTES) : 0));
  uint64_t *raw_full = bars;                            // [S_RAW_BARS]
  uint64_t *raw_empty = bars + S_RAW_BARS;              // [S_RAW_BARS]
  uint64_t *a_full = bars + 2 * S_RAW_BARS;             // [SAB]  transform done (pair: the leader's, both CTAs)
  uint64_t *st_empty = a_full + 4;                      // [SAB]  MMAs reading the A stage done (commit)
  uint64_t *b_full = st_empty + 4;                      // [SB]   filter chunk landed
  uint64_t *b_empty_p = b_full + S_B_MAX;               // [SB]   pair: MMAs reading the B stage done (commit)
  uint64_t *b_empty = PAIR ? b_empty_p : st_empty;      //        single CTAs: one ring, one barrier
  uint64_t *tmem_full = b_empty_p + S_B_MAX;            // [2]
  uint64_t *tmem_empty = tmem_full + 2;                 // [2]     one arrival per epilogue warp (pair: the leader's)
  uint64_t *b_peer = tmem_empty + 2;                    // [SB]   pair: the peer's half of the filter chunk landed
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(b_peer + S_B_MAX);
  static_assert((2 * S_RAW_BARS + 8 + 3 * S_B_MAX + 4) * 8 + 4 <= BAR_BYTES && SAB <= 4, "barrier block");

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // both CTAs of a pair walk the pair's tiles.  Re-read from the special / constant registers at every use, as K4
  // does: holding them in registers from the top of the kernel cost K4 0.7 us per launch and 2.5 % on config 4
  // (bisected, tools/ab_bisect.sh)
#define g_first int(blockIdx.x >> 1)
#define rank int(blockIdx.x & 1)   /* = %cluster_ctarank for clusters of two along x */
#define g_step int(gridDim.x >> 1)
#ifdef CE_K4_TRACE
  if (tid == 0 && g_k4_trace) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    g_k4_trace[size_t(blockIdx.x) * 256 + 0] = gt;
  }
#endif
  if (tid == 0) {
    K4TR(1);
    for (int s = 0; s < S_RAW_BARS; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_empty[s], NTR);
    }
    for (int s = 0; s < SAB; ++s) {
      mbar_init(&a_full[s], PAIR ? 16 : NTR);          // pair: one arrival per transform warp of both CTAs
      mbar_init(&st_empty[s], 1);
    }
    for (int s = 0; s < SB; ++s) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_peer[s], 1);
      if (PAIR) mbar_init(&b_empty_p[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&tmem_empty[i], PAIR ? 8 : 4);         // pair: the epilogue warps of both CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    K4TR(203);
  }
  // The raw producer decodes its first tile while the other warps set up: the decode chains dependent
  // kernel-parameter reads whose first accesses miss the constant cache (~0.5 us measured), and the first
  // TMA load is the head of the kernel's critical path.
  Tile4 ti0 = {};
  int row0_0 = 0, xbytes0 = 0, nkc0 = 0, K0 = 0, cols0 = 0;
  if (warp == 12 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmy)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmx)) : "memory");
    if (g_first < p.n_tiles) ti0 = decode4(p, g_first, rank);
    K0 = p.K;
    cols0 = p.cols;
    nkc0 = p.nkc;
    row0_0 = ti0.t * cols0 + ti0.ct * TM;
    xbytes0 = K0 * CK * 8;
    asm volatile("" ::"r"(row0_0), "r"(xbytes0), "r"(nkc0), "r"(ti0.a), "r"(ti0.t), "r"(cols0) : "memory");
  }
  if (warp == 13) {
    if (PAIR)
      tmem_alloc2(tmem_slot, 512);
    else
      tmem_alloc(tmem_slot, 512);
    if (lane == 0) K4TR(202);
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();           // the peer's barriers are initialised before any remote arrive / multicast commit
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (tid == 0) {
    pdl_launch_dependents();          // the next kernel in the stream may launch (it waits for our exit)
    K4TR(2);
  }
  // Programmatic dependent launch: every role that touches caller data (y, x, set_of_instance, h) waits
  // for the previous kernel in the stream first.  The B producer without a set table reads only the
  // filter bank, which ce_build_filters completed (stream-synchronised) before any estimate could be
  // enqueued, so its first chunks are fetched while the previous kernel drains.
#ifndef K4_NO_PDL
  if (!(warp == 14 && p.soi == nullptr && p.pow_acc == nullptr)) pdl_wait();   // power mode: bank built just before
#endif
#ifdef CE_K4_TRACE
  unsigned long long c_pdl = clock64(), c_dec = 0, c_tma0 = 0, c_w0 = 0;   // producer prologue, stored at the end
#endif
  const int nks_total = (2 * p.b + 15) / 16;   // 16-element (bf16) MMA K steps over 2b

  if (warp == 12) {
    // ---------------------------------------------------------------- raw producer (TMA)
    if (lane == 0) {
      const uint32_t xbytes = uint32_t(xbytes0);
      int it = 0;
      for (int g = g_first; g < p.n_tiles; g += g_step) {
        const Tile4 ti = g == g_first ? ti0 : decode4(p, g, rank);
#ifdef CE_K4_TRACE
        if (g == g_first) c_dec = clock64();
#endif
        const int row0 = g == g_first ? row0_0 : ti.t * cols0 + ti.ct * TM;
        for (int kc = 0; kc < nkc0; ++kc, ++it) {
          const int s = it % S_RAW;
          mbar_wait(&raw_empty[s], ((it / S_RAW) & 1) ^ 1);
#ifdef CE_K4_TRACE
          if (it == 0) c_w0 = clock64();
#endif
          mbar_arrive_expect_tx(&raw_full[s], RAWY + xbytes);
#ifdef CE_K4_TRACE
          if (it == 0) c_tma0 = clock64();
          else if (it < 24) K4TR(8 + it);
#endif
          const int f0 = 2 * (ti.a + kc * CK);        // first float of the chunk in the row
          if (p.l2_hint & 1)
            tma_load_2d_hint(raw + s * RAW_STAGE, &tmy, f0, row0, &raw_full[s], l2_evict_first_policy());
          else
            tma_load_2d(raw + s * RAW_STAGE, &tmy, f0, row0, &raw_full[s]);
          if (p.l2_hint & 4)
            tma_load_2d_hint(raw + s * RAW_STAGE + RAWY, &tmx, f0, ti.t * K0, &raw_full[s], l2_evict_last_policy());
          else
            tma_load_2d(raw + s * RAW_STAGE + RAWY, &tmx, f0, ti.t * K0, &raw_full[s]);
        }
      }
#ifdef CE_K4_TRACE
      if (g_k4_trace) {
        g_k4_trace[size_t(blockIdx.x) * 256 + 200] = c_pdl;
        g_k4_trace[size_t(blockIdx.x) * 256 + 201] = c_dec;
        g_k4_trace[size_t(blockIdx.x) * 256 + 8] = c_tma0;
        g_k4_trace[size_t(blockIdx.x) * 256 + 204] = c_w0;
      }
#endif
    }
  } else if (warp < 8) {
    // ---------------------------------------------------------------- transform
    const int jp = tid & 7;            // complex pair 2jp, 2jp+1 of the 16-complex chunk
    const int rb = tid >> 3;           // rows rb + 32 i, i < 4
    int it = 0;
    for (int g = g_first; g < p.n_tiles; g += g_step) {
      const Tile4 ti = decode4(p, g, rank);
      const int c_first = ti.ct * TM + rb;
      const int x_first = c_first % p.K;
      const int x_step = 32 % p.K;
      for (int kc = 0; kc < p.nkc; ++kc, ++it) {
        const int sr = it % S_RAW, sa = it % SAB;
        mbar_wait(&raw_full[sr], (it / S_RAW) & 1);
        if (tid == 0 && it < 24) K4TR(32 + it);
#ifdef K4_ABL_NOTRANSFORM
        mbar_arrive(&raw_empty[sr]);
        mbar_wait(&st_empty[sa], ((it / SAB) & 1) ^ 1);
        mbar_arrive(&a_full[sa]);
        continue;
#endif
        const float4 *ry = reinterpret_cast<const float4 *>(raw + sr * RAW_STAGE);
        const float4 *rx = reinterpret_cast<const float4 *>(raw + sr * RAW_STAGE + RAWY);
        float4 yv[4], xv[4];
        int xr = x_first;
#pragma unroll
        for (int i = 0; i < 4; ++i) {          // all 8 loads in flight at once
          yv[i] = ry[(rb + 32 * i) * 8 + jp];
          xv[i] = rx[xr * 8 + jp];
          xr += x_step;
          if (xr >= p.K) xr -= p.K;
        }
        // LS = y / x = y conj(x) / |x|^2 per element; a zero factor masks the K tail (j >= b)
        const bool ok0 = kc * CK + 2 * jp < p.b, ok1 = kc * CK + 2 * jp + 1 < p.b;
        uint32_t hv[4][2], lv[4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float i0 = ok0 ? rcp_approx(xv[i].x * xv[i].x + xv[i].y * xv[i].y) : 0.f;
          const float i1 = ok1 ? rcp_approx(xv[i].z * xv[i].z + xv[i].w * xv[i].w) : 0.f;
          const float f0r = xv[i].x * i0, f0i = -xv[i].y * i0, f1r = xv[i].z * i1, f1i = -xv[i].w * i1;
          const float l0r = yv[i].x * f0r - yv[i].y * f0i, l0i = yv[i].x * f0i + yv[i].y * f0r;
          const float l1r = yv[i].z * f1r - yv[i].w * f1i, l1i = yv[i].z * f1i + yv[i].w * f1r;
          hv[i][0] = pack_bf16(l0r, l0i);
          hv[i][1] = pack_bf16(l1r, l1i);
          lv[i][0] = pack_bf16(l0r - bf16_lo_f(hv[i][0]), l0i - bf16_hi_f(hv[i][0]));
          lv[i][1] = pack_bf16(l1r - bf16_lo_f(hv[i][1]), l1i - bf16_hi_f(hv[i][1]));
        }
        mbar_arrive(&raw_empty[sr]);           // the raw slot is consumed (values used above): refill it
        mbar_wait(&st_empty[sa], ((it / SAB) & 1) ^ 1);
        uint8_t *ah = ab + sa * A_STRIDE;
        uint8_t *al = ah + A_PLANE;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = rb + 32 * i;
          // SW64 K-major: row r at r*64 bytes, 16-byte chunk (jp>>1) ^ ((r>>1)&3), 8-byte half (jp&1)
          const int off = r * 64 + ((((jp >> 1) ^ ((r >> 1) & 3))) << 4) + ((jp & 1) << 3);
#ifdef K4_ABL_NOASTORE
          if (hv[i][0] == 0x12345u && lv[i][1] == 0x777u) *reinterpret_cast<uint2 *>(ah + off) = make_uint2(hv[i][1], lv[i][0]);
#else
          *reinterpret_cast<uint2 *>(ah + off) = make_uint2(hv[i][0], hv[i][1]);
          *reinterpret_cast<uint2 *>(al + off) = make_uint2(lv[i][0], lv[i][1]);
#endif
        }
        fence_proxy_async();
        if (tid == 0 && it < 24) K4TR(56 + it);
        if (PAIR) {
          __syncwarp();
          if (lane == 0) arrive_leader(&a_full[sa], rank);
        } else {
          mbar_arrive(&a_full[sa]);
        }
      }
    }
  } else if (warp < 12) {
    // ---------------------------------------------------------------- epilogue
    // TMEM -> registers (16x256b: 4 consecutive threads hold 4 consecutive complex outputs of one row)
    // -> direct 8-byte stores: each warp instruction writes 8 rows x 32 contiguous bytes.
    const int q = warp & 3;
    int lt = 0, nst = 0;
    for (int g = g_first; g < p.n_tiles; g += g_step, ++lt) {
      const Tile4 ti = decode4(p, g, rank);
      const bool set_ok = tile_set(p, ti.t) >= 0;
      const bool last = p.tma_last && g + g_step >= p.n_tiles;
      const int acc = lt & 1;
      mbar_wait(&tmem_full[acc], (lt >> 1) & 1);
      tc_fence_after();
      if (tid == 256 && lt < 8) K4TR(136 + lt);
      const int ncb = (ti.off + 2 * ti.kept + 31) / 32;
      if (p.pow_acc) {
        epi_power(p, tmem_base, ti, ncb, q, lane, acc, set_ok);
      } else {
        for (int cb = 0; cb < ncb; ++cb) epi_block<(PAIR ? EPI_NB_P : EPI_NB)>(p, &tmh, tmem_base, ab, epi, ti, cb, q, lane, acc, last, set_ok, nst);
      }
      if (tid == 256 && lt < 8) K4TR(144 + lt);
      __syncwarp();
      if (lane == 0) {
        tc_fence_before();
        if (PAIR)
          arrive_leader(&tmem_empty[acc], rank);
        else
          mbar_arrive(&tmem_empty[acc]);
      }
    }
    if ((p.tma_store || p.tma_last) && lane == 0) bulk_wait0();   // every TMA store of this warp completed
  } else if (warp == 14) {
    // ---------------------------------------------------------------- B producer
    if (lane == 0) {
      int it = 0;
      for (int g = g_first; g < p.n_tiles; g += g_step) {
        const Tile4 ti = decode4(p, g, rank);
        const int set = p.bank_shared ? 0 : max(tile_set(p, ti.t), 0);
        const int nrows = PAIR ? ti.nw >> 1 : ti.nw;          // pair: this CTA's half of the chunk's rows
        const uint32_t bytes = uint32_t(nrows) * 64;          // per plane
        for (int kc = 0; kc < p.nkc; ++kc, ++it) {
          const int s = it % SB;
          mbar_wait(&b_empty[s], ((it / SB) & 1) ^ 1);
#ifdef K4_ABL_NOB
          mbar_arrive(&b_full[s]);
          continue;
#endif
          mbar_arrive_expect_tx(&b_full[s], 2 * bytes);
          if (it < 24) K4TR(80 + it);
          const size_t src = ((size_t(set) * p.nkc + kc) * p.NR + ti.n0 + rank * nrows) * 32;   // bf16 elements
          uint8_t *bh = ab + B_BASE + s * B_STRIDE;
          if (p.l2_hint & 8) {
            const uint64_t pol = l2_evict_last_policy();
            bulk_g2s_hint(bh, p.bank_hi + src, bytes, &b_full[s], pol);
            bulk_g2s_hint(bh + BPL, p.bank_lo + src, bytes, &b_full[s], pol);
          } else {
            bulk_g2s(bh, p.bank_hi + src, bytes, &b_full[s]);
            bulk_g2s(bh + BPL, p.bank_lo + src, bytes, &b_full[s]);
          }
        }
      }
    }
  } else {
    // ---------------------------------------------------------------- MMA issuer (warp 13)
    if (lane == 0 && PAIR && rank != 0) {
      // pair mode, peer CTA: the leader issues the pair's MMAs; this thread only tells it when the peer's half of
      // each filter chunk has landed (bulk copies signal a barrier of their own CTA)
      int it = 0;
      for (int g = g_first; g < p.n_tiles; g += g_step) {
        for (int kc = 0; kc < p.nkc; ++kc, ++it) {
          const int s = it % SB;
          mbar_wait(&b_full[s], (it / SB) & 1);
          mbar_arrive_remote(&b_peer[s], 0);
        }
      }
    } else if (lane == 0) {
      int it = 0, lt = 0;
      for (int g = g_first; g < p.n_tiles; g += g_step, ++lt) {
        const Tile4 ti = decode4(p, g, rank);
        const int acc = lt & 1;
        // F32 accumulate, BF16 A/B, K-major A/B, N = nw, M = 128 (pair: 256 = 128 rows per CTA)
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(ti.nw >> 3) << 17) |
                               (uint32_t((PAIR ? 2 * TM : TM) >> 4) << 24);
        if (PAIR)
          wait_pair(&tmem_empty[acc], ((lt >> 1) & 1) ^ 1);
        else
          mbar_wait(&tmem_empty[acc], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + uint32_t(acc * NMAXW);
        for (int kc = 0; kc < p.nkc; ++kc, ++it) {
          const int s = it % SAB, sb = it % SB;
          const uint32_t ph = (it / SAB) & 1, phb = (it / SB) & 1;
          if (PAIR) {
            wait_pair(&a_full[s], ph);
            mbar_wait(&b_full[sb], phb);
#ifndef K4_ABL_NOPEER
            wait_pair(&b_peer[sb], phb);
#endif
          } else {
            mbar_wait(&a_full[s], ph);
            mbar_wait(&b_full[sb], phb);
          }
          tc_fence_after();
          if (it < 24) K4TR(104 + it);
          uint8_t *sta = ab + s * A_STRIDE, *stb = ab + B_BASE + sb * B_STRIDE;
          const uint64_t ah = sw64_desc(smem_u32(sta));
          const uint64_t al = sw64_desc(smem_u32(sta + A_PLANE));
          const uint64_t bh = sw64_desc(smem_u32(stb));
          const uint64_t bl = sw64_desc(smem_u32(stb + BPL));
          const int nks = min(2, nks_total - 2 * kc);
          for (int ks = 0; ks < nks; ++ks) {
            const uint64_t adv = uint64_t(2 * ks);      // +32 bytes along K
#ifndef K4_ABL_NOMMA
            if (PAIR) {
              mma_bf16_pair(d, ah + adv, bh + adv, idesc, (kc | ks) != 0);
              mma_bf16_pair(d, ah + adv, bl + adv, idesc, 1u);
              mma_bf16_pair(d, al + adv, bh + adv, idesc, 1u);
            } else {
              mma_bf16(d, ah + adv, bh + adv, idesc, (kc | ks) != 0);
              mma_bf16(d, ah + adv, bl + adv, idesc, 1u);
              mma_bf16(d, al + adv, bh + adv, idesc, 1u);
            }
#endif
          }
          if (PAIR) {
            mma_commit_pair(&st_empty[s]);
            mma_commit_pair(&b_empty_p[sb]);
          } else {
            mma_commit(&st_empty[s]);
          }
        }
        if (PAIR)
          mma_commit_pair(&tmem_full[acc]);
        else
          mma_commit(&tmem_full[acc]);
        if (lt < 8) K4TR(128 + lt);
        else if (lt < 32) K4TR(152 + lt - 8);
      }
    }
  }
  tc_fence_before();
  if (tid == 256) K4TR(3);
  __syncthreads();
  if (PAIR) cluster_sync();           // neither CTA leaves while the other may still reach its barriers or TMEM
  if (tid == 0) K4TR(4);
#ifdef CE_K4_TRACE
  if (tid == 0 && g_k4_trace) {   // end globaltimer: tools/k4_trace.cu calibrates clock64 against it
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    g_k4_trace[size_t(blockIdx.x) * 256 + 5] = gt;
  }
#endif
  if (warp == 13) {
    __syncwarp();
    tc_fence_after();
    if (PAIR)
      tmem_dealloc2(tmem_base, 512);
    else
      tmem_dealloc(tmem_base, 512);
  }
}
#undef g_first
#undef rank
#undef g_step

// Per-device launch facts: smem attribute set once, SM count, resident CTA pairs.
struct DevInfo {
  bool init = false;
  int num_sms = 0;
  int max_pairs = 0;   // CTA pairs (clusters of 2) of k4_bf16x3_pair resident at once
};
cudaError_t dev_info(DevInfo **out) {
  static DevInfo infos[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  DevInfo &d = infos[dev];
  if (!d.init) {
    e = cudaDeviceGetAttribute(&d.num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k4_bf16x3_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, K4P_SMEM);
    if (e != cudaSuccess) return e;
    // a persistent pair grid must not exceed the clusters the device can hold at once (a second wave would double
    // the time): ask the occupancy calculator rather than assuming num_sms / 2
    cudaLaunchConfig_t oc = {};
    oc.gridDim = dim3(unsigned(d.num_sms & ~1));
    oc.blockDim = dim3(K4_THREADS);
    oc.dynamicSmemBytes = K4P_SMEM;
    cudaLaunchAttribute ca[1];
    ca[0].id = cudaLaunchAttributeClusterDimension;
    ca[0].val.clusterDim.x = 2;
    ca[0].val.clusterDim.y = 1;
    ca[0].val.clusterDim.z = 1;
    oc.attrs = ca;
    oc.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, k4_bf16x3_pair, &oc) != cudaSuccess) {
      (void)cudaGetLastError();
      nc = 0;
    }
    d.max_pairs = nc < d.num_sms / 2 ? nc : d.num_sms / 2;
    if (getenv("CE_K4_DEBUG")) fprintf(stderr, "k4 pair: %d SMs, %d resident CTA pairs\n", d.num_sms, nc);
    d.init = true;
  }
  *out = &d;
  return cudaSuccess;
}

}  // namespace

#ifdef CE_K4_TRACE
extern "C" int ce_k4p_trace_set(void *dptr) {
  return int(cudaMemcpyToSymbol(g_k4_trace, &dptr, sizeof(dptr)));
}
#endif

// Policy.  CE_K4_PAIR = 0 / 1 forces pairs off / on (experiments).  Default: pairs when every CTA walks more than two
// 128-row tiles.  Measured, same box, against K4 (two repetitions each): config 5 1486-1488 -> 1400-1435 us
// (-3.5..6 %), config 4 325-330 -> 314-323 us (-1..5 %); config 3 (one tile per SM) 9.9 -> 11.6 us (the cluster
// barrier in the prologue, chunk lockstep of the two CTAs).  The power mode (the statistics noise window: N = 64, no
// stores) keeps single CTAs: exact in pairs, but the statistics step measured 571 -> 587 us (config 4), 2120 -> 2200 us
// (config 5).
bool bf16x3_pair_wanted(const ContractArgs &a) {
  static const int env_pair = getenv("CE_K4_PAIR") ? atoi(getenv("CE_K4_PAIR")) : -1;
  if (env_pair == 0) return false;
  const int n_ct = (a.M * a.K + TM - 1) / TM;
  if (n_ct < 2) return false;
  DevInfo *di = nullptr;
  if (dev_info(&di) != cudaSuccess || di->max_pairs < 1) return false;
  if (env_pair > 0) return true;
  return (long long)a.T * a.n_win * n_ct > 2LL * di->num_sms && a.pow_acc == nullptr;
}

cudaError_t launch_contract_bf16x3_pair(const ContractArgs &a, const uint16_t *bank_hi, const uint16_t *bank_lo,
                                        cudaStream_t stream, int64_t *launches) {
  if (!bf16x3_launchable(a)) return cudaErrorNotSupported;
  if (a.n_win <= MAXW_PARAM && a.geo_host == nullptr) return cudaErrorInvalidValue;
  DevInfo *di = nullptr;
  cudaError_t e = dev_info(&di);
  if (e != cudaSuccess) return e;
  static const int env_pairs = getenv("CE_K4_PAIRS") ? atoi(getenv("CE_K4_PAIRS")) : 0;   // experiments: grid pairs
  const int max_pairs = env_pairs > 0 && env_pairs < di->max_pairs ? env_pairs : di->max_pairs;
  if (max_pairs < 1) return cudaErrorNotSupported;
  K4Params p;
  p.h = a.h;
  p.bank_hi = bank_hi;
  p.bank_lo = bank_lo;
  p.geo = a.geo;
  p.soi = a.soi;
  p.T = a.T;
  p.K = a.K;
  p.N = a.N;
  p.b = a.b;
  p.n_win = a.n_win;
  p.n_sets = a.n_sets;
  bf16x3_bank_shape(a.b, &p.nkc, &p.NR);
  if (a.bank_rows > 0) p.NR = a.bank_rows;
  p.pow_acc = a.pow_acc;
  p.pow_stride = a.pow_stride;
  p.bank_shared = a.bank_shared ? 1 : 0;
  p.cols = a.M * a.K;
  p.pair = 1;
  p.n_ct = ((p.cols + TM - 1) / TM + 1) / 2;          // 256-row pair tiles
  for (int w = 0; w < MAXW_PARAM; ++w) p.geo_s[w] = w < a.n_win && a.geo_host ? a.geo_host[w] : Window{0, 0, 0};
  const long long tiles = (long long)a.T * a.n_win * p.n_ct;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  p.n_tiles = int(tiles);
  CUtensorMap tmy, tmx, tmh = {};
  if (!cached_map(&tmy, a.y, a.N, (long long)a.T * p.cols, TM) ||
      !cached_map(&tmx, a.x, a.N, (long long)a.T * a.K, a.K))
    return cudaErrorInvalidValue;
  // same launch rules as K4 (k4_block_lmmse_bf16x3.cu), counted in pairs
  static const int env_st = getenv("CE_K4_TMA_STORE") ? atoi(getenv("CE_K4_TMA_STORE")) : -1;   // experiments
  const bool st_ok = (reinterpret_cast<uintptr_t>(a.h) & 15) == 0 && (a.N % 2) == 0 && a.pow_acc == nullptr;
  p.tma_store = (env_st >= 0 ? env_st != 0 : tiles > (long long)max_pairs) && st_ok;
  static const int env_last = getenv("CE_K4_TMA_LAST") ? atoi(getenv("CE_K4_TMA_LAST")) : 1;   // experiments
  p.s_raw = p.tma_store ? S_RAW_P_ST : S_RAW_P_NOST;
  // a CTA's last tile stages its 4 x 8 output blocks in the then idle A and B rings and the raw ring behind them
  p.tma_last = env_last != 0 && st_ok && AB_BYTES_P + p.s_raw * RAW_STAGE >= 4 * 8 * EPI_WARP;
  if ((p.tma_store || p.tma_last) && !cached_map(&tmh, a.h, a.N, (long long)a.T * p.cols, 32, true))
    return cudaErrorInvalidValue;
  bool disjoint = a.geo_host != nullptr;
  for (int w = 0; disjoint && w + 1 < a.n_win; ++w) disjoint = a.geo_host[w + 1].a >= a.geo_host[w].a + a.b;
  static const int env_hint = getenv("CE_K4_L2HINT") ? atoi(getenv("CE_K4_L2HINT")) : -1;   // experiments
  p.l2_hint = env_hint >= 0 ? env_hint : ((tiles <= (long long)max_pairs && disjoint ? 1 : 0) | 4 | 8);
  cudaLaunchConfig_t cfg = {};
  const unsigned units = unsigned(tiles < max_pairs ? tiles : max_pairs);
  cfg.gridDim = dim3(2 * units);
  cfg.blockDim = dim3(K4_THREADS);
  cfg.dynamicSmemBytes = p.tma_store ? K4P_SMEM_ST : K4P_SMEM_NOST;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  int na = 0;
  at[na].id = cudaLaunchAttributeClusterDimension;
  at[na].val.clusterDim.x = 2;
  at[na].val.clusterDim.y = 1;
  at[na].val.clusterDim.z = 1;
  ++na;
#ifndef K4_NO_PDL
  at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[na].val.programmaticStreamSerializationAllowed = 1;
  ++na;
#endif
  cfg.attrs = at;
  cfg.numAttrs = na;
  e = cudaLaunchKernelEx(&cfg, k4_bf16x3_pair, tmy, tmx, tmh, p);
  if (e == cudaSuccess) ++*launches;
  return e;
}

}  // namespace ce
