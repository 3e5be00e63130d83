// K10 -- the paper's comb-pilot 12W-LMMSE (CE_COMB_FULL) on tcgen05: the same operation as K6b
// (Table II: group g outputs the S tones S*g + q from the G pilots [a_g, a_g + G) of its UE
// through W_s^(type), Eq. 17 weights; LS of Eq. 9 at the pilots), as a BF16x3 tensor-core GEMM.
//
// Why: per estimate the 12W is G = 12 complex MACs for 8 B of output -- 12 flop/B, beyond the FP32-SIMT ridge
// (69 TF/s / 6.6 TB/s = 10.5 flop/B), so the SIMT kernel K6b is ALU-bound.  On the tensor cores the same MACs
// cost a few percent of the tensor pipe and the kernel becomes a pure stream of its 8 B/estimate output.
//
// Formulation.  Groups are packed into blocks of ng consecutive groups whose pilot windows all lie inside one
// 16-pilot window [sw, sw + 16) with sw a multiple of 4 (host table, comb_tc_blocks; ng * S <= 64 outputs).
// Per (UE s, block) the block's outputs are one real GEMM
//     D[r][2o + c] = sum_k  L[r][k] * W_s,blk[2o + c][k],   k = 2j' + c'  (pilot sw + j', re / im)
// with L the LS of UE s at the window's pilots for M = 128 data rows r = (t, m) and W the block's weights embedded
// as 2x2 real blocks [[Re, -Im], [Im, Re]] (rows 2o / 2o + 1 of output o = i*S + q of group g0 + i; zero outside the
// group's own G taps).  M = 128 rows, N = 128 (<= 64 outputs), K = 32 (2 MMA K-steps), BF16x3
// (L_hi W_hi + L_hi W_lo + L_lo W_hi, FP32 accumulation in TMEM) as K4 (reading B1).
//
// Kernels:
//   k10_ls          LS = y conj(x) / |x|^2 of every tone of a row, de-interleaved per UE into bf16 hi / lo planes
//                   [n_ue][T*M][KP4] of (re, im) pairs (the strided comb pilots become contiguous K-major rows that
//                   TMA can load with SWIZZLE_64B straight into the MMA's B layout); 8 B per pilot written, kept
//                   in L2 for k10_comb_tc
//   k10_comb_tc     persistent, one CTA per SM over units (UE, block, 128-row tile), rows fastest:
//                     warp 0   : producer -- bulk copy of the (UE, block) weight image (pre-swizzled SW64, hi / lo)
//                                when it changes, 2 TMA loads of the LS tile per unit into a 6-deep ring
//                     warp 1   : TMEM allocator + MMA issuer (6 MMAs per unit, 2 TMEM accumulators of 128 columns)
//                     warps 2-9: epilogue -- tcgen05.ld 32x32b: lane = data row, column = output float, so each
//                                thread holds 128 contiguous bytes of h[t][m][s][.]: SW128 staging (16-byte shared
//                                stores) and 3-D TMA stores
//   k10_build_images (build time) the weight images from K6a's complex64 W.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "ce_internal.h"
#include "tc_ptx.cuh"
#include "tmap.cuh"

namespace ce {
namespace {

constexpr int K10_WIN = 16;                 // pilots per block window: K = 32 bf16 = one 64-byte SW64 row
constexpr int K10_NR = 128;                 // data rows per unit (MMA N)
constexpr int K10_PLANE = 128 * 64;         // [128 rows][32 bf16], SW64: 8 KB
#ifndef K10_SA_SLOTS
#define K10_SA_SLOTS 4       // interleaved units change the weight image almost every unit
#endif
constexpr int K10_SA = K10_SA_SLOTS;        // weight-image slots
#ifndef K10_CPS
#define K10_CPS 1
#endif
#ifndef K10_INTERLEAVE
#define K10_INTERLEAVE 1     // grid-stride units (measured: 74.3 -> 72.4 us with 4 image slots)
#endif
#ifndef K10_SB_STAGES
#define K10_SB_STAGES (K10_CPS == 1 ? 4 : 2)
#endif
constexpr int K10_SB = K10_SB_STAGES;       // LS-tile ring
// TMEM accumulators in flight: the 6 MMAs of a unit accumulate into one D and run back to back (~1.5 us from issue
// to commit), so two accumulators capped the kernel at ~0.8 us per unit with no epilogue at all (ablation); four
// fill the 512 TMEM columns
#ifndef K10_NACC_N
#define K10_NACC_N (K10_CPS == 1 ? 4 : 2)
#endif
constexpr int K10_NACC = K10_NACC_N;
#ifndef K10_ONE_COMMIT
#define K10_ONE_COMMIT 1
#endif
static_assert(!K10_ONE_COMMIT || K10_SB_STAGES == K10_NACC_N, "one commit per unit: LS stage i <-> accumulator i");
#ifndef K10_EPI_W
#define K10_EPI_W 16         // measured: 16 warps 71.3 us, 8 warps 72.4 us (interleaved units, 4 image slots)
#endif
constexpr int K10_EPI = K10_EPI_W;          // epilogue warps: 8 (two per TMEM lane quadrant, two column blocks each) or 16
constexpr int K10_NCBW = 16 / K10_EPI;      // 32-float column blocks per epilogue warp and unit
constexpr int K10_THREADS = 32 * (2 + K10_EPI);
constexpr int K10_STG = 4096;               // TMA-store staging box [32 rows][32 floats]
#ifndef K10_CPS
#define K10_CPS 1
#endif
constexpr int K10_CTAS = K10_CPS;           // CTAs per SM (2: half-size rings, one staging box per epilogue warp)
constexpr int K10_NSTG = (K10_CTAS == 1 && K10_EPI_W == 8) ? 2 : 1;   // staging boxes per epilogue warp
constexpr int K10_MAXBLK = 256;             // block table entries kept in shared memory (else read from global)
constexpr int K10_SMEM = (K10_SA + K10_SB) * 2 * K10_PLANE + K10_EPI * K10_NSTG * K10_STG + 256 + 1024;
static_assert(K10_SMEM <= 232448 - K10_MAXBLK * 16, "K10 shared memory");

struct K10Params {
  float *h;                     // [T*M][n_ue][N] complex64 as floats
  const uint16_t *img_hi;       // [n_ue][n_cls][128][32] bf16, SW64 image (blocks with equal tap patterns share one)
  const uint16_t *img_lo;
  const int4 *blk;              // [n_blk] {g0, ng, sw, image class}
  int R, n_ue, N, S, n_blk, n_cls, n_rt, u_total;
  int tma_st;                   // 1: full 32-float quadrant rows leave through staging + 3-D TMA stores
  int l2_hint;                  // (default 3) bit 0: LS tiles loaded evict_last (each is re-read by ~4 overlapping windows);
                                // bit 1: h TMA stores evict_first (the output stream must not push the LS planes out)
};

// Optional per-CTA event trace (tools/k10_trace.py builds with -DCE_K10_TRACE; the product build has none)
#ifdef CE_K10_TRACE
__device__ unsigned long long *g_k10_trace;
#define K10TR(slot)                                                                       \
  do {                                                                                    \
    const unsigned long long c_ = clock64();                                              \
    if (g_k10_trace) g_k10_trace[size_t(blockIdx.x) * 1024 + (slot)] = c_;                \
  } while (0)
#else
#define K10TR(slot) \
  do {              \
  } while (0)
#endif

struct Unit10 {
  int s, b, rt;
};
// units in (row tile, UE, block) order, blocks fastest: a CTA fills consecutive 480-byte output segments of the same
// 128 rows, so each row's DRAM pages are complete in L2 long before they are written back (rows-fastest order
// scattered every row's segments over the whole kernel and wrote partial pages)
__device__ __forceinline__ Unit10 decode10(const K10Params &p, int u) {
  Unit10 d;
  d.b = u % p.n_blk;
  const int rest = u / p.n_blk;
  d.s = rest % p.n_ue;
  d.rt = rest / p.n_ue;
  return d;
}
// the next unit without a division (the issue loops are single-thread latency chains: measured ~0.4 us of
// instruction overhead per unit with two decodes by division in the MMA issuer)
__device__ __forceinline__ void next10(const K10Params &p, Unit10 &d) {
  if (++d.b == p.n_blk) {
    d.b = 0;
    if (++d.s == p.n_ue) {
      d.s = 0;
      ++d.rt;
    }
  }
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo_addr, float hi_addr) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi_addr), "f"(lo_addr));
  return r;
}
__device__ __forceinline__ float bf16lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }

// k10_ls: LS at every tone (Eq. 9) of K10_LSR consecutive data rows per CTA, scattered into the
// per-UE bf16 hi / lo planes: plane[(s * R + r) * KP4 + p] = (re, im) of LS at tone S*p + s (pilots KP .. KP4-1
// zero).  Phase 1 streams the rows as float4 (two tones) with K10_LSJ independent loads per thread in flight and
// scatters LS into shared memory as [row][UE][pilot] (odd pilot pitch: consecutive tones land on distinct banks);
// the (row, tone) and (pilot, UE) coordinates advance by additions only.  Phase 2 writes one plane row per warp
// (128-byte stores).  N even and 16-byte aligned y / x (else the host takes K6b).
constexpr int K10_LSR = 6;                  // rows per CTA: R / 6 CTAs at 3 per SM is one wave for massive_12w
constexpr int K10_LSJ = 4;                  // float4 loads in flight per thread
constexpr int K10_LST = 256;                // threads
__device__ __forceinline__ float rcp_ftz(float v) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
__global__ void __launch_bounds__(K10_LST) k10_ls(const float4 *__restrict__ y, const float4 *__restrict__ x,
                                                  uint32_t *__restrict__ ls_hi, uint32_t *__restrict__ ls_lo, int M,
                                                  int R, int N, int S, int n_ue, int KP, int KP4) {
  extern __shared__ float2 lst[];                   // [K10_LSR][n_ue][KPS]
  pdl_wait();                                       // y, x (caller data) and the planes (read by the previous call)
#ifndef K10_LS_LATE_TRIGGER
  if (threadIdx.x == 0) pdl_launch_dependents();    // k10_comb_tc may start its weight-image loads
#endif
  const int KPS = KP4 + 1, N2 = N >> 1, t = threadIdx.x;
  const int rb = blockIdx.x * K10_LSR;
  const int nr = min(K10_LSR, R - rb);
  const int tot = nr * N2;                          // float4 (tone pairs) of the CTA's rows
  // coordinates of float4 i = t: row, tone pair k2 (tone k = 2 k2), pilot pp and UE ss of tone k
  int row = t / N2, k2 = t - (t / N2) * N2;
  int pp = (2 * k2) / S, ss = 2 * k2 - pp * S;
  const int d2 = K10_LST % N2, drow = K10_LST / N2;           // step of (row, k2) per K10_LST float4
  const int dq = (2 * d2) / S, dr = 2 * d2 - dq * S;           // tone step 2*d2 as (pilots, UEs)
  const float4 *yb = y + size_t(rb) * N2;
  const int t0 = rb / M, split = (t0 + 1) * M - rb;  // rows >= split belong to later instances (no division before)
  for (int i0 = t; i0 < tot; i0 += K10_LSJ * K10_LST) {
    float4 yv[K10_LSJ], xv[K10_LSJ];
    int rr[K10_LSJ], kk[K10_LSJ], pq[K10_LSJ], sq[K10_LSJ];
#pragma unroll
    for (int j = 0; j < K10_LSJ; ++j) {
      rr[j] = row;
      kk[j] = k2;
      pq[j] = pp;
      sq[j] = ss;
      if (i0 + j * K10_LST < tot) {
        yv[j] = yb[i0 + j * K10_LST];
        xv[j] = __ldg(x + size_t(row < split ? t0 : (rb + row) / M) * N2 + k2);
      }
      // advance by K10_LST float4: the tone moves by 2*d2 (and to the next row drow + carry times)
      k2 += d2;
      row += drow;
      pp += dq;
      ss += dr;
      if (ss >= S) {
        ss -= S;
        ++pp;
      }
      if (k2 >= N2) {
        k2 -= N2;
        ++row;
        pp -= KP;                                   // tone k - N: N = KP * S
      }
    }
#pragma unroll
    for (int j = 0; j < K10_LSJ; ++j) {
      if (i0 + j * K10_LST < tot) {
        const float i0f = rcp_ftz(xv[j].x * xv[j].x + xv[j].y * xv[j].y);
        const float i1f = rcp_ftz(xv[j].z * xv[j].z + xv[j].w * xv[j].w);
        const float f0r = xv[j].x * i0f, f0i = -xv[j].y * i0f, f1r = xv[j].z * i1f, f1i = -xv[j].w * i1f;
        float2 *base = lst + size_t(rr[j]) * n_ue * KPS;
        if (sq[j] < n_ue)
          base[sq[j] * KPS + pq[j]] = make_float2(yv[j].x * f0r - yv[j].y * f0i, yv[j].x * f0i + yv[j].y * f0r);
        int p1 = pq[j], s1 = sq[j] + 1;             // tone k + 1
        if (s1 == S) {
          s1 = 0;
          ++p1;
        }
        if (s1 < n_ue)
          base[s1 * KPS + p1] = make_float2(yv[j].z * f1r - yv[j].w * f1i, yv[j].z * f1i + yv[j].w * f1r);
      }
    }
  }
  __syncthreads();
  // phase 2: for each UE the CTA's nr plane rows are one contiguous run of nr * KP4 words per plane; thread t owns
  // words t, t + K10_LST, ... of every UE's run (row / pilot split once), so the UE loop is address increments only
  const int W = nr * KP4;
  const size_t ue_step = size_t(R) * KP4;
  for (int w = t; w < W; w += K10_LST) {
    const int r = w / KP4, p = w - r * KP4;
    const bool live = p < KP;
    const float2 *src = lst + r * n_ue * KPS + p;
    uint32_t *dh = ls_hi + size_t(rb) * KP4 + w, *dl = ls_lo + size_t(rb) * KP4 + w;
    for (int sc = 0; sc < n_ue; ++sc, src += KPS, dh += ue_step, dl += ue_step) {
      const float2 v = live ? *src : make_float2(0.f, 0.f);
      const uint32_t hv = pack_bf16x2(v.x, v.y);
      *dh = hv;
      *dl = pack_bf16x2(v.x - bf16lo(hv), v.y - bf16hi(hv));
    }
  }
#ifdef K10_LS_LATE_TRIGGER
  if (threadIdx.x == 0) pdl_launch_dependents();
#endif
}

// Weight image of (UE s, block b): A[m][kk], m = 2o + c (output o = i*S + q of group g0 + i, c = re / im row),
// kk = 2j' + c' (pilot sw + j'): the 2x2 real embedding of W_s^(type_g)[q][sw + j' - a_g] (zero outside the
// group's G taps and beyond the block's outputs); bf16 hi / lo planes in the SW64 image (row m at m*64 bytes,
// 16-byte chunk (kk/8) ^ ((m>>1)&3)).
__global__ void k10_build_images(const float2 *__restrict__ W, const int4 *__restrict__ rep, int n_cls, int S,
                                 int G, int K, int ml, uint16_t *__restrict__ img_hi, uint16_t *__restrict__ img_lo) {
  const int c = blockIdx.x, s = blockIdx.y;
  const int4 B = rep[c];                             // a block of image class c
  uint16_t *hi = img_hi + (size_t(s) * n_cls + c) * 128 * 32;
  uint16_t *lo = img_lo + (size_t(s) * n_cls + c) * 128 * 32;
  for (int e = threadIdx.x; e < 128 * 32; e += blockDim.x) {
    const int m = e / 32, kk = e % 32;
    const int o = m >> 1, ri = m & 1, jj = kk >> 1, cc = kk & 1;
    float v = 0.f;
    if (o < B.y * S) {
      const int i = o / S, q = o - i * S, g = B.x + i;
      const int a = min(max(g - ml, 0), K - G);
      const int j = B.z + jj - a;
      if (j >= 0 && j < G) {
        const float2 w = W[((size_t(s) * G + (g - a)) * S + q) * G + j];
        const int sel = (ri << 1) | cc;
        v = sel == 0 ? w.x : sel == 1 ? -w.y : sel == 2 ? w.y : w.x;
      }
    }
    const uint32_t h2 = pack_bf16x2(v, 0.f);
    const uint32_t l2 = pack_bf16x2(v - bf16lo(h2), 0.f);
    const int dst = m * 32 + (((kk >> 3) ^ ((m >> 1) & 3)) << 3) + (kk & 7);
    hi[dst] = uint16_t(h2 & 0xFFFFu);
    lo[dst] = uint16_t(l2 & 0xFFFFu);
  }
}

__global__ void __launch_bounds__(K10_THREADS, K10_CTAS)
    k10_comb_tc(const __grid_constant__ CUtensorMap tml_hi, const __grid_constant__ CUtensorMap tml_lo,
                const __grid_constant__ CUtensorMap tmh, const __grid_constant__ K10Params p) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ int4 blk_s[K10_MAXBLK];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sa = smem;                                         // [SA][hi | lo]
  uint8_t *sb = smem + K10_SA * 2 * K10_PLANE;                // [SB][hi | lo]
  uint8_t *stg = sb + K10_SB * 2 * K10_PLANE;                 // [EPI warps][2][32 rows][32 floats]
  uint64_t *bars = reinterpret_cast<uint64_t *>(stg + K10_EPI * K10_NSTG * K10_STG);
  uint64_t *a_full = bars, *a_empty = bars + K10_SA;
  uint64_t *b_full = bars + 2 * K10_SA, *b_empty = b_full + K10_SB;
  uint64_t *tmem_full = b_empty + K10_SB, *tmem_empty = tmem_full + K10_NACC;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_empty + K10_NACC);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) K10TR(0);
#if K10_INTERLEAVE
  // grid-stride units: at any moment the CTAs work on consecutive units (the blocks of the same rows and UE), so every
  // row's output pages are written by many SMs within a short window
  const int u0 = 0, u1 = (p.u_total - int(blockIdx.x) + int(gridDim.x) - 1) / int(gridDim.x);
  auto unit_at = [&](int j) { return decode10(p, int(blockIdx.x) + j * int(gridDim.x)); };
#else
  const int u0 = int((long long)blockIdx.x * p.u_total / gridDim.x);
  const int u1 = int((long long)(blockIdx.x + 1) * p.u_total / gridDim.x);
  auto unit_at = [&](int j) { return decode10(p, j); };
#endif
  const bool blk_in_smem = p.n_blk <= K10_MAXBLK;
  if (blk_in_smem)
    for (int i = tid; i < p.n_blk; i += blockDim.x) blk_s[i] = p.blk[i];   // built by ce_comb_init (not caller data)
  if (tid == 0) {
    for (int i = 0; i < K10_SA; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < K10_SB; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
    }
    for (int i = 0; i < K10_NACC; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&tmem_empty[i], K10_EPI);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, K10_NACC * K10_NR);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (tid == 0) pdl_launch_dependents();
  auto block_of = [&](int b) { return blk_in_smem ? blk_s[b] : __ldg(&p.blk[b]); };

#ifdef K10_ABL_STOREONLY
  if (warp < 2) {
  } else
#endif
  if (warp == 0) {
    // ------------------------------------------------------------------ producer (TMA / bulk copies)
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tml_hi)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tml_lo)) : "memory");
      const uint64_t pol = l2_evict_last_policy();
      int key_prev = -1, na = 0, ib = 0;
      bool waited = false;
      for (int u = u0; u < u1; ++u, ++ib) {
        const Unit10 d = unit_at(u);
        const int4 B = block_of(d.b);
        const int key = d.s * p.n_cls + B.w;           // weight image of (UE, class)
        if (key != key_prev) {                         // the weight image changes: next A slot
          const int sl = na % K10_SA;
          mbar_wait(&a_empty[sl], ((na / K10_SA) & 1) ^ 1);
          mbar_arrive_expect_tx(&a_full[sl], 2 * K10_PLANE);
          const size_t src = size_t(key) * 128 * 32;
          bulk_g2s(sa + sl * 2 * K10_PLANE, p.img_hi + src, K10_PLANE, &a_full[sl]);
          bulk_g2s(sa + sl * 2 * K10_PLANE + K10_PLANE, p.img_lo + src, K10_PLANE, &a_full[sl]);
          ++na;
          key_prev = key;
        }
        if (!waited) {                                 // the LS planes come from the preceding k10_ls
          pdl_wait();
          waited = true;
        }
        const int st = ib % K10_SB;
#if K10_ONE_COMMIT
        // one commit per unit: stage st was read by the MMAs of unit ib - SB, whose completion is tmem_full[st]
        if (ib >= K10_SB) mbar_wait(&tmem_full[st], ((ib - K10_SB) / K10_NACC) & 1);
#else
        mbar_wait(&b_empty[st], ((ib / K10_SB) & 1) ^ 1);
#endif
#ifdef K10_ABL_NOLOAD
        mbar_arrive(&b_full[st]);
        continue;
#endif
        mbar_arrive_expect_tx(&b_full[st], 2 * K10_PLANE);
        if (u - u0 < 40) K10TR(8 + u - u0);
        const int c0 = 2 * B.z, c1 = d.s * p.R + d.rt * K10_NR;
        if (p.l2_hint & 1) {
          tma_load_2d_hint(sb + st * 2 * K10_PLANE, &tml_hi, c0, c1, &b_full[st], pol);
          tma_load_2d_hint(sb + st * 2 * K10_PLANE + K10_PLANE, &tml_lo, c0, c1, &b_full[st], pol);
        } else {
          tma_load_2d(sb + st * 2 * K10_PLANE, &tml_hi, c0, c1, &b_full[st]);
          tma_load_2d(sb + st * 2 * K10_PLANE + K10_PLANE, &tml_lo, c0, c1, &b_full[st]);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      // F32 accumulate, BF16 A / B, both K-major, N = 128, M = 128
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(K10_NR >> 3) << 17) | (uint32_t(128 >> 4) << 24);
      int key_prev = -1, na = 0, ib = 0, lt = 0;
      Unit10 dn = unit_at(u0);
      int key_next = u0 < u1 ? dn.s * p.n_cls + block_of(dn.b).w : -1;
      for (int u = u0; u < u1; ++u, ++ib, ++lt) {
        const int key = key_next;
        if (key != key_prev) {
          mbar_wait(&a_full[na % K10_SA], (na / K10_SA) & 1);
          ++na;
          key_prev = key;
        }
        if (u + 1 < u1) {
          dn = unit_at(u + 1);
          key_next = dn.s * p.n_cls + block_of(dn.b).w;
        } else {
          key_next = -1;
        }
        const int sl = (na - 1) % K10_SA;
        const int acc = lt % K10_NACC;
        if (lt < 40) K10TR(168 + lt);
        mbar_wait(&tmem_empty[acc], ((lt / K10_NACC) & 1) ^ 1);
        if (lt < 40) K10TR(208 + lt);
        const int st = ib % K10_SB;
        mbar_wait(&b_full[st], (ib / K10_SB) & 1);
        tc_fence_after();
        if (lt < 40) K10TR(48 + lt);
        const uint32_t dt = tmem_base + uint32_t(acc * K10_NR);
        const uint64_t ah = sw64_desc(smem_u32(sa + sl * 2 * K10_PLANE));
        const uint64_t al = sw64_desc(smem_u32(sa + sl * 2 * K10_PLANE + K10_PLANE));
        const uint64_t bh = sw64_desc(smem_u32(sb + st * 2 * K10_PLANE));
        const uint64_t bl = sw64_desc(smem_u32(sb + st * 2 * K10_PLANE + K10_PLANE));
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint64_t adv = uint64_t(2 * ks);       // +32 bytes along K
          // A = the LS tile (M = 128 data rows), B = the weight image (N = 128 output floats): D[row][float]
          mma_bf16(dt, bh + adv, ah + adv, idesc, ks != 0);
          mma_bf16(dt, bh + adv, al + adv, idesc, 1u);
          mma_bf16(dt, bl + adv, ah + adv, idesc, 1u);
        }
#if !K10_ONE_COMMIT
        mma_commit(&b_empty[st]);
#endif
        if (key_next != key) mma_commit(&a_empty[sl]);   // last use of the image
        mma_commit(&tmem_full[acc]);
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue
    // TMEM lane = data row, column = output float: tcgen05.ld 32x32b gives each thread 32 consecutive output floats
    // (128 bytes of h) of its row; full 32-float blocks go through SW128 staging (8 conflict-free 16-byte shared stores
    // per thread) and one 3-D TMA store {32 floats, UE s, 32 rows}; a block cut by the block's output end (5-group
    // blocks: 120 floats) leaves through direct 16-byte stores of the valid floats
    pdl_wait();                                        // h may still be read by the previous kernel in the stream
    const int ew = warp - 2;
    const int q = warp & 3;                            // TMEM lane quadrant = rows 32q .. 32q + 31 of the unit
    const int part = ew >> 2;                          // column blocks part + (K10_EPI / 4) i
    uint8_t *mystg = stg + ew * K10_NSTG * K10_STG;
    const size_t row_floats = size_t(p.n_ue) * p.N * 2;
    int lt = 0, nst = 0;
    for (int u = u0; u < u1; ++u, ++lt) {
      const Unit10 d = unit_at(u);
      const int4 B = block_of(d.b);
      const int acc = lt % K10_NACC;
#ifndef K10_ABL_STOREONLY
      mbar_wait(&tmem_full[acc], (lt / K10_NACC) & 1);
      tc_fence_after();
#endif
      if (tid == 64 && lt < 40) K10TR(88 + lt);
      const int nf = 2 * B.y * p.S;                    // valid output floats of the block
#ifdef K10_ABL_NOEPI
      __syncwarp();
      if (lane == 0) {
        tc_fence_before();
        mbar_arrive(&tmem_empty[acc]);
      }
      continue;
#endif
      float v[K10_NCBW][32];
#ifdef K10_ABL_STOREONLY
#pragma unroll
      for (int i = 0; i < K10_NCBW; ++i)
#pragma unroll
        for (int c = 0; c < 32; ++c) v[i][c] = float(c + lane);
#else
#pragma unroll
      for (int i = 0; i < K10_NCBW; ++i)
        if (32 * (part + (K10_EPI / 4) * i) < nf)
          tmem_ld32(tmem_base + uint32_t(acc * K10_NR + 32 * (part + (K10_EPI / 4) * i)) + (uint32_t(32 * q) << 16), v[i]);
      __syncwarp();
      if (lane == 0) {
        tc_fence_before();
        mbar_arrive(&tmem_empty[acc]);               // the accumulator is in registers: the MMA may reuse it
      }
#endif
      if (tid == 64 && lt < 40) K10TR(256 + lt);
      const int r0 = d.rt * K10_NR + 32 * q;           // first row of this warp
      const int row = r0 + lane;
#pragma unroll
      for (int i = 0; i < K10_NCBW; ++i) {
        const int cb = part + (K10_EPI / 4) * i;
        const int f0 = 32 * cb;
        if (f0 >= nf || r0 >= p.R) continue;
        if (f0 + 32 <= nf && p.tma_st) {
          uint8_t *buf = mystg + (nst % K10_NSTG) * K10_STG;
          if (lane == 0) {                             // the store that used this buffer has read it
            if (K10_NSTG == 2)
              bulk_wait_read1();
            else
              bulk_wait_read0();
          }
          __syncwarp();
          if (tid == 64 && lt < 40) K10TR(296 + 40 * i + lt);
#pragma unroll
          for (int j = 0; j < 8; ++j)                  // SW128: 16-byte chunk j of row `lane` at chunk j ^ (lane & 7)
            *reinterpret_cast<float4 *>(buf + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                make_float4(v[i][4 * j], v[i][4 * j + 1], v[i][4 * j + 2], v[i][4 * j + 3]);
          if (tid == 64 && lt < 40) K10TR(376 + 40 * i + lt);
#ifdef K10_ST_LSU
          // coalesced LSU stores from the staged block: each instruction writes 4 rows x 128 B (full lines)
          __syncwarp();
          {
            float *hb = p.h + (size_t(d.s) * p.N + size_t(p.S) * B.x) * 2 + f0 + 4 * (lane & 7);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int rr = 4 * k + (lane >> 3), j = lane & 7;
              const float4 w = *reinterpret_cast<const float4 *>(buf + rr * 128 + ((j ^ (rr & 7)) << 4));
              if (r0 + rr < p.R) *reinterpret_cast<float4 *>(hb + size_t(r0 + rr) * row_floats) = w;
            }
          }
          __syncwarp();
          ++nst;
          continue;
#endif
          fence_proxy_async();
          __syncwarp();
          if (tid == 64 && lt < 40) K10TR(456 + 40 * i + lt);
          if (lane == 0) {
#ifndef K10_ABL_NOSTORE
            if (p.l2_hint & 2)
              tma_store_3d_hint(&tmh, buf, 2 * p.S * B.x + f0, d.s, r0, l2_evict_first_policy());
            else
#ifdef K10_ABL_ALIGNED
              tma_store_3d(&tmh, buf, ((2 * p.S * B.x) & ~31) + f0, d.s, r0);   // line-aligned (results wrong)
#else
              tma_store_3d(&tmh, buf, 2 * p.S * B.x + f0, d.s, r0);
#endif
#endif
            bulk_commit();
          }
          ++nst;
        } else if (row < p.R) {
          float *hr = p.h + size_t(row) * row_floats + (size_t(d.s) * p.N + size_t(p.S) * B.x) * 2 + f0;
          const int nv = min(32, nf - f0);             // a multiple of 4 (2 S ng floats, S * ng even)
          if ((reinterpret_cast<uintptr_t>(hr) & 15) == 0 && (nv & 3) == 0) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (4 * j < nv)
                *reinterpret_cast<float4 *>(hr + 4 * j) =
                    make_float4(v[i][4 * j], v[i][4 * j + 1], v[i][4 * j + 2], v[i][4 * j + 3]);
          } else {
#pragma unroll
            for (int c = 0; c < 32; ++c)
              if (c < nv) hr[c] = v[i][c];
          }
        }
      }
      if (tid == 64 && lt < 40) K10TR(128 + lt);
    }
    if (lane == 0) bulk_wait0();                       // every TMA store of this warp has completed
    if (tid == 64) K10TR(1);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem_base, K10_NACC * K10_NR);
  }
}

// [rows][2 KP] bf16 plane with row pitch KP4 * 4 bytes, box [128 rows][32 bf16], SWIZZLE_64B (the MMA's K-major
// SW64 B layout); pilots beyond KP and rows beyond `rows` read as zero.
bool make_map_ls(CUtensorMap *m, const void *ptr, int KP, int KP4, long long rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cuuint64_t(2) * KP, cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(KP4) * 4};
  cuuint32_t box[2] = {32, cuuint32_t(K10_NR)};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// h [R][n_ue][2N floats] as a 3-D tensor (2N, n_ue, R), box {32 floats, 1, 32 rows}, SWIZZLE_128B (store map).
bool make_map_h(CUtensorMap *m, const void *ptr, int N, int n_ue, long long R) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {cuuint64_t(2) * N, cuuint64_t(n_ue), cuuint64_t(R)};
  cuuint64_t strides[2] = {cuuint64_t(2) * N * 4, cuuint64_t(2) * N * 4 * n_ue};
  cuuint32_t box[3] = {32, 1, 32};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void *>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct K10Dev {
  bool init = false;
  int num_sms = 0;
};
cudaError_t k10_dev(K10Dev **out) {
  static K10Dev infos[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  K10Dev &d = infos[dev];
  if (!d.init) {
    e = cudaDeviceGetAttribute(&d.num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k10_comb_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, K10_SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k10_comb_tc, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
    d.init = true;
  }
  *out = &d;
  return cudaSuccess;
}

}  // namespace

#ifdef CE_K10_TRACE
extern "C" int ce_k10_trace_set(void *dptr) { return int(cudaMemcpyToSymbol(g_k10_trace, &dptr, sizeof(dptr))); }
#endif

bool comb_tc_supported(int32_t N, int32_t S, int32_t G, int32_t mode) {
  // a 16-pilot window at a multiple of 4 holds any G <= 13 window; a block's outputs fit M = 128 rows
  // k10_ls stages K10_LSR rows ([n_ue][KP4 + 1] complex each, n_ue <= S) in shared memory and reads float4 (N even)
  const long long KP4 = S >= 1 ? ((N / S) + 3) & ~3LL : 0;
  return mode == CE_COMB_FULL && G >= 1 && G <= K10_WIN - 3 && S >= 1 && S <= 64 && N % S == 0 && N % 2 == 0 &&
         (long long)K10_LSR * S * (KP4 + 1) * 8 <= 200 * 1024 && encode_fn() != nullptr;
}

std::vector<int4> comb_tc_blocks(int32_t K, int32_t G, int32_t S, std::vector<int4> *rep) {
  const int ml = (G - 1) / 2;
  auto a_of = [&](int g) { return std::min(std::max(g - ml, 0), K - G); };
  const int maxng = 64 / S;
  std::vector<int4> out;
  std::vector<std::vector<int>> sigs;                // per class: ng, then (type, a - sw) per group
  rep->clear();
  for (int g = 0; g < K;) {
    const int sw = a_of(g) & ~3;
    int ng = 1;
    while (g + ng < K && ng < maxng && a_of(g + ng) + G <= sw + K10_WIN) ++ng;
    std::vector<int> sig{ng};
    for (int i = 0; i < ng; ++i) {
      sig.push_back(g + i - a_of(g + i));
      sig.push_back(a_of(g + i) - sw);
    }
    int cls = int(std::find(sigs.begin(), sigs.end(), sig) - sigs.begin());
    if (cls == int(sigs.size())) {
      sigs.push_back(sig);
      rep->push_back(make_int4(g, ng, sw, cls));
    }
    out.push_back(make_int4(g, ng, sw, cls));
    g += ng;
  }
  return out;
}

size_t comb_tc_image_elems(int32_t n_ue, int32_t n_cls) { return size_t(n_ue) * n_cls * 128 * 32; }

size_t comb_tc_ls_bytes(int32_t N, int32_t S, int32_t n_ue, long long rows) {
  const long long KP4 = ((N / S) + 3) & ~3LL;
  return size_t(2) * n_ue * rows * KP4 * 4;       // hi and lo planes
}

cudaError_t launch_comb_tc_images(const float2 *W, const int4 *d_rep, int32_t n_cls, int32_t n_ue, int32_t N,
                                  int32_t S, int32_t G, uint16_t *img_hi, uint16_t *img_lo, cudaStream_t stream) {
  k10_build_images<<<dim3(n_cls, n_ue), 256, 0, stream>>>(W, d_rep, n_cls, S, G, N / S, (G - 1) / 2, img_hi, img_lo);
  return cudaGetLastError();
}

cudaError_t launch_comb_tc(const float2 *y, const float2 *x, float2 *h, int32_t T, int32_t M, int32_t N, int32_t S,
                           int32_t n_ue, const int4 *d_blk, int32_t n_blk, int32_t n_cls, const uint16_t *img_hi,
                           const uint16_t *img_lo, void *ls, cudaStream_t stream, int64_t *launches) {
  K10Dev *di = nullptr;
  cudaError_t e = k10_dev(&di);
  if (e != cudaSuccess) return e;
  const long long R = (long long)T * M;
  const int KP = N / S, KP4 = (KP + 3) & ~3;
  if (R * n_ue >= (1LL << 31) || (reinterpret_cast<uintptr_t>(ls) & 15)) return cudaErrorInvalidValue;
  uint32_t *ls_hi = static_cast<uint32_t *>(ls);
  uint32_t *ls_lo = ls_hi + size_t(n_ue) * R * KP4;
  CUtensorMap mh, ml;
  if (!make_map_ls(&mh, ls_hi, KP, KP4, R * n_ue) || !make_map_ls(&ml, ls_lo, KP, KP4, R * n_ue))
    return cudaErrorInvalidValue;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  // LS planes
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned((R + K10_LSR - 1) / K10_LSR));
    cfg.blockDim = dim3(K10_LST);
    cfg.dynamicSmemBytes = size_t(K10_LSR) * n_ue * (KP4 + 1) * sizeof(float2);
    cfg.stream = stream;
    cfg.attrs = at;
#ifdef K10_NO_PDL
    cfg.numAttrs = 0;
#else
    cfg.numAttrs = 1;
#endif
    e = smem_opt_in((const void *)k10_ls, cfg.dynamicSmemBytes);
    // the default carveout left room for 3 CTAs of 39 KB per SM (ncu occupancy limit): ask for the whole array
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k10_ls, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
    e = cudaLaunchKernelEx(&cfg, k10_ls, reinterpret_cast<const float4 *>(y), reinterpret_cast<const float4 *>(x),
                           ls_hi, ls_lo, int(M), int(R), int(N), int(S), int(n_ue), KP, KP4);
    if (e != cudaSuccess) return e;
    ++*launches;
  }
  K10Params p;
  p.h = reinterpret_cast<float *>(h);
  p.img_hi = img_hi;
  p.img_lo = img_lo;
  p.blk = d_blk;
  p.R = int(R);
  p.n_ue = n_ue;
  p.N = N;
  p.S = S;
  p.n_blk = n_blk;
  p.n_cls = n_cls;
  p.n_rt = int((R + K10_NR - 1) / K10_NR);
  const long long units = (long long)n_ue * n_blk * p.n_rt;
  if (units >= (1LL << 31)) return cudaErrorInvalidConfiguration;
  p.u_total = int(units);
  // 3-D TMA stores need a 16-byte aligned h and 16-byte row pitch (N even); else direct stores
  static const int env_st = getenv("CE_K10_TMA_STORE") ? atoi(getenv("CE_K10_TMA_STORE")) : -1;   // experiments
  static const int env_hint = getenv("CE_K10_L2HINT") ? atoi(getenv("CE_K10_L2HINT")) : -1;       // experiments
  CUtensorMap mhh = {};
  p.tma_st = env_st != 0 && (reinterpret_cast<uintptr_t>(h) & 15) == 0 && (N % 2) == 0 &&
             make_map_h(&mhh, h, N, n_ue, R);
  // evict_last LS loads + evict_first h stores: the LS planes stay in L2 (DRAM reads 23 -> 1.3 MB per launch)
  p.l2_hint = env_hint >= 0 ? env_hint : 3;
  cudaLaunchConfig_t cfg = {};
  const long long slots = (long long)K10_CTAS * di->num_sms;
  cfg.gridDim = dim3(unsigned(units < slots ? units : slots));
  cfg.blockDim = dim3(K10_THREADS);
  cfg.dynamicSmemBytes = K10_SMEM;
  cfg.stream = stream;
  cfg.attrs = at;
#ifdef K10_NO_PDL
  cfg.numAttrs = 0;
#else
  cfg.numAttrs = 1;
#endif
  e = cudaLaunchKernelEx(&cfg, k10_comb_tc, mh, ml, mhh, p);
  if (e == cudaSuccess) ++*launches;
  return e;
}

}  // namespace ce
