// K5 -- fused LS + block-LMMSE contraction on a CTA PAIR with the FILTER STATIONARY IN TENSOR MEMORY.
//
// Same operation as K2-K4 (Eq. 12 per block, the LS of Eq. 9 fused into the load,
// the filter of Eq. 17 built by K1) and the same error-compensated BF16x3 products as K4
// (reading B1): X_hi = bf16_rn(X), X_lo = bf16_rn(X - X_hi), D = W_hi L_hi + W_hi L_lo + W_lo L_hi,
// FP32 accumulation in TMEM.  What differs is the dataflow: the operands are swapped.
//
//   D^T [2 kept real output rows][columns c] = Wr [2 kept][2b]  x  Lr^T [2b][columns c]
//     Wr rows 2i / 2i+1 = (Re W_ij, -Im W_ij) / (Im W_ij, Re W_ij) over j  -- the real embedding of the filter rows
//     [o_w - a_w, o_w - a_w + kept) of window w (the paper's 12W edge clamping, selects rows)
//     Lr^T column c = the interleaved LS row of column c = (antenna m, user k) over the window's b input tones
//
// The filter is the MMA's A operand and lives in TMEM (tcgen05.mma ... [a_tmem]): a pair of CTAs
// (tcgen05 cta_group::2, M = 256 = 128 TMEM lanes per CTA) holds 256 real filter rows -- up to 128 complex outputs
// per window -- for the whole 2b-deep contraction, loaded once per (statistic set, row class) and reused by every
// column tile the pair walks.  Only the LS tile streams through shared memory (the B operand, N = NP columns: NB =
// NP / 2 per CTA).  Per 16 complex tones of a 64-column CTA tile the shared-memory traffic is the raw y box (8 KB
// in by TMA, 8 KB out to the transform), the LS planes (8 KB written) and the MMA reads of them (12 KB); K4 streams
// the filter bank through shared memory as well and reads both operands per MMA (~3x the bytes per output).
//
// Work unit: a pair tile = (instance t, window w, column block cb of NP columns).  Tiles are walked in the order
// (t, row class, cb, w) -- windows whose kept filter rows fit the same 256-row slice [R0, R0 + 256) of Wr form a
// row class and share the TMEM-resident A (the epilogue selects their lanes); consecutive tiles of a pair are
// adjacent windows over the same columns, so overlapping windows re-read y from L2.  Each pair walks a contiguous
// range of tiles; the filter is reloaded only when (set, class) changes.
//
// Roles (each CTA of the pair, 576 threads):
//   warp 12    : raw producer -- 2D TMA of the raw y box [NB rows x 16 complex] and the pilot box [K x 16 complex]
//   warps 0-7  : transform -- LS = y conj(x) / |x|^2, bf16 hi/lo -> SWIZZLE_64B K-major B planes; remote arrive
//                on the leader's b_full (16 arrivals: 8 warps x 2 CTAs)
//   warp 13    : TMEM allocation (cta_group::2, 512 columns); on the leader the MMA issuer: 3 MMAs per 16-deep K
//                step (M = 256, N = NP), commits multicast to both CTAs
//   warps 14-17: filter loaders -- bulk copies of the filter's TMEM image (4 KB pieces) through a staging ring,
//                then ld.shared + tcgen05.st into this CTA's 128 lanes; one lane quarter per warp
//   warps 8-11 : epilogue -- tcgen05.ld 32x32b (lane = real output row, 32 columns per load) -> each store
//                instruction writes 32 consecutive floats (one 128-byte segment) of one output row h[t][c][.]
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

constexpr int K5_THREADS = 576;           // 18 warps
constexpr int CK = 16;                    // complex per K chunk (32 real = 2 MMA K steps; 64-byte bf16 rows)
constexpr int MAX_RAW = 16;
constexpr int MAX_B = 8;
constexpr int MAX_WS = 32;
constexpr int WS_BYTES = 4096;            // one staging piece: (plane, K step), 2 halves x 128 rows x 16 B
constexpr int MAXW5 = 64;                 // windows carried in the kernel parameters
constexpr int MAXC5 = 8;                  // row classes
constexpr int SMEM_LIMIT = 232448;        // sm_100 opt-in maximum per CTA
constexpr int BAR_BYTES = 1024;

// Optional per-CTA event trace (tools/k4_trace.cu, built by tools/k4_trace.sh with -DCE_K4_TRACE; the product build
// has none): clock64 per event slot, slot 0 / 5 = %globaltimer at CTA start / end.
#ifdef CE_K4_TRACE
__device__ unsigned long long *g_k5_trace;
#define K5TR(slot)                                                                \
  do {                                                                            \
    const unsigned long long c_ = clock64();                                      \
    if (g_k5_trace) g_k5_trace[size_t(blockIdx.x) * 256 + (slot)] = c_;           \
  } while (0)
#define K5GT(slot)                                                                \
  do {                                                                            \
    unsigned long long gt_;                                                       \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));                       \
    if (g_k5_trace) g_k5_trace[size_t(blockIdx.x) * 256 + (slot)] = gt_;          \
  } while (0)
#else
#define K5TR(slot) \
  do {             \
  } while (0)
#define K5GT(slot) \
  do {             \
  } while (0)
#endif

struct Win5 {
  int a, o, kept, cls;
};

struct K5Params {
  float *hf;                 // output, as floats
  const uint4 *wimg;         // filter TMEM image [n_rep][n_sets][2 planes][nks][2 halves][RP rows] of 16 B
  long long rep_stride;      // uint4 elements per replica (pair p reads replica p % n_rep: spreads the all-SM reads)
  int n_rep;
  const Win5 *win_d;         // device window table (n_win > MAXW5), class-sorted
  const int32_t *soi;
  int T, K, N, b, n_sets, nks, nkc, RP, cols;
  int NP, NB, n_cb, n_acc, a_col0;
  int n_win, n_cls, n_tiles;
  int s_raw, s_b, s_w;
  int raw_stage, b_stage, xbytes;
  int off_b, off_w, off_e, off_bar;
  int epi_tma;               // 1: full, aligned 32 x 32 output blocks leave through smem staging + TMA stores
  int cls_start[MAXC5 + 1];  // windows of class c: [cls_start[c], cls_start[c+1]) in the (sorted) table
  int cls_r0[MAXC5];         // first real filter row held in TMEM lane 0 of CTA 0 for class c
  Win5 win[MAXW5];
};

struct Tile5 {
  int t, cb, w, cls, a, o, kept;
};

__device__ __forceinline__ Tile5 decode5(const K5Params &p, int g) {
  Tile5 ti;
  const int per_t = p.n_win * p.n_cb;
  ti.t = g / per_t;
  const int r = g - ti.t * per_t;
  int c = 0;
  while (c + 1 < p.n_cls && r >= p.cls_start[c + 1] * p.n_cb) ++c;
  const int r2 = r - p.cls_start[c] * p.n_cb;
  const int nwc = p.cls_start[c + 1] - p.cls_start[c];
  ti.cb = r2 / nwc;
  ti.w = p.cls_start[c] + (r2 - ti.cb * nwc);
  ti.cls = c;
  const Win5 wv = p.n_win <= MAXW5 ? p.win[ti.w] : p.win_d[ti.w];
  ti.a = wv.a;
  ti.o = wv.o;
  ti.kept = wv.kept;
  return ti;
}

// statistic set of instance t (clamped: an out-of-range index makes that instance's outputs NaN, reading B3)
__device__ __forceinline__ int raw_set(const K5Params &p, int t) { return p.soi ? p.soi[t] : 0; }
__device__ __forceinline__ int key_of(const K5Params &p, const Tile5 &ti) {
  int s = p.n_sets == 1 ? 0 : raw_set(p, ti.t);
  s = (s >= 0 && s < p.n_sets) ? s : 0;
  return s * MAXC5 + ti.cls;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo_addr, float hi_addr) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi_addr), "f"(lo_addr));
  return r;
}
__device__ __forceinline__ float bf16_lo_f(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi_f(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }
__device__ __forceinline__ float rcp_approx(float v) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
// tcgen05.mma, CTA pair, A from TMEM: D[256 x N] (+)= A[256 x 16] B[16 x N]
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint4 &u, const uint4 &v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(u.x), "r"(u.y), "r"(u.z), "r"(u.w), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// arrive on the leader's (rank 0) copy of `bar`: local for rank 0, remote (release, cluster scope) for rank 1
__device__ __forceinline__ void arrive_leader(uint64_t *bar, int rank) {
  if (rank == 0)
    asm volatile("mbarrier.arrive.release.cluster.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
  else
    mbar_arrive_remote(bar, 0);
}
__device__ __forceinline__ void tmem_ld32x32_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void st_f32(float *ptr, float v) {
  asm volatile("st.global.f32 [%0], %1;" ::"l"(ptr), "f"(v) : "memory");
}

__global__ void __launch_bounds__(K5_THREADS, 1)
    k5_pair(const __grid_constant__ CUtensorMap tmy, const __grid_constant__ CUtensorMap tmx,
            const __grid_constant__ CUtensorMap tmh, const __grid_constant__ K5Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *raw = smem;                                   // [s_raw][y box NB x 128 B | x box K x 128 B]
  uint8_t *bst = smem + p.off_b;                         // [s_b][B_hi NB x 64 B | B_lo NB x 64 B]  (SW64)
  uint8_t *wst = smem + p.off_w;                         // [s_w][4 KB]  filter staging
  uint8_t *est = smem + p.off_e;                         // [4 warps][2][4 KB]  output staging (epi_tma)
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + p.off_bar);
  uint64_t *raw_full = bars;                             // [MAX_RAW]
  uint64_t *raw_empty = raw_full + MAX_RAW;              // [MAX_RAW] 8 transform warps
  uint64_t *b_full = raw_empty + MAX_RAW;                // [MAX_B]   leader: 16 (8 warps x 2 CTAs)
  uint64_t *b_empty = b_full + MAX_B;                    // [MAX_B]   commit (multicast)
  uint64_t *ws_full = b_empty + MAX_B;                   // [MAX_WS]  bulk copy landed
  uint64_t *ws_empty = ws_full + MAX_WS;                 // [MAX_WS]  4 loader warps
  uint64_t *tmem_full = ws_empty + MAX_WS;               // [2]       commit (multicast)
  uint64_t *tmem_empty = tmem_full + 2;                  // [2]       leader: 8 (4 epilogue warps x 2 CTAs)
  uint64_t *w_full = tmem_empty + 2;                     // [1]       leader: 8 (4 loader warps x 2 CTAs)
  uint64_t *w_free = w_full + 1;                         // [1]       commit (multicast) after the last tile of a key
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(w_free + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = int(cluster_ctarank());
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int g_lo = int((long long)p.n_tiles * pair / n_pairs);
  const int g_hi = int((long long)p.n_tiles * (pair + 1) / n_pairs);

  if (tid == 0) {
    K5GT(0);
    K5TR(1);
    for (int s = 0; s < MAX_RAW; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_empty[s], 8);
    }
    for (int s = 0; s < MAX_B; ++s) {
      mbar_init(&b_full[s], 16);
      mbar_init(&b_empty[s], 1);
    }
    for (int s = 0; s < MAX_WS; ++s) {
      mbar_init(&ws_full[s], 1);
      mbar_init(&ws_empty[s], 4);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&tmem_empty[i], 8);
    }
    mbar_init(w_full, 8);
    mbar_init(w_free, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 12 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmy)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmx)) : "memory");
  }
  if (warp == 13) tmem_alloc2(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (tid == 0) {
    pdl_launch_dependents();
    K5TR(2);
  }

  if (warp == 12) {
    // ------------------------------------------------------------------ raw producer
    if (lane == 0) {
      pdl_wait();
      K5TR(200);
      const uint32_t bytes = uint32_t(p.NB) * 128 + uint32_t(p.xbytes);
      int it = 0;
      for (int g = g_lo; g < g_hi; ++g) {
        const Tile5 ti = decode5(p, g);
        const int row0 = ti.t * p.cols + ti.cb * p.NP + rank * p.NB;
        for (int kc = 0; kc < p.nkc; ++kc, ++it) {
          const int s = it % p.s_raw;
          mbar_wait(&raw_empty[s], ((it / p.s_raw) & 1) ^ 1);
          mbar_arrive_expect_tx(&raw_full[s], bytes);
          uint8_t *st = raw + size_t(s) * p.raw_stage;
          const int f0 = 2 * (ti.a + kc * CK);
          if (it < 24) K5TR(8 + it);
          tma_load_2d(st, &tmy, f0, row0, &raw_full[s]);
          tma_load_2d(st + p.NB * 128, &tmx, f0, ti.t * p.K, &raw_full[s]);
        }
      }
    }
  } else if (warp < 8) {
    // ------------------------------------------------------------------ transform
    const int jp = tid & 7;            // complex pair 2jp, 2jp+1 of the 16-complex chunk
    const int rb = tid >> 3;           // rows rb + 32 i
    const int nri = (p.NB + 31) >> 5;
    int it = 0;
    for (int g = g_lo; g < g_hi; ++g) {
      const Tile5 ti = decode5(p, g);
      const int c_first = ti.cb * p.NP + rank * p.NB + rb;
      const int x_first = c_first % p.K;
      const int x_step = 32 % p.K;
      for (int kc = 0; kc < p.nkc; ++kc, ++it) {
        const int sr = it % p.s_raw, sb = it % p.s_b;
        mbar_wait(&raw_full[sr], (it / p.s_raw) & 1);
        if (tid == 0 && it < 24) K5TR(32 + it);
        const float4 *ry = reinterpret_cast<const float4 *>(raw + size_t(sr) * p.raw_stage);
        const float4 *rx = reinterpret_cast<const float4 *>(raw + size_t(sr) * p.raw_stage + p.NB * 128);
        float4 yv[4], xv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) yv[i] = xv[i] = make_float4(0.f, 0.f, 0.f, 1.f);
        int xr = x_first;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = rb + 32 * i;
          if (i < nri && r < p.NB) {
            yv[i] = ry[r * 8 + jp];
            xv[i] = rx[xr * 8 + jp];
          }
          xr += x_step;
          if (xr >= p.K) xr -= p.K;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&raw_empty[sr]);       // values are in registers: the raw slot can refill
        const bool ok0 = kc * CK + 2 * jp < p.b, ok1 = kc * CK + 2 * jp + 1 < p.b;
        uint32_t hv[4][2], lv[4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (i < nri) {
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
        }
        mbar_wait(&b_empty[sb], ((it / p.s_b) & 1) ^ 1);
        uint8_t *bh = bst + size_t(sb) * p.b_stage;
        uint8_t *bl = bh + p.NB * 64;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = rb + 32 * i;
          if (i < nri && r < p.NB) {
            // SW64 K-major: row r at r*64 bytes, 16-byte chunk (jp>>1) ^ ((r>>1)&3), 8-byte half (jp&1)
            const int off = r * 64 + ((((jp >> 1) ^ ((r >> 1) & 3))) << 4) + ((jp & 1) << 3);
            *reinterpret_cast<uint2 *>(bh + off) = make_uint2(hv[i][0], hv[i][1]);
            *reinterpret_cast<uint2 *>(bl + off) = make_uint2(lv[i][0], lv[i][1]);
          }
        }
        fence_proxy_async();
        __syncwarp();
        if (tid == 0 && it < 24) K5TR(56 + it);
        if (lane == 0) arrive_leader(&b_full[sb], rank);
      }
    }
  } else if (warp < 12) {
    // ------------------------------------------------------------------ epilogue
    const int q = warp & 3;
    pdl_wait();                        // h may still be read by the previous kernel in the stream
    int lt = 0, epi_n = 0;
    for (int g = g_lo; g < g_hi; ++g, ++lt) {
      const Tile5 ti = decode5(p, g);
      const int sr = raw_set(p, ti.t);
      const bool set_ok = sr >= 0 && sr < p.n_sets;
      const int acc = p.n_acc == 2 ? (lt & 1) : 0;
      const int use = p.n_acc == 2 ? (lt >> 1) : lt;
      mbar_wait(&tmem_full[acc], use & 1);
      tc_fence_after();
      if (tid == 256 && lt < 8) K5TR(136 + lt);
      // this lane's real filter row and its place in the window's kept outputs
      const int rho = p.cls_r0[ti.cls] + 128 * rank + 32 * q + lane;
      const int i2 = rho - 2 * (ti.o - ti.a);
      const bool row_ok = i2 >= 0 && i2 < 2 * ti.kept;
      const int c0 = ti.cb * p.NP;
      float *hp = p.hf + (size_t(ti.t) * p.cols + c0) * size_t(2 * p.N) + 2 * ti.o + i2;
      const size_t cstride = size_t(2) * p.N;
      const int ncb = p.NP >> 5;
      // this warp's 32 lanes are all kept outputs, 16-byte aligned in h: its 32 x 32 blocks can leave through a TMA store
      const int fcol = 2 * ti.o + i2 - lane;           // float column of lane 0 in the h row
      const bool warp_full = p.epi_tma && (i2 - lane) >= 0 && (i2 - lane) + 32 <= 2 * ti.kept && (fcol & 3) == 0;
      for (int cbk = 0; cbk < ncb; ++cbk) {
        uint32_t v[32];
        __syncwarp();
        tmem_ld32x32_x32(tmem_base + uint32_t(acc * p.NP + cbk * 32) + (uint32_t(q * 32) << 16), v);
        tmem_ld_wait();
        const int cc = c0 + cbk * 32;
        if (warp_full && cc + 32 <= p.cols) {
          float *stg = reinterpret_cast<float *>(est + (q * 2 + (epi_n & 1)) * 4096);
          if (lane == 0) bulk_wait_read1();            // the store issued from this buffer two blocks ago has read it
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 32; ++j) stg[j * 32 + lane] = set_ok ? __uint_as_float(v[j]) : __int_as_float(0x7fc00000);
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmh, stg, fcol, ti.t * p.cols + cc);
            bulk_commit();
          }
          ++epi_n;
        } else if (row_ok) {
          const int nj = min(32, p.cols - cc);
          float *hq = hp + size_t(cbk * 32) * cstride;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < nj) st_f32(hq + size_t(j) * cstride, set_ok ? __uint_as_float(v[j]) : __int_as_float(0x7fc00000));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (tid == 256 && lt < 8) K5TR(144 + lt);
      if (lane == 0) arrive_leader(&tmem_empty[acc], rank);
    }
    if (lane == 0) bulk_wait0();         // every TMA store of this warp has completed
    if (tid == 256) K5TR(3);
  } else if (warp == 13) {
    // ------------------------------------------------------------------ MMA issuer (leader)
    if (rank == 0 && lane == 0) {
      // F32 accumulate, BF16 A/B, A (TMEM) and B K-major, N = NP, M = 256
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(p.NP >> 3) << 17) | (uint32_t(256 >> 4) << 24);
      const int nks_total = p.nks;
      if (p.n_sets > 1) pdl_wait();                     // the key reads set_of_instance
      int it = 0, lt = 0, epoch = 0, key_prev = -1;
      for (int g = g_lo; g < g_hi; ++g, ++lt) {
        const Tile5 ti = decode5(p, g);
        const int key = key_of(p, ti);
        if (key != key_prev) {                          // the filter rows of this (set, class) are in TMEM
          mbar_wait_cluster(w_full, epoch & 1);
          if (epoch < 8) K5TR(152 + epoch);
          ++epoch;
          key_prev = key;
          tc_fence_after();
        }
        const int acc = p.n_acc == 2 ? (lt & 1) : 0;
        const int use = p.n_acc == 2 ? (lt >> 1) : lt;
        mbar_wait_cluster(&tmem_empty[acc], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + uint32_t(acc * p.NP);
        for (int kc = 0; kc < p.nkc; ++kc, ++it) {
          const int s = it % p.s_b;
          mbar_wait_cluster(&b_full[s], (it / p.s_b) & 1);
          tc_fence_after();
          if (it < 24) K5TR(104 + it);
          uint8_t *bh = bst + size_t(s) * p.b_stage;
          const uint64_t dbh = sw64_desc(smem_u32(bh));
          const uint64_t dbl = sw64_desc(smem_u32(bh + p.NB * 64));
          const int nks = min(2, nks_total - 2 * kc);
          for (int ks = 0; ks < nks; ++ks) {
            const uint32_t ah = tmem_base + uint32_t(p.a_col0 + 8 * (2 * kc + ks));
            const uint32_t al = ah + uint32_t(8 * nks_total);
            const uint64_t adv = uint64_t(2 * ks);   // +32 bytes along K
#ifndef K5_ABL_NOMMA
            mma2_ts(d, ah, dbh + adv, idesc, (kc | ks) != 0);
            mma2_ts(d, ah, dbl + adv, idesc, 1u);
            mma2_ts(d, al, dbh + adv, idesc, 1u);
#endif
          }
          mma_commit_pair(&b_empty[s]);
        }
        mma_commit_pair(&tmem_full[acc]);
        // the filter of this key is no longer needed once these MMAs complete: tell the loaders (exactly one
        // w_free completion per reload, in order -- the loaders never skip a phase)
        if (g + 1 < g_hi && key_of(p, decode5(p, g + 1)) != key) mma_commit_pair(w_free);
        if (lt < 8) K5TR(128 + lt);
      }
    }
  } else {
    // ------------------------------------------------------------------ filter loaders (warps 14-17)
    const int qq = warp & 3;
    const bool issuer = warp == 14 && lane == 0;
    if (p.n_sets > 1) pdl_wait();                       // the key reads set_of_instance
    const int P = 2 * p.nks;                            // pieces per load: (plane, K step)
    int wit = 0, lt = 0, key_prev = -1, reload = 0;
    // pieces are loaded in a rotated order per pair: all CTAs read the same filter image, and rotation spreads the
    // simultaneous requests over different L2 lines
    const int rot = (pair * 7) % P;
    for (int g = g_lo; g < g_hi; ++g, ++lt) {
      const Tile5 ti = decode5(p, g);
      const int key = key_of(p, ti);
      if (key == key_prev) continue;
      if (reload > 0) {                                 // every MMA reading the previous filter has completed
        mbar_wait(w_free, (reload - 1) & 1);
        tc_fence_after();
      }
      ++reload;
      key_prev = key;
      if (warp == 14 && lane == 0 && wit / P < 8) K5TR(160 + wit / P);
      const int set = key / MAXC5;
      const int row0 = p.cls_r0[ti.cls] + 128 * rank;
      auto issue = [&](int pp) {
        const int u = wit + pp, s = u % p.s_w;
        mbar_wait(&ws_empty[s], ((u / p.s_w) & 1) ^ 1);
        const int pr = (pp + rot) % P;
        const int plane = pr / p.nks, ks = pr % p.nks;
        const size_t base = ((size_t(set) * 2 + plane) * p.nks + ks) * 2;
        uint8_t *dst = wst + size_t(s) * WS_BYTES;
        const uint4 *img = p.wimg + (pair % p.n_rep) * p.rep_stride;
#ifdef K5_ABL_NOW
        mbar_arrive(&ws_full[s]);                       // ablation: no filter copies (results wrong)
        (void)dst;
        (void)img;
        (void)base;
#else
        mbar_arrive_expect_tx(&ws_full[s], WS_BYTES);
        bulk_g2s(dst, img + base * p.RP + row0, 2048, &ws_full[s]);
        bulk_g2s(dst + 2048, img + (base + 1) * p.RP + row0, 2048, &ws_full[s]);
#endif
      };
      if (issuer)
        for (int pp = 0; pp < min(p.s_w, P); ++pp) issue(pp);
      for (int pp = 0; pp < P; ++pp) {
        const int u = wit + pp, s = u % p.s_w;
        mbar_wait(&ws_full[s], (u / p.s_w) & 1);
        const uint4 *st = reinterpret_cast<const uint4 *>(wst + size_t(s) * WS_BYTES);
        const uint4 w0 = st[32 * qq + lane], w1 = st[128 + 32 * qq + lane];
        const int pr = (pp + rot) % P;
        const int plane = pr / p.nks, ks = pr % p.nks;
        if (warp == 14 && lane == 0 && wit == 0 && pp < 24) K5TR(80 + pp);
        __syncwarp();
        tmem_st8(tmem_base + (uint32_t(32 * qq) << 16) + uint32_t(p.a_col0 + plane * 8 * p.nks + 8 * ks), w0, w1);
        __syncwarp();
        if (lane == 0) mbar_arrive(&ws_empty[s]);
        if (issuer && pp + p.s_w < P) issue(pp + p.s_w);
      }
      wit += P;
      __syncwarp();
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (warp == 14 && lane == 0 && wit / P <= 8) K5TR(168 + wit / P - 1);
      if (lane == 0) arrive_leader(w_full, rank);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (tid == 0) {
    K5TR(4);
    K5GT(5);
  }
  if (warp == 13) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc2(tmem_base, 512);
  }
}

// Filter TMEM image: wimg[set][plane][ks][half][row] = 16 bytes = bf16 values of Wr[row][16 ks + 8 half + 0..7]
// (two per 32-bit word, the even K index in the low half), Wr = the real embedding of W (rows 2i / 2i+1, columns
// 2j / 2j+1 as in the header); plane 0 = bf16_rn(v), plane 1 = bf16_rn(v - hi).  Rows >= 2b and K >= 2b are zero.
__global__ void k5_build_wimg(const float2 *__restrict__ W, int b, int nks, int RP, long long rep_stride,
                              uint4 *__restrict__ wimg) {
  const int set = blockIdx.x;
  wimg += blockIdx.z * rep_stride;
  const int seg = blockIdx.y;                 // (plane, ks, half)
  const int half = seg & 1, ks = (seg >> 1) % nks, plane = (seg >> 1) / nks;
  const float2 *Ws = W + size_t(set) * b * b;
  uint4 *dst = wimg + ((size_t(set) * 2 + plane) * nks + ks) * 2 * size_t(RP) + size_t(half) * RP;
  for (int row = threadIdx.x; row < RP; row += blockDim.x) {
    uint32_t wv[4];
    for (int e = 0; e < 4; ++e) {
      float v2[2];
      for (int u = 0; u < 2; ++u) {
        const int k = 16 * ks + 8 * half + 2 * e + u;
        const int i = row >> 1, j = k >> 1;
        float v = 0.f;
        if (row < 2 * b && k < 2 * b) {
          const float2 w = Ws[size_t(i) * b + j];
          const int sel = ((row & 1) << 1) | (k & 1);
          v = sel == 0 ? w.x : sel == 1 ? -w.y : sel == 2 ? w.y : w.x;
        }
        const uint32_t hi2 = pack_bf16(v, 0.f);
        const float hi = bf16_lo_f(hi2);
        const uint32_t lo2 = pack_bf16(v - hi, 0.f);
        v2[u] = __uint_as_float(plane == 0 ? hi2 : lo2);
      }
      wv[e] = (__float_as_uint(v2[0]) & 0xFFFFu) | (__float_as_uint(v2[1]) << 16);
    }
    dst[row] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
  }
}

struct Dev5 {
  bool init = false;
  int num_sms = 0;
  int max_pairs = 0;
};

cudaError_t dev5(Dev5 **out) {
  static Dev5 infos[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  Dev5 &d = infos[dev];
  if (!d.init) {
    e = cudaDeviceGetAttribute(&d.num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k5_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k5_pair, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
    cudaGetLastError();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(d.num_sms / 2 * 2));
    cfg.blockDim = dim3(K5_THREADS);
    cfg.dynamicSmemBytes = SMEM_LIMIT;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k5_pair, &cfg) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    d.max_pairs = n;
    d.init = true;
  }
  *out = &d;
  return cudaSuccess;
}

struct Plan5 {
  int nks, nkc, RP, NP, NB, n_acc, a_col0;
  int s_raw, s_b, s_w, raw_stage, b_stage, xbytes, off_b, off_w, off_e, off_bar, smem, epi_tma;
  std::vector<Win5> win;     // class-sorted
  std::vector<int> cls_start, cls_r0;
};

// Windows with more than 128 kept outputs are split into output sub-windows over the same input (M = 256 real rows
// per pair tile); each piece's kept filter rows [2(o - a), 2(o - a) + 2 kept) pick a row class: R0 = 0 when they
// lie below row 256, else R0 = 2(o - a).  Windows are stably sorted by class.
bool plan5_windows(const ContractArgs &a, Plan5 *pl) {
  if (a.geo_host == nullptr || a.b < 1) return false;
  std::vector<Win5> pieces;
  std::vector<int> r0s;
  for (int w = 0; w < a.n_win; ++w) {
    const Window &g = a.geo_host[w];
    for (int o = g.o; o < g.o_next;) {
      const int kept = std::min(128, g.o_next - o);
      const int lo = 2 * (o - g.a), hi = lo + 2 * kept;
      const int r0 = hi <= 256 ? 0 : lo;
      int c = int(std::find(r0s.begin(), r0s.end(), r0) - r0s.begin());
      if (c == int(r0s.size())) r0s.push_back(r0);
      pieces.push_back(Win5{g.a, o, kept, c});
      o += kept;
    }
  }
  if (int(r0s.size()) > MAXC5) return false;
  pl->win.clear();
  pl->cls_start.assign(r0s.size() + 1, 0);
  for (int c = 0; c < int(r0s.size()); ++c) {
    pl->cls_start[c] = int(pl->win.size());
    for (const Win5 &w5 : pieces)
      if (w5.cls == c) pl->win.push_back(w5);
  }
  pl->cls_start[r0s.size()] = int(pl->win.size());
  pl->cls_r0 = r0s;
  return true;
}

bool plan5(const ContractArgs &a, Plan5 *pl) {
  if (a.geo_host == nullptr || !a.even_starts || a.b < 1) return false;
  pl->nks = (2 * a.b + 15) / 16;
  pl->nkc = (a.b + CK - 1) / CK;
  pl->RP = 2 * a.b + 256;
  const int a_cols = 16 * pl->nks;
  if (a_cols > 512 - 64) return false;
  static const int env_np = getenv("CE_K5_NP") ? atoi(getenv("CE_K5_NP")) : 0;   // experiments
  const int budget = 512 - ((a_cols + 31) & ~31);
  int NP = std::min(256, (budget / 2) / 32 * 32);
  int n_acc = 2;
  if (NP < 64) {
    NP = std::min(256, budget / 32 * 32);
    n_acc = 1;
  }
  if (env_np >= 32 && env_np % 32 == 0 && env_np <= NP) NP = env_np;
  const int cols = a.M * a.K;
  NP = std::min(NP, std::max(32, (cols + 31) & ~31));          // tiny column counts: narrower tiles (multiple of 32)
  pl->NP = NP;
  pl->NB = NP / 2;
  pl->n_acc = n_acc;
  pl->a_col0 = n_acc * NP;
  if (pl->a_col0 + a_cols > 512) return false;
  if (!plan5_windows(a, pl)) return false;
  // shared memory: raw ring | B ring | filter staging | barriers
  pl->xbytes = a.K * CK * 8;
  pl->raw_stage = (pl->NB * 128 + pl->xbytes + 127) & ~127;
  pl->b_stage = pl->NB * 128;
  static const int env_epi = getenv("CE_K5_EPI") ? atoi(getenv("CE_K5_EPI")) : 1;     // experiments
  pl->epi_tma = env_epi != 0;
  const int epi_bytes = pl->epi_tma ? 4 * 2 * 4096 : 0;
  pl->s_b = 6;
  static const int env_raw = getenv("CE_K5_RAW") ? atoi(getenv("CE_K5_RAW")) : 8;     // experiments
  pl->s_raw = std::max(3, std::min(MAX_RAW, env_raw));
  // the filter staging ring takes what is left, up to one whole load (2 nks pieces) in flight; at least 4 pieces
  // (the raw ring gives way)
  auto raw_bytes = [&]() { return ((pl->s_raw * pl->raw_stage) + 1023) & ~1023; };
  const int fixed = 1024 /*align*/ + BAR_BYTES + epi_bytes + pl->s_b * pl->b_stage;
  pl->s_w = std::min({MAX_WS, 2 * pl->nks, (SMEM_LIMIT - fixed - raw_bytes()) / WS_BYTES});
  while (pl->s_w < 4 && pl->s_raw > 3) {
    --pl->s_raw;
    pl->s_w = std::min({MAX_WS, 2 * pl->nks, (SMEM_LIMIT - fixed - raw_bytes()) / WS_BYTES});
  }
  if (pl->s_w < 2) return false;
  pl->off_b = ((pl->s_raw * pl->raw_stage) + 1023) & ~1023;
  pl->off_w = pl->off_b + pl->s_b * pl->b_stage;
  pl->off_e = pl->off_w + pl->s_w * WS_BYTES;
  pl->off_bar = pl->off_e + epi_bytes;
  pl->smem = pl->off_bar + BAR_BYTES + 1024;
  return pl->smem <= SMEM_LIMIT;
}

}  // namespace

#ifdef CE_K4_TRACE
extern "C" int ce_k5_trace_set(void *dptr) { return int(cudaMemcpyToSymbol(g_k5_trace, &dptr, sizeof(dptr))); }
#endif

static size_t wimg_one(int32_t b, int32_t n_sets) {   // uint4 elements of one replica
  const int nks = (2 * b + 15) / 16;
  return size_t(n_sets) * 2 * nks * 2 * (2 * size_t(b) + 256);
}
// replicas of the filter image: up to 16, within 64 MB
int pair_wimg_reps(int32_t b, int32_t n_sets) {
  static const int env = getenv("CE_K5_REPS") ? atoi(getenv("CE_K5_REPS")) : 16;   // experiments
  const size_t one = wimg_one(b, n_sets) * 16;
  int r = std::max(1, std::min(env, int((64u << 20) / std::max<size_t>(one, 1))));
  return std::min(r, 16);
}
size_t pair_wimg_elems(int32_t b, int32_t n_sets) { return wimg_one(b, n_sets) * pair_wimg_reps(b, n_sets); }

bool pair_supported(int32_t b) { return b >= 1 && 16 * ((2 * b + 15) / 16) <= 512 - 64 - 32; }

cudaError_t launch_build_wimg(const float2 *d_W, int32_t b, int32_t n_sets, void *wimg, cudaStream_t stream,
                              int64_t *launches) {
  const int nks = (2 * b + 15) / 16;
  k5_build_wimg<<<dim3(n_sets, 2 * nks * 2, pair_wimg_reps(b, n_sets)), 256, 0, stream>>>(
      d_W, b, nks, 2 * b + 256, (long long)wimg_one(b, n_sets), static_cast<uint4 *>(wimg));
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) ++*launches;
  return e;
}

bool pair_launchable(const ContractArgs &a) {
  Plan5 pl;
  return a.K <= 32 && (a.N % 2) == 0 && (reinterpret_cast<uintptr_t>(a.y) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(a.x) & 15) == 0 && (long long)a.T * a.M * a.K < (1LL << 31) &&
         encode_fn() != nullptr && plan5(a, &pl);
}

bool pair_window_table(const ContractArgs &a, std::vector<uint8_t> *bytes) {
  Plan5 pl;
  if (!plan5_windows(a, &pl)) return false;
  bytes->assign(reinterpret_cast<const uint8_t *>(pl.win.data()),
                reinterpret_cast<const uint8_t *>(pl.win.data()) + pl.win.size() * sizeof(Win5));
  return true;
}

cudaError_t launch_contract_pair(const ContractArgs &a, const void *wimg, const void *win_dev, cudaStream_t stream,
                                 int64_t *launches) {
  if (!pair_launchable(a)) return cudaErrorNotSupported;
  Plan5 pl;
  plan5(a, &pl);
  Dev5 *di = nullptr;
  cudaError_t e = dev5(&di);
  if (e != cudaSuccess) return e;
  if (di->max_pairs < 1) return cudaErrorNotSupported;
  K5Params p = {};
  p.hf = reinterpret_cast<float *>(a.h);
  p.wimg = static_cast<const uint4 *>(wimg);
  p.n_rep = pair_wimg_reps(a.b, a.n_sets);
  p.rep_stride = (long long)wimg_one(a.b, a.n_sets);
  p.soi = a.soi;
  p.T = a.T;
  p.K = a.K;
  p.N = a.N;
  p.b = a.b;
  p.n_sets = a.n_sets;
  p.nks = pl.nks;
  p.nkc = pl.nkc;
  p.RP = pl.RP;
  p.cols = a.M * a.K;
  p.NP = pl.NP;
  p.NB = pl.NB;
  p.n_cb = (p.cols + pl.NP - 1) / pl.NP;
  p.n_acc = pl.n_acc;
  p.a_col0 = pl.a_col0;
  p.n_win = int(pl.win.size());
  p.n_cls = int(pl.cls_r0.size());
  const long long tiles = (long long)a.T * p.n_win * p.n_cb;
  if (tiles > 0x7fffffffLL || tiles < 1) return cudaErrorInvalidConfiguration;
  p.n_tiles = int(tiles);
  p.s_raw = pl.s_raw;
  p.s_b = pl.s_b;
  p.s_w = pl.s_w;
  p.raw_stage = pl.raw_stage;
  p.b_stage = pl.b_stage;
  p.xbytes = pl.xbytes;
  p.off_b = pl.off_b;
  p.off_w = pl.off_w;
  p.off_e = pl.off_e;
  p.off_bar = pl.off_bar;
  for (int c = 0; c <= p.n_cls; ++c) p.cls_start[c] = pl.cls_start[c];
  for (int c = 0; c < p.n_cls; ++c) p.cls_r0[c] = pl.cls_r0[c];
  for (int w = 0; w < MAXW5; ++w) p.win[w] = w < p.n_win ? pl.win[w] : Win5{0, 0, 0, 0};
  // long tables: the handle's device copy of the same class-sorted table (pair_window_table at ce_init)
  p.win_d = static_cast<const Win5 *>(win_dev);
  if (p.n_win > MAXW5 && win_dev == nullptr) return cudaErrorInvalidValue;
  CUtensorMap tmy, tmx, tmh = {};
  if (!cached_map(&tmy, a.y, a.N, (long long)a.T * p.cols, pl.NB) ||
      !cached_map(&tmx, a.x, a.N, (long long)a.T * a.K, a.K))
    return cudaErrorInvalidValue;
  p.epi_tma = pl.epi_tma && (reinterpret_cast<uintptr_t>(a.h) & 15) == 0;
  if (p.epi_tma && !cached_map(&tmh, a.h, a.N, (long long)a.T * p.cols, 32)) return cudaErrorInvalidValue;
  static const int env_pairs = getenv("CE_K5_PAIRS") ? atoi(getenv("CE_K5_PAIRS")) : 0;   // experiments / tests
  long long n_pairs = std::min<long long>(tiles, di->max_pairs);
  if (env_pairs > 0) n_pairs = std::min<long long>(n_pairs, env_pairs);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(2 * n_pairs));
  cfg.blockDim = dim3(K5_THREADS);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = 2;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  e = cudaLaunchKernelEx(&cfg, k5_pair, tmy, tmx, tmh, p);
  if (e == cudaSuccess) ++*launches;
  return e;
}

}  // namespace ce
