// K5 -- fused LS + block-LMMSE contraction on a CTA PAIR (tcgen05 cta_group::2, M = 256) with the filter
// operand RESIDENT in shared memory.  Same arithmetic as K4 (BF16x3 error-compensated products, FP32
// accumulation in TMEM; reading B1) and the same complex -> real embedding:
//   D[c][2i + q] = sum_k A_r[c][k] B_r^T[2i + q][k],  A_r = interleaved LS row (Eq. 9),
//   B_r^T rows 2i / 2i+1 = (Re W_ij, -Im W_ij) / (Im W_ij, Re W_ij)  (W of PAPER.md:306-309, Eq. 17),
// applied per window as in Eq. 12 with the 12W edge clamping.
//
// Why: per 16 complex of y (16 KB) a K4 tile streams 32 KB of filter planes through shared memory; the
// filter re-reads, not the y/h traffic, set K4's pace (measured: 1.5x faster with them removed).  Here
// the two CTAs of a pair each own 128 A rows (two column blocks of the same (t, w)) and HALF of the
// filter's N rows; the pair MMA reads B from both CTAs.  With the half-bank resident (loaded once per
// (set, window row range) -- once per launch for the paper's single fixed design), shared memory holds
// only the y stream: a unified ring where each stage's raw y box is converted IN PLACE into the bf16
// hi/lo A tiles.
//
// Roles (each CTA of the pair, 480 threads):
//   warp 12   : raw producer -- 2D TMA y box [128 rows x 16 complex] + pilot box [K x 16] per K chunk
//   warps 0-7 : transform -- LS factors in place (x area), then y -> registers, named barrier, bf16
//               hi/lo A tiles written over the y area (SWIZZLE_64B K-major); arrive a_full
//   warp 14   : B producer -- loads this CTA's half of the bank for the current (set, n0, nw) key into
//               the resident region (per-chunk b_full barriers); reloads only when the key changes,
//               after every earlier tile's MMAs completed (tiles_done counter kept by the epilogue)
//   warp 13   : leader: TMEM alloc (pair) + MMA issuer (waits own a_full, peer_ready, b_full);
//               follower: forwards "my A and B of this stage are ready" to the leader (remote arrive)
//   warps 8-11: epilogue -- tcgen05.ld 16x256b of this CTA's 128 accumulator lanes, direct stores;
//               one arrival per warp on the leader's tmem_empty
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ce_internal.h"
#include "tc_ptx.cuh"
#include "tmap.cuh"

namespace ce {
namespace {

#ifdef CE_K4_TRACE
__device__ unsigned long long *g_k5_trace;
#define K5TR(slot)                                                             \
  do {                                                                         \
    if (g_k5_trace) g_k5_trace[size_t(blockIdx.x) * 256 + (slot)] = clock64(); \
  } while (0)
#else
#define K5TR(slot) \
  do {             \
  } while (0)
#endif

constexpr int K5_THREADS = 480;
constexpr int NTR = 256;                   // transform threads
constexpr int CK = 16;                     // complex per K chunk (64-byte bf16 rows)
constexpr int TM = 128;                    // A rows per CTA
constexpr int NMAXW = 256;                 // MMA N max
constexpr int RAWY = TM * CK * 8;          // 16 KB: raw y box, later A_hi (8 KB) | A_lo (8 KB)
constexpr int A_PLANE = TM * 64;
constexpr int MAXW_PARAM = 32;
constexpr int MAX_STAGES = 8;
constexpr int MAX_NKC = 24;                // b <= 376
constexpr int SMEM_LIMIT = 232448;         // sm_100 opt-in maximum per CTA
constexpr int BAR_REGION = 1024;

struct K5Params {
  float2 *h;
  const uint16_t *bank_hi;   // bf16 [n_sets][nkc][NR][32] SW64 images
  const uint16_t *bank_lo;
  const Window *geo;         // device window table (n_win > MAXW_PARAM)
  const int32_t *soi;
  int T, K, N, b, n_win, n_sets, nkc, NR, cols, n_ct;
  int n_ctg;                 // column-block pairs per (t, w)
  int n_groups;              // T * n_win * n_ctg
  int nrh;                   // resident rows per CTA (max over windows of nw / 2)
  int stages;                // ring stages
  int stage_bytes;           // RAWY + x area
  int b_bytes;               // resident bank half: nkc * 2 * nrh * 64
  Window geo_s[MAXW_PARAM];
};

struct Tile5 {
  int t, w, ct, a, o, kept, n0, off, nw;
};

__device__ __forceinline__ Tile5 decode5(const K5Params &p, int g, int rank) {
  Tile5 ti;
  const int ctg = g % p.n_ctg;
  const int rest = g / p.n_ctg;
  ti.w = rest % p.n_win;
  ti.t = rest / p.n_win;
  ti.ct = 2 * ctg + rank;
  const Window gw = p.n_win <= MAXW_PARAM ? p.geo_s[ti.w] : p.geo[ti.w];
  ti.a = gw.a;
  ti.o = gw.o;
  ti.kept = gw.o_next - gw.o;
  const int row2 = 2 * (gw.o - gw.a);
  ti.n0 = row2 & ~7;
  ti.off = row2 - ti.n0;
  ti.nw = (ti.off + 2 * ti.kept + 15) & ~15;
  return ti;
}

__device__ __forceinline__ int raw_set(const K5Params &p, int t) { return p.soi ? p.soi[t] : 0; }

// resident-bank key of a tile: the bank rows it needs depend on (set, n0, nw)
__device__ __forceinline__ long long bkey(const K5Params &p, const Tile5 &ti) {
  const int s = raw_set(p, ti.t);
  const int sc = (s >= 0 && s < p.n_sets) ? s : 0;
  return ((long long)sc << 32) | ((long long)ti.n0 << 16) | ti.nw;
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

// this pair's contiguous range of groups [g_lo, g_hi): consecutive groups share (t, w), so the resident
// bank is reloaded only at set / window-type changes
__device__ __forceinline__ void unit_range(const K5Params &p, int unit, int n_units, int *g_lo, int *g_hi) {
  const long long G = p.n_groups;
  *g_lo = int(G * unit / n_units);
  *g_hi = int(G * (unit + 1) / n_units);
}

__global__ void __launch_bounds__(K5_THREADS, 1)
    k5_pair(const __grid_constant__ CUtensorMap tmy, const __grid_constant__ CUtensorMap tmx,
            const __grid_constant__ K5Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *bres = smem;                                  // [nkc][hi | lo][nrh rows][64 B]
  uint8_t *ring = smem + p.b_bytes;                      // [stages][y/A 16 KB | x]
  uint64_t *bars = reinterpret_cast<uint64_t *>(ring + size_t(p.stages) * p.stage_bytes);
  uint64_t *ring_full = bars;                            // [MAX_STAGES] TMA y + x landed
  uint64_t *ring_empty = ring_full + MAX_STAGES;         // [MAX_STAGES] pair MMAs done with the stage
  uint64_t *a_full = ring_empty + MAX_STAGES;            // [MAX_STAGES] local A tiles written
  uint64_t *peer_ready = a_full + MAX_STAGES;            // [MAX_STAGES] (leader) follower's stage ready
  uint64_t *b_full = peer_ready + MAX_STAGES;            // [MAX_NKC]    resident chunk kc loaded
  uint64_t *tmem_full = b_full + MAX_NKC;                // [2]
  uint64_t *tmem_empty = tmem_full + 2;                  // [2] 8 arrivals: 4 epilogue warps x 2 CTAs
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_empty + 2);
  volatile int *tiles_done = reinterpret_cast<volatile int *>(tmem_slot + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = int(cluster_ctarank());
  const int unit = blockIdx.x >> 1, n_units = gridDim.x >> 1;
  int g_lo, g_hi;
  unit_range(p, unit, n_units, &g_lo, &g_hi);
  const int S = p.stages;
#ifdef CE_K4_TRACE
  if (tid == 0 && g_k5_trace) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    g_k5_trace[size_t(blockIdx.x) * 256 + 0] = gt;
  }
#endif
  if (tid == 0) {
    K5TR(1);
    for (int s = 0; s < MAX_STAGES; ++s) {
      mbar_init(&ring_full[s], 1);
      mbar_init(&ring_empty[s], 1);
      mbar_init(&a_full[s], NTR);
      mbar_init(&peer_ready[s], 1);
    }
    for (int k = 0; k < MAX_NKC; ++k) mbar_init(&b_full[k], 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&tmem_empty[i], 8);
    }
    *tiles_done = 0;
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
  pdl_wait();
  const int nks_total = (2 * p.b + 15) / 16;

  if (warp == 12) {
    // ------------------------------------------------------------------ raw producer
    if (lane == 0) {
      const uint32_t xbytes = uint32_t(p.K) * CK * 8;
      int it = 0;
      for (int g = g_lo; g < g_hi; ++g) {
        const Tile5 ti = decode5(p, g, rank);
        const int row0 = ti.t * p.cols + ti.ct * TM;
        for (int kc = 0; kc < p.nkc; ++kc, ++it) {
          const int s = it % S;
          mbar_wait(&ring_empty[s], ((it / S) & 1) ^ 1);
          mbar_arrive_expect_tx(&ring_full[s], RAWY + xbytes);
          if (it < 24) K5TR(8 + it);
          uint8_t *st = ring + size_t(s) * p.stage_bytes;
          const int f0 = 2 * (ti.a + kc * CK);
          tma_load_2d(st, &tmy, f0, row0, &ring_full[s]);
          tma_load_2d(st + RAWY, &tmx, f0, ti.t * p.K, &ring_full[s]);
        }
      }
      // drain: the leader's commits for the last use of every stage have arrived before teardown
      for (int i = 0; i < S; ++i, ++it) mbar_wait(&ring_empty[it % S], ((it / S) & 1) ^ 1);
    }
  } else if (warp < 8) {
    // ------------------------------------------------------------------ transform (in place)
    const int jp = tid & 7;
    const int rb = tid >> 3;
    int it = 0;
    for (int g = g_lo; g < g_hi; ++g) {
      const Tile5 ti = decode5(p, g, rank);
      const int c_first = ti.ct * TM + rb;
      const int x_first = c_first % p.K;
      const int x_step = 32 % p.K;
      for (int kc = 0; kc < p.nkc; ++kc, ++it) {
        const int s = it % S;
        mbar_wait(&ring_full[s], (it / S) & 1);
        if (tid == 0 && it < 24) K5TR(32 + it);
        uint8_t *st = ring + size_t(s) * p.stage_bytes;
        const float4 *ry = reinterpret_cast<const float4 *>(st);
        float4 *rx = reinterpret_cast<float4 *>(st + RAWY);
        if (tid < p.K * 8) {
          const float4 xv = rx[tid];
          const float i0 = rcp_approx(xv.x * xv.x + xv.y * xv.y);
          const float i1 = rcp_approx(xv.z * xv.z + xv.w * xv.w);
          const bool ok0 = kc * CK + 2 * (tid & 7) < p.b, ok1 = kc * CK + 2 * (tid & 7) + 1 < p.b;
          rx[tid] = make_float4(ok0 ? xv.x * i0 : 0.f, ok0 ? -xv.y * i0 : 0.f, ok1 ? xv.z * i1 : 0.f,
                                ok1 ? -xv.w * i1 : 0.f);
        }
        named_bar_sync(1, NTR);
        uint32_t hv[4][2], lv[4][2];
        int xr = x_first;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = rb + 32 * i;
          const float4 yv = ry[r * 8 + jp];
          const float4 fv = rx[xr * 8 + jp];
          const float l0r = yv.x * fv.x - yv.y * fv.y, l0i = yv.x * fv.y + yv.y * fv.x;
          const float l1r = yv.z * fv.z - yv.w * fv.w, l1i = yv.z * fv.w + yv.w * fv.z;
          hv[i][0] = pack_bf16(l0r, l0i);
          hv[i][1] = pack_bf16(l1r, l1i);
          lv[i][0] = pack_bf16(l0r - bf16_lo_f(hv[i][0]), l0i - bf16_hi_f(hv[i][0]));
          lv[i][1] = pack_bf16(l1r - bf16_lo_f(hv[i][1]), l1i - bf16_hi_f(hv[i][1]));
          xr += x_step;
          if (xr >= p.K) xr -= p.K;
        }
        named_bar_sync(2, NTR);                          // every thread has read the raw y of this stage
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = rb + 32 * i;
          const int off = r * 64 + ((((jp >> 1) ^ ((r >> 1) & 3))) << 4) + ((jp & 1) << 3);
          *reinterpret_cast<uint2 *>(st + off) = make_uint2(hv[i][0], hv[i][1]);
          *reinterpret_cast<uint2 *>(st + A_PLANE + off) = make_uint2(lv[i][0], lv[i][1]);
        }
        fence_proxy_async();
        if (tid == 0 && it < 24) K5TR(56 + it);
        mbar_arrive(&a_full[s]);
      }
    }
  } else if (warp < 12) {
    // ------------------------------------------------------------------ epilogue
    const int q = warp & 3;
    const int rA = lane >> 2, cq = lane & 3;
    int lt = 0;
    for (int g = g_lo; g < g_hi; ++g, ++lt) {
      const Tile5 ti = decode5(p, g, rank);
      const int s_raw = raw_set(p, ti.t);
      const bool set_ok = s_raw >= 0 && s_raw < p.n_sets;
      const int acc = lt & 1;
      mbar_wait(&tmem_full[acc], (lt >> 1) & 1);
      tc_fence_after();
      if (tid == 256 && lt < 8) K5TR(136 + lt);
      if (tid == 256) *tiles_done = lt + 1;              // every MMA of tiles 0..lt has completed
      const int nf = 2 * ti.kept;
      const int ncb = (ti.off + nf + 31) / 32;
      const int c0 = ti.ct * TM + q * 32 + rA;
      float2 *hrow = p.h + (size_t(ti.t) * p.cols + c0) * p.N + ti.o;
      const size_t row8 = size_t(8) * p.N;
      const float qnan = __int_as_float(0x7fc00000);
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
            const int ci = f >> 1;
            float2 a0 = make_float2(__uint_as_float(v0[4 * m]), __uint_as_float(v0[4 * m + 1]));
            float2 a1 = make_float2(__uint_as_float(v0[4 * m + 2]), __uint_as_float(v0[4 * m + 3]));
            float2 a2 = make_float2(__uint_as_float(v1[4 * m]), __uint_as_float(v1[4 * m + 1]));
            float2 a3 = make_float2(__uint_as_float(v1[4 * m + 2]), __uint_as_float(v1[4 * m + 3]));
            if (!set_ok) a0 = a1 = a2 = a3 = make_float2(qnan, qnan);
            if (c0 < p.cols) hrow[ci] = a0;
            if (c0 + 8 < p.cols) hrow[row8 + ci] = a1;
            if (c0 + 16 < p.cols) hrow[2 * row8 + ci] = a2;
            if (c0 + 24 < p.cols) hrow[3 * row8 + ci] = a3;
          }
        }
      }
      __syncwarp();
      if (tid == 256 && lt < 8) K5TR(144 + lt);
      if (lane == 0) {
        tc_fence_before();
        if (rank == 0)
          mbar_arrive(&tmem_empty[acc]);
        else
          mbar_arrive_remote(&tmem_empty[acc], 0);
      }
    }
  } else if (warp == 14) {
    // ------------------------------------------------------------------ resident bank producer
    if (lane == 0) {
      long long cur = -1;
      int epoch = 0, lt = 0;
      for (int g = g_lo; g < g_hi; ++g, ++lt) {
        const Tile5 ti = decode5(p, g, rank);
        const long long key = bkey(p, ti);
        if (key == cur) continue;
        // every earlier tile's MMAs (which read the resident bank) must be complete before overwriting it
        while (*tiles_done < lt) {
        }
        cur = key;
        ++epoch;
        const int set = int(key >> 32);
        const int rows = ti.nw / 2;
        const uint32_t bytes = uint32_t(rows) * 64;
        for (int kc = 0; kc < p.nkc; ++kc) {
          mbar_arrive_expect_tx(&b_full[kc], 2 * bytes);
          const size_t src = ((size_t(set) * p.nkc + kc) * p.NR + ti.n0 + rank * rows) * 32;
          uint8_t *dst = bres + size_t(kc) * 2 * p.nrh * 64;
          bulk_g2s(dst, p.bank_hi + src, bytes, &b_full[kc]);
          bulk_g2s(dst + size_t(p.nrh) * 64, p.bank_lo + src, bytes, &b_full[kc]);
        }
      }
    }
  } else {
    // ------------------------------------------------------------------ MMA issuer (leader) / forwarder
    if (lane == 0) {
      long long cur = -1;
      int epoch = 0;
      int it = 0, lt = 0;
      for (int g = g_lo; g < g_hi; ++g, ++lt) {
        const Tile5 ti = decode5(p, g, rank);
        const long long key = bkey(p, ti);
        if (key != cur) {
          cur = key;
          ++epoch;
        }
        const uint32_t bph = uint32_t(epoch - 1) & 1;
        if (rank == 1) {
          for (int kc = 0; kc < p.nkc; ++kc, ++it) {
            const int s = it % S;
            mbar_wait(&a_full[s], (it / S) & 1);
            mbar_wait(&b_full[kc], bph);
            if (it < 24) K5TR(80 + it);
            mbar_arrive_remote(&peer_ready[s], 0);
          }
          continue;
        }
        const int acc = lt & 1;
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(ti.nw >> 3) << 17) |
                               (uint32_t(256 >> 4) << 24);
        mbar_wait_cluster(&tmem_empty[acc], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + uint32_t(acc * NMAXW);
        for (int kc = 0; kc < p.nkc; ++kc, ++it) {
          const int s = it % S;
          const uint32_t ph = (it / S) & 1;
          mbar_wait(&a_full[s], ph);
          if (it < 24) K5TR(152 + it);
          mbar_wait(&b_full[kc], bph);
          if (it < 24) K5TR(176 + it);
          mbar_wait_cluster(&peer_ready[s], ph);
          tc_fence_after();
          if (it < 24) K5TR(104 + it);
          uint8_t *st = ring + size_t(s) * p.stage_bytes;
          uint8_t *bb = bres + size_t(kc) * 2 * p.nrh * 64;
          const uint64_t ah = sw64_desc(smem_u32(st));
          const uint64_t al = sw64_desc(smem_u32(st + A_PLANE));
          const uint64_t bh = sw64_desc(smem_u32(bb));
          const uint64_t bl = sw64_desc(smem_u32(bb + size_t(p.nrh) * 64));
          const int nks = min(2, nks_total - 2 * kc);
          for (int ks = 0; ks < nks; ++ks) {
            const uint64_t adv = uint64_t(2 * ks);
            mma_bf16_pair(d, ah + adv, bh + adv, idesc, (kc | ks) != 0);
            mma_bf16_pair(d, ah + adv, bl + adv, idesc, 1u);
            mma_bf16_pair(d, al + adv, bh + adv, idesc, 1u);
          }
          mma_commit_pair(&ring_empty[s]);
        }
        mma_commit_pair(&tmem_full[acc]);
        if (lt < 8) K5TR(128 + lt);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 13) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc2(tmem_base, 512);
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

// Shared-memory plan: resident half bank + as many ring stages as fit (>= 3), or false.
bool plan5(const ContractArgs &a, int *nrh, int *b_bytes, int *stage_bytes, int *stages) {
  int32_t nkc, NR;
  bf16x3_bank_shape(a.b, &nkc, &NR);
  if (nkc > MAX_NKC || a.geo_host == nullptr) return false;
  int nw_max = 0;
  for (int w = 0; w < a.n_win; ++w) {
    const Window &g = a.geo_host[w];
    const int row2 = 2 * (g.o - g.a), off = row2 - (row2 & ~7);
    const int nw = (off + 2 * (g.o_next - g.o) + 15) & ~15;
    if (nw > NMAXW) return false;
    nw_max = nw > nw_max ? nw : nw_max;
  }
  *nrh = nw_max / 2;
  *b_bytes = nkc * 2 * (*nrh) * 64;
  *stage_bytes = RAWY + ((a.K * CK * 8 + 1023) & ~1023);
  const int avail = SMEM_LIMIT - 1024 /*align*/ - BAR_REGION - *b_bytes;
  int s = avail / *stage_bytes;
  if (s > MAX_STAGES) s = MAX_STAGES;
  *stages = s;
  return s >= 3;
}

}  // namespace

#ifdef CE_K4_TRACE
extern "C" int ce_k5_trace_set(void *dptr) { return int(cudaMemcpyToSymbol(g_k5_trace, &dptr, sizeof(dptr))); }
#endif

bool pair_launchable(const ContractArgs &a) {
  int nrh, bb, sb, st;
  return bf16x3_launchable(a) && plan5(a, &nrh, &bb, &sb, &st);
}

cudaError_t launch_contract_pair(const ContractArgs &a, const uint16_t *bank_hi, const uint16_t *bank_lo,
                                 cudaStream_t stream, int64_t *launches) {
  K5Params p;
  if (!bf16x3_launchable(a) || !plan5(a, &p.nrh, &p.b_bytes, &p.stage_bytes, &p.stages))
    return cudaErrorNotSupported;
  Dev5 *di = nullptr;
  cudaError_t e = dev5(&di);
  if (e != cudaSuccess) return e;
  if (di->max_pairs < 1) return cudaErrorNotSupported;
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
  p.cols = a.M * a.K;
  p.n_ct = (p.cols + TM - 1) / TM;
  p.n_ctg = (p.n_ct + 1) / 2;
  for (int w = 0; w < MAXW_PARAM; ++w) p.geo_s[w] = w < a.n_win ? a.geo_host[w] : Window{0, 0, 0};
  const long long groups = (long long)a.T * a.n_win * p.n_ctg;
  if (groups > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  p.n_groups = int(groups);
  CUtensorMap tmy, tmx;
  if (!cached_map(&tmy, a.y, a.N, (long long)a.T * p.cols, TM) ||
      !cached_map(&tmx, a.x, a.N, (long long)a.T * a.K, a.K))
    return cudaErrorInvalidValue;
  const int n_units = int(groups < di->max_pairs ? groups : di->max_pairs);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(2 * n_units));
  cfg.blockDim = dim3(K5_THREADS);
  cfg.dynamicSmemBytes = SMEM_LIMIT;
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
  e = cudaLaunchKernelEx(&cfg, k5_pair, tmy, tmx, p);
  if (e == cudaSuccess) ++*launches;
  return e;
}

}  // namespace ce
