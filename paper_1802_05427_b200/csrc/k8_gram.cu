// K8 -- the lag correlation of the statistics estimator (NEXT-3, reading D1) on tcgen05 tensor cores:
//   S[d] = sum_c sum_n conj(H_LS[c, n]) H_LS[c, n + d],   0 <= d < D,
// summed over the columns c = (t, m, k) of a statistic set (K7b divides by C (N - d)).  This is the band
// 0 <= n' - n < D of the Gram matrix G = H^H H of the set's LS rows (H_LS = y / x, Eq. 9), read
// along its diagonals.
//
// Tiling: tone tiles of 128.  A unit is (instance t, tile pair (i, j) with 0 <= j - i < JJ, a range of the
// instance's columns).  Its product is one real GEMM tile: M = the 128 tones n of tile i, N = 256 = the 128 tones
// n' of tile j embedded as rows (b_re, b_im) / (b_im, -b_re), K = 2 x the unit's columns:
//   D[n][2n'] = sum_c Re(conj(a) b),  D[n][2n' + 1] = sum_c Im(conj(a) b),   a = H_LS[c, n], b = H_LS[c, n'],
// with K4's BF16x3 error compensation (A_hi B_hi + A_hi B_lo + A_lo B_hi, FP32 accumulation in TMEM).  The
// epilogue adds every element with 0 <= d = n' - n < D into per-CTA shared bins, then the bins into the set's
// FP64 accumulator (K7's layout: K7 adds the noise floor and the column count, K7b normalises).
//
// Roles (persistent CTAs, 448 threads):
//   warp 12   : TMA of the raw y boxes [16 antennas of one user][128 tones] of tiles i and j (4-D map, so a
//               chunk's columns share one user and one LS factor per tone) into a 2-deep raw ring
//   warps 0-7 : transform -- per unit the LS factors conj(x)/|x|^2 of tiles i and j for every user; per
//               16-column chunk the LS values transposed into the K-major A tile (row n: the chunk's 16 columns)
//               and B tile (rows 2n', 2n'+1), bf16 hi/lo, SWIZZLE_64B, 2-deep A/B ring
//   warp 13   : TMEM (2 x 256 columns) + MMA issuer: 2 K steps x 3 MMAs per chunk
//   warps 8-11: epilogue -- tcgen05.ld 32x32b (thread = tone n of tile i), diagonal bins, FP64 atomics
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <vector>

#include "ce_internal.h"
#include "tc_ptx.cuh"
#include "tmap.cuh"

namespace ce {
namespace {

constexpr int K8_THREADS = 448;
constexpr int NTR8 = 256;                 // transform threads
constexpr int TT = 128;                   // tones per tile
constexpr int CC8 = 16;                   // columns per chunk (K = 32 real)
constexpr int RAW_TILE = CC8 * TT * 8;    // 16 KB: [16 columns][128 complex]
constexpr int RAW8 = 2 * RAW_TILE;        // tiles i and j
constexpr int S_RAW8 = 2;
constexpr int A8_PLANE = TT * 64;         // [128 rows][32 bf16]
constexpr int B8_PLANE = 2 * TT * 64;     // [256 rows][32 bf16]
constexpr int AB8 = 2 * A8_PLANE + 2 * B8_PLANE;   // 48 KB
constexpr int S_AB8 = 2;
constexpr int KMAX8 = 24;                 // users (LS-factor table rows)
constexpr int MAXP8 = 160;                // tile pairs carried in the parameters
constexpr int DMAX8 = 512;                // lags (bins) per launch
constexpr int K8_SMEM = 1024 + S_AB8 * AB8 + S_RAW8 * RAW8 + 2 * KMAX8 * TT * 8 + 2 * DMAX8 * 4 + 256;
static_assert(K8_SMEM <= 232448, "K8 shared memory");

struct K8Params {
  const int32_t *soi;
  const float2 *x;
  double *acc;                            // [n_sets][2D + 2]
  int T, M, K, N, D, n_sets;
  int nmc;                                // 16-antenna chunks per user: chunk q of an instance = (k = q / nmc, m0 = 16 (q % nmc))
  int n_pairs, n_cc, cq, n_units;         // units = T x n_cc x n_pairs (pair fastest), cq chunks per unit
  short2 pairs[MAXP8];                    // (i, j) tone tiles
};

struct Unit8 {
  int t, q0, q1, i, j;
};

__device__ __forceinline__ Unit8 decode8(const K8Params &p, int u) {
  Unit8 un;
  const int pr = u % p.n_pairs;
  const int rest = u / p.n_pairs;
  const int cc = rest % p.n_cc;
  un.t = rest / p.n_cc;
  un.q0 = cc * p.cq;
  un.q1 = min(p.K * p.nmc, un.q0 + p.cq);
  un.i = p.pairs[pr].x;
  un.j = p.pairs[pr].y;
  return un;
}

__device__ __forceinline__ uint32_t pk_bf16(float lo_addr, float hi_addr) {   // lo_addr -> low 16 bits
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi_addr), "f"(lo_addr));
  return r;
}
__device__ __forceinline__ float lo_f(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float hi_f(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }
// (hi, lo) bf16x2 words of the pair (e0 at the lower address, e1)
__device__ __forceinline__ void split2(float e0, float e1, uint32_t &h, uint32_t &l) {
  h = pk_bf16(e0, e1);
  l = pk_bf16(e0 - lo_f(h), e1 - hi_f(h));
}
__device__ __forceinline__ void tmem_ld32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,"
      "%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// SWIZZLE_64B K-major tile: row r at r*64 bytes, 16-byte chunk c (of 4) stored at (c ^ ((r >> 1) & 3)) * 16
__device__ __forceinline__ int sw64_off(int r, int c) { return r * 64 + ((c ^ ((r >> 1) & 3)) << 4); }

__global__ void __launch_bounds__(K8_THREADS, 1)
    k8_gram(const __grid_constant__ CUtensorMap tmy, const __grid_constant__ K8Params p) {
  extern __shared__ uint8_t smem_raw8[];
  uint8_t *smem = smem_raw8 + ((1024u - (smem_u32(smem_raw8) & 1023u)) & 1023u);
  uint8_t *ab = smem;                                        // [S_AB8][A_hi | A_lo | B_hi | B_lo]
  uint8_t *raw = ab + S_AB8 * AB8;                           // [S_RAW8][tile i | tile j]
  float2 *fac = reinterpret_cast<float2 *>(raw + S_RAW8 * RAW8);   // [2 tiles][K][128] LS factors
  float *bins = reinterpret_cast<float *>(fac + 2 * KMAX8 * TT);   // [2 D]
  uint64_t *bars = reinterpret_cast<uint64_t *>(bins + 2 * DMAX8);
  uint64_t *raw_full = bars, *raw_empty = bars + S_RAW8;
  uint64_t *a_full = bars + 2 * S_RAW8, *st_empty = a_full + S_AB8;
  uint64_t *tmem_full = st_empty + S_AB8, *tmem_empty = tmem_full + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_empty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < S_RAW8; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_empty[s], NTR8);
    }
    for (int s = 0; s < S_AB8; ++s) {
      mbar_init(&a_full[s], NTR8);
      mbar_init(&st_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&tmem_empty[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int q = tid; q < 2 * DMAX8; q += K8_THREADS) bins[q] = 0.f;
  if (warp == 12 && lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmy)) : "memory");
  if (warp == 13) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 12) {
    // ------------------------------------------------------------------ raw producer (TMA)
    if (lane == 0) {
      int it = 0;
      for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
        const Unit8 un = decode8(p, u);
        for (int q = un.q0; q < un.q1; ++q, ++it) {
          const int s = it % S_RAW8;
          mbar_wait(&raw_empty[s], ((it / S_RAW8) & 1) ^ 1);
          mbar_arrive_expect_tx(&raw_full[s], RAW8);
          // 16 antennas m0.. of user k (rows beyond M are zero-filled: zero LS values)
          const int k = q / p.nmc, m0 = CC8 * (q % p.nmc);
          tma_load_4d(raw + s * RAW8, &tmy, 2 * TT * un.i, k, m0, un.t, &raw_full[s]);
          tma_load_4d(raw + s * RAW8 + RAW_TILE, &tmy, 2 * TT * un.j, k, m0, un.t, &raw_full[s]);
        }
      }
    }
  } else if (warp < 8) {
    // ------------------------------------------------------------------ transform
    const int n = tid & (TT - 1), hc = tid >> 7;     // tone n of both tiles; columns 8 hc .. 8 hc + 7 of a chunk
    int it = 0;
    for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
      const Unit8 un = decode8(p, u);
      // LS factors of this instance, tiles i and j, every user.  The barrier keeps the previous unit's chunks
      // (transformed by these same threads) from reading a factor that is being overwritten.
      named_bar_sync(1, NTR8);
      for (int e = tid; e < 2 * p.K * TT; e += NTR8) {
        const int tile = e / (p.K * TT), k = (e / TT) % p.K, nn = e % TT;
        const int tone = TT * (tile ? un.j : un.i) + nn;
        float2 f = make_float2(0.f, 0.f);
        if (tone < p.N) {
          const float2 xv = p.x[(size_t(un.t) * p.K + k) * p.N + tone];
          const float inv = 1.0f / (xv.x * xv.x + xv.y * xv.y);
          f = make_float2(xv.x * inv, -xv.y * inv);
        }
        fac[e] = f;
      }
      named_bar_sync(1, NTR8);
      for (int q = un.q0; q < un.q1; ++q, ++it) {
        const int sr = it % S_RAW8, sa = it % S_AB8;
        // every column of the chunk belongs to user k: one pair of LS factors per thread and chunk
        const int k = q / p.nmc;
        const float2 fi = fac[k * TT + n], fj = fac[(p.K + k) * TT + n];
        mbar_wait(&raw_full[sr], (it / S_RAW8) & 1);
        const float2 *ri = reinterpret_cast<const float2 *>(raw + sr * RAW8);
        const float2 *rj = reinterpret_cast<const float2 *>(raw + sr * RAW8 + RAW_TILE);
        // 8 columns -> 8 words per row and plane: A row n, B rows 2n (b_re, b_im) and 2n+1 (b_im, -b_re)
        uint32_t ah[8], al[8], b0h[8], b0l[8], b1h[8], b1l[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int cl = 8 * hc + e;
          const float2 yi = ri[cl * TT + n], yj = rj[cl * TT + n];
          const float2 a = make_float2(yi.x * fi.x - yi.y * fi.y, yi.x * fi.y + yi.y * fi.x);
          const float2 b = make_float2(yj.x * fj.x - yj.y * fj.y, yj.x * fj.y + yj.y * fj.x);
          split2(a.x, a.y, ah[e], al[e]);
          split2(b.x, b.y, b0h[e], b0l[e]);
          split2(b.y, -b.x, b1h[e], b1l[e]);
        }
        mbar_arrive(&raw_empty[sr]);
        mbar_wait(&st_empty[sa], ((it / S_AB8) & 1) ^ 1);
        uint8_t *st = ab + sa * AB8;
        uint8_t *pah = st, *pal = st + A8_PLANE, *pbh = st + 2 * A8_PLANE, *pbl = pbh + B8_PLANE;
#pragma unroll
        for (int h = 0; h < 2; ++h) {                  // 16-byte chunks 2 hc + h of the 64-byte rows
          const int ch = 2 * hc + h;
          *reinterpret_cast<uint4 *>(pah + sw64_off(n, ch)) = make_uint4(ah[4 * h], ah[4 * h + 1], ah[4 * h + 2], ah[4 * h + 3]);
          *reinterpret_cast<uint4 *>(pal + sw64_off(n, ch)) = make_uint4(al[4 * h], al[4 * h + 1], al[4 * h + 2], al[4 * h + 3]);
          // rows 2n and 2n+1: lanes with n & 4 store the odd row first, so each quarter-warp's 16-byte stores
          // cover both 64-byte halves of the 128-byte bank window (all rows 2n sit in the lower half)
          const uint4 e0h = make_uint4(b0h[4 * h], b0h[4 * h + 1], b0h[4 * h + 2], b0h[4 * h + 3]);
          const uint4 e0l = make_uint4(b0l[4 * h], b0l[4 * h + 1], b0l[4 * h + 2], b0l[4 * h + 3]);
          const uint4 e1h = make_uint4(b1h[4 * h], b1h[4 * h + 1], b1h[4 * h + 2], b1h[4 * h + 3]);
          const uint4 e1l = make_uint4(b1l[4 * h], b1l[4 * h + 1], b1l[4 * h + 2], b1l[4 * h + 3]);
          const bool sw = (n & 4) != 0;
          const int r0 = 2 * n + (sw ? 1 : 0), r1 = 2 * n + (sw ? 0 : 1);
          *reinterpret_cast<uint4 *>(pbh + sw64_off(r0, ch)) = sw ? e1h : e0h;
          *reinterpret_cast<uint4 *>(pbl + sw64_off(r0, ch)) = sw ? e1l : e0l;
          *reinterpret_cast<uint4 *>(pbh + sw64_off(r1, ch)) = sw ? e0h : e1h;
          *reinterpret_cast<uint4 *>(pbl + sw64_off(r1, ch)) = sw ? e0l : e1l;
        }
        fence_proxy_async();
        mbar_arrive(&a_full[sa]);
      }
    }
  } else if (warp < 12) {
    // ------------------------------------------------------------------ epilogue
    const int q = warp & 3;
    const int r = 32 * q + lane;                      // TMEM lane = tone n of tile i
    const int etid = tid - 256;                       // 0..127
    int lu = 0;
    for (int u = blockIdx.x; u < p.n_units; u += gridDim.x, ++lu) {
      const Unit8 un = decode8(p, u);
      const int set = p.soi ? p.soi[un.t] : 0;
      const bool set_ok = set >= 0 && set < p.n_sets;
      const int acc = lu & 1;
      mbar_wait(&tmem_full[acc], (lu >> 1) & 1);
      tc_fence_after();
      const int nt = TT * un.i + r;                  // this thread's tone of tile i
      const int dbase = TT * (un.j - un.i) - r;      // d = dbase + m for tone m of tile j
      for (int cb = 0; cb < 8; ++cb) {
        uint32_t v[32];
        tmem_ld32x32b_x32(tmem_base + uint32_t(acc * 256 + 32 * cb) + (uint32_t(32 * q) << 16), v);
        tmem_ld_wait();
        if (!set_ok || nt >= p.N) continue;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const int col = 32 * cb + e, m = col >> 1;
          const int d = dbase + m;
          if (d >= 0 && d < p.D && TT * un.j + m < p.N) atomicAdd(&bins[2 * d + (col & 1)], __uint_as_float(v[e]));
        }
      }
      tc_fence_before();
      named_bar_sync(2, 128);                        // all rows binned
      if (lane == 0) mbar_arrive(&tmem_empty[acc]);  // the accumulator is free for the unit after next
      if (set_ok) {
        double *acc_s = p.acc + size_t(set) * (2 * p.D + 2);
        for (int qd = etid; qd < 2 * p.D; qd += 128) {
          const float bv = bins[qd];
          if (bv != 0.f) atomicAdd(&acc_s[qd], double(bv));
          bins[qd] = 0.f;
        }
      }
      named_bar_sync(2, 128);                        // bins cleared before the next unit
    }
  } else {
    // ------------------------------------------------------------------ MMA issuer (warp 13)
    if (lane == 0) {
      // F32 accumulate, BF16 A/B, K-major A/B, N = 256, M = 128
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(256 >> 3) << 17) | (uint32_t(TT >> 4) << 24);
      int it = 0, lu = 0;
      for (int u = blockIdx.x; u < p.n_units; u += gridDim.x, ++lu) {
        const Unit8 un = decode8(p, u);
        const int acc = lu & 1;
        mbar_wait(&tmem_empty[acc], ((lu >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + uint32_t(acc * 256);
        bool first = true;
        for (int q = un.q0; q < un.q1; ++q, ++it) {
          const int s = it % S_AB8;
          mbar_wait(&a_full[s], (it / S_AB8) & 1);
          tc_fence_after();
          uint8_t *st = ab + s * AB8;
          const uint64_t ahd = sw64_desc(smem_u32(st)), ald = sw64_desc(smem_u32(st + A8_PLANE));
          const uint64_t bhd = sw64_desc(smem_u32(st + 2 * A8_PLANE)),
                         bld = sw64_desc(smem_u32(st + 2 * A8_PLANE + B8_PLANE));
          for (int ks = 0; ks < 2; ++ks) {
            const uint64_t adv = uint64_t(2 * ks);      // +32 bytes along K
            mma_bf16(d, ahd + adv, bhd + adv, idesc, first ? 0u : 1u);
            first = false;
            mma_bf16(d, ahd + adv, bld + adv, idesc, 1u);
            mma_bf16(d, ald + adv, bhd + adv, idesc, 1u);
          }
          mma_commit(&st_empty[s]);
        }
        mma_commit(&tmem_full[acc]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 13) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace

bool gram_launchable(const float2 *y, int32_t K, int32_t N, int32_t D) {
  const int n_tiles = (N + TT - 1) / TT;
  const int jj = (D + TT - 2) / TT + 1;
  return K >= 1 && K <= KMAX8 && D >= 1 && D <= DMAX8 && N % 2 == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0 &&
         n_tiles * jj <= MAXP8 && encode_fn() != nullptr;
}

cudaError_t launch_gram(const float2 *y, const float2 *x, int32_t T, int32_t M, int32_t K, int32_t N,
                        const int32_t *soi, int32_t n_sets, int32_t D, double *acc, cudaStream_t stream) {
  if (!gram_launchable(y, K, N, D)) return cudaErrorNotSupported;
  int dev = 0, nsm = 148;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // the shared-memory opt-in is per device (a process may drive several GPUs)
  static std::atomic<uint64_t> attr_set{0};
  const uint64_t bit = dev < 64 ? (uint64_t(1) << dev) : 0;
  if (!bit || !(attr_set.load() & bit)) {
    e = cudaFuncSetAttribute(k8_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, K8_SMEM);
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(bit);
  }
  K8Params p;
  p.soi = soi;
  p.x = x;
  p.acc = acc;
  p.T = T;
  p.M = M;
  p.nmc = (M + CC8 - 1) / CC8;
  p.K = K;
  p.N = N;
  p.D = D;
  p.n_sets = n_sets;
  const int n_tiles = (N + TT - 1) / TT;
  const int jj = (D + TT - 2) / TT + 1;            // j - i < jj covers every 0 <= n' - n < D
  int np = 0;
  for (int i = 0; i < n_tiles; ++i)
    for (int dj = 0; dj < jj && i + dj < n_tiles; ++dj) p.pairs[np++] = make_short2(short(i), short(i + dj));
  p.n_pairs = np;
  // columns per unit: about one unit per SM (each unit pays a factor table and 2D atomics), whole 16-column
  // chunks, at most one instance
  // chunks per unit: about one unit per SM (each unit pays a factor table and 2D atomics), at most one instance
  const int nq = K * p.nmc;                        // 16-column chunks per instance
  const long long work = (long long)T * np * nq;
  static const int env_upsm = getenv("CE_K8_UPSM") ? atoi(getenv("CE_K8_UPSM")) : 1;   // experiments
  long long cq = work / (std::max(1, env_upsm) * (long long)nsm);
  cq = std::max<long long>(1, std::min<long long>(cq, std::min(256, nq)));
  p.cq = int(cq);
  p.n_cc = (nq + p.cq - 1) / p.cq;
  const long long units = (long long)T * p.n_cc * np;
  if (units > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  p.n_units = int(units);
  CUtensorMap tmy;
  if (!make_map_kmajor(&tmy, y, N, K, M, T, CC8, 2 * TT)) return cudaErrorInvalidValue;
  k8_gram<<<unsigned(std::min<long long>(units, nsm)), K8_THREADS, K8_SMEM, stream>>>(tmy, p);
  return cudaGetLastError();
}

}  // namespace ce
