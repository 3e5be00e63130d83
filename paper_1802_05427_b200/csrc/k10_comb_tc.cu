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
//     D[2o + c][r] = sum_k  A_s,blk[2o + c][k] * B[r][k],   k = 2j' + c'  (pilot sw + j', re / im)
// with A the block's weights embedded as 2x2 real blocks [[Re, -Im], [Im, Re]] (rows 2o / 2o + 1 of output o =
// i*S + q of group g0 + i; zero outside the group's own G taps) and B the LS of UE s at the window's pilots
// for N = 128 data rows r = (t, m).  M = 128 (<= 64 outputs), N = 128 rows, K = 32 (2 MMA K-steps), BF16x3
// (A_hi B_hi + A_hi B_lo + A_lo B_hi, FP32 accumulation in TMEM) as K4 (reading B1).
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
//                     warps 2-9: epilogue -- tcgen05.ld 32x32b: lane = output component, column = data row, so for
//                                each data row a warp holds 16 consecutive complex outputs and writes them as one
//                                128-byte coalesced segment of h[t][m][s][.]
//   k10_build_images (build time) the weight images from K6a's complex64 W.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "ce_internal.h"
#include "tc_ptx.cuh"
#include "tmap.cuh"

namespace ce {
namespace {

constexpr int K10_WIN = 16;                 // pilots per block window: K = 32 bf16 = one 64-byte SW64 row
constexpr int K10_NR = 128;                 // data rows per unit (MMA N)
constexpr int K10_PLANE = 128 * 64;         // [128 rows][32 bf16], SW64: 8 KB
constexpr int K10_SA = 2;                   // weight-image slots
#ifndef K10_SB_STAGES
#define K10_SB_STAGES 6
#endif
constexpr int K10_SB = K10_SB_STAGES;       // LS-tile ring
#ifndef K10_EPI_WARPS
#define K10_EPI_WARPS 8
#endif
constexpr int K10_EPI = K10_EPI_WARPS;      // 4 or 8 epilogue warps (two per TMEM lane quadrant)
constexpr int K10_THREADS = 32 * (2 + K10_EPI);
constexpr int K10_SMEM = (K10_SA + K10_SB) * 2 * K10_PLANE + 256 + 1024;
static_assert(K10_EPI == 4 || K10_EPI == 8, "K10 epilogue warps");
static_assert(K10_SMEM <= 232448, "K10 shared memory");

struct K10Params {
  float *h;                     // [T*M][n_ue][N] complex64 as floats
  const uint16_t *img_hi;       // [n_ue][n_blk][128][32] bf16, SW64 image
  const uint16_t *img_lo;
  const int4 *blk;              // [n_blk] {g0, ng, sw, 0}
  int R, n_ue, N, S, n_blk, n_rt, u_total;
};

struct Unit10 {
  int s, b, rt, key;
};
__device__ __forceinline__ Unit10 decode10(const K10Params &p, int u) {
  Unit10 d;
  d.rt = u % p.n_rt;
  d.key = u / p.n_rt;           // s * n_blk + b: the weight image
  d.b = d.key % p.n_blk;
  d.s = d.key / p.n_blk;
  return d;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo_addr, float hi_addr) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi_addr), "f"(lo_addr));
  return r;
}
__device__ __forceinline__ float bf16lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }

// LS at every tone of data row r (Eq. 9), scattered into the per-UE bf16 hi / lo planes:
// plane[(s * R + r) * KP4 + p] = (re, im) of LS at tone S*p + s.  One CTA per row (grid-stride).
__global__ void __launch_bounds__(256) k10_ls(const float2 *__restrict__ y, const float2 *__restrict__ x,
                                              uint32_t *__restrict__ ls_hi, uint32_t *__restrict__ ls_lo, int M,
                                              int R, int N, int S, int n_ue, int KP, int KP4) {
  extern __shared__ float2 lsrow[];                 // [N]
  pdl_wait();                                       // y, x (caller data) and the planes (read by the previous call)
  if (threadIdx.x == 0) pdl_launch_dependents();    // k10_comb_tc may start its weight-image loads
  for (int r = blockIdx.x; r < R; r += gridDim.x) {
    const int t = r / M;
    const float2 *yr = y + size_t(r) * N;
    const float2 *xr = x + size_t(t) * N;
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
      const float2 yv = yr[k], xv = __ldg(xr + k);
      const float inv = 1.0f / (xv.x * xv.x + xv.y * xv.y);
      lsrow[k] = make_float2((yv.x * xv.x + yv.y * xv.y) * inv, (yv.y * xv.x - yv.x * xv.y) * inv);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n_ue * KP; e += blockDim.x) {
      const int s = e / KP, p = e - s * KP;
      const float2 v = lsrow[S * p + s];
      const uint32_t hi = pack_bf16x2(v.x, v.y);
      const uint32_t lo = pack_bf16x2(v.x - bf16lo(hi), v.y - bf16hi(hi));
      const size_t idx = (size_t(s) * R + r) * KP4 + p;
      ls_hi[idx] = hi;
      ls_lo[idx] = lo;
    }
    __syncthreads();
  }
}

// Weight image of (UE s, block b): A[m][kk], m = 2o + c (output o = i*S + q of group g0 + i, c = re / im row),
// kk = 2j' + c' (pilot sw + j'): the 2x2 real embedding of W_s^(type_g)[q][sw + j' - a_g] (zero outside the
// group's G taps and beyond the block's outputs); bf16 hi / lo planes in the SW64 image (row m at m*64 bytes,
// 16-byte chunk (kk/8) ^ ((m>>1)&3)).
__global__ void k10_build_images(const float2 *__restrict__ W, const int4 *__restrict__ blk, int n_blk, int S,
                                 int G, int K, int ml, uint16_t *__restrict__ img_hi, uint16_t *__restrict__ img_lo) {
  const int b = blockIdx.x, s = blockIdx.y;
  const int4 B = blk[b];
  uint16_t *hi = img_hi + (size_t(s) * n_blk + b) * 128 * 32;
  uint16_t *lo = img_lo + (size_t(s) * n_blk + b) * 128 * 32;
  for (int e = threadIdx.x; e < 128 * 32; e += blockDim.x) {
    const int m = e / 32, kk = e % 32;
    const int o = m >> 1, c = m & 1, jj = kk >> 1, cc = kk & 1;
    float v = 0.f;
    if (o < B.y * S) {
      const int i = o / S, q = o - i * S, g = B.x + i;
      const int a = min(max(g - ml, 0), K - G);
      const int j = B.z + jj - a;
      if (j >= 0 && j < G) {
        const float2 w = W[((size_t(s) * G + (g - a)) * S + q) * G + j];
        const int sel = (c << 1) | cc;
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

__global__ void __launch_bounds__(K10_THREADS, 1)
    k10_comb_tc(const __grid_constant__ CUtensorMap tml_hi, const __grid_constant__ CUtensorMap tml_lo,
                const __grid_constant__ K10Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sa = smem;                                         // [SA][hi | lo]
  uint8_t *sb = smem + K10_SA * 2 * K10_PLANE;                // [SB][hi | lo]
  uint64_t *bars = reinterpret_cast<uint64_t *>(sb + K10_SB * 2 * K10_PLANE);
  uint64_t *a_full = bars, *a_empty = bars + K10_SA;
  uint64_t *b_full = bars + 2 * K10_SA, *b_empty = b_full + K10_SB;
  uint64_t *tmem_full = b_empty + K10_SB, *tmem_empty = tmem_full + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_empty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int u0 = int((long long)blockIdx.x * p.u_total / gridDim.x);
  const int u1 = int((long long)(blockIdx.x + 1) * p.u_total / gridDim.x);
  if (tid == 0) {
    for (int i = 0; i < K10_SA; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < K10_SB; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&tmem_empty[i], K10_EPI);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (tid == 0) pdl_launch_dependents();

  if (warp == 0) {
    // ------------------------------------------------------------------ producer (TMA / bulk copies)
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tml_hi)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tml_lo)) : "memory");
      int key_prev = -1, na = 0, ib = 0;
      bool waited = false;
      for (int u = u0; u < u1; ++u, ++ib) {
        const Unit10 d = decode10(p, u);
        if (d.key != key_prev) {                       // the weight image changes: next A slot
          const int sl = na % K10_SA;
          mbar_wait(&a_empty[sl], ((na / K10_SA) & 1) ^ 1);
          mbar_arrive_expect_tx(&a_full[sl], 2 * K10_PLANE);
          const size_t src = size_t(d.key) * 128 * 32;
          bulk_g2s(sa + sl * 2 * K10_PLANE, p.img_hi + src, K10_PLANE, &a_full[sl]);
          bulk_g2s(sa + sl * 2 * K10_PLANE + K10_PLANE, p.img_lo + src, K10_PLANE, &a_full[sl]);
          ++na;
          key_prev = d.key;
        }
        if (!waited) {                                 // the LS planes come from the preceding k10_ls
          pdl_wait();
          waited = true;
        }
        const int st = ib % K10_SB;
        mbar_wait(&b_empty[st], ((ib / K10_SB) & 1) ^ 1);
        mbar_arrive_expect_tx(&b_full[st], 2 * K10_PLANE);
        const int4 B = __ldg(&p.blk[d.b]);
        const int c0 = 2 * B.z, c1 = d.s * p.R + d.rt * K10_NR;
        tma_load_2d(sb + st * 2 * K10_PLANE, &tml_hi, c0, c1, &b_full[st]);
        tma_load_2d(sb + st * 2 * K10_PLANE + K10_PLANE, &tml_lo, c0, c1, &b_full[st]);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      // F32 accumulate, BF16 A / B, both K-major, N = 128, M = 128
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(K10_NR >> 3) << 17) | (uint32_t(128 >> 4) << 24);
      int key_prev = -1, na = 0, ib = 0, lt = 0;
      for (int u = u0; u < u1; ++u, ++ib, ++lt) {
        const Unit10 d = decode10(p, u);
        if (d.key != key_prev) {
          mbar_wait(&a_full[na % K10_SA], (na / K10_SA) & 1);
          ++na;
          key_prev = d.key;
        }
        const int sl = (na - 1) % K10_SA;
        const int acc = lt & 1;
        mbar_wait(&tmem_empty[acc], ((lt >> 1) & 1) ^ 1);
        const int st = ib % K10_SB;
        mbar_wait(&b_full[st], (ib / K10_SB) & 1);
        tc_fence_after();
        const uint32_t dt = tmem_base + uint32_t(acc * K10_NR);
        const uint64_t ah = sw64_desc(smem_u32(sa + sl * 2 * K10_PLANE));
        const uint64_t al = sw64_desc(smem_u32(sa + sl * 2 * K10_PLANE + K10_PLANE));
        const uint64_t bh = sw64_desc(smem_u32(sb + st * 2 * K10_PLANE));
        const uint64_t bl = sw64_desc(smem_u32(sb + st * 2 * K10_PLANE + K10_PLANE));
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint64_t adv = uint64_t(2 * ks);       // +32 bytes along K
          mma_bf16(dt, ah + adv, bh + adv, idesc, ks != 0);
          mma_bf16(dt, ah + adv, bl + adv, idesc, 1u);
          mma_bf16(dt, al + adv, bh + adv, idesc, 1u);
        }
        mma_commit(&b_empty[st]);
        if (u + 1 >= u1 || decode10(p, u + 1).key != d.key) mma_commit(&a_empty[sl]);   // last use of the image
        mma_commit(&tmem_full[acc]);
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue
    pdl_wait();                                        // h may still be read by the previous kernel in the stream
    const int q = warp & 3;                            // TMEM lane quadrant this warp may access
    const int part = (warp - 2) >> 2;                  // 8 warps: column blocks {part, part + 2}; 4 warps: all four
    constexpr int NCB = K10_EPI == 8 ? 2 : 4;
    const int comp = 32 * q + lane;                    // output float (2o + c) held by this thread
    const size_t row_floats = size_t(p.n_ue) * p.N * 2;
    int lt = 0;
    for (int u = u0; u < u1; ++u, ++lt) {
      const Unit10 d = decode10(p, u);
      const int4 B = __ldg(&p.blk[d.b]);
      const int acc = lt & 1;
      mbar_wait(&tmem_full[acc], (lt >> 1) & 1);
      tc_fence_after();
      float v[NCB][32];
#pragma unroll
      for (int i = 0; i < NCB; ++i) {
        const int cb = K10_EPI == 8 ? part + 2 * i : i;
        tmem_ld32(tmem_base + uint32_t(acc * K10_NR + 32 * cb) + (uint32_t(32 * q) << 16), v[i]);
      }
      __syncwarp();
      if (lane == 0) {
        tc_fence_before();
        mbar_arrive(&tmem_empty[acc]);               // the accumulator is in registers: the MMA may reuse it
      }
      if (comp < 2 * B.y * p.S) {
        float *hb = p.h + (size_t(d.s) * p.N + size_t(p.S) * B.x) * 2 + comp;
        const int rbase = d.rt * K10_NR;
#pragma unroll
        for (int i = 0; i < NCB; ++i) {
          const int cb = K10_EPI == 8 ? part + 2 * i : i;
          const int r0 = rbase + 32 * cb;
          const int nr = min(32, p.R - r0);
          float *hr = hb + size_t(r0) * row_floats;
          if (nr >= 32) {
#pragma unroll
            for (int c = 0; c < 32; ++c) hr[size_t(c) * row_floats] = v[i][c];
          } else {
#pragma unroll
            for (int c = 0; c < 32; ++c)
              if (c < nr) hr[size_t(c) * row_floats] = v[i][c];
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem_base, 256);
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
    if (e != cudaSuccess) return e;
    d.init = true;
  }
  *out = &d;
  return cudaSuccess;
}

}  // namespace

bool comb_tc_supported(int32_t N, int32_t S, int32_t G, int32_t mode) {
  // a 16-pilot window at a multiple of 4 holds any G <= 13 window; a block's outputs fit M = 128 rows
  return mode == CE_COMB_FULL && G >= 1 && G <= K10_WIN - 3 && S >= 1 && S <= 64 && N % S == 0 &&
         encode_fn() != nullptr;
}

std::vector<int4> comb_tc_blocks(int32_t K, int32_t G, int32_t S) {
  const int ml = (G - 1) / 2;
  auto a_of = [&](int g) { return std::min(std::max(g - ml, 0), K - G); };
  const int maxng = 64 / S;
  std::vector<int4> out;
  for (int g = 0; g < K;) {
    const int sw = a_of(g) & ~3;
    int ng = 1;
    while (g + ng < K && ng < maxng && a_of(g + ng) + G <= sw + K10_WIN) ++ng;
    out.push_back(make_int4(g, ng, sw, 0));
    g += ng;
  }
  return out;
}

size_t comb_tc_image_elems(int32_t n_ue, int32_t n_blk) { return size_t(n_ue) * n_blk * 128 * 32; }

size_t comb_tc_ls_bytes(int32_t N, int32_t S, int32_t n_ue, long long rows) {
  const long long KP4 = ((N / S) + 3) & ~3LL;
  return size_t(2) * n_ue * rows * KP4 * 4;       // hi and lo planes
}

cudaError_t launch_comb_tc_images(const float2 *W, const int4 *d_blk, int32_t n_blk, int32_t n_ue, int32_t N,
                                  int32_t S, int32_t G, uint16_t *img_hi, uint16_t *img_lo, cudaStream_t stream) {
  k10_build_images<<<dim3(n_blk, n_ue), 256, 0, stream>>>(W, d_blk, n_blk, S, G, N / S, (G - 1) / 2, img_hi, img_lo);
  return cudaGetLastError();
}

cudaError_t launch_comb_tc(const float2 *y, const float2 *x, float2 *h, int32_t T, int32_t M, int32_t N, int32_t S,
                           int32_t n_ue, const int4 *d_blk, int32_t n_blk, const uint16_t *img_hi,
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
    const long long g = R < 8LL * di->num_sms * 4 ? R : 8LL * di->num_sms * 4;
    cfg.gridDim = dim3(unsigned(g));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = size_t(N) * sizeof(float2);
    cfg.stream = stream;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = smem_opt_in((const void *)k10_ls, cfg.dynamicSmemBytes);
    if (e != cudaSuccess) return e;
    e = cudaLaunchKernelEx(&cfg, k10_ls, y, x, ls_hi, ls_lo, int(M), int(R), int(N), int(S), int(n_ue), KP, KP4);
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
  p.n_rt = int((R + K10_NR - 1) / K10_NR);
  const long long units = (long long)n_ue * n_blk * p.n_rt;
  if (units >= (1LL << 31)) return cudaErrorInvalidConfiguration;
  p.u_total = int(units);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(units < di->num_sms ? units : di->num_sms));
  cfg.blockDim = dim3(K10_THREADS);
  cfg.dynamicSmemBytes = K10_SMEM;
  cfg.stream = stream;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, k10_comb_tc, mh, ml, p);
  if (e == cudaSuccess) ++*launches;
  return e;
}

}  // namespace ce
