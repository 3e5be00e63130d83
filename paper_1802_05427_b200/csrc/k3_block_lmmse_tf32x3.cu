// K3 -- fused LS + block-LMMSE contraction on the 5th-gen tensor cores (tcgen05, kind::tf32),
// error-compensated "3xTF32": D = A_hi B_hi + A_hi B_lo + A_lo B_hi (FP32 accumulate in TMEM).
//
// Same operation as K2 (Eq. 12 per block, LS of Eq. 9 fused into the load):
//   h[t, c, o+i] = sum_j W[o-a+i][j] * y[t,c,a+j] / x[t,k,a+j]
//
// Complex -> real embedding.  With the LS row stored interleaved (re, im) the per-window
// complex GEMM C[cols x kept] = A[cols x b] W_rows^T becomes ONE real GEMM
//   D[cols x 2kept] = A_r[cols x 2b] . B_r[2b x 2kept]
//   A_r[c][2j+q]              = (re, im)(H_LS[c][j])            <- the interleaved LS row itself
//   B_r^T[2i][2j], [2i][2j+1]  = Re W_ij, -Im W_ij
//   B_r^T[2i+1][2j], [2i+1][2j+1] = Im W_ij,  Re W_ij
//   D[c][2i], D[c][2i+1]       = (re, im)(h[c][o+i])            <- the interleaved output row
// (8 real MACs... 4 per complex MAC, no waste).  MMA M = 128 columns (c), N = 2*kept padded to
// 16, K = 2b in 32-float chunks (128-byte K-major rows, SWIZZLE_128B).
//
// B (the filter) is built once by K1 as a "bank" already split into hi/lo TF32 planes and laid
// out in global memory as the exact shared-memory image of each K chunk (rows 128 B apart,
// 16-byte chunks XOR-swizzled by row % 8), so a plain cp.async.bulk lands it ready for the
// UMMA descriptor.  Window row offsets are handled by starting the copy at the 8-row aligned
// bank row n0 <= 2*row0 and reading the accumulator from column off = 2*row0 - n0.
//
// Warp roles (320 threads, persistent CTAs, one per SM):
//   warps 0-3 : transform -- load y, x from HBM, LS = y conj(x)/|x|^2, split hi/lo (cvt.rna.tf32),
//               write the swizzled A_hi/A_lo tiles, fence.proxy.async, arrive a_full[s]
//   warps 4-7 : epilogue  -- tcgen05.ld the TMEM accumulator (32 lanes per warp), transpose
//               through shared memory, coalesced stores of the kept output tones
//   warp 8    : B producer -- cp.async.bulk of the bank chunk (hi + lo) -> b_full[s]
//   warp 9    : TMEM allocator + MMA issuer (one lane): 3 tcgen05.mma per 8-float K step,
//               tcgen05.commit -> empty[s]; per tile tcgen05.commit -> tmem_full[acc]
// Two smem stages (A_hi, A_lo, B_hi, B_lo), two TMEM accumulators of 256 columns.
#include <cuda_runtime.h>
#include <stdint.h>

#include "ce_internal.h"
#include "tc_ptx.cuh"

namespace ce {
namespace {

constexpr int K3_THREADS = 320;
constexpr int KC = 32;             // floats per K chunk (one 128-byte swizzle row)
constexpr int STAGES = 2;
constexpr int TILE_M = 128;
constexpr int NMAX = 256;
constexpr int A_BYTES = TILE_M * KC * 4;   // 16 KB
constexpr int B_BYTES = NMAX * KC * 4;     // 32 KB
constexpr int EPI_STRIDE = 34;             // floats per row of the epilogue transpose buffer
constexpr int SMEM_BYTES = STAGES * (2 * A_BYTES + 2 * B_BYTES) + 4 * 32 * EPI_STRIDE * 4 + 256 + 1024;

struct K3Params {
  const float2 *y;
  const float2 *x;
  float2 *h;
  const float *bank_hi;
  const float *bank_lo;
  const Window *geo;
  const int32_t *soi;
  int T, K, N, b, n_win, n_sets, nkc, NR, cols, n_ct, n_tiles;
};

// ------------------------------------------------------------------------------ tile geometry
struct TileInfo {
  int t, w, ct, a, o, kept, n0, off, nw, set;
  bool set_ok;
};

__device__ __forceinline__ TileInfo decode(const K3Params &p, int tile) {
  TileInfo ti;
  ti.ct = tile % p.n_ct;
  const int rest = tile / p.n_ct;
  ti.w = rest % p.n_win;
  ti.t = rest / p.n_win;
  const Window g = p.geo[ti.w];
  ti.a = g.a;
  ti.o = g.o;
  ti.kept = g.o_next - g.o;
  const int row2 = 2 * (g.o - g.a);
  ti.n0 = row2 & ~7;
  ti.off = row2 - ti.n0;
  ti.nw = (ti.off + 2 * ti.kept + 15) & ~15;
  const int s = p.soi ? p.soi[ti.t] : 0;
  ti.set_ok = s >= 0 && s < p.n_sets;
  ti.set = ti.set_ok ? s : 0;
  return ti;
}

__global__ void __launch_bounds__(K3_THREADS, 1) k3_tf32x3(K3Params p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment by pointer arithmetic on the __shared__ array (keeps the shared address space
  // visible to the compiler: LDS/STS instead of generic LD/ST)
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float *A_hi = reinterpret_cast<float *>(smem);
  float *A_lo = A_hi + STAGES * TILE_M * KC;
  float *B_hi = A_lo + STAGES * TILE_M * KC;
  float *B_lo = B_hi + STAGES * NMAX * KC;
  float *epi = B_lo + STAGES * NMAX * KC;                       // [4 warps][32][EPI_STRIDE]
  uint64_t *bars = reinterpret_cast<uint64_t *>(epi + 4 * 32 * EPI_STRIDE);
  uint64_t *a_full = bars;                                      // [STAGES]
  uint64_t *b_full = bars + STAGES;                             // [STAGES]
  uint64_t *empty = bars + 2 * STAGES;                          // [STAGES]
  uint64_t *tmem_full = bars + 3 * STAGES;                      // [2]
  uint64_t *tmem_empty = bars + 3 * STAGES + 2;                 // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 3 * STAGES + 4);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&a_full[s], 128);
      mbar_init(&b_full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&tmem_empty[i], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int nks_total = (2 * p.b + 7) / 8;   // 8-float MMA K steps over the 2b real K extent

  if (warp < 4) {
    // ------------------------------------------------------------------ transform (A operand)
    const int j = tid & 15;          // complex index inside the 16-complex chunk
    const int rb = tid >> 4;         // row base 0..7 ; rows rb + 8 i
    const int phys = (((j >> 1) ^ (rb & 7)) << 2) + ((j & 1) << 1);   // swizzled float offset in the row
    int it = 0;
    for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
      const TileInfo ti = decode(p, tile);
      const float2 *yb = p.y + size_t(ti.t) * p.cols * p.N + ti.a;
      const float2 *xb = p.x + size_t(ti.t) * p.K * p.N + ti.a;
      const int c_first = ti.ct * TILE_M + rb;     // column of row rb; rows step by 8
      const int x_first = c_first % p.K;
      const int x_step = 8 % p.K;
      float2 yv[16], xv[16];
      auto load = [&](int kc) {
        const int jj = kc * 16 + j;
        const bool kok = jj < p.b;
        int xr = x_first;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int c = c_first + 8 * i;
          yv[i] = make_float2(0.f, 0.f);
          xv[i] = make_float2(1.f, 0.f);
          if (kok && c < p.cols) {
            yv[i] = __ldg(yb + size_t(c) * p.N + jj);
            xv[i] = __ldg(xb + size_t(xr) * p.N + jj);
          }
          xr += x_step;
          if (xr >= p.K) xr -= p.K;
        }
      };
      load(0);
      for (int kc = 0; kc < p.nkc; ++kc, ++it) {
        const int s = it % STAGES;
        mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
        float *ah = A_hi + s * TILE_M * KC;
        float *al = A_lo + s * TILE_M * KC;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float inv = 1.0f / (xv[i].x * xv[i].x + xv[i].y * xv[i].y);
          const float lre = (yv[i].x * xv[i].x + yv[i].y * xv[i].y) * inv;
          const float lim = (yv[i].y * xv[i].x - yv[i].x * xv[i].y) * inv;
          const int r = rb + 8 * i;
          const float hr = tf32_rna(lre), hi_ = tf32_rna(lim);
          *reinterpret_cast<float2 *>(ah + r * KC + phys) = make_float2(hr, hi_);
          *reinterpret_cast<float2 *>(al + r * KC + phys) = make_float2(tf32_rna(lre - hr), tf32_rna(lim - hi_));
        }
        fence_proxy_async();
        mbar_arrive(&a_full[s]);
        if (kc + 1 < p.nkc) load(kc + 1);   // prefetch: in flight while the MMAs of this chunk run
      }
    }
  } else if (warp < 8) {
    // ------------------------------------------------------------------ epilogue
    const int q = warp & 3;                  // TMEM lane quarter
    float *stage = epi + q * 32 * EPI_STRIDE;
    int lt = 0;
    for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++lt) {
      const TileInfo ti = decode(p, tile);
      const int acc = lt & 1;
      mbar_wait(&tmem_full[acc], (lt >> 1) & 1);
      tc_fence_after();
      const int nf = 2 * ti.kept;                     // valid floats per row
      const int ncb = (ti.off + nf + 31) / 32;        // 32-column TMEM chunks holding them
      const int row_base = ti.ct * TILE_M + q * 32;   // column c of lane 0 of this warp
      const float qnan = __int_as_float(0x7fc00000);
      for (int cb = 0; cb < ncb; ++cb) {
        float v[32];
        tmem_ld32(tmem_base + uint32_t(acc * NMAX + cb * 32) + (uint32_t(q * 32) << 16), v);
#pragma unroll
        for (int u = 0; u < 32; u += 2)
          *reinterpret_cast<float2 *>(stage + lane * EPI_STRIDE + u) = make_float2(v[u], v[u + 1]);
        __syncwarp();
        // rows of this warp: 2 per instruction, 16 lanes x 8 bytes each = 128 contiguous bytes
        const int f = cb * 32 - ti.off + 2 * (lane & 15);   // float index inside the kept row
        const bool fok = f >= 0 && f < nf;
#pragma unroll 4
        for (int rr = 0; rr < 32; rr += 2) {
          const int r = rr + (lane >> 4);
          const int c = row_base + r;
          if (fok && c < p.cols) {
            float2 val = *reinterpret_cast<const float2 *>(stage + r * EPI_STRIDE + 2 * (lane & 15));
            if (!ti.set_ok) val = make_float2(qnan, qnan);
            p.h[(size_t(ti.t) * p.cols + c) * p.N + ti.o + (f >> 1)] = val;
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      mbar_arrive(&tmem_empty[acc]);
    }
  } else if (warp == 8) {
    // ------------------------------------------------------------------ B producer
    if (lane == 0) {
      int it = 0;
      for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
        const TileInfo ti = decode(p, tile);
        const uint32_t bytes = uint32_t(ti.nw) * KC * 4;
        for (int kc = 0; kc < p.nkc; ++kc, ++it) {
          const int s = it % STAGES;
          mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          mbar_arrive_expect_tx(&b_full[s], 2 * bytes);
          const size_t src = ((size_t(ti.set) * p.nkc + kc) * p.NR + ti.n0) * KC;
          bulk_g2s(B_hi + s * NMAX * KC, p.bank_hi + src, bytes, &b_full[s]);
          bulk_g2s(B_lo + s * NMAX * KC, p.bank_lo + src, bytes, &b_full[s]);
        }
      }
    }
  } else {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int it = 0, lt = 0;
      for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++lt) {
        const TileInfo ti = decode(p, tile);
        const int acc = lt & 1;
        // instruction descriptor: F32 accum, TF32 A/B, K-major A/B, N = nw, M = 128
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(ti.nw >> 3) << 17) |
                               (uint32_t(TILE_M >> 4) << 24);
        mbar_wait(&tmem_empty[acc], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + uint32_t(acc * NMAX);
        for (int kc = 0; kc < p.nkc; ++kc, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&a_full[s], ph);
          mbar_wait(&b_full[s], ph);
          tc_fence_after();
          const uint64_t ah = sw128_desc(smem_u32(A_hi + s * TILE_M * KC));
          const uint64_t al = sw128_desc(smem_u32(A_lo + s * TILE_M * KC));
          const uint64_t bh = sw128_desc(smem_u32(B_hi + s * NMAX * KC));
          const uint64_t bl = sw128_desc(smem_u32(B_lo + s * NMAX * KC));
          const int nks = min(4, nks_total - 4 * kc);
          for (int ks = 0; ks < nks; ++ks) {
            const uint64_t adv = uint64_t(2 * ks);     // +32 bytes along K (start address >> 4)
            mma_tf32(d, ah + adv, bh + adv, idesc, (kc | ks) != 0);
            mma_tf32(d, ah + adv, bl + adv, idesc, 1u);
            mma_tf32(d, al + adv, bh + adv, idesc, 1u);
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&tmem_full[acc]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    __syncwarp();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512) : "memory");
  }
}

// ------------------------------------------------------------------------ filter bank (K1 tail)
// bank[set][kc][n][32] = swizzled TF32 hi/lo planes of B_r^T[n][32 kc + kk] (see header comment).
__global__ void k3_build_bank(const float2 *__restrict__ W, int b, int nkc, int NR, float *__restrict__ bank_hi,
                              float *__restrict__ bank_lo) {
  const int set = blockIdx.x, kc = blockIdx.y;
  const float2 *Ws = W + size_t(set) * b * b;
  float *bh = bank_hi + (size_t(set) * nkc + kc) * NR * KC;
  float *bl = bank_lo + (size_t(set) * nkc + kc) * NR * KC;
  for (int e = threadIdx.x; e < NR * KC; e += blockDim.x) {
    const int n = e / KC, kk = e % KC;
    const int k = kc * KC + kk;
    const int i = n >> 1, jw = k >> 1;
    float v = 0.f;
    if (i < b && jw < b) {
      const float2 w = Ws[size_t(i) * b + jw];
      const int sel = ((n & 1) << 1) | (k & 1);   // (row parity, col parity)
      v = sel == 0 ? w.x : sel == 1 ? -w.y : sel == 2 ? w.y : w.x;
    }
    const float hi = tf32_rna(v);
    const float lo = tf32_rna(v - hi);
    const int dst = n * KC + ((((kk >> 2) ^ (n & 7)) << 2) | (kk & 3));
    bh[dst] = hi;
    bl[dst] = lo;
  }
}

}  // namespace

bool tf32x3_supported(int32_t b, const std::vector<Window> &geo) {
  for (const auto &g : geo) {
    const int row2 = 2 * (g.o - g.a);
    const int off = row2 & 7;
    if (((off + 2 * (g.o_next - g.o) + 15) & ~15) > NMAX) return false;
  }
  return b >= 1;
}

void tf32x3_bank_shape(int32_t b, int32_t *nkc, int32_t *NR) {
  *nkc = (2 * b + KC - 1) / KC;
  *NR = ((2 * b + 16) + 7) & ~7;
}

cudaError_t launch_build_bank(const float2 *d_W, int32_t b, int32_t n_sets, float *bank_hi, float *bank_lo,
                              cudaStream_t stream, int64_t *launches) {
  int32_t nkc, NR;
  tf32x3_bank_shape(b, &nkc, &NR);
  k3_build_bank<<<dim3(n_sets, nkc), 256, 0, stream>>>(d_W, b, nkc, NR, bank_hi, bank_lo);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) ++*launches;
  return e;
}

cudaError_t launch_contract_tf32x3(const ContractArgs &a, const float *bank_hi, const float *bank_lo,
                                   cudaStream_t stream, int64_t *launches) {
  K3Params p;
  p.y = a.y;
  p.x = a.x;
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
  tf32x3_bank_shape(a.b, &p.nkc, &p.NR);
  p.cols = a.M * a.K;
  p.n_ct = (p.cols + TILE_M - 1) / TILE_M;
  const long long tiles = (long long)a.T * a.n_win * p.n_ct;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  p.n_tiles = int(tiles);
  static int num_sms = 0;
  if (num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  cudaError_t e = cudaFuncSetAttribute(k3_tf32x3, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int grid = int(tiles < num_sms ? tiles : num_sms);
  k3_tf32x3<<<grid, K3_THREADS, SMEM_BYTES, stream>>>(p);
  e = cudaGetLastError();
  if (e == cudaSuccess) ++*launches;
  return e;
}

}  // namespace ce
