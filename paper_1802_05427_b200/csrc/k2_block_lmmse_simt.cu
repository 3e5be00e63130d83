// K2 -- fused LS + block-LMMSE contraction, FP32 SIMT (CUDA cores).
//
// For every instance t, window w = (a, o, o_next) and column c = (m, k):
//   h[t, c, o + i] = sum_{j < b} W[o - a + i][j] * H_LS[t, c, a + j],   0 <= i < o_next - o
//   H_LS[t, c, n]  = y[t, c, n] / x[t, k, n] = y conj(x) / |x|^2
// PAPER.md:186-190 (Eq. 12) applied per block as in 12W, with the LS of
// Eq. 9 fused into the operand load (PAPER.md:438 multiplies by the conjugated
// pilot; the 1/|x|^2 factor keeps it a true division for non-unit pilots).
//
// Per (t, w) this is a complex GEMM  C[cols x kept] = A[cols x b] * W_rows^T[b x kept].
// CTA tile: 64 columns x 64 kept rows, K chunks of 16 complex, register double buffering.
// Thread tile: 4 columns x 4 rows (complex) = 32 FP32 accumulators; W operands are warp
// broadcasts (8 lanes share a row group), A operands are 128-bit loads of (k, k+1) pairs.
// 4 FFMA per complex MAC; FP32 accumulation in a fixed order per (window, row, column),
// independent of the launch geometry -> bitwise shard invariance (reading A11).
#include <cuda_runtime.h>
#include <stdint.h>

#include "ce_internal.h"

namespace ce {
namespace {

constexpr int BM = 64;        // columns per CTA tile
constexpr int BN = 64;        // kept rows per CTA tile
constexpr int BK = 16;        // complex K chunk
constexpr int AS = BK + 2;    // As row stride (float2): 144 B -> conflict-free 128-bit reads
constexpr int NT = 256;

__device__ __forceinline__ float2 ls_div(float2 y, float2 x) {
  const float inv = 1.0f / (x.x * x.x + x.y * x.y);
  return make_float2((y.x * x.x + y.y * x.y) * inv, (y.y * x.x - y.x * x.y) * inv);
}

struct Tile {
  float2 y[4];  // raw y prefetch (LS applied at stash time, after the compute phase)
  float2 x[4];  // matching pilots
  float2 w[4];  // W^T prefetch
};

union __align__(16) Smem {
  struct {
    float2 As[2][BM][AS];
    float2 Ws[2][BK][BN];
  } k;
  float2 Cs[BM][BN + 1];  // output staging for coalesced row stores
};

__global__ void __launch_bounds__(NT, 2) k2_simt(ContractArgs p, int row_tiles) {
  __shared__ Smem sm;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lc = lane & 7, lr = lane >> 3, wc = warp & 1, wr = warp >> 1;
  const int cols = p.M * p.K;
  const int c0 = blockIdx.x * BM;
  const int w = blockIdx.y / row_tiles, rt = blockIdx.y % row_tiles;
  const Window g = p.geo[w];
  const int kept = g.o_next - g.o;
  const int r_base = rt * BN;
  if (r_base >= kept) return;
  const int rows = min(BN, kept - r_base);
  const int row0 = g.o - g.a + r_base;  // first W row of this tile
  const int b = p.b, N = p.N;
  const int nk = (b + BK - 1) / BK;
  const bool warp_active = wr * 16 < rows;

  // load mapping
  const int a_kk = tid & 15, a_c = tid >> 4;   // A: 16 tones x 16 columns per pass, 4 passes
  const int w_r = tid & 63, w_kk = tid >> 6;   // W: 64 rows x 4 tones per pass, 4 passes
  size_t y_off[4], x_off[4];
  bool c_ok[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c = c0 + a_c + 16 * q;
    c_ok[q] = c < cols;
    y_off[q] = size_t(c) * N;
    x_off[q] = size_t(c_ok[q] ? c % p.K : 0) * N;
  }

  for (int t = blockIdx.z; t < p.T; t += gridDim.z) {
    const int set = p.soi ? p.soi[t] : 0;
    const size_t y_inst = size_t(t) * cols * N;
    if (set < 0 || set >= p.n_sets) {  // documented: out-of-range set -> NaN outputs
      const float qnan = __int_as_float(0x7fc00000);
      for (int e = tid; e < BM * rows; e += NT) {
        const int c = c0 + e / rows, i = e % rows;
        if (c < cols) p.h[y_inst + size_t(c) * N + g.o + r_base + i] = make_float2(qnan, qnan);
      }
      continue;
    }
    const float2 *__restrict__ Wt = p.Wt + size_t(set) * b * b;
    const float2 *__restrict__ yb = p.y + y_inst + g.a;
    const float2 *__restrict__ xb = p.x + size_t(t) * p.K * N + g.a;

    auto fetch = [&](int k0, Tile &f) {
      const int k = k0 + a_kk;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        f.y[q] = make_float2(0.f, 0.f);
        f.x[q] = make_float2(1.f, 0.f);
        if (c_ok[q] && k < b) {
          f.y[q] = __ldg(yb + y_off[q] + k);
          f.x[q] = __ldg(xb + x_off[q] + k);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int kw = k0 + w_kk + 4 * q;
        f.w[q] = make_float2(0.f, 0.f);
        if (w_r < rows && kw < b) f.w[q] = __ldg(Wt + size_t(kw) * b + row0 + w_r);
      }
    };
    auto stash = [&](int buf, const Tile &f) {
#pragma unroll
      for (int q = 0; q < 4; ++q) sm.k.As[buf][a_c + 16 * q][a_kk] = ls_div(f.y[q], f.x[q]);
#pragma unroll
      for (int q = 0; q < 4; ++q) sm.k.Ws[buf][w_kk + 4 * q][w_r] = f.w[q];
    };

    float acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.f;

    Tile f;
    fetch(0, f);
    __syncthreads();  // previous instance's readers are done with the shared buffers
    stash(0, f);
    __syncthreads();
    for (int kc = 0; kc < nk; ++kc) {
      const int buf = kc & 1;
      const int klim = b - kc * BK;  // >= BK except in the last chunk
      if (kc + 1 < nk) fetch((kc + 1) * BK, f);
      if (warp_active) {
#pragma unroll
        for (int kk = 0; kk < BK; kk += 2) {
          if (kk >= klim) break;  // warp-uniform: skip the zero padding of the K tail
          float4 av[4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            av[i] = *reinterpret_cast<const float4 *>(&sm.k.As[buf][wc * 32 + lc + 8 * i][kk]);
          float4 wv0[2], wv1[2];
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            wv0[jj] = *reinterpret_cast<const float4 *>(&sm.k.Ws[buf][kk][wr * 16 + lr * 4 + 2 * jj]);
            wv1[jj] = *reinterpret_cast<const float4 *>(&sm.k.Ws[buf][kk + 1][wr * 16 + lr * 4 + 2 * jj]);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float wr0 = (j & 1) ? wv0[j >> 1].z : wv0[j >> 1].x;
              const float wi0 = (j & 1) ? wv0[j >> 1].w : wv0[j >> 1].y;
              const float wr1 = (j & 1) ? wv1[j >> 1].z : wv1[j >> 1].x;
              const float wi1 = (j & 1) ? wv1[j >> 1].w : wv1[j >> 1].y;
              acc[i][j][0] = fmaf(wr0, av[i].x, acc[i][j][0]);
              acc[i][j][0] = fmaf(-wi0, av[i].y, acc[i][j][0]);
              acc[i][j][1] = fmaf(wr0, av[i].y, acc[i][j][1]);
              acc[i][j][1] = fmaf(wi0, av[i].x, acc[i][j][1]);
              acc[i][j][0] = fmaf(wr1, av[i].z, acc[i][j][0]);
              acc[i][j][0] = fmaf(-wi1, av[i].w, acc[i][j][0]);
              acc[i][j][1] = fmaf(wr1, av[i].w, acc[i][j][1]);
              acc[i][j][1] = fmaf(wi1, av[i].z, acc[i][j][1]);
            }
          }
        }
      }
      if (kc + 1 < nk) {
        stash(buf ^ 1, f);
        __syncthreads();
      }
    }

    // stage the 64 x 64 tile in shared memory, then write each column's kept rows contiguously
    __syncthreads();
    if (warp_active) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          sm.Cs[wc * 32 + lc + 8 * i][wr * 16 + lr * 4 + j] = make_float2(acc[i][j][0], acc[i][j][1]);
    }
    __syncthreads();
    float2 *hb = p.h + y_inst + g.o + r_base;
    for (int cc = warp; cc < BM; cc += NT / 32) {
      const int c = c0 + cc;
      if (c >= cols) break;
      for (int r = lane; r < rows; r += 32) hb[size_t(c) * N + r] = sm.Cs[cc][r];
    }
  }
}

}  // namespace

cudaError_t launch_contract_simt(const ContractArgs &a, cudaStream_t stream, int64_t *launches) {
  const int cols = a.M * a.K;
  const int row_tiles = (a.max_kept + BN - 1) / BN;
  const long long gy = (long long)a.n_win * row_tiles;
  if (gy > 65535) return cudaErrorInvalidConfiguration;
  dim3 grid((cols + BM - 1) / BM, unsigned(gy), unsigned(a.T < 65535 ? a.T : 65535));
  k2_simt<<<grid, NT, 0, stream>>>(a, row_tiles);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) ++*launches;
  return e;
}

}  // namespace ce
