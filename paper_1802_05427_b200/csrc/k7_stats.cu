// K7 -- statistics that feed the filter build, estimated from the received pilots (NEXT-3), and the C-ABI
// ce_stats_estimate of include/ce.h.
//
// The paper designs W from an ASSUMED path count L and SNR_fixed and fixes the
// detector's sigma^2 "for the lack of SNR estimation module".  Here, per statistic set s
// and from the LS estimates H_LS = y / x (Eq. 9) of every column c = (t, m, k) of the set's instances:
//   R_hat[d]   = sum_c sum_{n<N-d} H_LS[c,n+d] conj(H_LS[c,n]) / (C_s (N-d))            d < D
//   sigma2_hat = sum_c sum_{kappa in window} |IDFT_N(H_LS[c])[kappa]|^2 / (C_s B)     (unitary IDFT)
//   r_hat[d]   = R_hat[d] - sigma2_hat delta[d]
// The noise window is the B delay bins centred on N/2, far from the channel's delay support (reading D2).
//
// K7a: one CTA per cpb columns of one instance: the N twiddles exp(j 2 pi n / N) and, G columns at a time, the LS
// rows in shared memory; threads own blocks of 4 lags (x as many n-ranges as fit in 256 threads, partial sums
// carried in registers across the columns; skipped when K8 computes the lags) and then warps own (column,
// tone range) with one noise bin per lane (a per-32-tone Horner recursion); one FP64 reduction + atomics per
// CTA into the per-set accumulators.  K7b: one thread per (set, lag) normalises.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

#include "ce_internal.h"
#include "tc_ptx.cuh"

namespace ce {
namespace {

constexpr int K7_THREADS = 256;

constexpr int K7_CPB = 1;      // columns per CTA, same instance (measured on config 3: 1 -> 139 us, 2 -> 143, 8 -> 184)
constexpr int LB = 4;          // lags per thread

__device__ __forceinline__ float2 cmulf(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}

// packed FP32x2 (FFMA2): one instruction per complex multiply-add half, the scalar operand broadcast
__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 upk2(uint64_t v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
// z * w + v for complex z, w, v packed (re, im): w given as wab = (w.re, w.im), wba = (-w.im, w.re)
__device__ __forceinline__ uint64_t cmac2(uint64_t z, uint64_t wab, uint64_t wba, uint64_t v) {
  const float2 zf = upk2(z);
  return fma2(pk2(zf.x, zf.x), wab, fma2(pk2(zf.y, zf.y), wba, v));
}

// e^{+j 2 pi r / N} for 0 <= r < N (the exact integer reduction keeps the FP32 argument 2r/N in [0, 2))
__device__ __forceinline__ float2 twiddle(int r, int N) {
  float sv, cv;
  sincospif(2.0f * float(r) / float(N), &sv, &cv);
  return make_float2(cv, sv);
}

// ls rows are padded with zeros to NP = N rounded up to 32 tones (16-byte aligned, whole 32-tone noise blocks)
__global__ void __launch_bounds__(K7_THREADS) k7_accumulate(const float2 *__restrict__ y, const float2 *__restrict__ x,
                                                            int M, int K, int N, const int32_t *__restrict__ soi,
                                                            int n_sets, int D, int B, double *__restrict__ acc,
                                                            int lags, int cpb, int G, int noise) {
  extern __shared__ __align__(16) float2 sm7[];
  const int NP = (N + 31) & ~31;
  float2 *ls0 = sm7;                                 // [G][NP] LS rows of the resident columns
  float2 *tw = sm7 + size_t(G) * NP;                 // [N] exp(+j 2 pi n / N)
  __shared__ double part[2 * LB * K7_THREADS];       // [lag in block][thread][re, im]
  const int MK = M * K;
  const int n_cb = (MK + cpb - 1) / cpb;
  const int t = blockIdx.x / n_cb, c_lo = (blockIdx.x % n_cb) * cpb, c_hi = min(MK, c_lo + cpb);
  const int set = soi ? soi[t] : 0;
  if (set < 0 || set >= n_sets) return;              // out-of-range set: the instance is skipped
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    // FP32 twiddle (|error| < 2^-23); the exact reduction 2n/N in [0, 2) keeps the argument small
    float sv, cv;
    sincospif(2.0f * float(n) / float(N), &sv, &cv);
    tw[n] = make_float2(cv, sv);
  }
  double *acc_s = acc + size_t(set) * (2 * D + 2);   // [re, im] x D lags, noise power, column count
  // lag work split: thread -> (block of LB consecutive lags, n-range); partial sums stay in registers
  // across the CTA's columns and are reduced once at the end
  const int n_lb = (lags + LB - 1) / LB;               // 0 when K8 computes the lags on the tensor cores
  const int nparts = max(1, int(blockDim.x) / max(1, n_lb));
  const int lanes = blockDim.x / nparts;
  const int lb = int(threadIdx.x) % lanes, pr = int(threadIdx.x) / lanes;
  const bool lag_thread = lb < n_lb && pr < nparts && lanes >= n_lb;
  float re[LB] = {0.f, 0.f, 0.f, 0.f}, im[LB] = {0.f, 0.f, 0.f, 0.f};
  // noise work split: warp -> (resident column g, 32-tone-block range p), lane -> bin
  const int warp = int(threadIdx.x) >> 5, lane = int(threadIdx.x) & 31;
  const int nwarps = int(blockDim.x) >> 5;
  const int P = max(1, nwarps / G);                  // tone ranges per column
  const int g_w = warp % G, p_w = warp / G;
  const int nblk = NP / 32, bchunk = (nblk + P - 1) / P;
  const int blk0 = min(nblk, p_w * bchunk), blk1 = min(nblk, blk0 + bchunk);
  const int lo = N / 2 - B / 2;
  double pw = 0;
  for (int cg = c_lo; cg < c_hi; cg += G) {
    const int ng = min(G, c_hi - cg);
    __syncthreads();                                 // previous group's ls fully consumed
    for (int g = 0; g < ng; ++g) {
      const int c = cg + g;
      const float2 *yr = y + (size_t(t) * MK + c) * N;
      const float2 *xr = x + (size_t(t) * K + c % K) * N;
      float2 *ls = ls0 + size_t(g) * NP;
      for (int n = threadIdx.x; n < NP; n += blockDim.x) {
        float2 v = make_float2(0.f, 0.f);
        if (n < N) {
          const float2 yv = yr[n], xv = xr[n];
          const float inv = 1.0f / (xv.x * xv.x + xv.y * xv.y);
          v = make_float2((yv.x * xv.x + yv.y * xv.y) * inv, (yv.y * xv.x - yv.x * xv.y) * inv);
        }
        ls[n] = v;
      }
    }
    __syncthreads();
    // lags: ls[n] is shared by LB lags and ls[n+d..n+d+LB-1] slides (8 FMA per shared-memory read)
    for (int g = 0; g < ng && n_lb > 0; ++g) {
      const float2 *ls = ls0 + size_t(g) * NP;
      for (int l0 = 0; l0 < n_lb; l0 += lanes) {
        const int lbk = l0 + lb;
        if (lanes >= n_lb ? lag_thread : (lbk < n_lb && pr < nparts)) {
          const int d = lbk * LB;
          const int len = N - d, chunk = (len + nparts - 1) / nparts;
          const int n0 = pr * chunk, n1 = min(len, n0 + chunk);
          float2 win[LB];
#pragma unroll
          for (int i = 0; i < LB; ++i) win[i] = (n0 + d + i < N) ? ls[n0 + d + i] : make_float2(0.f, 0.f);
          // packed FFMA2: acc = (re, -im) of sum win * conj(b) += win.x (b.x, b.y) + win.y (b.y, -b.x); the two
          // packed forms of b are shared by the LB lags, the window components are broadcast scalar operands
          uint64_t acc4[LB] = {0ull, 0ull, 0ull, 0ull};
          for (int n = n0; n < n1; ++n) {
            const float2 bv = ls[n];
            const uint64_t bab = pk2(bv.x, bv.y), bba = pk2(bv.y, -bv.x);
#pragma unroll
            for (int i = 0; i < LB; ++i)             // win[i] = ls[n + d + i] (zero beyond N)
              acc4[i] = fma2(pk2(win[i].x, win[i].x), bab, fma2(pk2(win[i].y, win[i].y), bba, acc4[i]));
#pragma unroll
            for (int i = 0; i < LB - 1; ++i) win[i] = win[i + 1];
            win[LB - 1] = (n + d + LB < N) ? ls[n + d + LB] : make_float2(0.f, 0.f);
          }
          float r4[LB], i4[LB];
#pragma unroll
          for (int i = 0; i < LB; ++i) {
            const float2 a = upk2(acc4[i]);
            r4[i] = a.x;
            i4[i] = -a.y;
          }
          if (lanes >= n_lb) {
#pragma unroll
            for (int i = 0; i < LB; ++i) {
              re[i] += r4[i];
              im[i] += i4[i];
            }
          } else {                                   // D > 4 * 256: no register carry, add directly
            for (int i = 0; i < LB && d + i < D; ++i) {
              atomicAdd(&acc_s[2 * (d + i)], double(r4[i]));
              atomicAdd(&acc_s[2 * (d + i) + 1], double(i4[i]));
            }
          }
        }
      }
    }
    // noise window X[kap] = sum_n ls[n] e^{+j 2 pi n kap / N}: per 32-tone block a Horner recursion in w = e^{j 2 pi
    // kap / N} (two chains, even and odd tones, in w^2: 4 FMA per tone, ls read as broadcast 2-tone vectors), the
    // block's sum rotated by the tabled e^{j 2 pi 32 blk kap / N}; the complex partial sums of a bin are combined
    // before taking |.|^2
    const float2 *lsw = ls0 + size_t(g_w) * NP;
    for (int b0 = 0; b0 < (noise ? B : 0); b0 += 32) {
      const int bin = b0 + lane;
      const int kap = lo + min(bin, B - 1);
      const float2 w1 = tw[kap], w2 = cmulf(w1, w1);
      const int step = int((32LL * kap) % N);
      int idx = int((32LL * blk0 * kap) % N);
      float xr = 0.f, xi = 0.f;
      if (g_w < ng) {
        for (int blk = blk0; blk < blk1; ++blk) {
          const float4 *vp = reinterpret_cast<const float4 *>(lsw + blk * 32);
          float4 v = vp[15];                         // tones 30 (x, y) and 31 (z, w)
          float er = v.x, ei = v.y, orr = v.z, oi = v.w;
#pragma unroll
          for (int q = 14; q >= 0; --q) {
            v = vp[q];
            const float ner = fmaf(er, w2.x, fmaf(-ei, w2.y, v.x));
            const float nei = fmaf(er, w2.y, fmaf(ei, w2.x, v.y));
            const float nor = fmaf(orr, w2.x, fmaf(-oi, w2.y, v.z));
            const float noi = fmaf(orr, w2.y, fmaf(oi, w2.x, v.w));
            er = ner; ei = nei; orr = nor; oi = noi;
          }
          const float pr_ = er + fmaf(orr, w1.x, -oi * w1.y), pi_ = ei + fmaf(orr, w1.y, oi * w1.x);
          const float2 s = tw[idx];
          xr = fmaf(s.x, pr_, fmaf(-s.y, pi_, xr));
          xi = fmaf(s.x, pi_, fmaf(s.y, pr_, xi));
          idx += step;
          if (idx >= N) idx -= N;
        }
      }
      if (P == 1) {
        if (bin < B && g_w < ng) pw += double(xr) * xr + double(xi) * xi;
      } else {
        __syncthreads();                             // part[] free
        part[2 * threadIdx.x] = xr;
        part[2 * threadIdx.x + 1] = xi;
        __syncthreads();
        if (p_w == 0 && bin < B && g_w < ng) {
          double sr = 0, si = 0;
          for (int q = 0; q < P; ++q) {
            sr += part[2 * ((q * G + g_w) * 32 + lane)];
            si += part[2 * ((q * G + g_w) * 32 + lane) + 1];
          }
          pw += sr * sr + si * si;
        }
      }
    }
  }
  // one reduction and one set of atomics per CTA
  __syncthreads();
#pragma unroll
  for (int i = 0; i < LB; ++i) {
    part[2 * (i * K7_THREADS + threadIdx.x)] = re[i];
    part[2 * (i * K7_THREADS + threadIdx.x) + 1] = im[i];
  }
  __syncthreads();
  if (lanes >= n_lb && threadIdx.x < n_lb) {
    for (int i = 0; i < LB; ++i) {
      const int dd = int(threadIdx.x) * LB + i;
      if (dd >= D) break;
      double sr = 0, si = 0;
      for (int q = 0; q < nparts; ++q) {
        sr += part[2 * (i * K7_THREADS + q * lanes + threadIdx.x)];
        si += part[2 * (i * K7_THREADS + q * lanes + threadIdx.x) + 1];
      }
      atomicAdd(&acc_s[2 * dd], sr);
      atomicAdd(&acc_s[2 * dd + 1], si);
    }
  }
  if (!noise) return;                                // K7c adds the noise floor and the column count
  __syncthreads();
  part[threadIdx.x] = pw;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) part[threadIdx.x] += part[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    atomicAdd(&acc_s[2 * D], part[0] / N);            // unitary IDFT: |sum|^2 / N
    atomicAdd(&acc_s[2 * D + 1], double(c_hi - c_lo));
  }
}

// K7c -- the noise window on its own, streamed: one CTA per (instance t, user k, range of antennas m), so one x
// row (the LS factors conj(x)/|x|^2) serves all its columns c = (m, k).  Each warp owns every 8th group of 4
// columns of the range and streams the group's y rows in 128-tone chunks into its own 2-deep ring by 1-D bulk
// copies (no CTA barrier in the loop), converts the chunk to LS values in place, then runs a per-block (64-tone) Horner
// recursion: lane l works on column l / 8 of the group and on NB bins (l % 8) + 8 j, so every broadcast 2-tone
// shared-memory read (a quarter-warp per column) feeds 4 NB FMAs -- broadcast 16-byte reads cost one wavefront
// per quarter-warp, so one bin per lane left the kernel bound by shared-memory wavefronts.  Bins beyond 8 NB run
// in further passes over the columns.  Needs N even and y 16-byte aligned (whole 16-byte bulk copies).
constexpr int NZ_CH = 128;     // tones per chunk
constexpr int NZ_CPW = 4;      // columns per warp job
constexpr int NZ_R = 2;        // chunks in flight per warp
constexpr int NZ_WARPS = 8;
constexpr int NZ_NB = 4;       // bins per lane per pass (8 NB bins per pass)
#ifndef K7C_BLK
#define K7C_BLK 64
#endif
constexpr int NZ_BLK = K7C_BLK; // tones per Horner block (the per-block rotation and sum are the overhead)

__global__ void __launch_bounds__(NZ_WARPS * 32) k7_noise(const float2 *__restrict__ y, const float2 *__restrict__ x,
                                                          int M, int K, int N, const int32_t *__restrict__ soi,
                                                          int n_sets, int D, int B, double *__restrict__ acc, int mpb) {
  constexpr int NB = NZ_NB;
  extern __shared__ __align__(128) unsigned char smz[];
  const int nch = (N + NZ_CH - 1) / NZ_CH;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smz);                  // [warp][R]
  float2 *ring = reinterpret_cast<float2 *>(smz + 1024);               // [warp][R][CPW][CH]
  float2 *fac = ring + NZ_WARPS * NZ_R * NZ_CPW * NZ_CH;               // [nch * CH] conj(x)/|x|^2, zero beyond N
  const int n_mc = (M + mpb - 1) / mpb;
  const int mc = blockIdx.x % n_mc, tk = blockIdx.x / n_mc, k = tk % K, t = tk / K;
  const int set = soi ? soi[t] : 0;
  if (set < 0 || set >= n_sets) return;              // out-of-range set: the instance is skipped
  const int warp = int(threadIdx.x) >> 5, lane = int(threadIdx.x) & 31;
  const int MK = M * K;
  const int m_lo = mc * mpb, m_hi = min(M, m_lo + mpb);
  const int ngrp = (m_hi - m_lo + NZ_CPW - 1) / NZ_CPW;
  const int ngrp_w = max(0, (ngrp - warp + NZ_WARPS - 1) / NZ_WARPS);
  const int npass = (B + 8 * NB - 1) / (8 * NB);     // bins per pass 8 NB; the columns are re-streamed per pass
  const int jpp = ngrp_w * nch;                       // jobs (column group, chunk) per pass
  const int jobs = npass * jpp;
  uint64_t *wb = bars + warp * NZ_R;
  float2 *wr = ring + size_t(warp) * NZ_R * NZ_CPW * NZ_CH;
  auto issue = [&](int j) {                          // lane 0: job j into slot j % R
    const int ch = j % nch, m0 = m_lo + NZ_CPW * (warp + NZ_WARPS * ((j % jpp) / nch));
    const int nv = min(NZ_CPW, m_hi - m0);
    const uint32_t bytes = uint32_t(min(NZ_CH, N - ch * NZ_CH)) * 8u;
    uint64_t *bar = &wb[j % NZ_R];
    mbar_arrive_expect_tx(bar, bytes * uint32_t(nv));
    for (int i = 0; i < nv; ++i) {
      const float2 *src = y + (size_t(t) * MK + size_t(m0 + i) * K + k) * N + size_t(ch) * NZ_CH;
      bulk_g2s(wr + ((j % NZ_R) * NZ_CPW + i) * NZ_CH, src, bytes, bar);
    }
  };
  if (lane == 0) {
    for (int s = 0; s < NZ_R; ++s) mbar_init(&wb[s], 1);
    fence_proxy_async();
  }
  __syncwarp();
  if (lane == 0)
    for (int j = 0; j < min(NZ_R, jobs); ++j) issue(j);
  const float2 *xr = x + (size_t(t) * K + k) * N;
  for (int n = threadIdx.x; n < nch * NZ_CH; n += blockDim.x) {
    float2 f = make_float2(0.f, 0.f);
    if (n < N) {
      const float2 xv = xr[n];
      const float inv = 1.0f / (xv.x * xv.x + xv.y * xv.y);
      f = make_float2(xv.x * inv, -xv.y * inv);
    }
    fac[n] = f;
  }
  __syncthreads();
  const int lo = N / 2 - B / 2;
  const int ci = lane >> 3, bl = lane & 7;            // column of the group, bin lane
  float2 w1[NB], w32[NB];
  uint64_t w2ab[NB], w2ba[NB];
  int kap[NB];
  float xr_[NB], xi_[NB];
  float2 rot[NB];
  int bin0 = 0;
  double pw = 0;
  for (int j = 0; j < jobs; ++j) {
    const int s = j % NZ_R, ch = j % nch;
    if (j % jpp == 0) {                              // a pass starts: bins bin0 .. bin0 + 8 NB - 1
      bin0 = (j / jpp) * 8 * NB;
#pragma unroll
      for (int g = 0; g < NB; ++g) {
        kap[g] = lo + min(bin0 + bl + 8 * g, B - 1);
        w1[g] = twiddle(kap[g], N);
        const float2 w2 = cmulf(w1[g], w1[g]);
        w2ab[g] = pk2(w2.x, w2.y);
        w2ba[g] = pk2(-w2.y, w2.x);
        w32[g] = twiddle(int((static_cast<long long>(NZ_BLK) * kap[g]) % N), N);
        xr_[g] = xi_[g] = 0.f;
      }
    }
    mbar_wait(&wb[s], uint32_t(j / NZ_R) & 1u);
    float2 *rb = wr + s * NZ_CPW * NZ_CH;
    const int m0 = m_lo + NZ_CPW * (warp + NZ_WARPS * ((j % jpp) / nch));
    const int nv = min(NZ_CPW, m_hi - m0);
    const int n0 = ch * NZ_CH, len = min(NZ_CH, N - n0);
#pragma unroll 4
    for (int e = 2 * lane; e < NZ_CPW * NZ_CH; e += 64) {   // LS values in place, 2 tones per access (len is even);
      const int i = e / NZ_CH, nn = e % NZ_CH;              // zero beyond N and for absent columns
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i < nv && nn < len) {
        const float4 r = *reinterpret_cast<const float4 *>(rb + e), f = *reinterpret_cast<const float4 *>(fac + n0 + nn);
        const float2 a = cmulf(make_float2(r.x, r.y), make_float2(f.x, f.y)), b = cmulf(make_float2(r.z, r.w), make_float2(f.z, f.w));
        v = make_float4(a.x, a.y, b.x, b.y);
      }
      *reinterpret_cast<float4 *>(rb + e) = v;
    }
    __syncwarp();
    const int nb = (len + NZ_BLK - 1) / NZ_BLK;   // zero-padded to whole blocks by the conversion
    const float2 *rc = rb + ci * NZ_CH;
    // rot = e^{j 2 pi n kap / N} at the block start n: 1 at the column start, advanced by e^{j 2 pi 32 kap / N} per
    // block and re-seeded exactly every 8 chunks (at most 8 CH / NZ_BLK FP32 rotation steps between exact values)
    if (ch % 8 == 0) {
#pragma unroll
      for (int g = 0; g < NB; ++g)
        rot[g] = ch == 0 ? make_float2(1.f, 0.f) : twiddle(int((static_cast<long long>(n0) * kap[g]) % N), N);
    }
    for (int bb = 0; bb < nb; ++bb) {
      const ulonglong2 *vp = reinterpret_cast<const ulonglong2 *>(rc + bb * NZ_BLK);   // (tone 2q, tone 2q+1)
      uint64_t ev[NB], od[NB];                       // even / odd tone chains, packed (re, im)
      ulonglong2 v = vp[NZ_BLK / 2 - 1];             // the block's last two tones
#pragma unroll
      for (int g = 0; g < NB; ++g) {
        ev[g] = v.x;
        od[g] = v.y;
      }
#pragma unroll
      for (int q = NZ_BLK / 2 - 2; q >= 0; --q) {
        v = vp[q];
#pragma unroll
        for (int g = 0; g < NB; ++g) {
          ev[g] = cmac2(ev[g], w2ab[g], w2ba[g], v.x);
          od[g] = cmac2(od[g], w2ab[g], w2ba[g], v.y);
        }
      }
#pragma unroll
      for (int g = 0; g < NB; ++g) {
        const float2 e2 = upk2(ev[g]), o2 = upk2(od[g]);
        const float pr_ = e2.x + fmaf(o2.x, w1[g].x, -o2.y * w1[g].y);
        const float pi_ = e2.y + fmaf(o2.x, w1[g].y, o2.y * w1[g].x);
        const float2 sv = rot[g];
        xr_[g] = fmaf(sv.x, pr_, fmaf(-sv.y, pi_, xr_[g]));
        xi_[g] = fmaf(sv.x, pi_, fmaf(sv.y, pr_, xi_[g]));
        rot[g] = cmulf(rot[g], w32[g]);
      }
    }
    fence_proxy_async();                             // the in-place writes before the slot's next bulk copy
    __syncwarp();
    if (lane == 0 && j + NZ_R < jobs) issue(j + NZ_R);
    if (ch == nch - 1) {                             // the group's columns complete
#pragma unroll
      for (int g = 0; g < NB; ++g) {
        if (ci < nv && bin0 + bl + 8 * g < B) pw += double(xr_[g]) * xr_[g] + double(xi_[g]) * xi_[g];
        xr_[g] = xi_[g] = 0.f;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pw += __shfl_xor_sync(0xffffffffu, pw, o);
  __shared__ double wpw[NZ_WARPS];
  if (lane == 0) wpw[warp] = pw;
  __syncthreads();
  if (threadIdx.x == 0) {
    double sum = 0;
    for (int w = 0; w < NZ_WARPS; ++w) sum += wpw[w];
    double *acc_s = acc + size_t(set) * (2 * D + 2);
    atomicAdd(&acc_s[2 * D], sum / N);                // unitary IDFT: |sum|^2 / N
    atomicAdd(&acc_s[2 * D + 1], double(m_hi - m_lo));
  }
}

// one thread per (set, lag), lag D standing for sigma^2
__global__ void k7_finalize(const double *__restrict__ acc, int n_sets, int N, int D, int B, double *__restrict__ r,
                            double *__restrict__ sigma2) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)n_sets * (D + 1)) return;
  const int s = int(i / (D + 1)), d = int(i % (D + 1));
  const double *a = acc + size_t(s) * (2 * D + 2);
  const double C = a[2 * D + 1];
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  const double s2 = C > 0 ? a[2 * D] / (C * B) : nan;
  if (d == D) {
    sigma2[s] = s2;
    return;
  }
  const double den = C * (N - d);
  r[(size_t(s) * D + d) * 2] = C > 0 ? a[2 * d] / den - (d == 0 ? s2 : 0.0) : nan;
  r[(size_t(s) * D + d) * 2 + 1] = C > 0 ? a[2 * d + 1] / den : nan;
}

}  // namespace
}  // namespace ce

namespace {
// workspace layout: the per-set accumulators (K7's layout) then, 256-byte aligned, K9's per-set spectra
size_t stats_acc_bytes(int32_t n_sets, int32_t D) {
  return ((size_t(n_sets) * (2 * size_t(D) + 2) * sizeof(double)) + 255) & ~size_t(255);
}
size_t stats_spectrum_bytes(int32_t N, int32_t n_sets, int32_t D) {
  const int l = ce::spectrum_log2(N, D);
  return ((l < 0 ? 0 : size_t(n_sets) * (size_t(1) << l) * sizeof(double)) + 255) & ~size_t(255);
}
// K4's inverse-DFT bank for the noise window: hi and lo bf16 planes
size_t stats_bank_plane_bytes(int32_t N, int32_t B) {
  int32_t nkc, NR;
  ce::dft_bank_shape(N, B, &nkc, &NR);
  return ((size_t(nkc) * NR * 32 * sizeof(uint16_t)) + 255) & ~size_t(255);
}
constexpr int32_t K4_NOISE_MAX_B = 32 * 128;   // windows of 128 bins carried in K4's kernel parameters
}  // namespace

extern "C" {

int ce_stats_workspace_bytes(int32_t N, int32_t n_sets, int32_t D, int32_t B, int64_t *out) {
  if (out == nullptr || N < 2 || n_sets < 1 || D < 1 || B < 1) {
    ce::set_last_error("ce_stats_workspace_bytes: need N >= 2, n_sets >= 1, D >= 1, B >= 1, out != NULL");
    return CE_EINVAL;
  }
  *out = int64_t(stats_acc_bytes(n_sets, D) + stats_spectrum_bytes(N, n_sets, D) +
                 (B <= K4_NOISE_MAX_B ? 2 * stats_bank_plane_bytes(N, B) : 0));
  return CE_OK;
}

int ce_stats_estimate(const void *d_y, const void *d_x, int32_t T, int32_t M, int32_t K, int32_t N,
                      const int32_t *d_set_of_instance, int32_t n_sets, int32_t D, int32_t B, void *d_r,
                      void *d_sigma2, void *d_work, void *stream) {
  auto fail = [](int st, const char *m) {
    ce::set_last_error(m);
    return st;
  };
  if (!d_y || !d_x || !d_r || !d_sigma2 || !d_work) return fail(CE_EINVAL, "ce_stats_estimate: NULL pointer");
  if (T < 1 || M < 1 || K < 1 || N < 2 || n_sets < 1) return fail(CE_EINVAL, "ce_stats_estimate: bad sizes");
  if (D < 1 || D > N || D > 4096 || B < 1 || B > N) return fail(CE_EINVAL, "ce_stats_estimate: need 1 <= D, B <= N");
  if ((reinterpret_cast<uintptr_t>(d_y) | reinterpret_cast<uintptr_t>(d_x)) & 7u)
    return fail(CE_EINVAL, "ce_stats_estimate: y, x must be 8-byte aligned");
  if ((reinterpret_cast<uintptr_t>(d_r) | reinterpret_cast<uintptr_t>(d_sigma2) | reinterpret_cast<uintptr_t>(d_work)) & 7u)
    return fail(CE_EINVAL, "ce_stats_estimate: outputs / workspace must be 8-byte aligned");
  const long long cols = (long long)T * M * K;
  // columns per CTA: 1 when K7 also runs the lags (measured: more is slower there); with the lags on K8 the
  // per-CTA twiddle table and row-load latency are amortised over several columns
  static const int env_cpb = getenv("CE_K7_CPB") ? atoi(getenv("CE_K7_CPB")) : 0;   // experiments
  static const int env_gram = getenv("CE_K8_GRAM") ? atoi(getenv("CE_K8_GRAM")) : -1;   // experiments: 0 off, 1 force
  const bool gram = env_gram != 0;
  // K8 pays a per-unit factor table and diagonal-bin epilogue: measured faster from config 4's 61440 columns
  // up (config 4: 2.4 vs 4.1 ms, config 5: 9.7 vs 17.2 ms) and slower on config 3's 1536 (164 vs 147 us)
  const bool k8 = gram && (cols >= 16384 || env_gram == 1) && ce::gram_launchable(static_cast<const float2 *>(d_y), K, N, D);
  static const int env_k9 = getenv("CE_K9") ? atoi(getenv("CE_K9")) : -1;   // experiments: 0 off
  const bool k9 = env_k9 != 0 && ce::spectrum_log2(N, D) >= 0 && n_sets <= 65535;
  int cpb = (k8 || k9) ? 8 : ce::K7_CPB;
  if (env_cpb > 0) cpb = env_cpb;
  cpb = std::max(1, std::min(cpb, M * K));
  const long long ctas = (long long)T * ((static_cast<long long>(M) * K + cpb - 1) / cpb);
  if (cols > 0x7fffffffLL || ctas > 0x7fffffffLL) return fail(CE_EINVAL, "ce_stats_estimate: too many columns");
  // resident LS rows per CTA (1, 2, 4 or 8: whole warps per column in the noise window), bounded by shared memory
  const int NP = (N + 31) & ~31;
  if (size_t(NP + N) * sizeof(float2) > 200 * 1024) return fail(CE_EINVAL, "ce_stats_estimate: N too large (N <= 12800)");
  int G = 1;
  while (G < 8 && 2 * G <= cpb && size_t(2 * G * NP + N) * sizeof(float2) <= 200 * 1024) G *= 2;
  const size_t smem = size_t(G * NP + N) * sizeof(float2);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double *acc = static_cast<double *>(d_work);
  cudaError_t e = cudaMemsetAsync(acc, 0, size_t(n_sets) * (2 * D + 2) * sizeof(double), st);
  // K7a also holds static shared memory: ce::smem_opt_in reads its size from the compiled kernel
  if (e == cudaSuccess) e = ce::smem_opt_in((const void *)ce::k7_accumulate, smem);
  if (e != cudaSuccess) {
    ce::set_last_error(std::string("ce_stats_estimate: ") + cudaGetErrorString(e));
    return CE_ECUDA;
  }
  // the lag correlation: through the power spectrum (K9, FFT of the zero-padded LS rows) when L = 2^l >= N + D - 1
  // fits 8192, else on the tensor cores (K8) from 16384 columns, else inside K7a's pass (direct sums); K7 then adds
  // the noise floor and the column count
  int k7_lags = D;
  if (k9) {
    double *P = reinterpret_cast<double *>(static_cast<char *>(d_work) + stats_acc_bytes(n_sets, D));
    e = ce::launch_spectrum_lags(static_cast<const float2 *>(d_y), static_cast<const float2 *>(d_x), T, M, K, N,
                                 d_set_of_instance, n_sets, D, P, acc, st);
    if (e != cudaSuccess) {
      ce::set_last_error(std::string("ce_stats_estimate: K9 launch: ") + cudaGetErrorString(e));
      return CE_ECUDA;
    }
    k7_lags = 0;
  } else if (k8) {
    e = ce::launch_gram(static_cast<const float2 *>(d_y), static_cast<const float2 *>(d_x), T, M, K, N,
                        d_set_of_instance, n_sets, D, acc, st);
    if (e != cudaSuccess) {
      ce::set_last_error(std::string("ce_stats_estimate: K8 launch: ") + cudaGetErrorString(e));
      return CE_ECUDA;
    }
    k7_lags = 0;
  }
  // the noise window when the lags ran elsewhere: on the tensor cores by K4 in power mode (the unitary inverse DFT at
  // the B bins as a BF16x3 bank, LS division fused, sum of |.|^2 per set; needs K4's TMA conditions), else streamed
  // by K7c (N even, y 16-byte aligned; bins in passes of 32), else inside K7a's pass (measured: K7a alone 116 us vs
  // K7a lags + K7c 133 us on config 3; with K8, config 4 2.15 -> 1.60 ms, config 5 11.9 -> 6.1 ms)
  static const int env_nz = getenv("CE_K7_NOISE") ? atoi(getenv("CE_K7_NOISE")) : -1;   // experiments: 0 off, 1 force
  static const int env_mpb = getenv("CE_K7_MPB") ? atoi(getenv("CE_K7_MPB")) : 0;
  static const int env_k4n = getenv("CE_K4_NOISE") ? atoi(getenv("CE_K4_NOISE")) : -1;   // experiments: 0 off
  std::vector<ce::Window> nwin;
  for (int32_t o = 0; o < B; o += 128) nwin.push_back(ce::Window{0, o, std::min(B, o + 128)});
  ce::ContractArgs na;
  na.y = static_cast<const float2 *>(d_y);
  na.x = static_cast<const float2 *>(d_x);
  na.h = nullptr;
  na.Wt = nullptr;
  na.geo = nullptr;
  na.geo_host = nwin.data();
  na.soi = d_set_of_instance;
  na.T = T;
  na.M = M;
  na.K = K;
  na.N = N;
  na.b = N;
  na.n_win = int32_t(nwin.size());
  na.n_sets = n_sets;
  na.max_kept = std::min(B, 128);
  na.even_starts = true;
  na.pow_acc = acc + 2 * D;
  na.pow_stride = 2 * D + 2;
  int32_t bank_nkc = 0, bank_NR = 0;
  ce::dft_bank_shape(N, B, &bank_nkc, &bank_NR);
  na.bank_rows = bank_NR;
  na.bank_shared = true;
  const bool k4n = env_k4n != 0 && env_nz != 1 && k7_lags == 0 && B <= K4_NOISE_MAX_B && ce::bf16x3_launchable(na);
  if (k4n) {
    char *wb = static_cast<char *>(d_work) + stats_acc_bytes(n_sets, D) + stats_spectrum_bytes(N, n_sets, D);
    uint16_t *bank_hi = reinterpret_cast<uint16_t *>(wb);
    uint16_t *bank_lo = reinterpret_cast<uint16_t *>(wb + stats_bank_plane_bytes(N, B));
    e = ce::launch_build_dft_bank(N, B, N / 2 - B / 2, bank_hi, bank_lo, st);
    int64_t nl = 0;
    if (e == cudaSuccess) e = ce::launch_contract_bf16x3(na, bank_hi, bank_lo, st, &nl);
    if (e != cudaSuccess) {
      ce::set_last_error(std::string("ce_stats_estimate: K4 noise-window launch: ") + cudaGetErrorString(e));
      return CE_ECUDA;
    }
  }
  const bool k7c = !k4n && (env_nz == 1 || (env_nz != 0 && k7_lags == 0)) && N % 2 == 0 &&
                   (reinterpret_cast<uintptr_t>(d_y) & 15u) == 0;
  if (!k4n && (k7_lags > 0 || !k7c)) {   // K7a: the lags (unless K9 / K8 ran) and the noise window (unless K7c runs)
    ce::k7_accumulate<<<unsigned(ctas), ce::K7_THREADS, smem, st>>>(static_cast<const float2 *>(d_y),
                                                                    static_cast<const float2 *>(d_x), M, K, N,
                                                                    d_set_of_instance, n_sets, D, B, acc, k7_lags, cpb,
                                                                    G, k7c ? 0 : 1);
  }
  if (k7c) {
    const int nch = (N + ce::NZ_CH - 1) / ce::NZ_CH;
    const size_t zsm = 1024 + size_t(ce::NZ_WARPS) * ce::NZ_R * ce::NZ_CPW * ce::NZ_CH * 8 + size_t(nch) * ce::NZ_CH * 8;
    if (zsm > 200 * 1024) return fail(CE_EINVAL, "ce_stats_estimate: N too large for the noise kernel");
    // antennas per CTA: enough CTAs for several waves, whole warps of 4-column groups
    int nsm = 148;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    int mpb = env_mpb > 0 ? env_mpb
                          : int(std::min<long long>(M, std::max<long long>(32, (cols / (long long)(nsm * 12)) & ~31LL)));
    mpb = std::max(1, std::min(mpb, M));
    const long long zctas = (long long)T * K * ((M + mpb - 1) / mpb);
    if (zctas > 0x7fffffffLL) return fail(CE_EINVAL, "ce_stats_estimate: too many columns");
    e = ce::smem_opt_in((const void *)ce::k7_noise, zsm);
    if (e != cudaSuccess) {
      ce::set_last_error(std::string("ce_stats_estimate: ") + cudaGetErrorString(e));
      return CE_ECUDA;
    }
    ce::k7_noise<<<unsigned(zctas), ce::NZ_WARPS * 32, zsm, st>>>(static_cast<const float2 *>(d_y),
                                                                  static_cast<const float2 *>(d_x), M, K, N,
                                                                  d_set_of_instance, n_sets, D, B, acc, mpb);
  }
  ce::k7_finalize<<<unsigned((static_cast<long long>(n_sets) * (D + 1) + 127) / 128), 128, 0, st>>>(acc, n_sets, N, D, B, static_cast<double *>(d_r),
                                                       static_cast<double *>(d_sigma2));
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    ce::set_last_error(std::string("ce_stats_estimate: launch: ") + cudaGetErrorString(e));
    return CE_ECUDA;
  }
  return CE_OK;
}

}  // extern "C"
