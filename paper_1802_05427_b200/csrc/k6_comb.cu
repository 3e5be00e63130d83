// K6 -- the paper's own comb-pilot grouped LMMSE estimators (3W-LMMSE / 12W-LMMSE, NEXT-1), plus the
// C-ABI of include/ce.h's ce_comb_* entry points.
//
//   comb pilots          UE s owns tones S*j + s                       PAPER.md:85 (Fig. fig1), Eq. 6
//   LS at its pilots     H_LS = Y / X                                  PAPER.md:179 (Eq. 9)
//   group weights        W = R_{H,H_LS} (R_{H_LS,H_LS} + sigma^2 I)^-1  PAPER.md:306-309 (Eq. 17)
//   3W mapping           3 outputs / group, 3 weights for all UEs      PAPER.md:345-385 (Table I, Eq. W1-W3, P)
//   12W mapping          S outputs / group, 12 weights per UE          PAPER.md:400-403 (Table II)
//   zero-order hold      un-estimated tones hold the last estimate
//
// Geometry (readings C1-C4): K = N/S pilots per UE; group g (one per pilot position) uses the
// pilot window [a_g, a_g + G), a_g = clamp(g - (G-1)/2, 0, K - G) -- the main path's window rule in pilot
// units, stride 1 -- and weight type g - a_g.  Output tones of group g: S*g + q (full / 12W, q < S) or
// S*g + s + (S/G) q (sub / 3W, q < G).
//
// K6a (filter build, FP64): one CTA per (UE, type): A = R_pp + sigma^2 I (G x G, Toeplitz at pilot
// spacing), Cholesky, W^H = A^-1 R_{in,out} by two triangular solves per output column.
// K6b (estimate, FP32 SIMT): one CTA per received row (t, m): the row and the comb pilot symbol go to
// shared memory, LS is formed for every tone (each tone is some UE's pilot), then every thread produces
// outputs h[t][m][s][k] = sum_j W[s][type][q][j] LS[S(a+j)+s] (3W: at the held tone e(k)), written
// coalesced along k.  The op is HBM-bound on the n_ue x N output row (8 B per estimate).
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <cmath>
#include <new>
#include <string>

#include "ce_internal.h"

namespace ce {
namespace {

constexpr int GMAX = 32;     // pilots per group window
constexpr int OMAX = 64;     // outputs per group (S in full mode)

struct CombGeo {
  int N, S, n_ue, G, mode, K, n_out, n_ue_f, ml;
};

__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {   // a * conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ double2 rhh(const double2 *r, int d) {    // r_d, r_{-d} = conj(r_d)
  if (d >= 0) return r[d];
  const double2 v = r[-d];
  return make_double2(v.x, -v.y);
}

// K6a: one CTA (32 threads) per (UE filter index sf, type).
__global__ void k6_build(const double2 *__restrict__ r, double sigma2, CombGeo g, float2 *__restrict__ W,
                         int32_t *__restrict__ flag) {
  __shared__ double2 L[GMAX][GMAX];
  __shared__ double2 Z[GMAX][OMAX];
  const int sf = blockIdx.x, typ = blockIdx.y, tid = threadIdx.x;
  const int s = sf;                                    // sub mode: sf = 0 (UE-independent weights)
  const int G = g.G;
  // relative tones (window start = tone 0): inputs S*j + s, outputs S*typ + q or S*typ + s + (S/G) q
  for (int e = tid; e < G * G; e += blockDim.x) {
    const int i = e / G, j = e % G;
    double2 v = rhh(r, g.S * (i - j));
    if (i == j) v.x += sigma2;
    L[i][j] = v;
  }
  for (int e = tid; e < G * g.n_out; e += blockDim.x) {
    const int j = e / g.n_out, q = e % g.n_out;
    const int out = g.mode == 0 ? g.S * typ + q : g.S * typ + s + (g.S / G) * q;
    const int in = g.S * j + s;
    Z[j][q] = rhh(r, in - out);                         // R[in, out] = conj(R[out, in])
  }
  __syncthreads();
  if (tid == 0) {                                       // Cholesky A = L L^H (lower, in place)
    for (int k = 0; k < G; ++k) {
      double d = L[k][k].x;
      for (int p = 0; p < k; ++p) d -= L[k][p].x * L[k][p].x + L[k][p].y * L[k][p].y;
      if (!(d > 0.0) || !isfinite(d)) {
        atomicOr(flag, 1);
        d = 1.0;
      }
      const double lkk = sqrt(d);
      L[k][k] = make_double2(lkk, 0.0);
      for (int i = k + 1; i < G; ++i) {
        double2 v = L[i][k];
        for (int p = 0; p < k; ++p) {
          const double2 t = cmulc(L[i][p], L[k][p]);
          v.x -= t.x;
          v.y -= t.y;
        }
        L[i][k] = make_double2(v.x / lkk, v.y / lkk);
      }
    }
  }
  __syncthreads();
  for (int q = tid; q < g.n_out; q += blockDim.x) {     // solve L L^H z = R[in, out_q]
    for (int i = 0; i < G; ++i) {
      double2 v = Z[i][q];
      for (int p = 0; p < i; ++p) {
        const double2 l = L[i][p], z = Z[p][q];
        v.x -= l.x * z.x - l.y * z.y;
        v.y -= l.x * z.y + l.y * z.x;
      }
      Z[i][q] = make_double2(v.x / L[i][i].x, v.y / L[i][i].x);
    }
    for (int i = G - 1; i >= 0; --i) {
      double2 v = Z[i][q];
      for (int p = i + 1; p < G; ++p) {
        const double2 t = cmulc(Z[p][q], L[p][i]);     // conj(L[p][i]) * z_p
        v.x -= t.x;
        v.y -= t.y;
      }
      Z[i][q] = make_double2(v.x / L[i][i].x, v.y / L[i][i].x);
    }
    // W[q][j] = conj(Z[j][q])
    float2 *Wq = W + ((size_t(sf) * G + typ) * g.n_out + q) * G;
    for (int j = 0; j < G; ++j) Wq[j] = make_float2(float(Z[j][q].x), float(-Z[j][q].y));
  }
}

// K6b (generic shapes): one CTA per row (t, m).
__global__ void __launch_bounds__(256) k6_estimate(const float2 *__restrict__ y, const float2 *__restrict__ x,
                                                   const float2 *__restrict__ W, float2 *__restrict__ h, int M,
                                                   CombGeo g) {
  extern __shared__ float2 ls[];                        // [N]
  const int row = blockIdx.x;                           // t * M + m
  const int t = row / M;
  const float2 *yr = y + size_t(row) * g.N;
  const float2 *xr = x + size_t(t) * g.N;
  for (int k = threadIdx.x; k < g.N; k += blockDim.x) {
    const float2 yv = yr[k], xv = xr[k];
    const float inv = 1.0f / (xv.x * xv.x + xv.y * xv.y);
    ls[k] = make_float2((yv.x * xv.x + yv.y * xv.y) * inv, (yv.y * xv.x - yv.x * xv.y) * inv);
  }
  __syncthreads();
  const int G = g.G, S = g.S, K = g.K;
  const int step = g.mode == 0 ? 1 : S / G;             // sub: estimated tones every S/G
  for (int e = threadIdx.x; e < g.n_ue * g.N; e += blockDim.x) {
    const int s = e / g.N, k = e % g.N;
    int gq, q;                                          // group and output index of the (held) tone
    if (g.mode == 0) {
      gq = k / S;
      q = k % S;
    } else {
      const int i = k >= s ? (k - s) / step : 0;        // ZOH: last estimated tone <= k (first if none)
      gq = i / G;
      q = i % G;
    }
    const int a = min(max(gq - g.ml, 0), K - G);
    const int typ = gq - a;
    const float2 *w = W + ((size_t(g.mode == 0 ? s : 0) * G + typ) * g.n_out + q) * G;
    const float2 *l = ls + S * a + s;
    float re = 0.f, im = 0.f;
    for (int j = 0; j < G; ++j) {
      const float2 wv = __ldg(w + j), lv = l[S * j];
      re = fmaf(wv.x, lv.x, re);
      re = fmaf(-wv.y, lv.y, re);
      im = fmaf(wv.x, lv.y, im);
      im = fmaf(wv.y, lv.x, im);
    }
    h[(size_t(row) * g.n_ue + s) * g.N + k] = make_float2(re, im);
  }
}

// K6b (specialised G, the paper's 12W: mode 0, G = 12; 3W: mode 1, G = 3): one CTA per (t, block of RB
// antennas, UE s).  The UE's weights sit in shared memory for RB rows; per row the UE's K pilot LS values
// are formed into a contiguous smem vector, each thread computes one group (12W: 12 outputs from 12
// register-held LS values with warp-broadcast weight reads) or one estimated tone (3W), the row is staged
// in shared memory and written out coalesced (3W: with the zero-order hold applied on the way out).
constexpr int RB = 4;
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
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {   // a * b + c, FP32x2
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
template <int MODE, int GG, int SS>
__global__ void __launch_bounds__(128, 4) k6_estimate_g(const float2 *__restrict__ y, const float2 *__restrict__ x,
                                                     const float2 *__restrict__ W, float2 *__restrict__ h,
                                                     int M, CombGeo g) {
  extern __shared__ float2 sm6[];
  constexpr int n_out = MODE == 0 ? SS : GG;
  const int K = g.K, N = g.N;
  const int per_row = MODE == 0 ? n_out * (K + 1) : K * GG;   // staged outputs per row
  float2 *Ws = sm6;                                     // [GG types][n_out][GG]
  float2 *lsu = Ws + GG * n_out * GG;                   // [RB][K]
  float2 *outs = lsu + RB * K;                          // [RB][per_row]  (12W: transposed [q][g], padded)
  const int n_mb = (M + RB - 1) / RB;
  const int s = blockIdx.x % g.n_ue;
  const int mb = (blockIdx.x / g.n_ue) % n_mb;
  const int t = blockIdx.x / (g.n_ue * n_mb);
  const int rows = min(RB, M - mb * RB);
  const size_t row0 = size_t(t) * M + size_t(mb) * RB;
  const float2 *Wg = W + size_t(MODE == 0 ? s : 0) * GG * n_out * GG;
  for (int e = threadIdx.x; e < GG * n_out * GG; e += blockDim.x) Ws[e] = __ldg(Wg + e);
  const float2 *xr = x + size_t(t) * N;
  // phase 1: LS at this UE's pilots for all rows of the block (rows beyond M are zero)
  for (int e = threadIdx.x; e < RB * K; e += blockDim.x) {
    const int r = e / K, j = e % K;
    const int k = SS * j + s;
    float2 v = make_float2(0.f, 0.f);
    if (r < rows) {
      const float2 yv = y[(row0 + r) * N + k], xv = __ldg(xr + k);
      const float inv = 1.0f / (xv.x * xv.x + xv.y * xv.y);
      v = make_float2((yv.x * xv.x + yv.y * xv.y) * inv, (yv.y * xv.x - yv.x * xv.y) * inv);
    }
    lsu[r * K + j] = v;
  }
  __syncthreads();
  // phase 2: one (group, output) column of the weight per thread and all RB rows at once: every weight
  // element read from shared memory feeds RB complex MACs
  const int tasks = MODE == 0 ? K : K * GG;
  for (int e = threadIdx.x; e < tasks; e += blockDim.x) {
    const int gq = MODE == 0 ? e : e / GG;
    const int a = min(max(gq - g.ml, 0), K - GG);
    float2 l[RB][GG];
#pragma unroll
    for (int r = 0; r < RB; ++r)
#pragma unroll
      for (int j = 0; j < GG; ++j) l[r][j] = lsu[r * K + a + j];
    const int q0 = MODE == 0 ? 0 : e % GG, q1 = MODE == 0 ? n_out : q0 + 1;
    for (int q = q0; q < q1; ++q) {
      const float2 *w = Ws + ((gq - a) * n_out + q) * GG;
      // packed FP32x2 complex MACs with the l components as FFMA2's broadcast scalar operand and the weight as
      // loaded (one 8-byte (re, im) pair): P += l.re w, Q += l.im w, then w l = (P.re - Q.im, P.im + Q.re) --
      // no (-im, re) weight copy per tap (-DK6_NO_PQ: the earlier (re, im) / (-im, re) pair form)
#ifndef K6_NO_PQ
      uint64_t P[RB], Q[RB];
#pragma unroll
      for (int r = 0; r < RB; ++r) P[r] = Q[r] = 0ull;
#pragma unroll
      for (int j = 0; j < GG; ++j) {
        const uint64_t wab = *reinterpret_cast<const uint64_t *>(w + j);
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          P[r] = fma2(pk2(l[r][j].x, l[r][j].x), wab, P[r]);
          Q[r] = fma2(pk2(l[r][j].y, l[r][j].y), wab, Q[r]);
        }
      }
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const float2 pv = upk2(P[r]), qv = upk2(Q[r]);
        outs[r * per_row + (MODE == 0 ? q * (K + 1) + gq : e)] = make_float2(pv.x - qv.y, pv.y + qv.x);
      }
#else
      uint64_t acc[RB];
#pragma unroll
      for (int r = 0; r < RB; ++r) acc[r] = 0ull;
#pragma unroll
      for (int j = 0; j < GG; ++j) {
        const float2 wv = w[j];
        const uint64_t wab = pk2(wv.x, wv.y), wba = pk2(-wv.y, wv.x);
#pragma unroll
        for (int r = 0; r < RB; ++r)
          acc[r] = fma2(pk2(l[r][j].x, l[r][j].x), wab, fma2(pk2(l[r][j].y, l[r][j].y), wba, acc[r]));
      }
#pragma unroll
      for (int r = 0; r < RB; ++r)
        outs[r * per_row + (MODE == 0 ? q * (K + 1) + gq : e)] = upk2(acc[r]);
#endif
    }
  }
  __syncthreads();
  // phase 3: coalesced rows out (3W: zero-order hold on the way out).  12W: threads 0 .. 8 SS - 1 each own one
  // output phase q = tid % SS and group offset tid / SS, and stride by 8 groups: tone k = SS g + q = tid + 8 SS i,
  // so every pass writes 8 SS consecutive tones with no division in the loop
  constexpr int step = SS / GG;
  if (MODE == 0) {
    constexpr int GS = 8;
    if (threadIdx.x < GS * SS) {
      const int q = threadIdx.x % SS, go = threadIdx.x / SS;
      for (int r = 0; r < rows; ++r) {
        float2 *hr = h + ((row0 + r) * g.n_ue + s) * N + threadIdx.x;
        const float2 *o = outs + r * per_row + q * (K + 1);
        for (int gq = go, i = 0; gq < K; gq += GS, i += GS * SS) hr[i] = o[gq];
      }
    }
  } else {
    for (int r = 0; r < rows; ++r) {
      float2 *hr = h + ((row0 + r) * g.n_ue + s) * N;
      const float2 *o = outs + r * per_row;
      for (int k = threadIdx.x; k < N; k += blockDim.x) hr[k] = o[k >= s ? (k - s) / step : 0];
    }
  }
}

}  // namespace
}  // namespace ce

struct ce_comb_handle {
  int device = -1;
  ce::CombGeo g{};
  double sigma2 = 0;
  bool built = false;
  double2 *d_r = nullptr;
  float2 *d_W = nullptr;
  int32_t *d_flag = nullptr;
  int64_t launches = 0;
  // K10 (tcgen05 12W): block table, weight images, LS-plane workspace
  int kernel = CE_COMB_KERNEL_AUTO;
  bool tc_ok = false;
  int n_blk = 0, n_cls = 0;
  int4 *d_blk = nullptr;          // [n_blk] blocks, then [n_cls] class representatives
  uint16_t *d_img = nullptr;      // [hi | lo] images
  void *d_ls = nullptr;
  size_t ls_bytes = 0;
};

namespace {

int cfail(int st, const std::string &m) {
  ce::set_last_error(m);
  return st;
}
int ccuda(cudaError_t e, const char *what) {
  ce::set_last_error(std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
  return e == cudaErrorMemoryAllocation ? CE_ENOMEM : CE_ECUDA;
}
size_t filt_elems(const ce::CombGeo &g) { return size_t(g.n_ue_f) * g.G * g.n_out * g.G; }
// K10 under AUTO only with enough units (128-row tile, UE, block) for ~4 per SM: small calls are latency-bound and two
// launches (k10_ls + k10_comb_tc) cost more than K6b's one (paper_12w, 1152 (row, UE) pairs: K10 25.4 us, K6b 19.2 us;
// massive_12w: 76 vs 155 us)
bool use_tc(const ce_comb_handle *h, long long T, long long M) {
  if (!h->tc_ok || h->kernel == CE_COMB_KERNEL_SIMT) return false;
  if (h->kernel == CE_COMB_KERNEL_TC) return true;
  int dev = h->device, nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const long long units = ((T * M + 127) / 128) * h->g.n_ue * h->n_blk;
  return units >= 4LL * nsm;
}
void free_comb(ce_comb_handle *h) {
  cudaFree(h->d_r);
  cudaFree(h->d_W);
  cudaFree(h->d_flag);
  cudaFree(h->d_blk);
  cudaFree(h->d_img);
  cudaFree(h->d_ls);
}

}  // namespace

extern "C" {

int ce_comb_init(const ce_comb_params *p, ce_comb_handle **out) {
  if (p == nullptr || out == nullptr) return cfail(CE_EINVAL, "ce_comb_init: NULL params or out");
  if (p->N < 1 || p->S < 1 || p->N % p->S) return cfail(CE_EINVAL, "ce_comb_init: need N >= 1, S >= 1, N % S == 0");
  const int K = p->N / p->S;
  if (p->n_ue < 1 || p->n_ue > p->S) return cfail(CE_EINVAL, "ce_comb_init: need 1 <= n_ue <= S");
  if (p->G < 1 || p->G > K || p->G > ce::GMAX) return cfail(CE_EINVAL, "ce_comb_init: need 1 <= G <= min(N/S, 32)");
  if (p->mode != CE_COMB_FULL && p->mode != CE_COMB_SUB) return cfail(CE_EINVAL, "ce_comb_init: unknown mode");
  if (p->mode == CE_COMB_SUB && p->S % p->G) return cfail(CE_EINVAL, "ce_comb_init: sub mode needs S % G == 0");
  if (p->mode == CE_COMB_FULL && p->S > ce::OMAX) return cfail(CE_EINVAL, "ce_comb_init: full mode needs S <= 64");
  if (p->r_hh == nullptr) return cfail(CE_EINVAL, "ce_comb_init: NULL r_hh");
  if (!std::isfinite(p->sigma2) || !(p->sigma2 > 0.0)) return cfail(CE_EINVAL, "ce_comb_init: sigma2 must be finite and > 0");
  for (int d = 0; d < p->N; ++d)
    if (!std::isfinite(p->r_hh[2 * d]) || !std::isfinite(p->r_hh[2 * d + 1]))
      return cfail(CE_EINVAL, "ce_comb_init: r_hh must be finite");
  if (!(p->r_hh[0] > 0.0) || std::fabs(p->r_hh[1]) > 1e-9 * p->r_hh[0])
    return cfail(CE_EINVAL, "ce_comb_init: r[0] must be real and > 0");
  int dev = -1, ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1 || cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return cfail(CE_ENODEV, "ce_comb_init: no CUDA device");
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess || prop.major != 10)
    return cfail(CE_ENODEV, "ce_comb_init: libce is built for sm_100a (compute capability 10.x)");
  ce_comb_handle *h = new (std::nothrow) ce_comb_handle();
  if (!h) return cfail(CE_ENOMEM, "ce_comb_init: host allocation");
  h->device = dev;
  h->g = ce::CombGeo{p->N, p->S, p->n_ue, p->G, p->mode, K, p->mode == CE_COMB_FULL ? p->S : p->G,
                     p->mode == CE_COMB_FULL ? p->n_ue : 1, (p->G - 1) / 2};
  h->sigma2 = p->sigma2;
  // only |d| <= max relative tone distance inside one group is needed: < S * (G + 1) + S
  const int need = std::min(p->N, p->S * (p->G + 2));
  cudaError_t e = cudaMalloc(&h->d_r, size_t(need) * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc(&h->d_W, filt_elems(h->g) * sizeof(float2));
  if (e == cudaSuccess) e = cudaMalloc(&h->d_flag, sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMemcpy(h->d_r, p->r_hh, size_t(need) * sizeof(double2), cudaMemcpyHostToDevice);
  h->tc_ok = ce::comb_tc_supported(p->N, p->S, p->G, p->mode);
  if (e == cudaSuccess && h->tc_ok) {
    std::vector<int4> rep;
    std::vector<int4> blk = ce::comb_tc_blocks(K, p->G, p->S, &rep);
    h->n_blk = int(blk.size());
    h->n_cls = int(rep.size());
    blk.insert(blk.end(), rep.begin(), rep.end());
    e = cudaMalloc(&h->d_blk, blk.size() * sizeof(int4));
    if (e == cudaSuccess) e = cudaMemcpy(h->d_blk, blk.data(), blk.size() * sizeof(int4), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&h->d_img, 2 * ce::comb_tc_image_elems(p->n_ue, h->n_cls) * sizeof(uint16_t));
  }
  if (e != cudaSuccess) {
    int st = ccuda(e, "ce_comb_init");
    free_comb(h);
    delete h;
    return st;
  }
  *out = h;
  return CE_OK;
}

int ce_comb_build_filters(ce_comb_handle *h, void *stream) {
  if (h == nullptr) return cfail(CE_EINVAL, "ce_comb_build_filters: NULL handle");
  ce::DeviceGuard dg(h->device);
  if (!dg.ok) return cfail(CE_ECUDA, "ce_comb_build_filters: cannot select the handle's device");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  h->built = false;
  cudaError_t e = cudaMemsetAsync(h->d_flag, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return ccuda(e, "ce_comb_build_filters: memset");
  ce::k6_build<<<dim3(h->g.n_ue_f, h->g.G), 32, 0, st>>>(h->d_r, h->sigma2, h->g, h->d_W, h->d_flag);
  e = cudaGetLastError();
  if (e != cudaSuccess) return ccuda(e, "ce_comb_build_filters: launch");
  ++h->launches;
  int32_t flag = 0;
  e = cudaMemcpyAsync(&flag, h->d_flag, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return ccuda(e, "ce_comb_build_filters: synchronize");
  if (flag) return cfail(CE_ENOTPD, "ce_comb_build_filters: R_pp + sigma^2 I not positive definite");
  if (h->tc_ok) {                                     // K10 weight images from the complex64 weights
    const size_t ie = ce::comb_tc_image_elems(h->g.n_ue, h->n_cls);
    e = ce::launch_comb_tc_images(h->d_W, h->d_blk + h->n_blk, h->n_cls, h->g.n_ue, h->g.N, h->g.S, h->g.G, h->d_img,
                                  h->d_img + ie, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return ccuda(e, "ce_comb_build_filters: K10 images");
    ++h->launches;
  }
  h->built = true;
  return CE_OK;
}

int ce_comb_estimate(ce_comb_handle *h, const void *d_y, const void *d_x, void *d_h, int32_t T, int32_t M,
                     void *stream) {
  if (h == nullptr) return cfail(CE_EINVAL, "ce_comb_estimate: NULL handle");
  if (!h->built) return cfail(CE_ESTATE, "ce_comb_estimate: call ce_comb_build_filters first");
  if (!d_y || !d_x || !d_h) return cfail(CE_EINVAL, "ce_comb_estimate: NULL pointer");
  if (T < 1 || M < 1) return cfail(CE_EINVAL, "ce_comb_estimate: T and M must be >= 1");
  if ((reinterpret_cast<uintptr_t>(d_y) | reinterpret_cast<uintptr_t>(d_x) | reinterpret_cast<uintptr_t>(d_h)) & 7u)
    return cfail(CE_EINVAL, "ce_comb_estimate: pointers must be 8-byte aligned (complex64)");
  const size_t rows = size_t(T) * M;
  if (rows > 0x7fffffffULL) return cfail(CE_EINVAL, "ce_comb_estimate: too many rows");
  const uintptr_t hy = reinterpret_cast<uintptr_t>(d_h), yy = reinterpret_cast<uintptr_t>(d_y),
                  xx = reinterpret_cast<uintptr_t>(d_x);
  const size_t nh = rows * h->g.n_ue * h->g.N * 8, ny = rows * h->g.N * 8, nx = size_t(T) * h->g.N * 8;
  if ((hy < yy + ny && yy < hy + nh) || (hy < xx + nx && xx < hy + nh))
    return cfail(CE_EINVAL, "ce_comb_estimate: output aliases an input");
  ce::DeviceGuard dg(h->device);
  if (!dg.ok) return cfail(CE_ECUDA, "ce_comb_estimate: cannot select the handle's device");
  const ce::CombGeo &g = h->g;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const float2 *yp = static_cast<const float2 *>(d_y), *xp = static_cast<const float2 *>(d_x);
  float2 *hp = static_cast<float2 *>(d_h);
  if (use_tc(h, T, M)) {
    const size_t need = ce::comb_tc_ls_bytes(g.N, g.S, g.n_ue, (long long)rows);
    if (need > h->ls_bytes) {                         // grow the LS-plane workspace (ce.h: outside stream order)
      cudaFree(h->d_ls);
      h->d_ls = nullptr;
      h->ls_bytes = 0;
      cudaError_t e = cudaMalloc(&h->d_ls, need);
      if (e != cudaSuccess) return ccuda(e, "ce_comb_estimate: K10 workspace");
      h->ls_bytes = need;
    }

    cudaError_t e = ce::launch_comb_tc(yp, xp, hp, T, M, g.N, g.S, g.n_ue, h->d_blk, h->n_blk, h->n_cls, h->d_img,
                                       h->d_img + ce::comb_tc_image_elems(g.n_ue, h->n_cls), h->d_ls, st,
                                       &h->launches);
    if (e != cudaSuccess) return ccuda(e, "ce_comb_estimate: K10 launch");
    return CE_OK;
  }
  const bool spec = g.S == 12 && ((g.mode == CE_COMB_FULL && g.G == 12) || (g.mode == CE_COMB_SUB && g.G == 3));
  const size_t smem_g = (size_t(g.G) * g.n_out * g.G + size_t(ce::RB) * g.K +
                         size_t(ce::RB) * (g.mode == CE_COMB_FULL ? size_t(g.n_out) * (g.K + 1) : size_t(g.K) * g.G)) *
                        sizeof(float2);
  if (spec && smem_g <= 200 * 1024) {
    const size_t n_mb = (size_t(M) + ce::RB - 1) / ce::RB;
    const size_t blocks = size_t(T) * n_mb * g.n_ue;
    if (blocks > 0x7fffffffULL) return cfail(CE_EINVAL, "ce_comb_estimate: too many rows");
    cudaError_t e;
    if (g.mode == CE_COMB_FULL) {
      e = ce::smem_opt_in((const void *)ce::k6_estimate_g<0, 12, 12>, smem_g);
      if (e == cudaSuccess)
        ce::k6_estimate_g<0, 12, 12><<<unsigned(blocks), 128, smem_g, st>>>(yp, xp, h->d_W, hp, M, g);
    } else {
      e = ce::smem_opt_in((const void *)ce::k6_estimate_g<1, 3, 12>, smem_g);
      if (e == cudaSuccess)
        ce::k6_estimate_g<1, 3, 12><<<unsigned(blocks), 128, smem_g, st>>>(yp, xp, h->d_W, hp, M, g);
    }
    if (e != cudaSuccess) return ccuda(e, "ce_comb_estimate: smem attribute");
  } else {
    const size_t smem = size_t(g.N) * sizeof(float2);
    cudaError_t e = ce::smem_opt_in((const void *)ce::k6_estimate, smem);
    if (e != cudaSuccess) return ccuda(e, "ce_comb_estimate: smem attribute");
    ce::k6_estimate<<<unsigned(rows), 256, smem, st>>>(yp, xp, h->d_W, hp, M, g);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return ccuda(e, "ce_comb_estimate: launch");
  ++h->launches;
  return CE_OK;
}

int ce_comb_get_filters(ce_comb_handle *h, void *host_W) {
  if (h == nullptr || host_W == nullptr) return cfail(CE_EINVAL, "ce_comb_get_filters: NULL argument");
  if (!h->built) return cfail(CE_ESTATE, "ce_comb_get_filters: filters not built");
  ce::DeviceGuard dg(h->device);
  if (!dg.ok) return cfail(CE_ECUDA, "ce_comb_get_filters: cannot select the handle's device");
  cudaError_t e = cudaMemcpy(host_W, h->d_W, filt_elems(h->g) * sizeof(float2), cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? CE_OK : ccuda(e, "ce_comb_get_filters");
}

int ce_comb_launch_count(const ce_comb_handle *h, int64_t *out) {
  if (h == nullptr || out == nullptr) return cfail(CE_EINVAL, "ce_comb_launch_count: NULL argument");
  *out = h->launches;
  return CE_OK;
}

int ce_comb_set_kernel(ce_comb_handle *h, int32_t kernel) {
  if (h == nullptr) return cfail(CE_EINVAL, "ce_comb_set_kernel: NULL handle");
  if (kernel != CE_COMB_KERNEL_AUTO && kernel != CE_COMB_KERNEL_SIMT && kernel != CE_COMB_KERNEL_TC)
    return cfail(CE_EINVAL, "ce_comb_set_kernel: unknown kernel");
  if (kernel == CE_COMB_KERNEL_TC && !h->tc_ok)
    return cfail(CE_EINVAL, "ce_comb_set_kernel: K10 needs mode FULL, G <= 13 and the TMA encoder");
  h->kernel = kernel;
  return CE_OK;
}

int ce_comb_selected_kernel(const ce_comb_handle *h, int32_t T, int32_t M, int32_t *out) {
  if (h == nullptr || out == nullptr) return cfail(CE_EINVAL, "ce_comb_selected_kernel: NULL argument");
  if (T < 1 || M < 1) return cfail(CE_EINVAL, "ce_comb_selected_kernel: T and M must be >= 1");
  *out = use_tc(h, T, M) ? CE_COMB_KERNEL_TC : CE_COMB_KERNEL_SIMT;
  return CE_OK;
}

int ce_comb_free(ce_comb_handle *h) {
  if (h == nullptr) return CE_OK;
  {
    ce::DeviceGuard dg(h->device);
    free_comb(h);
  }
  delete h;
  return CE_OK;
}

}  // extern "C"
