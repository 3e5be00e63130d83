// K1 -- block LMMSE filter build on device, FP64.
//
//   W_b = R_b (R_b + sigma^2 I)^-1            PAPER.md:306-309 (Eq. 17), square case (reading A2)
//
// R_b is the b x b leading block of the Hermitian Toeplitz R_hh built from its first column r[d] (PAPER.md:287,
// "only depends on the difference"); with Toeplitz R_hh one W_b serves every window.  A = R_b + sigma^2 I is
// Hermitian Toeplitz too, and R_b = A - sigma^2 I, so
//   W_b = (A - sigma^2 I) A^-1 = I - sigma^2 A^-1.
// The paper solves its Hermitian PD systems by Cholesky (LAPACKE_cposv), O(b^3); here the Toeplitz
// structure gives A^-1 in O(b^2):
//   K1a (one warp per set): Levinson-Durbin recursion for x = A^-1 e_0.  Order-k forward vector f_k (f_k[0] = 1,
//       T_{k+1} f_k = eps_k e_0): eta = sum_{m<k} c[k-m] f_{k-1}[m], gamma = -eta / eps_{k-1},
//       f_k[m] = f_{k-1}[m] + gamma conj(f_{k-1}[k-m]) (m = 0..k, f_{k-1}[k] = 0), eps_k = eps_{k-1} (1 - |gamma|^2);
//       x = f_{b-1} / eps_{b-1}.  A is PD iff every eps_k > 0 (leading minors): the CE_ENOTPD flag.
//   K1b (one thread per diagonal): Gohberg-Semencul / Trench.  With B = A^-1 and x its first column,
//       B = (1/x_0) (L1 L1^H - L2 L2^H),  L1 lower-triangular Toeplitz with first column x, L2 with first column
//       (0, conj(x_{b-1}), ..., conj(x_1)), so along every diagonal
//       B[i+1][j+1] = B[i][j] + (x[i+1] conj(x[j+1]) - conj(x[b-1-i]) x[b-1-j]) / x_0,   B[0][j] = conj(x[j]);
//       thread d walks the diagonal j - i = d and writes W = I - sigma^2 B (Hermitian) to the upper triangles of W
//       and of W^T = conj(W) (K2's coalesced layout), rounded to complex64; K1m mirrors them to the lower triangles.
//   K1r between them: one step of iterative refinement of x (Levinson-Durbin is only weakly stable).
// FP64 throughout: an FP32 build alone exceeds the 1e-4 budget at the config-4 condition numbers.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <cstdlib>

#include "ce_internal.h"

namespace ce {
namespace {

constexpr int K1B_THREADS = 128;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

__device__ __forceinline__ double2 warp_sum(double2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// K1a: one warp per set.  c = first column of A (r[d], plus sigma^2 on d = 0); f in shared memory.
// Writes x = A^-1 e_0 to ws[s][0..b-1].
__global__ void __launch_bounds__(32) k1_levinson(const double2 *__restrict__ d_r, const double *__restrict__ d_sigma2,
                                                  int b, double2 *__restrict__ ws, int in_smem, int32_t *__restrict__ flag) {
  extern __shared__ double2 sm1[];
  const int s = blockIdx.x, lane = threadIdx.x;
  double2 *wss = ws + size_t(s) * (4 * size_t(b) + 1);   // [x: b + 1][c: b][f: b][-: b]
  double2 *c = in_smem ? sm1 : wss + b + 1;          // [b]
  double2 *f = c + b;                                // [b]
  const double2 *r = d_r + size_t(s) * b;
  const double sigma2 = d_sigma2[s];
  for (int m = lane; m < b; m += 32) {
    double2 v = r[m];
    if (m == 0) v = make_double2(v.x + sigma2, 0.0);   // A is Hermitian: c[0] real
    c[m] = v;
    f[m] = make_double2(m == 0 ? 1.0 : 0.0, 0.0);
  }
  __syncwarp();
  double eps = c[0].x;
  bool bad = !(eps > 0.0) || !isfinite(eps);
  for (int k = 1; k < b && !bad; ++k) {
    double2 acc = make_double2(0.0, 0.0);
    for (int m = lane; m < k; m += 32) {             // eta = sum_{m<k} c[k-m] f[m]
      const double2 p = cmul(c[k - m], f[m]);
      acc.x += p.x;
      acc.y += p.y;
    }
    const double2 eta = warp_sum(acc);
    const double2 gamma = make_double2(-eta.x / eps, -eta.y / eps);
    // in-place pair update (m, k - m), m = 0..k/2: f[m] += gamma conj(f[k-m]), f[k-m] += gamma conj(f[m])
    for (int m = lane; 2 * m <= k; m += 32) {
      const double2 fm = f[m], fk = f[k - m];
      const double2 um = cmul(gamma, cconj(fk));
      if (2 * m == k) {
        f[m] = make_double2(fm.x + um.x, fm.y + um.y);
      } else {
        const double2 uk = cmul(gamma, cconj(fm));
        f[m] = make_double2(fm.x + um.x, fm.y + um.y);
        f[k - m] = make_double2(fk.x + uk.x, fk.y + uk.y);
      }
    }
    __syncwarp();
    eps *= 1.0 - (gamma.x * gamma.x + gamma.y * gamma.y);
    bad = !(eps > 0.0) || !isfinite(eps);
  }
  if (bad && lane == 0) atomicOr(flag, 1);
  const double inv = bad ? nan("") : 1.0 / eps;
  __syncwarp();
  for (int m = lane; m < b; m += 32) wss[m] = make_double2(f[m].x * inv, f[m].y * inv);
}

// K1r: one step of iterative refinement of x (one CTA per set).  Levinson-Durbin is only weakly stable: at
// condition numbers ~1e8 its x is off by ~1e-6 relative (W by ~5e-6) where a backward-stable solve gives ~1e-8.
// With the residual res = e_0 - A x (exact Toeplitz products in FP64) and the Gohberg-Semencul form of the
// current inverse, x += (1/x_0) (L1 L1^H res - L2 L2^H res) brings x to the backward-stable level (4 triangular
// Toeplitz products and one Toeplitz product, O(b^2), one thread per output index).
constexpr int K1R_THREADS = 1024;
__global__ void __launch_bounds__(K1R_THREADS) k1_refine(const double2 *__restrict__ d_r,
                                                         const double *__restrict__ d_sigma2, int b,
                                                         double2 *__restrict__ ws) {
  extern __shared__ double2 sr[];
  double2 *c = sr, *x = sr + b, *res = sr + 2 * b, *u = sr + 3 * b, *u2 = sr + 4 * b;
  const int s = blockIdx.x, tid = threadIdx.x;
  double2 *xg = ws + size_t(s) * (4 * size_t(b) + 1);
  const double2 *r = d_r + size_t(s) * b;
  for (int m = tid; m < b; m += blockDim.x) {
    double2 v = r[m];
    if (m == 0) v = make_double2(v.x + d_sigma2[s], 0.0);
    c[m] = v;
    x[m] = xg[m];
  }
  __syncthreads();
  // res[i] = delta_i0 - sum_j A[i][j] x[j],  A[i][j] = c[i-j] (i >= j), conj(c[j-i]) (i < j)
  for (int i = tid; i < b; i += blockDim.x) {
    double2 acc = make_double2(i == 0 ? 1.0 : 0.0, 0.0);
    for (int j = 0; j <= i; ++j) {
      const double2 p = cmul(c[i - j], x[j]);
      acc.x -= p.x;
      acc.y -= p.y;
    }
    for (int j = i + 1; j < b; ++j) {
      const double2 p = cmul(cconj(c[j - i]), x[j]);
      acc.x -= p.x;
      acc.y -= p.y;
    }
    res[i] = acc;
  }
  __syncthreads();
  // u = L1^H res: u[k] = sum_{i>=k} conj(x[i-k]) res[i];  u2 = L2^H res: u2[k] = sum_{i>k} x[b-(i-k)] res[i]
  for (int k = tid; k < b; k += blockDim.x) {
    double2 a = make_double2(0.0, 0.0), a2 = make_double2(0.0, 0.0);
    for (int i = k; i < b; ++i) {
      const double2 p = cmul(cconj(x[i - k]), res[i]);
      a.x += p.x;
      a.y += p.y;
      if (i > k) {
        const double2 q = cmul(x[b - (i - k)], res[i]);
        a2.x += q.x;
        a2.y += q.y;
      }
    }
    u[k] = a;
    u2[k] = a2;
  }
  __syncthreads();
  // delta[i] = (sum_{k<=i} x[i-k] u[k] - sum_{k<i} conj(x[b-i+k]) u2[k]) / x_0
  const double ix0 = 1.0 / x[0].x;
  for (int i = tid; i < b; i += blockDim.x) {
    double2 a = make_double2(0.0, 0.0);
    for (int k = 0; k <= i; ++k) {
      const double2 p = cmul(x[i - k], u[k]);
      a.x += p.x;
      a.y += p.y;
      if (k < i) {
        const double2 q = cmul(cconj(x[b - i + k]), u2[k]);
        a.x -= q.x;
        a.y -= q.y;
      }
    }
    xg[i] = make_double2(x[i].x + a.x * ix0, x[i].y + a.y * ix0);
  }
}

// K1a for large b (one CTA per set): the same recursion with the dot product spread over the CTA -- per step a
// warp reduction, one barrier, every thread summing the per-warp partials in the same order (identical gamma
// and eps everywhere), the pair update, and a second barrier.
constexpr int K1L_THREADS = 512;
__global__ void __launch_bounds__(K1L_THREADS) k1_levinson_cta(const double2 *__restrict__ d_r,
                                                               const double *__restrict__ d_sigma2, int b,
                                                               double2 *__restrict__ ws, int in_smem,
                                                               int32_t *__restrict__ flag) {
  extern __shared__ double2 sm1[];
  __shared__ double2 part[2][K1L_THREADS / 32];
  const int s = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = blockDim.x >> 5;
  double2 *wss = ws + size_t(s) * (4 * size_t(b) + 1);   // [x: b + 1][c: b][f: b][-: b]
  double2 *c = in_smem ? sm1 : wss + b + 1;
  double2 *f = c + b;
  const double2 *r = d_r + size_t(s) * b;
  const double sigma2 = d_sigma2[s];
  for (int m = tid; m < b; m += blockDim.x) {
    double2 v = r[m];
    if (m == 0) v = make_double2(v.x + sigma2, 0.0);
    c[m] = v;
    f[m] = make_double2(m == 0 ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  double eps = c[0].x;
  bool bad = !(eps > 0.0) || !isfinite(eps);
  for (int k = 1; k < b && !bad; ++k) {
    double2 acc = make_double2(0.0, 0.0);
    for (int m = tid; m < k; m += blockDim.x) {
      const double2 p = cmul(c[k - m], f[m]);
      acc.x += p.x;
      acc.y += p.y;
    }
    acc = warp_sum(acc);
    if (lane == 0) part[k & 1][warp] = acc;
    __syncthreads();
    double2 eta = make_double2(0.0, 0.0);
    for (int w = 0; w < nw; ++w) {
      eta.x += part[k & 1][w].x;
      eta.y += part[k & 1][w].y;
    }
    const double2 gamma = make_double2(-eta.x / eps, -eta.y / eps);
    for (int m = tid; 2 * m <= k; m += blockDim.x) {
      const double2 fm = f[m], fk = f[k - m];
      const double2 um = cmul(gamma, cconj(fk));
      if (2 * m == k) {
        f[m] = make_double2(fm.x + um.x, fm.y + um.y);
      } else {
        const double2 uk = cmul(gamma, cconj(fm));
        f[m] = make_double2(fm.x + um.x, fm.y + um.y);
        f[k - m] = make_double2(fk.x + uk.x, fk.y + uk.y);
      }
    }
    eps *= 1.0 - (gamma.x * gamma.x + gamma.y * gamma.y);
    bad = !(eps > 0.0) || !isfinite(eps);
    __syncthreads();
  }
  if (bad && tid == 0) atomicOr(flag, 1);
  const double inv = bad ? nan("") : 1.0 / eps;
  __syncthreads();
  for (int m = tid; m < b; m += blockDim.x) wss[m] = make_double2(f[m].x * inv, f[m].y * inv);
}

// K1a' (Schur form, default): the same reflection coefficients without a per-step reduction.  With the residuals
// of the forward and backward vectors, e_k[i] = (A [f_k; 0])[i] and r_k[i] = (A [b_k; 0])[i] (b_k = J conj(f_k)),
// gamma_{k+1} = -e_k[k+1] / r_k[k] and, by the Toeplitz shift invariance, for i > k
//   e_{k+1}[i] = e_k[i] + gamma r_k[i-1],   r_{k+1}[i] = r_k[i-1] + conj(gamma) e_k[i],
// kept in place as R_k[j] = r_k[j + k] (thread j owns the pair (e[j+k+1], R[j])); f is updated by the same pair rule
// as in K1a.  One barrier per step; the next step's two pivots go to a ping-pong slot.  e_0 = r_0 = c.
__global__ void __launch_bounds__(K1L_THREADS) k1_schur(const double2 *__restrict__ d_r,
                                                        const double *__restrict__ d_sigma2, int b,
                                                        double2 *__restrict__ ws, int in_smem,
                                                        int32_t *__restrict__ flag) {
  extern __shared__ double2 sm1[];
  __shared__ double2 piv[2][2];                      // [step parity][e_k[k+1], R_k[0]]
  const int s = blockIdx.x, tid = threadIdx.x;
  double2 *wss = ws + size_t(s) * (4 * size_t(b) + 1);   // [x: b + 1][e: b][R: b] (f in x's slot when not in smem)
  double2 *e = in_smem ? sm1 : wss + b + 1;
  double2 *R = e + b;
  double2 *f = in_smem ? sm1 + 2 * b : wss;
  const double2 *r = d_r + size_t(s) * b;
  const double sigma2 = d_sigma2[s];
  for (int m = tid; m < b; m += blockDim.x) {
    double2 v = r[m];
    if (m == 0) v = make_double2(v.x + sigma2, 0.0);
    e[m] = v;
    R[m] = v;
    f[m] = make_double2(m == 0 ? 1.0 : 0.0, 0.0);
    if (m == 0) piv[0][1] = v;
    if (m == 1) piv[0][0] = v;
  }
  __syncthreads();
  double eps = piv[0][1].x;
  bool bad = !(eps > 0.0) || !isfinite(eps);
  for (int k = 0; k + 1 < b && !bad; ++k) {
    const double2 ek = piv[k & 1][0], r0 = piv[k & 1][1];
    const double den = r0.x * r0.x + r0.y * r0.y;
    const double2 gamma = make_double2(-(ek.x * r0.x + ek.y * r0.y) / den, -(ek.y * r0.x - ek.x * r0.y) / den);
    const double2 gc = cconj(gamma);
    for (int j = tid; j < b - 1 - k; j += blockDim.x) {
      const double2 eo = e[j + k + 1], ro = R[j];
      const double2 p = cmul(gamma, ro), q = cmul(gc, eo);
      const double2 en = make_double2(eo.x + p.x, eo.y + p.y), rn = make_double2(ro.x + q.x, ro.y + q.y);
      e[j + k + 1] = en;
      R[j] = rn;
      if (j == 0) piv[(k + 1) & 1][1] = rn;            // R_{k+1}[0] = eps_{k+1}
      if (j == 1) piv[(k + 1) & 1][0] = en;            // e_{k+1}[k+2]
    }
    for (int m = tid; 2 * m <= k + 1; m += blockDim.x) {   // f_{k+1}[m] = f_k[m] + gamma conj(f_k[k+1-m])
      const int mk = k + 1 - m;
      const double2 fm = f[m], fk = f[mk];
      const double2 um = cmul(gamma, cconj(fk));
      if (m == mk) {
        f[m] = make_double2(fm.x + um.x, fm.y + um.y);
      } else {
        const double2 uk = cmul(gamma, cconj(fm));
        f[m] = make_double2(fm.x + um.x, fm.y + um.y);
        f[mk] = make_double2(fk.x + uk.x, fk.y + uk.y);
      }
    }
    eps *= 1.0 - (gamma.x * gamma.x + gamma.y * gamma.y);
    bad = !(eps > 0.0) || !isfinite(eps);
    __syncthreads();
  }
  if (bad && tid == 0) atomicOr(flag, 1);
  const double inv = bad ? nan("") : 1.0 / eps;
  for (int m = tid; m < b; m += blockDim.x) {
    const double2 v = f[m];
    wss[m] = make_double2(v.x * inv, v.y * inv);       // in place when f lives in x's slot
  }
}

// K1r split over CTAs for large b (grid (sets, ceil(b / 256)), three launches): the refinement's three phases each
// need the whole previous vector, so each phase is one kernel; every CTA stages the vectors it reads in shared
// memory and computes 256 outputs.  ws per set: [x: b + 1][res: b][u: b][u2: b].
constexpr int K1P_THREADS = 256;
__device__ __forceinline__ double2 first_col(const double2 *r, double sigma2, int m) {
  const double2 v = r[m];
  return m == 0 ? make_double2(v.x + sigma2, 0.0) : v;
}
// in_smem = 0 (b beyond the shared-memory range): the same arithmetic on the vectors in the set's workspace and
// the statistics column in global memory (L2-resident at these sizes)
__global__ void __launch_bounds__(K1P_THREADS) k1_refine_res(const double2 *__restrict__ d_r,
                                                             const double *__restrict__ d_sigma2, int b,
                                                             double2 *__restrict__ ws, int in_smem) {
  extern __shared__ double2 sp[];
  const int s = blockIdx.x;
  double2 *wss = ws + size_t(s) * (4 * size_t(b) + 1);
  const double2 *r = d_r + size_t(s) * b;
  const double sigma2 = d_sigma2[s];
  double2 *c = sp;
  const double2 *x = in_smem ? sp + b : wss;
  if (in_smem) {
    for (int m = threadIdx.x; m < b; m += blockDim.x) {
      c[m] = first_col(r, sigma2, m);
      sp[b + m] = wss[m];
    }
    __syncthreads();
  }
  const int i = blockIdx.y * blockDim.x + threadIdx.x;
  if (i >= b) return;
  double2 acc = make_double2(i == 0 ? 1.0 : 0.0, 0.0);
  for (int j = 0; j <= i; ++j) {
    const double2 p = cmul(in_smem ? c[i - j] : first_col(r, sigma2, i - j), x[j]);
    acc.x -= p.x;
    acc.y -= p.y;
  }
  for (int j = i + 1; j < b; ++j) {
    const double2 p = cmul(cconj(in_smem ? c[j - i] : first_col(r, sigma2, j - i)), x[j]);
    acc.x -= p.x;
    acc.y -= p.y;
  }
  wss[b + 1 + i] = acc;                              // res
}
__global__ void __launch_bounds__(K1P_THREADS) k1_refine_u(int b, double2 *__restrict__ ws, int in_smem) {
  extern __shared__ double2 sp[];
  const int s = blockIdx.x;
  double2 *wss = ws + size_t(s) * (4 * size_t(b) + 1);
  const double2 *x = in_smem ? sp : wss, *res = in_smem ? sp + b : wss + b + 1;
  if (in_smem) {
    for (int m = threadIdx.x; m < b; m += blockDim.x) {
      sp[m] = wss[m];
      sp[b + m] = wss[b + 1 + m];
    }
    __syncthreads();
  }
  const int k = blockIdx.y * blockDim.x + threadIdx.x;
  if (k >= b) return;
  double2 a = make_double2(0.0, 0.0), a2 = make_double2(0.0, 0.0);
  for (int i = k; i < b; ++i) {                      // u[k] = sum_{i>=k} conj(x[i-k]) res[i]
    const double2 p = cmul(cconj(x[i - k]), res[i]);
    a.x += p.x;
    a.y += p.y;
  }
  for (int i = k + 1; i < b; ++i) {                  // u2[k] = sum_{i>k} x[b-(i-k)] res[i]
    const double2 q = cmul(x[b - (i - k)], res[i]);
    a2.x += q.x;
    a2.y += q.y;
  }
  wss[2 * b + 1 + k] = a;
  wss[3 * b + 1 + k] = a2;
}
__global__ void __launch_bounds__(K1P_THREADS) k1_refine_x(int b, double2 *__restrict__ ws, int in_smem) {
  extern __shared__ double2 sp[];
  const int s = blockIdx.x;
  double2 *wss = ws + size_t(s) * (4 * size_t(b) + 1);
  const double2 *x = in_smem ? sp : wss, *u = in_smem ? sp + b : wss + 2 * b + 1,
                *u2 = in_smem ? sp + 2 * b : wss + 3 * b + 1;
  if (in_smem) {
    for (int m = threadIdx.x; m < b; m += blockDim.x) {
      sp[m] = wss[m];
      sp[b + m] = wss[2 * b + 1 + m];
      sp[2 * b + m] = wss[3 * b + 1 + m];
    }
    __syncthreads();
  }
  const int i = blockIdx.y * blockDim.x + threadIdx.x;
  if (i >= b) return;
  double2 a = make_double2(0.0, 0.0);
  for (int k = 0; k <= i; ++k) {                     // delta[i] = (sum_{k<=i} x[i-k] u[k] - sum_{k<i} conj(x[b-i+k]) u2[k]) / x_0
    const double2 p = cmul(x[i - k], u[k]);
    a.x += p.x;
    a.y += p.y;
  }
  for (int k = 0; k < i; ++k) {
    const double2 q = cmul(cconj(x[b - i + k]), u2[k]);
    a.x -= q.x;
    a.y -= q.y;
  }
  const double ix0 = 1.0 / x[0].x;
  // the refined x goes to the (now free) res slot: other CTAs of this launch may still be reading x
  wss[b + 1 + i] = make_double2(x[i].x + a.x * ix0, x[i].y + a.y * ix0);
}

// K1m: lower triangles of W and W^T from the upper ones through 32 x 32 shared-memory tiles (coalesced reads and
// writes): W[r][c] = conj(W[c][r]), W^T[r][c] = W[c][r] for r > c.  grid (sets, nb, nb), block (32, 8).
__global__ void __launch_bounds__(256) k1_mirror(int b, float2 *__restrict__ W, float2 *__restrict__ Wt) {
  __shared__ float2 tile[32][33];
  const int s = blockIdx.x, bi = blockIdx.y, bj = blockIdx.z;   // output block row bi, column bj (bi >= bj)
  if (bi < bj) return;
  float2 *Ws = W + size_t(s) * b * b;
  float2 *Wts = Wt + size_t(s) * b * b;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int yy = ty; yy < 32; yy += 8) {              // source: upper block (bj, bi), rows bj*32 + yy
    const int r = bj * 32 + yy, c = bi * 32 + tx;
    if (r < b && c < b) tile[yy][tx] = Ws[size_t(r) * b + c];
  }
  __syncthreads();
  for (int yy = ty; yy < 32; yy += 8) {              // destination: lower block (bi, bj), rows bi*32 + yy
    const int r = bi * 32 + yy, c = bj * 32 + tx;
    if (r < b && c < b && r > c) {
      const float2 u = tile[tx][yy];                 // W[c][r]
      Ws[size_t(r) * b + c] = make_float2(u.x, -u.y);
      Wts[size_t(r) * b + c] = u;
    }
  }
}

// K1b: grid (sets, ceil(b / 128)); thread d walks the diagonal j - i = d of B = A^-1.
__global__ void __launch_bounds__(K1B_THREADS) k1_trench(const double *__restrict__ d_sigma2, int b,
                                                         const double2 *__restrict__ ws, int in_smem, int xoff,
                                                         float2 *__restrict__ W, float2 *__restrict__ Wt) {
  extern __shared__ double2 sx[];                    // [b] x, when it fits
  const int s = blockIdx.x;
  const double2 *xg = ws + size_t(s) * (4 * size_t(b) + 1) + xoff;
  if (in_smem)
    for (int m = threadIdx.x; m < b; m += blockDim.x) sx[m] = xg[m];
  __syncthreads();
  const double2 *xs = in_smem ? sx : xg;
  const int d = blockIdx.y * blockDim.x + threadIdx.x;
  if (d >= b) return;
  const double sigma2 = d_sigma2[s];
  const double ix0 = 1.0 / xs[0].x;
  float2 *Ws = W + size_t(s) * b * b;
  float2 *Wts = Wt + size_t(s) * b * b;
  double2 v = cconj(xs[d]);                          // B[0][d]
  for (int i = 0; i + d < b; ++i) {
    const int j = i + d;
    // W = I - sigma^2 B: upper element (i, j) and, by Hermitian symmetry, lower element (j, i)
    const double2 w = make_double2((i == j ? 1.0 : 0.0) - sigma2 * v.x, -sigma2 * v.y);
    const float2 wu = make_float2(__double2float_rn(w.x), __double2float_rn(w.y));
    const float2 wl = make_float2(wu.x, -wu.y);
    // upper triangle only (coalesced across the threads of a step); W is Hermitian, so W^T = conj(W) and the
    // lower triangles are filled by K1m from these
    Ws[size_t(i) * b + j] = wu;                      // W[i][j]
    Wts[size_t(i) * b + j] = wl;                     // W^T[i][j] = W[j][i] = conj(W[i][j])
    if (j + 1 < b) {                                 // B[i+1][j+1] = B[i][j] + (x[i+1] x*[j+1] - x*[b-1-i] x[b-1-j]) / x0
      const double2 p = cmul(xs[i + 1], cconj(xs[j + 1]));
      const double2 q = cmul(cconj(xs[b - 1 - i]), xs[b - 1 - j]);
      v.x += (p.x - q.x) * ix0;
      v.y += (p.y - q.y) * ix0;
    }
  }
}

}  // namespace

cudaError_t launch_filter_build(const double2 *d_r, const double *d_sigma2, int32_t N, int32_t b, int32_t n_sets,
                                double2 *d_ws, float2 *d_W, float2 *d_Wt, int32_t *d_flag, cudaStream_t stream,
                                int64_t *launches) {
  (void)N;
  cudaError_t e;
  // f and c in shared memory up to b = 6400, else in the set's workspace (ws: [n_sets][4b + 1] double2)
  const int lev_in_smem = size_t(2) * b * sizeof(double2) <= 200 * 1024;
  const size_t lev_smem = lev_in_smem ? size_t(2) * b * sizeof(double2) : 0;
  // b <= 256: Levinson-Durbin in one warp (config 4, b = 150: 62 us; the Schur form in one warp: 125 us);
  // b > 256: the Schur form in a 512-thread CTA (config 6, b = 1200: 0.87 ms; 128 / 256 threads: 1.32 / 0.98 ms;
  // the CTA Levinson form: 1.34 ms, one warp: 1.74 ms).  CE_K1_SCHUR (experiments): 0 never, 1 always.
  static const int env_schur = getenv("CE_K1_SCHUR") ? atoi(getenv("CE_K1_SCHUR")) : -1;
  const bool lev_cta = b > 256;
  if (env_schur == 1 || (env_schur != 0 && lev_cta)) {
    const int schur_in_smem = size_t(3) * b * sizeof(double2) <= 200 * 1024;
    const size_t sch_smem = schur_in_smem ? size_t(3) * b * sizeof(double2) : 0;
    if ((e = smem_opt_in((const void *)k1_schur, sch_smem)) != cudaSuccess) return e;
    static const int env_st = getenv("CE_K1_SCHUR_T") ? atoi(getenv("CE_K1_SCHUR_T")) : K1L_THREADS;   // experiments
    k1_schur<<<n_sets, std::min(std::max(env_st, 32), K1L_THREADS) / 32 * 32, sch_smem, stream>>>(d_r, d_sigma2, b,
                                                                                                 d_ws, schur_in_smem, d_flag);
  } else {
    e = smem_opt_in(lev_cta ? (const void *)k1_levinson_cta : (const void *)k1_levinson, lev_smem);
    if (e != cudaSuccess) return e;
    if (lev_cta)
      k1_levinson_cta<<<n_sets, K1L_THREADS, lev_smem, stream>>>(d_r, d_sigma2, b, d_ws, lev_in_smem, d_flag);
    else
      k1_levinson<<<n_sets, 32, lev_smem, stream>>>(d_r, d_sigma2, b, d_ws, lev_in_smem, d_flag);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  ++*launches;
  // one refinement step of x: split over CTAs (three launches) above b = 256, one CTA per set below
  int xoff = 0;
  const size_t ref_smem = size_t(5) * b * sizeof(double2);
  const size_t rp_smem = size_t(3) * b * sizeof(double2);
  if (b > 256) {
    // every b: the vectors in shared memory up to b = 4266 (3b double2 <= 200 KB), else read from the workspace
    const int rp_in = rp_smem <= 200 * 1024;
    const dim3 pg(n_sets, (b + K1P_THREADS - 1) / K1P_THREADS);
    const size_t s2b = rp_in ? 2 * size_t(b) * sizeof(double2) : 0, s3b = rp_in ? rp_smem : 0;
    if ((e = smem_opt_in((const void *)k1_refine_res, s2b)) != cudaSuccess) return e;
    if ((e = smem_opt_in((const void *)k1_refine_u, s2b)) != cudaSuccess) return e;
    if ((e = smem_opt_in((const void *)k1_refine_x, s3b)) != cudaSuccess) return e;
    k1_refine_res<<<pg, K1P_THREADS, s2b, stream>>>(d_r, d_sigma2, b, d_ws, rp_in);
    k1_refine_u<<<pg, K1P_THREADS, s2b, stream>>>(b, d_ws, rp_in);
    k1_refine_x<<<pg, K1P_THREADS, s3b, stream>>>(b, d_ws, rp_in);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    *launches += 3;
    xoff = b + 1;
  } else if (ref_smem <= 200 * 1024) {
    if ((e = smem_opt_in((const void *)k1_refine, ref_smem)) != cudaSuccess) return e;
    k1_refine<<<n_sets, K1R_THREADS, ref_smem, stream>>>(d_r, d_sigma2, b, d_ws);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ++*launches;
  }
  const int tr_in_smem = size_t(b) * sizeof(double2) <= 200 * 1024;
  const size_t tr_smem = tr_in_smem ? size_t(b) * sizeof(double2) : 0;
  if ((e = smem_opt_in((const void *)k1_trench, tr_smem)) != cudaSuccess) return e;
  dim3 grid(n_sets, (b + K1B_THREADS - 1) / K1B_THREADS);
  k1_trench<<<grid, K1B_THREADS, tr_smem, stream>>>(d_sigma2, b, d_ws, tr_in_smem, xoff, d_W, d_Wt);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  ++*launches;
  const int nbk = (b + 31) / 32;
  k1_mirror<<<dim3(n_sets, nbk, nbk), dim3(32, 8), 0, stream>>>(b, d_W, d_Wt);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  ++*launches;
  return cudaSuccess;
}

}  // namespace ce
