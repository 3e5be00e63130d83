// K1 -- block LMMSE filter build on device, FP64.
//
//   W_b = R_b (R_b + sigma^2 I)^-1            PAPER.md:306-309 (Eq. 17), square case (reading A2)
//
// R_b is the b x b leading block of the Hermitian Toeplitz R_hh built from its first column
// r[d] ("only depends on the difference"); with Toeplitz R_hh one W_b serves
// every window.  As in the paper's detector (LAPACKE_cposv) the Hermitian PD
// system is solved by Cholesky:  A = R_b + sigma^2 I = L L^H, then W = A^-1 R_b by forward
// (L Z = R_b) and back (L^H W = Z) substitution for the b right-hand sides.  A and R_b commute,
// so A^-1 R_b = R_b A^-1 = W.  FP64 is required: an FP32 build alone exceeds the 1e-4 budget
// at the config-4 condition numbers (SURVEY.md §7 "Accuracy").
//
// Kernel 1 (one CTA per set): packed lower-triangular Cholesky, in shared memory when it fits
//   (b <= 168), else in the global workspace; writes L (packed) to the workspace.
// Kernel 2 (grid sets x ceil(b/8), one warp per right-hand side): loads packed L into shared
//   memory, forward/back substitution, writes W (row-major) and W^T (for K2's coalesced loads)
//   rounded to complex64.
#include <cuda_runtime.h>
#include <math.h>

#include "ce_internal.h"

namespace ce {
namespace {

constexpr int K1_THREADS = 256;
constexpr int K1S_WARPS = 8;
constexpr size_t SMEM_LIMIT = 220 * 1024;

__device__ __forceinline__ size_t pk(int i, int j) { return size_t(i) * (i + 1) / 2 + j; }  // i >= j

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmul_conj_b(double2 a, double2 b) {  // a * conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}

// R_b[i][j] of the Hermitian Toeplitz block: r[i-j] for i >= j, conj(r[j-i]) otherwise.
__device__ __forceinline__ double2 toeplitz(const double2 *r, int i, int j) {
  if (i >= j) return r[i - j];
  double2 v = r[j - i];
  return make_double2(v.x, -v.y);
}

__global__ void __launch_bounds__(K1_THREADS) k1_cholesky(const double2 *__restrict__ d_r,
                                                          const double *__restrict__ d_sigma2, int b,
                                                          double2 *__restrict__ ws, int use_smem,
                                                          int32_t *__restrict__ flag) {
  extern __shared__ double2 sm[];
  const int s = blockIdx.x;
  const size_t packed = size_t(b) * (b + 1) / 2;
  double2 *L = use_smem ? sm : ws + size_t(s) * packed;
  const double2 *r = d_r + size_t(s) * b;
  const double sigma2 = d_sigma2[s];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  __shared__ double s_inv;

  // A = R_b + sigma^2 I, lower triangle, packed by rows
  for (int i = warp; i < b; i += nwarp)
    for (int j = lane; j <= i; j += 32) {
      double2 v = toeplitz(r, i, j);
      if (i == j) v.x += sigma2;
      L[pk(i, j)] = v;
    }
  __syncthreads();

  for (int k = 0; k < b; ++k) {
    if (tid == 0) {
      const double d = L[pk(k, k)].x;
      const bool bad = !(d > 0.0) || !isfinite(d);
      if (bad) atomicOr(flag, 1);
      const double lkk = bad ? nan("") : sqrt(d);
      L[pk(k, k)] = make_double2(lkk, 0.0);
      s_inv = 1.0 / lkk;
    }
    __syncthreads();
    const double inv = s_inv;
    for (int i = k + 1 + tid; i < b; i += blockDim.x) {
      double2 v = L[pk(i, k)];
      L[pk(i, k)] = make_double2(v.x * inv, v.y * inv);
    }
    __syncthreads();
    // trailing update of the lower triangle: L(i,j) -= L(i,k) conj(L(j,k)), k < j <= i
    for (int i = k + 1 + warp; i < b; i += nwarp) {
      const double2 lik = L[pk(i, k)];
      for (int j = k + 1 + lane; j <= i; j += 32) {
        const double2 p = cmul_conj_b(lik, L[pk(j, k)]);
        double2 v = L[pk(i, j)];
        L[pk(i, j)] = make_double2(v.x - p.x, v.y - p.y);
      }
    }
    __syncthreads();
  }
  if (use_smem) {
    double2 *out = ws + size_t(s) * packed;
    for (size_t e = tid; e < packed; e += blockDim.x) out[e] = L[e];
  }
}

__device__ __forceinline__ double2 warp_sum(double2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

__global__ void __launch_bounds__(K1S_WARPS * 32) k1_solve(const double2 *__restrict__ d_r, int b,
                                                           const double2 *__restrict__ ws, int l_in_smem,
                                                           float2 *__restrict__ W, float2 *__restrict__ Wt) {
  extern __shared__ double2 sm[];
  const int s = blockIdx.x;
  const size_t packed = size_t(b) * (b + 1) / 2;
  const double2 *Lg = ws + size_t(s) * packed;
  double2 *z_all = sm;                                  // [K1S_WARPS][b]
  double2 *Ls = sm + size_t(K1S_WARPS) * b;             // packed L copy (if it fits)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (l_in_smem)
    for (size_t e = tid; e < packed; e += blockDim.x) Ls[e] = Lg[e];
  __syncthreads();
  const double2 *L = l_in_smem ? Ls : Lg;
  const double2 *r = d_r + size_t(s) * b;
  const int j = blockIdx.y * K1S_WARPS + warp;          // right-hand side (column of R_b)
  if (j >= b) return;
  double2 *z = z_all + size_t(warp) * b;
  for (int i = lane; i < b; i += 32) z[i] = toeplitz(r, i, j);
  __syncwarp();
  // forward: L Z = R_b[:, j]
  for (int i = 0; i < b; ++i) {
    double2 acc = make_double2(0.0, 0.0);
    for (int k = lane; k < i; k += 32) {
      const double2 p = cmul(L[pk(i, k)], z[k]);
      acc.x += p.x;
      acc.y += p.y;
    }
    acc = warp_sum(acc);
    if (lane == 0) {
      const double inv = 1.0 / L[pk(i, i)].x;
      z[i] = make_double2((z[i].x - acc.x) * inv, (z[i].y - acc.y) * inv);
    }
    __syncwarp();
  }
  // back: L^H W = Z
  for (int i = b - 1; i >= 0; --i) {
    double2 acc = make_double2(0.0, 0.0);
    for (int k = i + 1 + lane; k < b; k += 32) {
      const double2 p = cmul_conj_b(z[k], L[pk(k, i)]);  // conj(L(k,i)) * z[k]
      acc.x += p.x;
      acc.y += p.y;
    }
    acc = warp_sum(acc);
    if (lane == 0) {
      const double inv = 1.0 / L[pk(i, i)].x;
      z[i] = make_double2((z[i].x - acc.x) * inv, (z[i].y - acc.y) * inv);
    }
    __syncwarp();
  }
  float2 *Ws = W + size_t(s) * b * b;
  float2 *Wts = Wt + size_t(s) * b * b;
  for (int i = lane; i < b; i += 32) {
    const float2 v = make_float2(__double2float_rn(z[i].x), __double2float_rn(z[i].y));
    Ws[size_t(i) * b + j] = v;   // W[i][j]
    Wts[size_t(j) * b + i] = v;  // W^T[j][i]
  }
}

}  // namespace

cudaError_t launch_filter_build(const double2 *d_r, const double *d_sigma2, int32_t N, int32_t b, int32_t n_sets,
                                double2 *d_ws, float2 *d_W, float2 *d_Wt, int32_t *d_flag, cudaStream_t stream,
                                int64_t *launches) {
  (void)N;
  const size_t packed_bytes = size_t(b) * (b + 1) / 2 * sizeof(double2);
  const int chol_smem = packed_bytes <= SMEM_LIMIT;
  cudaError_t e;
  if (chol_smem) {
    e = cudaFuncSetAttribute(k1_cholesky, cudaFuncAttributeMaxDynamicSharedMemorySize, int(packed_bytes));
    if (e != cudaSuccess) return e;
  }
  k1_cholesky<<<n_sets, K1_THREADS, chol_smem ? packed_bytes : 0, stream>>>(d_r, d_sigma2, b, d_ws, chol_smem,
                                                                              d_flag);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  ++*launches;
  const size_t z_bytes = size_t(K1S_WARPS) * b * sizeof(double2);
  const int l_smem = z_bytes + packed_bytes <= SMEM_LIMIT;
  const size_t solve_smem = z_bytes + (l_smem ? packed_bytes : 0);
  e = cudaFuncSetAttribute(k1_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, int(solve_smem));
  if (e != cudaSuccess) return e;
  dim3 grid(n_sets, (b + K1S_WARPS - 1) / K1S_WARPS);
  k1_solve<<<grid, K1S_WARPS * 32, solve_smem, stream>>>(d_r, b, d_ws, l_smem, d_W, d_Wt);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  ++*launches;
  return cudaSuccess;
}

}  // namespace ce
