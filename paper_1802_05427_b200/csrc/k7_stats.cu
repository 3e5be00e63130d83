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
// K7a: one CTA per column: LS row and the N twiddles exp(j 2 pi n / N) in shared memory; threads split the
// D lags (x as many n-ranges as fit in 256 threads) and then the B noise bins; per-CTA partial sums are
// added in FP64 to per-set accumulators.  K7b: one thread per set normalises.
#include <cuda_runtime.h>
#include <math.h>

#include <string>

#include "ce_internal.h"

namespace ce {
namespace {

constexpr int K7_THREADS = 256;

__global__ void __launch_bounds__(K7_THREADS) k7_accumulate(const float2 *__restrict__ y, const float2 *__restrict__ x,
                                                            int M, int K, int N, const int32_t *__restrict__ soi,
                                                            int n_sets, int D, int B, double *__restrict__ acc) {
  extern __shared__ float2 sm7[];
  float2 *ls = sm7;                                  // [N]
  float2 *tw = sm7 + N;                              // [N] exp(+j 2 pi n / N)
  __shared__ double part[2 * K7_THREADS];
  const int col = blockIdx.x;                        // (t * M + m) * K + k
  const int t = col / (M * K), k = col % K;
  const int set = soi ? soi[t] : 0;
  if (set < 0 || set >= n_sets) return;              // out-of-range set: the instance is skipped
  const float2 *yr = y + size_t(col) * N;
  const float2 *xr = x + (size_t(t) * K + k) * N;
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    const float2 yv = yr[n], xv = xr[n];
    const float inv = 1.0f / (xv.x * xv.x + xv.y * xv.y);
    ls[n] = make_float2((yv.x * xv.x + yv.y * xv.y) * inv, (yv.y * xv.x - yv.x * xv.y) * inv);
    double sv, cv;
    sincospi(2.0 * n / N, &sv, &cv);
    tw[n] = make_float2(float(cv), float(sv));
  }
  __syncthreads();
  double *acc_s = acc + size_t(set) * (2 * D + 2);   // [re, im] x D lags, noise power, column count
  // lags: thread -> (d, n-range)
  const int nparts = max(1, int(blockDim.x) / D);
  for (int d0 = 0; d0 < D; d0 += blockDim.x / nparts) {
    const int d = d0 + int(threadIdx.x) % (blockDim.x / nparts), pr = int(threadIdx.x) / (blockDim.x / nparts);
    float re = 0.f, im = 0.f;
    if (d < D && pr < nparts) {
      const int len = N - d, chunk = (len + nparts - 1) / nparts;
      const int n1 = min(len, (pr + 1) * chunk);
      for (int n = pr * chunk; n < n1; ++n) {
        const float2 a = ls[n + d], b = ls[n];     // a conj(b)
        re = fmaf(a.x, b.x, fmaf(a.y, b.y, re));
        im = fmaf(a.y, b.x, fmaf(-a.x, b.y, im));
      }
    }
    part[2 * threadIdx.x] = re;
    part[2 * threadIdx.x + 1] = im;
    __syncthreads();
    if (threadIdx.x < blockDim.x / nparts) {
      const int dd = d0 + threadIdx.x;
      if (dd < D) {
        double sr = 0, si = 0;
        for (int q = 0; q < nparts; ++q) {
          sr += part[2 * (q * (blockDim.x / nparts) + threadIdx.x)];
          si += part[2 * (q * (blockDim.x / nparts) + threadIdx.x) + 1];
        }
        atomicAdd(&acc_s[2 * dd], sr);
        atomicAdd(&acc_s[2 * dd + 1], si);
      }
    }
    __syncthreads();
  }
  // noise window: B delay bins centred on N/2
  const int lo = N / 2 - B / 2;
  double pw = 0;
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    const int kap = lo + i;
    float re = 0.f, im = 0.f;
    int idx = 0;                                      // (n * kap) mod N
    for (int n = 0; n < N; ++n) {
      const float2 w = tw[idx], v = ls[n];
      re = fmaf(v.x, w.x, fmaf(-v.y, w.y, re));
      im = fmaf(v.x, w.y, fmaf(v.y, w.x, im));
      idx += kap;
      if (idx >= N) idx -= N;
    }
    pw += double(re) * re + double(im) * im;
  }
  part[threadIdx.x] = pw;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) part[threadIdx.x] += part[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    atomicAdd(&acc_s[2 * D], part[0] / N);            // unitary IDFT: |sum|^2 / N
    atomicAdd(&acc_s[2 * D + 1], 1.0);
  }
}

__global__ void k7_finalize(const double *__restrict__ acc, int n_sets, int N, int D, int B, double *__restrict__ r,
                            double *__restrict__ sigma2) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_sets) return;
  const double *a = acc + size_t(s) * (2 * D + 2);
  const double C = a[2 * D + 1];
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  const double s2 = C > 0 ? a[2 * D] / (C * B) : nan;
  sigma2[s] = s2;
  for (int d = 0; d < D; ++d) {
    const double den = C * (N - d);
    r[(size_t(s) * D + d) * 2] = C > 0 ? a[2 * d] / den - (d == 0 ? s2 : 0.0) : nan;
    r[(size_t(s) * D + d) * 2 + 1] = C > 0 ? a[2 * d + 1] / den : nan;
  }
}

}  // namespace
}  // namespace ce

extern "C" {

int ce_stats_workspace_bytes(int32_t n_sets, int32_t D, int64_t *out) {
  if (out == nullptr || n_sets < 1 || D < 1) {
    ce::set_last_error("ce_stats_workspace_bytes: need n_sets >= 1, D >= 1, out != NULL");
    return CE_EINVAL;
  }
  *out = int64_t(n_sets) * (2 * int64_t(D) + 2) * int64_t(sizeof(double));
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
  if (cols > 0x7fffffffLL) return fail(CE_EINVAL, "ce_stats_estimate: too many columns");
  const size_t smem = size_t(2) * N * sizeof(float2);
  if (smem > 200 * 1024) return fail(CE_EINVAL, "ce_stats_estimate: N too large (N <= 12800)");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double *acc = static_cast<double *>(d_work);
  cudaError_t e = cudaMemsetAsync(acc, 0, size_t(n_sets) * (2 * D + 2) * sizeof(double), st);
  if (e == cudaSuccess && smem > 48 * 1024)
    e = cudaFuncSetAttribute(ce::k7_accumulate, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) {
    ce::set_last_error(std::string("ce_stats_estimate: ") + cudaGetErrorString(e));
    return CE_ECUDA;
  }
  ce::k7_accumulate<<<unsigned(cols), ce::K7_THREADS, smem, st>>>(static_cast<const float2 *>(d_y),
                                                                  static_cast<const float2 *>(d_x), M, K, N,
                                                                  d_set_of_instance, n_sets, D, B, acc);
  ce::k7_finalize<<<(n_sets + 127) / 128, 128, 0, st>>>(acc, n_sets, N, D, B, static_cast<double *>(d_r),
                                                       static_cast<double *>(d_sigma2));
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    ce::set_last_error(std::string("ce_stats_estimate: launch: ") + cudaGetErrorString(e));
    return CE_ECUDA;
  }
  return CE_OK;
}

}  // extern "C"
