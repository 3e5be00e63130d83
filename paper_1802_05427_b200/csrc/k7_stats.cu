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
// K7a: one CTA per K7_CPB columns of one instance: the N twiddles exp(j 2 pi n / N) and, column by column, the LS
// row in shared memory; threads own blocks of 4 lags (x as many n-ranges as fit in 256 threads, partial sums
// carried in registers across the columns) and then (bin, n-range) pairs of the noise window; one FP64
// reduction + atomics per CTA into the per-set accumulators.  K7b: one thread per set normalises.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "ce_internal.h"

namespace ce {
namespace {

constexpr int K7_THREADS = 256;

constexpr int K7_CPB = 1;      // columns per CTA, same instance (measured on config 3: 1 -> 139 us, 2 -> 143, 8 -> 184)
constexpr int LB = 4;          // lags per thread

__global__ void __launch_bounds__(K7_THREADS) k7_accumulate(const float2 *__restrict__ y, const float2 *__restrict__ x,
                                                            int M, int K, int N, const int32_t *__restrict__ soi,
                                                            int n_sets, int D, int B, double *__restrict__ acc,
                                                            int lags, int cpb) {
  extern __shared__ float2 sm7[];
  float2 *ls = sm7;                                  // [N]
  float2 *tw = sm7 + N;                              // [N] exp(+j 2 pi n / N)
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
  // noise work split: thread -> (bin, n-range)
  const int lo = N / 2 - B / 2;
  const int bparts = max(1, int(blockDim.x) / min(B, int(blockDim.x)));
  const int bins_per_pass = blockDim.x / bparts;
  double pw = 0;
  for (int c = c_lo; c < c_hi; ++c) {
    const float2 *yr = y + (size_t(t) * MK + c) * N;
    const float2 *xr = x + (size_t(t) * K + c % K) * N;
    __syncthreads();                                 // previous column's ls fully consumed
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
      const float2 yv = yr[n], xv = xr[n];
      const float inv = 1.0f / (xv.x * xv.x + xv.y * xv.y);
      ls[n] = make_float2((yv.x * xv.x + yv.y * xv.y) * inv, (yv.y * xv.x - yv.x * xv.y) * inv);
    }
    __syncthreads();
    // lags: ls[n] is shared by LB lags and ls[n+d..n+d+LB-1] slides (8 FMA per shared-memory read)
    for (int l0 = 0; l0 < n_lb; l0 += lanes) {
      const int lbk = l0 + lb;
      if (lanes >= n_lb ? lag_thread : (lbk < n_lb && pr < nparts)) {
        const int d = lbk * LB;
        const int len = N - d, chunk = (len + nparts - 1) / nparts;
        const int n0 = pr * chunk, n1 = min(len, n0 + chunk);
        float2 win[LB];
#pragma unroll
        for (int i = 0; i < LB; ++i) win[i] = (n0 + d + i < N) ? ls[n0 + d + i] : make_float2(0.f, 0.f);
        float r4[LB] = {0.f, 0.f, 0.f, 0.f}, i4[LB] = {0.f, 0.f, 0.f, 0.f};
        for (int n = n0; n < n1; ++n) {
          const float2 bv = ls[n];
#pragma unroll
          for (int i = 0; i < LB; ++i) {             // win[i] = ls[n + d + i] (zero beyond N)
            r4[i] = fmaf(win[i].x, bv.x, fmaf(win[i].y, bv.y, r4[i]));
            i4[i] = fmaf(win[i].y, bv.x, fmaf(-win[i].x, bv.y, i4[i]));
          }
#pragma unroll
          for (int i = 0; i < LB - 1; ++i) win[i] = win[i + 1];
          win[LB - 1] = (n + d + LB < N) ? ls[n + d + LB] : make_float2(0.f, 0.f);
        }
        if (lanes >= n_lb) {
#pragma unroll
          for (int i = 0; i < LB; ++i) {
            re[i] += r4[i];
            im[i] += i4[i];
          }
        } else {                                     // D > 4 * 256: no register carry, add directly
          for (int i = 0; i < LB && d + i < D; ++i) {
            atomicAdd(&acc_s[2 * (d + i)], double(r4[i]));
            atomicAdd(&acc_s[2 * (d + i) + 1], double(i4[i]));
          }
        }
      }
    }
    // noise window: the complex partial sums of a bin are combined before taking |.|^2
    for (int b0 = 0; b0 < B; b0 += bins_per_pass) {
      const int bi = b0 + int(threadIdx.x) % bins_per_pass, bp = int(threadIdx.x) / bins_per_pass;
      float nre = 0.f, nim = 0.f;
      if (bi < B && bp < bparts) {
        const int kap = lo + bi;
        const int chunk = (N + bparts - 1) / bparts;
        const int n0 = bp * chunk, n1 = min(N, n0 + chunk);
        // the twiddle e^{+j 2 pi n kap / N} advances by a register rotation, re-seeded from the table at the
        // start of every 32-tone block (FP32 rotation error <= ~32 * 2^-23): the inner loop is one broadcast
        // shared-memory read (ls[n]) and 8 FP32 operations per tone, no gathers and no index arithmetic
        const float2 rot = tw[kap % N];
        const int step32 = int((32LL * kap) % N);
        int idx = int((static_cast<long long>(n0) * kap) % N);   // (n * kap) mod N at the block start
        const float2 *lp = ls + n0;
        for (int nb = n0; nb < n1; nb += 32) {
          float2 w = tw[idx];
          const int cnt = min(32, n1 - nb);
#pragma unroll 4
          for (int q = 0; q < cnt; ++q) {
            const float2 v = lp[q];
            nre = fmaf(v.x, w.x, fmaf(-v.y, w.y, nre));
            nim = fmaf(v.x, w.y, fmaf(v.y, w.x, nim));
            w = make_float2(fmaf(w.x, rot.x, -w.y * rot.y), fmaf(w.x, rot.y, w.y * rot.x));
          }
          lp += 32;
          idx += step32;
          if (idx >= N) idx -= N;
        }
      }
      __syncthreads();                               // part[] free
      part[2 * threadIdx.x] = nre;
      part[2 * threadIdx.x + 1] = nim;
      __syncthreads();
      if (threadIdx.x < bins_per_pass && b0 + int(threadIdx.x) < B) {
        double sr = 0, si = 0;
        for (int q = 0; q < bparts; ++q) {
          sr += part[2 * (q * bins_per_pass + threadIdx.x)];
          si += part[2 * (q * bins_per_pass + threadIdx.x) + 1];
        }
        pw += sr * sr + si * si;
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
  // columns per CTA: 1 when K7 also runs the lags (measured: more is slower there); with the lags on K8 the
  // per-CTA twiddle table and row-load latency are amortised over several columns
  static const int env_cpb = getenv("CE_K7_CPB") ? atoi(getenv("CE_K7_CPB")) : 0;   // experiments
  static const int env_gram = getenv("CE_K8_GRAM") ? atoi(getenv("CE_K8_GRAM")) : -1;   // experiments: 0 off, 1 force
  const bool gram = env_gram != 0;
  // K8 pays a per-unit factor table and diagonal-bin epilogue: measured faster from config 4's 61440 columns
  // up (config 4: 2.4 vs 4.1 ms, config 5: 9.7 vs 17.2 ms) and slower on config 3's 1536 (164 vs 147 us)
  const bool k8 = gram && (cols >= 16384 || env_gram == 1) && ce::gram_launchable(static_cast<const float2 *>(d_y), K, N, D);
  int cpb = k8 ? 8 : ce::K7_CPB;
  if (env_cpb > 0) cpb = env_cpb;
  cpb = std::max(1, std::min(cpb, M * K));
  const long long ctas = (long long)T * ((static_cast<long long>(M) * K + cpb - 1) / cpb);
  if (cols > 0x7fffffffLL || ctas > 0x7fffffffLL) return fail(CE_EINVAL, "ce_stats_estimate: too many columns");
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
  // the lag correlation on the tensor cores (K8) when it fits; K7 then adds the noise floor and column count
  int k7_lags = D;
  if (k8) {
    e = ce::launch_gram(static_cast<const float2 *>(d_y), static_cast<const float2 *>(d_x), T, M, K, N,
                        d_set_of_instance, n_sets, D, acc, st);
    if (e != cudaSuccess) {
      ce::set_last_error(std::string("ce_stats_estimate: K8 launch: ") + cudaGetErrorString(e));
      return CE_ECUDA;
    }
    k7_lags = 0;
  }
  ce::k7_accumulate<<<unsigned(ctas), ce::K7_THREADS, smem, st>>>(static_cast<const float2 *>(d_y),
                                                                  static_cast<const float2 *>(d_x), M, K, N,
                                                                  d_set_of_instance, n_sets, D, B, acc, k7_lags, cpb);
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
