// K9 -- the lag correlation of the statistics estimator (NEXT-3, reading D1) through the power spectrum
// of the LS rows (Wiener-Khinchin):
//   S[d] = sum_c sum_n H[c, n+d] conj(H[c, n]) = (1/L) sum_f P[f] e^{+2 pi i f d / L},   P[f] = sum_c |X_c[f]|^2,
// X_c = the L-point DFT of the LS row H[c] = y / x (Eq. 9) zero-padded from N to a power of two
// L >= N + D - 1, so that no circular wrap reaches a lag d < D.  Same quantity K7a (direct sums) and K8 (banded Gram
// matrix on the tensor cores) compute, in O(L log L) per row instead of O(N D): config 4 (N = 1200, D = 150) does
// ~0.11 Mflop per row here against 1.4 Mflop per row in the direct sum.
//
// K9a (k9_spectrum): a team of L/16 threads per LS row (16 complex values per thread), several rows per CTA from one
// instance (one statistic set).  A Stockham autosort FFT in radix-16 passes (a final radix 2/4/8 pass when log2 L
// is not a multiple of 4): the first pass reads y and x straight from global memory (coalesced, LS division fused,
// zero beyond N), intermediate passes go through a padded shared-memory row (index i + i/16: conflict-free for the
// pass patterns), and the last pass squares its outputs into per-thread FP32 accumulators (a fixed set of
// frequencies per thread).  Per CTA, the teams' accumulators are summed in shared memory and added to the set's
// FP64 spectrum P[s][f] with one atomic per frequency.
// K9b (k9_lags): per (set, 8 lags) the direct inverse DFT of P at d < D in FP64 over an FP64 twiddle table, written
// into K7's accumulator layout (acc[s][2d], acc[s][2d+1]); K7 adds the noise floor and the column count, K7b
// normalises.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "ce_internal.h"
#include "tc_ptx.cuh"

namespace ce {
namespace {

constexpr int K9_MIN_LOG2 = 6;    // L >= 64 (at least one radix-16 pass before the last one)
constexpr int K9_MAX_LOG2 = 13;   // L <= 8192 (one row of 8704 padded complex values in shared memory)

// complex arithmetic on packed FP32 pairs (FADD2 / FMUL2 / FFMA2, one instruction per complex add and two per
// complex multiply; a scalar operand is broadcast, a pair read with its halves swapped)
__device__ __forceinline__ uint64_t u64(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 f2(uint64_t v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ float2 c_add(float2 a, float2 b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(u64(a.x, a.y)), "l"(u64(b.x, b.y)));
  return f2(r);
}
__device__ __forceinline__ float2 c_sub(float2 a, float2 b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(u64(a.x, a.y)), "l"(u64(b.x, b.y)));
  return f2(r);
}
// a * w with w given as (w.x, w.y) and its companion ny = (-w.y, w.y):  (a.x, a.y) w.x + (a.y, a.x) ny
__device__ __forceinline__ float2 c_mul_t(float2 a, float wx, uint64_t ny) {
  uint64_t t, r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(u64(a.y, a.x)), "l"(ny));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(u64(a.x, a.y)), "l"(u64(wx, wx)), "l"(t));
  return f2(r);
}
__device__ __forceinline__ float2 c_mul(float2 a, float2 w) { return c_mul_t(a, w.x, u64(-w.y, w.y)); }

// d * e^{-2 pi i k / 16}; k is a compile-time constant once the callers' loops are unrolled
__device__ __forceinline__ float2 rot16(float2 d, int k) {
  switch (k & 15) {
    case 0: return d;
    case 4: return make_float2(d.y, -d.x);
    case 8: return make_float2(-d.x, -d.y);
    case 12: return make_float2(-d.y, d.x);
    default: break;
  }
  const float c1 = 0.92387953251128674f, c2 = 0.70710678118654752f, c3 = 0.38268343236508977f;
  float c = 0.f, s = 0.f;   // cos, sin of 2 pi k / 16
  switch (k & 15) {
    case 1: c = c1; s = c3; break;
    case 2: c = c2; s = c2; break;
    case 3: c = c3; s = c1; break;
    case 5: c = -c3; s = c1; break;
    case 6: c = -c2; s = c2; break;
    case 7: c = -c1; s = c3; break;
    case 9: c = -c1; s = -c3; break;
    case 10: c = -c2; s = -c2; break;
    case 11: c = -c3; s = -c1; break;
    case 13: c = c3; s = -c1; break;
    case 14: c = c2; s = -c2; break;
    case 15: c = c1; s = -c3; break;
  }
  // (x + i y)(c - i s)
  return c_mul_t(d, c, u64(s, -s));
}

__host__ __device__ constexpr int bitrev(int i, int bits) {
  int r = 0;
  for (int b = 0; b < bits; ++b) r |= ((i >> b) & 1) << (bits - 1 - b);
  return r;
}
__host__ __device__ constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v >> 1); }

// in-register forward DFT_R (e^{-2 pi i n k / R}), natural order in and out: radix-2 decimation in frequency, then
// the bit-reversal permutation (register renaming)
template <int R>
__device__ __forceinline__ void dft_reg(float2 *v) {
#pragma unroll
  for (int h = R / 2; h >= 1; h >>= 1) {
#pragma unroll
    for (int s = 0; s < R; s += 2 * h) {
#pragma unroll
      for (int i = 0; i < h; ++i) {
        const float2 a = v[s + i], b = v[s + i + h];
        v[s + i] = c_add(a, b);
        v[s + i + h] = rot16(c_sub(a, b), i * (8 / h));   // e^{-2 pi i i / (2h)} = e^{-2 pi i (8 i / h) / 16}
      }
    }
  }
  float2 t[R];
#pragma unroll
  for (int i = 0; i < R; ++i) t[bitrev(i, ilog2(R))] = v[i];
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = t[i];
}

// v[r] *= w^r, w = e^{-2 pi i k / (Ns R)}, 0 < r < R: FP32 sincospi at r = 1 and r = 8, running products in between
// (at most 7 roundings from an exact value: ~1e-6 relative, far inside the 1e-4 bar on the lags)
template <int R>
__device__ __forceinline__ void apply_twiddles(float2 *v, int k, int NsR) {
  // angle -2 pi k / (Ns R) reduced to (-pi, pi] for the MUFU sine / cosine (abs. error ~5e-7)
  const int kk = 2 * k > NsR ? k - NsR : k;
  const float a = -6.28318530717958648f * float(kk) / float(NsR);
  float s, c;
  __sincosf(a, &s, &c);
  const float2 w1 = make_float2(c, s);
  const uint64_t w1n = u64(-s, s);
  float2 w = w1;
#pragma unroll
  for (int r = 1; r < R && r < 8; ++r) {
    v[r] = c_mul(v[r], w);
    if (r + 1 < R && r + 1 < 8) w = c_mul_t(w, w1.x, w1n);
  }
  if constexpr (R > 8) {
    // e^{8 i a} from the integer angle 8 k mod (Ns R), again reduced to (-pi, pi]
    int k8 = (8 * k) % NsR;
    k8 = 2 * k8 > NsR ? k8 - NsR : k8;
    __sincosf(-6.28318530717958648f * float(k8) / float(NsR), &s, &c);
    w = make_float2(c, s);
#pragma unroll
    for (int r = 8; r < R; ++r) {
      v[r] = c_mul(v[r], w);
      if (r + 1 < R) w = c_mul_t(w, w1.x, w1n);
    }
  }
}

__device__ __forceinline__ int pad(int i) { return i + (i >> 4); }


// One Stockham pass of radix R over a team's row: butterflies j = jt + q L/16 (q < 16/R), inputs j + r L/R, outputs
// ((j / Ns) Ns R) + (j mod Ns) + r Ns.  v holds the thread's 16 values [q][r].
template <int R, int L>
__device__ __forceinline__ void pass_compute(float2 *v, int jt, int lNs) {
  const int Ns = 1 << lNs;
#pragma unroll
  for (int q = 0; q < 16 / R; ++q) {
    const int j = jt + q * (L / 16);
    const int k = j & (Ns - 1);
    if (lNs > 0) apply_twiddles<R>(v + q * R, k, Ns * R);
    dft_reg<R>(v + q * R);
  }
}
template <int R, int L>
__device__ __forceinline__ void pass_load(float2 *v, const float2 *buf, int jt) {
#pragma unroll
  for (int q = 0; q < 16 / R; ++q) {
    const int j = jt + q * (L / 16);
#pragma unroll
    for (int r = 0; r < R; ++r) v[q * R + r] = buf[pad(j + r * (L / R))];
  }
}
template <int R, int L>
__device__ __forceinline__ int out_index(int j, int lNs, int r) {
  return ((j >> lNs) << (lNs + ilog2(R))) + (j & ((1 << lNs) - 1)) + (r << lNs);
}
template <int R, int L>
__device__ __forceinline__ void pass_store(const float2 *v, float2 *buf, int jt, int lNs) {
#pragma unroll
  for (int q = 0; q < 16 / R; ++q) {
    const int j = jt + q * (L / 16);
#pragma unroll
    for (int r = 0; r < R; ++r) buf[pad(out_index<R, L>(j, lNs, r))] = v[q * R + r];
  }
}

template <int LOG2L>
struct K9Shape {
  static constexpr int L = 1 << LOG2L;
  static constexpr int TEAM = L / 16;                       // threads per row
  static constexpr int NT = TEAM >= 256 ? TEAM : 256;       // threads per CTA
  static constexpr int TEAMS = NT / TEAM;                   // rows in flight per CTA
  static constexpr int LP = L + L / 16;                     // padded row
  static constexpr int N16 = LOG2L / 4;                     // radix-16 passes
  static constexpr int RLAST = 1 << (LOG2L % 4);            // final pass radix (1: the last radix-16 pass is last)
};

// P[set][f] += sum over this CTA's rows of |X_row[f]|^2.  CTA = (instance t, rows [g cpb, (g + 1) cpb)).
// PF (N even, 16-byte aligned y): each team's y rows are bulk-copied (cp.async.bulk, one mbarrier per stage) into a
// 2-stage shared-memory ring two rows ahead, so pass 0 reads shared memory instead of waiting on DRAM (ncu, config 4
// without it: long_scoreboard 37 % of the stall samples, FMA pipe 50 %)
template <int LOG2L, bool PF>
__global__ void __launch_bounds__(K9Shape<LOG2L>::NT, K9Shape<LOG2L>::NT >= 512 ? 1 : 2) k9_spectrum(const float2 *__restrict__ y, const float2 *__restrict__ x,
                                                                   int M, int K, int N, const int32_t *__restrict__ soi,
                                                                   int n_sets, int cpb, double *__restrict__ P) {
  using S = K9Shape<LOG2L>;
  constexpr int L = S::L, TEAM = S::TEAM, TEAMS = S::TEAMS;
  extern __shared__ float2 sm9[];
  float2 *ystg = sm9 + TEAMS * S::LP;                       // PF: [TEAMS][2][N] y rows
  uint64_t *ybar = reinterpret_cast<uint64_t *>(ystg + (PF ? size_t(TEAMS) * 2 * N : 0));   // PF: [TEAMS][2]
  const int MK = M * K;
  const int groups = (MK + cpb - 1) / cpb;
  const int t = blockIdx.x / groups, g = blockIdx.x % groups;
  const int set = soi ? soi[t] : 0;
  if (set < 0 || set >= n_sets) return;                     // instances with an out-of-range set are skipped
  const int team = threadIdx.x / TEAM, jt = threadIdx.x % TEAM;
  float2 *buf = sm9 + team * S::LP;
  const int c_lo = g * cpb, c_hi = min(MK, c_lo + cpb);
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.f;
  const uint32_t ybytes = uint32_t(N) * 8u;
  if constexpr (PF) {
    if (jt == 0) {
      mbar_init(&ybar[2 * team], 1);
      mbar_init(&ybar[2 * team + 1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
      for (int st = 0; st < 2; ++st) {
        const int cr = c_lo + st * TEAMS + team;
        if (cr < c_hi) {
          mbar_arrive_expect_tx(&ybar[2 * team + st], ybytes);
          bulk_g2s(ystg + (2 * team + st) * N, y + (size_t(t) * MK + cr) * N, ybytes, &ybar[2 * team + st]);
        }
      }
    }
    __syncthreads();                                        // barriers initialised before any team waits on them
  }
  int it = 0;
  for (int c0 = c_lo; c0 < c_hi; c0 += TEAMS, ++it) {
    const int c = c0 + team;
    const bool ok = c < c_hi;
    float2 v[16];
    // pass 0 (radix 16, Ns = 1): LS values from global memory (PF: y from the team's ring), zero beyond N and for
    // absent rows
    {
      const float2 *yr = y + (size_t(t) * MK + (ok ? c : c_lo)) * N;
      if constexpr (PF) {
        yr = ystg + (2 * team + (it & 1)) * N;
        if (ok) mbar_wait(&ybar[2 * team + (it & 1)], (it >> 1) & 1);
      }
      const float2 *xr = x + (size_t(t) * K + (ok ? c : c_lo) % K) * N;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int n = jt + r * TEAM;
        float2 h = make_float2(0.f, 0.f);
        if (ok && n < N) {
          const float2 yv = yr[n], xv = xr[n];
          float inv;
          asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(fmaf(xv.x, xv.x, xv.y * xv.y)));
          h = make_float2(fmaf(yv.x, xv.x, yv.y * xv.y) * inv, fmaf(yv.y, xv.x, -yv.x * xv.y) * inv);
        }
        v[r] = h;
      }
      dft_reg<16>(v);
    }
    int lNs = 4;
    pass_store<16, L>(v, buf, jt, 0);
    __syncthreads();
    if constexpr (PF) {                                     // every thread has read this stage: refill it two rows ahead
      const int cr = c + 2 * TEAMS;
      if (jt == 0 && cr < c_hi) {
        mbar_arrive_expect_tx(&ybar[2 * team + (it & 1)], ybytes);
        bulk_g2s(ystg + (2 * team + (it & 1)) * N, y + (size_t(t) * MK + cr) * N, ybytes, &ybar[2 * team + (it & 1)]);
      }
    }
    // middle radix-16 passes
#pragma unroll 1
    for (int p = 1; p < S::N16 - (S::RLAST == 1 ? 1 : 0); ++p) {
      pass_load<16, L>(v, buf, jt);
      __syncthreads();
      pass_compute<16, L>(v, jt, lNs);
      pass_store<16, L>(v, buf, jt, lNs);
      __syncthreads();
      lNs += 4;
    }
    // last pass: squares into the accumulators (frequency out_index(j, lNs, r) for slot q R + r)
    constexpr int RL = S::RLAST == 1 ? 16 : S::RLAST;
    pass_load<RL, L>(v, buf, jt);
    __syncthreads();                                        // the next row's pass 0 may overwrite buf
    pass_compute<RL, L>(v, jt, lNs);
    if (ok) {
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = fmaf(v[i].x, v[i].x, fmaf(v[i].y, v[i].y, acc[i]));
    }
  }
  // teams' accumulators -> shared memory (float view of the rows), summed per frequency, FP64 atomics
  constexpr int RL = S::RLAST == 1 ? 16 : S::RLAST;
  int lNs_last = 4 * (S::N16 - (S::RLAST == 1 ? 1 : 0));
  float *red = reinterpret_cast<float *>(sm9);
#pragma unroll
  for (int q = 0; q < 16 / RL; ++q) {
    const int j = jt + q * (L / 16);
#pragma unroll
    for (int r = 0; r < RL; ++r) red[team * L + out_index<RL, L>(j, lNs_last, r)] = acc[q * RL + r];
  }
  __syncthreads();
  double *Ps = P + size_t(set) * L;
  for (int f = threadIdx.x; f < L; f += blockDim.x) {
    float s = 0.f;
#pragma unroll
    for (int tm = 0; tm < TEAMS; ++tm) s += red[tm * L + f];
    atomicAdd(&Ps[f], double(s));
  }
}

// acc[s][2d], acc[s][2d + 1] = Re, Im of (1/L) sum_f P[s][f] e^{+2 pi i f d / L}, d < D; one warp per lag
constexpr int K9B_LAGS = 8;
__global__ void __launch_bounds__(32 * K9B_LAGS) k9_lags(const double *__restrict__ P, int L, int D,
                                                         double *__restrict__ acc) {
  extern __shared__ double2 tab[];                          // [L] (cos, sin)(2 pi k / L)
  for (int k = threadIdx.x; k < L; k += blockDim.x) {
    double s, c;
    sincospi(2.0 * double(k) / double(L), &s, &c);
    tab[k] = make_double2(c, s);
  }
  __syncthreads();
  const int s = blockIdx.y;
  const int d = blockIdx.x * K9B_LAGS + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (d >= D) return;
  const double *Ps = P + size_t(s) * L;
  double re = 0, im = 0;
  for (int f = lane; f < L; f += 32) {
    const double p = Ps[f];
    const double2 w = tab[(static_cast<long long>(f) * d) & (L - 1)];
    re = fma(p, w.x, re);
    im = fma(p, w.y, im);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    re += __shfl_xor_sync(0xffffffffu, re, o);
    im += __shfl_xor_sync(0xffffffffu, im, o);
  }
  if (lane == 0) {
    double *a = acc + size_t(s) * (2 * D + 2);
    a[2 * d] = re / L;
    a[2 * d + 1] = im / L;
  }
}

template <int LOG2L>
cudaError_t launch_spectrum_t(const float2 *y, const float2 *x, int T, int M, int K, int N, const int32_t *soi,
                              int n_sets, double *P, cudaStream_t st) {
  using S = K9Shape<LOG2L>;
  static const int env_pf = getenv("CE_K9_PF") ? atoi(getenv("CE_K9_PF")) : 1;   // experiments
  const size_t smem0 = size_t(S::TEAMS) * S::LP * sizeof(float2);
  const size_t smem_pf = smem0 + size_t(S::TEAMS) * 2 * N * sizeof(float2) + size_t(S::TEAMS) * 2 * sizeof(uint64_t);
  const bool pf = env_pf != 0 && N % 2 == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0 && smem_pf <= 220 * 1024;
  const size_t smem = pf ? smem_pf : smem0;
  const void *fn = pf ? (const void *)k9_spectrum<LOG2L, true> : (const void *)k9_spectrum<LOG2L, false>;
  cudaError_t e = smem_opt_in(fn, smem);
  if (e != cudaSuccess) return e;
  int nsm = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // rows per CTA: about 4 waves of 2 CTAs per SM (each CTA adds L FP64 atomics at its end), whole teams
  const long long rows = (long long)T * M * K;
  long long cpb = (rows + 8LL * nsm - 1) / (8LL * nsm);
  cpb = ((cpb + S::TEAMS - 1) / S::TEAMS) * S::TEAMS;
  cpb = std::max<long long>(cpb, S::TEAMS);
  cpb = std::min<long long>(cpb, (long long)M * K);
  const long long groups = ((long long)M * K + cpb - 1) / cpb;
  const long long ctas = (long long)T * groups;
  if (ctas > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  if (pf)
    k9_spectrum<LOG2L, true><<<unsigned(ctas), S::NT, smem, st>>>(y, x, M, K, N, soi, n_sets, int(cpb), P);
  else
    k9_spectrum<LOG2L, false><<<unsigned(ctas), S::NT, smem, st>>>(y, x, M, K, N, soi, n_sets, int(cpb), P);
  return cudaGetLastError();
}

}  // namespace

int spectrum_log2(int32_t N, int32_t D) {
  int l = K9_MIN_LOG2;
  while (l <= K9_MAX_LOG2 && (1 << l) < N + D - 1) ++l;
  return l <= K9_MAX_LOG2 ? l : -1;
}

cudaError_t launch_spectrum_lags(const float2 *y, const float2 *x, int32_t T, int32_t M, int32_t K, int32_t N,
                                 const int32_t *soi, int32_t n_sets, int32_t D, double *P, double *acc,
                                 cudaStream_t st) {
  const int l = spectrum_log2(N, D);
  if (l < 0) return cudaErrorInvalidValue;
  const int L = 1 << l;
  cudaError_t e = cudaMemsetAsync(P, 0, size_t(n_sets) * L * sizeof(double), st);
  if (e != cudaSuccess) return e;
  switch (l) {
    case 6: e = launch_spectrum_t<6>(y, x, T, M, K, N, soi, n_sets, P, st); break;
    case 7: e = launch_spectrum_t<7>(y, x, T, M, K, N, soi, n_sets, P, st); break;
    case 8: e = launch_spectrum_t<8>(y, x, T, M, K, N, soi, n_sets, P, st); break;
    case 9: e = launch_spectrum_t<9>(y, x, T, M, K, N, soi, n_sets, P, st); break;
    case 10: e = launch_spectrum_t<10>(y, x, T, M, K, N, soi, n_sets, P, st); break;
    case 11: e = launch_spectrum_t<11>(y, x, T, M, K, N, soi, n_sets, P, st); break;
    case 12: e = launch_spectrum_t<12>(y, x, T, M, K, N, soi, n_sets, P, st); break;
    case 13: e = launch_spectrum_t<13>(y, x, T, M, K, N, soi, n_sets, P, st); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  const size_t tsm = size_t(L) * sizeof(double2);
  e = smem_opt_in((const void *)k9_lags, tsm);
  if (e != cudaSuccess) return e;
  k9_lags<<<dim3((D + K9B_LAGS - 1) / K9B_LAGS, n_sets), 32 * K9B_LAGS, tsm, st>>>(P, L, D, acc);
  return cudaGetLastError();
}

}  // namespace ce
