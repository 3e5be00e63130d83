/*
 * ce.h -- C ABI of libce, the B200 (sm_100a) block-LMMSE pilot channel estimator.
 *
 * Method (arXiv 1802.05427, "Implementation of Massive MIMO Uplink Receiver on
 * RaPro Prototyping Platform"; line numbers refer to /root/reference/PAPER.md):
 *
 *   LS at the pilots        H_LS = Y / X                      PAPER.md:173-180 (Eq. 8-9), 438
 *   block LMMSE filter      W_b  = R_b (R_b + sigma^2 I)^-1    PAPER.md:306-309 (Eq. 17), 345-349
 *   block application       H    = W_b H_LS  per window        PAPER.md:186-190 (Eq. 12), 400-403
 *
 * generalised from the paper's 12x12 "12W" groups to
 * b x b blocks of the N x N Toeplitz frequency autocorrelation R_hh, laid out as
 * non-overlapping blocks (stride == b) or overlapping windows that keep their
 * centre `stride` outputs (stride < b), with the paper's edge clamping
 * (Table II).
 *
 * Window geometry (reading A7): n_windows = ceil((N-b)/stride) + 1;
 * window w reads LS tones [a_w, a_w+b) with a_w = min(w*stride, N-b) and keeps
 * outputs [o_w, o_{w+1}) with o_0 = 0, o_w = w*stride + floor((b-stride)/2),
 * o_{n_windows} = N.  The kept ranges partition [0, N).
 *
 * Data layout (all complex values are interleaved {re, im}):
 *   y  : complex64 [T][M][K][N]  received pilot symbols, antenna-major   (caller-owned)
 *   x  : complex64 [T][K][N]     pilots, shared by all antennas           (caller-owned)
 *   h  : complex64 [T][M][K][N]  channel estimates                        (caller-owned)
 *   W  : complex64 [n_sets][b][b] filters, row-major                     (library-owned)
 * T = estimation instances (slots x pilot symbols), M = BS antennas, K = users,
 * N = subcarriers (contiguous tones 0..N-1, reading A10).
 *
 * Conventions
 *   - Every function returns a ce_status (0 = OK, < 0 = error); ce_last_error()
 *     gives a human-readable detail of the calling thread's last failure.
 *   - A handle is bound to the CUDA device that is current at ce_init and is used
 *     from one host thread at a time.  Multi-GPU = one handle per device/rank.
 *   - `stream` arguments are cudaStream_t values passed as void* (NULL = legacy
 *     default stream).  Device entry points are asynchronous on that stream.
 *   - There is no CPU fallback: without a usable sm_100 device, calls that need the
 *     GPU return CE_ENODEV / CE_ECUDA.
 */
#ifndef CE_H
#define CE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CE_OK = 0,
  CE_EINVAL = -1,  /* invalid argument: sizes, pointers, alignment, aliasing, sigma^2 */
  CE_ENOMEM = -2,  /* host or device allocation failed */
  CE_ECUDA = -3,   /* a CUDA runtime call failed (detail in ce_last_error) */
  CE_ENOTPD = -4,  /* filter build: R_b + sigma^2 I not positive definite (a pivot <= 0 or NaN) */
  CE_ESTATE = -5,  /* ce_estimate before a successful ce_build_filters */
  CE_ENODEV = -6   /* no CUDA device, or not compute capability 10.x */
} ce_status;

typedef enum {
  CE_KERNEL_AUTO = 0,   /* library picks the fastest kernel meeting the 1e-4 parity bar */
  CE_KERNEL_SIMT = 1,   /* K2: FP32 SIMT complex FMA contraction (fallback when the tensor-core filter banks do not
                           fit; north_star's SIMT design, kept for parity and as the FP32 reference path) */
  CE_KERNEL_TF32X3 = 2, /* K3: tcgen05 kind::tf32, error-compensated hi/lo split (3 MMAs) */
  CE_KERNEL_BF16X3 = 3  /* K4: tcgen05 kind::f16 (BF16), hi/lo split (3 MMAs), TMA-fed input ring; launches whose CTAs
                           walk more than two tiles run its CTA-pair variant (cta_group::2, M = 256, half of each
                           filter chunk per CTA): the same products in the same order, still reported as BF16X3 */
  /* 4 was the CTA-pair kernel K5 (filter stationary in TMEM): removed in round 2 -- exact, but pair MMAs with the
   * A operand in TMEM cost 180 cycles flat and it ran 2.6-4.5x slower than K4; 4 is now CE_EINVAL */
} ce_kernel;

typedef struct ce_handle ce_handle; /* opaque */

typedef struct {
  int32_t N;      /* subcarriers, >= 1 */
  int32_t b;      /* block / window length, 1 <= b <= N (b == N gives the full LMMSE) */
  int32_t stride; /* window stride s, 1 <= s <= b: s == b non-overlapping, s < b overlapping */
  int32_t n_sets; /* statistic sets, >= 1 (1 = the paper's fixed design) */
  /* host, [n_sets][N][2] float64: Toeplitz first column r[d] = E{H(n+d) H*(n)}, d = 0..N-1,
   * complex128 interleaved.  Only d < b is used by the filters; r[0]
   * must be real and finite.  Copied by ce_init. */
  const double *r_hh;
  /* host, [n_sets] float64: sigma^2 / sigma_s^2 (Eq. 13), finite and > 0. Copied. */
  const double *sigma2;
} ce_params;

/* Validate `p`, compute the window table on the host, copy the statistics to the
 * current device and allocate W[n_sets][b][b] plus its workspace.
 * Returns CE_EINVAL (nothing allocated, *out untouched) for: p or out NULL, N < 1,
 * b < 1 or b > N, stride < 1 or stride > b, n_sets < 1, r_hh or sigma2 NULL,
 * non-finite r_hh, r[0] not real and > 0, sigma2 <= 0 or non-finite.
 * CE_ENODEV if no compute-capability-10 device is current; CE_ENOMEM on allocation failure. */
int ce_init(const ce_params *p, ce_handle **out);

/* K1 (Eq. 17): per set, A = R_b + sigma^2 I from the Toeplitz first column (Hermitian
 * Toeplitz), W = R_b A^-1 = I - sigma^2 A^-1 in FP64 by the Toeplitz structure in O(b^2): Levinson-Durbin for
 * A^-1 e_0, then the Gohberg-Semencul (Trench) recurrence for every entry (the paper's own solver is a Cholesky,
 * cposv); rounded to complex64.  Enqueued on `stream`, then synchronises that stream once to read
 * the positive-definite flag.  Returns CE_ENOTPD (handle stays unbuilt) if a Levinson prediction-error power
 * (a ratio of leading minors of A) is <= 0 or not finite. */
int ce_build_filters(ce_handle *h, void *stream);

/* K2/K3 hot path (a3-a5 of SURVEY.md §8(a)): for every instance t, window w and column (m,k)
 *   h[t,m,k, o_w:o_{w+1}] = W_{set(t)}[o_w-a_w : o_{w+1}-a_w, :] . (y[t,m,k, a_w:a_w+b] / x[t,k, a_w:a_w+b])
 * with the LS division fused into the operand load.  Device pointers, asynchronous on
 * `stream`: no allocation and no host synchronisation.
 *   d_y, d_x, d_h : device, complex64, 8-byte aligned, layouts above; d_h must not overlap
 *                   d_y or d_x.  Sub-tensors (e.g. an antenna shard [T][M'][K][N] with the
 *                   matching instance range) are passed as offset pointers.
 *   T, M, K       : >= 1.
 *   d_set_of_instance : device int32 [T] with values in [0, n_sets), or NULL (all set 0).
 *                   An out-of-range value makes that instance's outputs NaN.
 * Returns CE_ESTATE before a successful ce_build_filters, CE_EINVAL for bad sizes, NULL or
 * misaligned pointers and aliasing, CE_ECUDA if the launch fails. */
int ce_estimate(ce_handle *h, const void *d_y, const void *d_x, void *d_h,
                int32_t T, int32_t M, int32_t K, const int32_t *d_set_of_instance, void *stream);

/* Same computation on HOST buffers (end-to-end path): copies y and x to device staging buffers
 * owned by the handle (grown on demand), runs the hot path in antenna chunks pipelined over
 * internal streams so host<->device copies overlap compute, copies h back, and returns after
 * the results are in `h_host` (synchronous).  Pinned host memory gives full copy bandwidth.
 * set_of_instance is HOST int32 [T] or NULL. */
int ce_estimate_host(ce_handle *h, const void *y_host, const void *x_host, void *h_host,
                     int32_t T, int32_t M, int32_t K, const int32_t *set_of_instance, void *stream);

/* Asynchronous form of ce_estimate_host: the same copies and kernels, ordered after the work enqueued on `stream`
 * before this call, on the handle's internal streams; the call returns once everything is enqueued, and `stream`
 * does NOT wait for it -- call ce_estimate_host_wait (or synchronise the device) before reading h_host.  y_host,
 * x_host, set_of_instance and h_host must stay valid (and h_host unread) until then.  The handle alternates two
 * device staging slots, so consecutive calls overlap (one call's device->host copies with the next call's
 * host->device copies); a call on a slot waits on the device for the previous user of that slot.  Pinned host
 * memory is required for the copies to be asynchronous.  Same validation and errors as ce_estimate_host. */
int ce_estimate_host_async(ce_handle *h, const void *y_host, const void *x_host, void *h_host,
                           int32_t T, int32_t M, int32_t K, const int32_t *set_of_instance, void *stream);

/* Make `stream` wait (on the device) for every ce_estimate_host_async call enqueued on the handle so far. */
int ce_estimate_host_wait(ce_handle *h, void *stream);

/* Free W, workspace, staging buffers and the handle.  NULL is allowed (no-op). */
int ce_free(ce_handle *h);

/* Choose the contraction kernel (ce_kernel).  CE_EINVAL for an unknown value (including the retired 4), for a
 * tensor-core kernel when its filter banks would exceed 8 GB (very large b x n_sets), and for BF16X3 when some
 * window start a_w is odd (16-byte TMA boxes).  Windows wider than one 256-column accumulator are split into
 * output sub-windows over the same input, so every b fits the tensor-core tiles.
 * CE_KERNEL_AUTO (default): BF16X3 when the call is launchable (K <= 32, N even, every window start a_w even,
 * 16-byte aligned y/x), else TF32X3, else SIMT.  All meet the 1e-4 parity bar.
 * An explicit BF16X3 is also rejected by ce_estimate (CE_EINVAL) when the call itself is not launchable for it. */
int ce_set_kernel(ce_handle *h, int32_t kernel);

/* The kernel the most recent ce_estimate launched (CE_KERNEL_SIMT / _TF32X3 / _BF16X3); before
 * the first estimate, the kernel AUTO/the setting prefers for this geometry. */
int ce_selected_kernel(const ce_handle *h, int32_t *out);

/* Copy the built filters to host memory: complex64 [n_sets][b][b] row-major (W[i][j] multiplies
 * H_LS[a_w + j] for output a_w + i).  Synchronous.  CE_ESTATE if not built. */
int ce_get_filters(ce_handle *h, void *host_W);

/* Host-only (no CUDA): write the window table for (N, b, stride) as int32 triples
 * {a_w, o_w, o_{w+1}} into out[0 .. 3*n_windows).  Returns n_windows (>= 1), or CE_EINVAL for
 * invalid sizes or if capacity (in triples) < n_windows (out may be NULL to query the count
 * with capacity 0 -> returns n_windows). */
int ce_window_table(int32_t N, int32_t b, int32_t stride, int32_t *out, int32_t capacity);

/* Number of CUDA kernels this handle has launched (K1 + K2/K3), for launch accounting. */
int ce_launch_count(const ce_handle *h, int64_t *out);

/* ---------------------------------------------------------------------------------------------------
 * NEXT-1: the paper's own comb-pilot grouped estimators, 3W-LMMSE and 12W-LMMSE (PAPER.md:345-403,
 * Tables I-II; zero-order hold of PAPER.md:519).  UE s (0-based) owns pilot tones S*j + s, j < K = N/S
 * (Eq. 6).  Group g in [0, K) uses the pilot window [a_g, a_g + G),
 * a_g = clamp(g - (G-1)/2, 0, K - G), and weight type g - a_g; its weight is
 *   W = R[out, in] (R[in, in] + sigma^2 I)^-1     (Eq. 17, R[p, q] = r[p - q], r[-d] = conj(r[d]))
 * CE_COMB_FULL (12W): group g outputs the S tones S*g + q (every tone); one weight set per UE.
 * CE_COMB_SUB  (3W):  group g outputs the G tones S*g + s + (S/G) q; weights shared by all UEs; every
 *                     other tone holds the last estimate at or before it (the first estimate before it).
 * Readings C1-C6 in DESIGN.md (C6: under K10 a non-finite LS value -- a zero pilot symbol -- reaches every output of
 * the 16-pilot block windows that hold it, not only the groups whose G-pilot windows use it).
 * ------------------------------------------------------------------------------------------------- */
typedef enum { CE_COMB_FULL = 0, CE_COMB_SUB = 1 } ce_comb_mode;

typedef struct ce_comb_handle ce_comb_handle; /* opaque */

typedef struct {
  int32_t N;      /* used subcarriers, N % S == 0 */
  int32_t S;      /* comb spacing: pilot-interleaved UE slots (12 in PAPER.md Fig. fig1) */
  int32_t n_ue;   /* UEs estimated: comb offsets 0 .. n_ue-1, 1 <= n_ue <= S */
  int32_t G;      /* pilots per group window, 1 <= G <= min(N/S, 32); SUB needs S % G == 0 */
  int32_t mode;   /* ce_comb_mode; FULL needs S <= 64 */
  const double *r_hh; /* host [N][2] complex128 first column of R_hh (same statistics for all UEs); copied */
  double sigma2;      /* sigma^2 / sigma_s^2 > 0 */
} ce_comb_params;

/* Validate, copy the statistics to the current device, allocate the weights.  CE_EINVAL / CE_ENODEV /
 * CE_ENOMEM as ce_init. */
int ce_comb_init(const ce_comb_params *p, ce_comb_handle **out);
/* K6a: FP64 Cholesky build of every (UE, type) weight, rounded to complex64; synchronises the stream
 * once to read the positive-definite flag (CE_ENOTPD); for K10-capable shapes also builds K10's bf16 hi / lo weight
 * images from those weights (one more kernel and stream synchronisation). */
int ce_comb_build_filters(ce_comb_handle *h, void *stream);
/* Hot path on device pointers (K10, or K6b: ce_comb_set_kernel), asynchronous on `stream`:
 *   d_y : complex64 [T][M][N]     received pilot OFDM symbol of each antenna (all UEs on their combs)
 *   d_x : complex64 [T][N]        comb pilot symbol: tone k carries UE (k % S)'s pilot
 *   d_h : complex64 [T][M][n_ue][N] estimates (caller-owned, must not alias d_y / d_x)
 * CE_ESTATE before a successful build; CE_EINVAL for NULL / misaligned (8 B) pointers, T or M < 1,
 * aliasing. */
int ce_comb_estimate(ce_comb_handle *h, const void *d_y, const void *d_x, void *d_h, int32_t T, int32_t M,
                     void *stream);
/* Copy the weights to host: complex64 [n_w][G types][n_out][G], n_w = n_ue (FULL) or 1 (SUB),
 * n_out = S (FULL) or G (SUB).  Synchronous. */
int ce_comb_get_filters(ce_comb_handle *h, void *host_W);
/* Kernels launched by this handle (K6a + K6b / K10). */
int ce_comb_launch_count(const ce_comb_handle *h, int64_t *out);
/* Estimator kernel of ce_comb_estimate.  AUTO (default): K10 -- the 12W on tcgen05 (BF16x3 products, FP32
 * accumulation; LS de-interleaved per UE by k10_ls, then one GEMM per (UE, block of groups, 128 rows)) -- when
 * mode == CE_COMB_FULL, G <= 13, N even and the call has at least 4 units of work per SM
 * (ceil(T*M / 128) * n_ue * blocks; a block is up to floor(64/S) groups whose pilot windows fit one 16-pilot window:
 * ~N/(4S) blocks for the 12W), else K6b (FP32 SIMT; one launch, faster on small calls).  SIMT
 * forces K6b; TC forces K10 for every call (CE_EINVAL when the shape is not supported).  K10 keeps a per-handle
 * device workspace for the LS planes (2 * n_ue * T*M * ceil4(N/S) * 4 bytes), grown on the first call that needs
 * more (a cudaMalloc outside any stream order, so a handle's calls must not overlap on different streams). */
typedef enum { CE_COMB_KERNEL_AUTO = 0, CE_COMB_KERNEL_SIMT = 1, CE_COMB_KERNEL_TC = 2 } ce_comb_kernel;
int ce_comb_set_kernel(ce_comb_handle *h, int32_t kernel);
/* The kernel ce_comb_estimate will use for a call with T instances of M antennas (CE_COMB_KERNEL_SIMT or
 * CE_COMB_KERNEL_TC); CE_EINVAL for T or M < 1. */
int ce_comb_selected_kernel(const ce_comb_handle *h, int32_t T, int32_t M, int32_t *out);
/* Free; NULL allowed. */
int ce_comb_free(ce_comb_handle *h);

/* ---------------------------------------------------------------------------------------------------
 * NEXT-3: the statistics the filter build needs, estimated from the received pilots (the paper designs W
 * from an assumed L and SNR_fixed, and fixes sigma^2 "for the lack of SNR estimation module",
 * PAPER.md:519).  Per statistic set s, from the LS estimates H_LS = y / x (Eq. 9) of every column
 * c = (t, m, k) of the set's instances (readings D1-D3 in DESIGN.md):
 *   r_hat[d]   = sum_c sum_{n<N-d} H_LS[c,n+d] conj(H_LS[c,n]) / (C_s (N-d)) - sigma2_hat delta[d],  d < D
 *   sigma2_hat = mean over c and over the B delay bins centred on N/2 of |IDFT_N(H_LS[c])|^2 (unitary)
 * The results can be handed (via the host) to ce_init as r_hh (entries d >= D may be zero when D >= b:
 * the filters use d < b only) and sigma2.
 * ------------------------------------------------------------------------------------------------- */
/* Bytes of device workspace ce_stats_estimate needs for (N, n_sets, D, B): the per-set accumulators
 * (n_sets * (2 D + 2) doubles, rounded up to 256 bytes) plus, when L = the smallest power of two >= max(64, N + D - 1)
 * is at most 8192, the per-set power spectra (n_sets * L doubles).  CE_EINVAL for N < 2, n_sets, D or B < 1, NULL out. */
int ce_stats_workspace_bytes(int32_t N, int32_t n_sets, int32_t D, int32_t B, int64_t *out);
/* Device pointers, asynchronous on `stream`.  The lag sums: when L (above) is at most 8192 and n_sets <= 65535,
 * through the power spectrum of the zero-padded LS rows (K9: FP32 FFT of length L per row, |X|^2 summed per set in
 * FP64, then the FP64 inverse DFT at d < D -- the Wiener-Khinchin identity, no wrap for L >= N + D - 1); else from
 * 16384 columns T*M*K up, with K <= 24, D <= 512, N even and d_y 16-byte aligned, on the tensor cores as a banded
 * Gram matrix (K8, BF16x3); else as direct sums (K7a).  The noise floor: streamed by K7c (N even, d_y 16-byte
 * aligned) when the lags ran elsewhere, else inside K7a; K7b normalises.  Every path meets the same 1e-4 parity bar:
 *   d_y [T][M][K][N], d_x [T][K][N] complex64 (8-byte aligned); d_set_of_instance int32 [T] or NULL (all
 *   set 0; instances with an out-of-range set are skipped); d_r out: complex128 [n_sets][D] interleaved;
 *   d_sigma2 out: float64 [n_sets]; d_work: ce_stats_workspace_bytes(N, n_sets, D, B) bytes, 8-byte aligned.  A set with no instance gets
 *   NaN.  CE_EINVAL for NULL / misaligned pointers, sizes < 1, D or B > N, N > 12800. */
int ce_stats_estimate(const void *d_y, const void *d_x, int32_t T, int32_t M, int32_t K, int32_t N,
                      const int32_t *d_set_of_instance, int32_t n_sets, int32_t D, int32_t B, void *d_r,
                      void *d_sigma2, void *d_work, void *stream);

/* Static description of a status code; never NULL. */
const char *ce_status_string(int status);

/* Detail of the calling thread's last failed call ("" if none); never NULL. */
const char *ce_last_error(void);

/* Library version string, e.g. "libce 0.1 sm_100a". */
const char *ce_version(void);

#ifdef __cplusplus
}
#endif

#endif /* CE_H */
