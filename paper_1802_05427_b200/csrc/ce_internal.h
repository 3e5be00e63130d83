// Internal declarations shared by the libce translation units (host API, K1, K2, K3).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/ce.h"

namespace ce {

// One window of the geometry table (reading A7).
struct Window {
  int32_t a;       // first LS tone read
  int32_t o;       // first output tone kept
  int32_t o_next;  // one past the last output tone kept
};

// Host-side window table; returns false for invalid sizes.
bool window_table(int32_t N, int32_t b, int32_t s, std::vector<Window> *out);
// The same windows with every window too wide for one 256-column MMA tile split into output sub-windows.
std::vector<Window> split_for_tensor_tiles(const std::vector<Window> &geo);

// Arguments of one contraction launch (K2 / K3).
struct ContractArgs {
  const float2 *y;         // [T][M][K][N]
  const float2 *x;         // [T][K][N]
  float2 *h;               // [T][M][K][N]
  const float2 *Wt;        // [n_sets][b][b] transposed filters: Wt[s][j][i] = W[s][i][j]
  const Window *geo;       // [n_win] (device)
  const Window *geo_host;  // [n_win] (host copy; K4 passes small tables in its kernel parameters)
  const int32_t *soi;      // [T] device or nullptr
  int32_t T, M, K, N, b, n_win, n_sets, max_kept;
  bool even_starts;        // every window start a_w is even (16-byte aligned TMA boxes, K4)
  // K4 power mode (the statistics estimator's noise window, k7_stats.cu): no h stores; each tile adds the sum of
  // |output|^2 over its rows to pow_acc[set * pow_stride] and, for window 0, its row count to
  // pow_acc[set * pow_stride + 1].  bank_rows (> 0) overrides the bank's rows per K chunk; bank_shared: one bank for
  // every set.
  double *pow_acc = nullptr;
  int32_t pow_stride = 0;
  int32_t bank_rows = 0;
  bool bank_shared = false;
};

// K1: filter build.  Returns cudaError_t of the launches.
cudaError_t launch_filter_build(const double2 *d_r, const double *d_sigma2, int32_t N, int32_t b,
                                int32_t n_sets, double2 *d_ws, float2 *d_W, float2 *d_Wt,
                                int32_t *d_flag, cudaStream_t stream,
                                int64_t *launches);

// K2: FP32 SIMT contraction.
cudaError_t launch_contract_simt(const ContractArgs &a, cudaStream_t stream, int64_t *launches);

// K3: tcgen05 3xTF32 contraction over the pre-split, pre-swizzled filter bank.
bool tf32x3_supported(int32_t b, const std::vector<Window> &geo);
void tf32x3_bank_shape(int32_t b, int32_t *nkc, int32_t *NR);
cudaError_t launch_build_bank(const float2 *d_W, int32_t b, int32_t n_sets, float *bank_hi, float *bank_lo,
                              cudaStream_t stream, int64_t *launches);
cudaError_t launch_contract_tf32x3(const ContractArgs &a, const float *bank_hi, const float *bank_lo,
                                   cudaStream_t stream, int64_t *launches);

// K4: tcgen05 BF16x3 contraction with TMA-fed raw ring (same bank geometry as K3, bf16 planes).
void bf16x3_bank_shape(int32_t b, int32_t *nkc, int32_t *NR);
bool bf16x3_launchable(const ContractArgs &a);
cudaError_t launch_build_bank_bf16(const float2 *d_W, int32_t b, int32_t n_sets, uint16_t *bank_hi,
                                   uint16_t *bank_lo, cudaStream_t stream, int64_t *launches);
cudaError_t launch_contract_bf16x3(const ContractArgs &a, const uint16_t *bank_hi, const uint16_t *bank_lo,
                                   cudaStream_t stream, int64_t *launches);
// K4 on CTA pairs (k4p_block_lmmse_pair.cu: tcgen05 cta_group::2, each CTA of a cluster holds half of the filter
// chunk); bf16x3_pair_wanted is the policy launch_contract_bf16x3 consults (CE_K4_PAIR = 0 / 1 overrides it).
bool bf16x3_pair_wanted(const ContractArgs &a);
cudaError_t launch_contract_bf16x3_pair(const ContractArgs &a, const uint16_t *bank_hi, const uint16_t *bank_lo,
                                        cudaStream_t stream, int64_t *launches);
// K4's bank for the unitary N-point inverse DFT at the B delay bins lo .. lo + B - 1 (rows = bins, K = tones): one
// set, nkc = ceil(2N / 32) chunks of NR = ceil(2B / 16) * 16 rows, bf16 hi / lo planes.
void dft_bank_shape(int32_t N, int32_t B, int32_t *nkc, int32_t *NR);
cudaError_t launch_build_dft_bank(int32_t N, int32_t B, int32_t lo, uint16_t *bank_hi, uint16_t *bank_lo,
                                  cudaStream_t stream);


// K8: the statistics estimator's lag correlation (banded Gram matrix) on tcgen05; adds into K7's accumulator.
bool gram_launchable(const float2 *y, int32_t K, int32_t N, int32_t D);
cudaError_t launch_gram(const float2 *y, const float2 *x, int32_t T, int32_t M, int32_t K, int32_t N,
                        const int32_t *soi, int32_t n_sets, int32_t D, double *acc, cudaStream_t stream);

// K9: the lag correlation through the power spectrum of the zero-padded LS rows (FFT of length L = 2^l >= N + D - 1);
// spectrum_log2 returns l, or -1 when L would exceed 8192.  P: [n_sets][L] FP64 workspace; writes acc[s][0 .. 2D).
int spectrum_log2(int32_t N, int32_t D);
cudaError_t launch_spectrum_lags(const float2 *y, const float2 *x, int32_t T, int32_t M, int32_t K, int32_t N,
                                 const int32_t *soi, int32_t n_sets, int32_t D, double *P, double *acc,
                                 cudaStream_t stream);

// K10: the comb-pilot 12W (CE_COMB_FULL) on tcgen05 (k10_comb_tc.cu).  Blocks {g0, ng, sw, 0}: ng consecutive
// groups from g0 whose pilot windows lie in [sw, sw + 16), sw % 4 == 0, ng * S <= 64; cls = the block's weight-image
// class (blocks with the same groups-per-block, types and tap offsets share one image); rep[cls] = a block of it.
bool comb_tc_supported(int32_t N, int32_t S, int32_t G, int32_t mode);
std::vector<int4> comb_tc_blocks(int32_t K, int32_t G, int32_t S, std::vector<int4> *rep);
size_t comb_tc_image_elems(int32_t n_ue, int32_t n_cls);
size_t comb_tc_ls_bytes(int32_t N, int32_t S, int32_t n_ue, long long rows);
cudaError_t launch_comb_tc_images(const float2 *W, const int4 *d_rep, int32_t n_cls, int32_t n_ue, int32_t N,
                                  int32_t S, int32_t G, uint16_t *img_hi, uint16_t *img_lo, cudaStream_t stream);
cudaError_t launch_comb_tc(const float2 *y, const float2 *x, float2 *h, int32_t T, int32_t M, int32_t N, int32_t S,
                           int32_t n_ue, const int4 *d_blk, int32_t n_blk, int32_t n_cls, const uint16_t *img_hi,
                           const uint16_t *img_lo, void *ls, cudaStream_t stream, int64_t *launches);

void set_last_error(const std::string &msg);

// Selects a handle's device for the duration of an entry point and restores the caller's current device on exit.
struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) { ok = false; return; }
    if (prev != dev && cudaSetDevice(dev) != cudaSuccess) ok = false;
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard &) = delete;
  DeviceGuard &operator=(const DeviceGuard &) = delete;
};

// Dynamic shared-memory opt-in: a launch needs cudaFuncAttributeMaxDynamicSharedMemorySize >= dyn whenever dyn plus
// the kernel's own static __shared__ storage exceeds the 48 KB default.  The static size is read from the compiled
// kernel (cudaFuncGetAttributes), so a later change to a kernel's __shared__ arrays cannot silently break the launch.
inline cudaError_t smem_opt_in(const void *fn, size_t dyn) {
  if (dyn == 0) return cudaSuccess;
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return e;
  if (dyn + fa.sharedSizeBytes <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn));
}

}  // namespace ce
