// libce host side: parameter validation, window geometry, handle/memory management,
// launch selection and the host-buffer (end-to-end) pipeline.  See include/ce.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "ce_internal.h"

namespace ce {

static thread_local std::string g_last_error;

void set_last_error(const std::string &msg) { g_last_error = msg; }

// Reading A7; generalises PAPER.md:242-257 (Table II edge clamping).
bool window_table(int32_t N, int32_t b, int32_t s, std::vector<Window> *out) {
  if (N < 1 || b < 1 || b > N || s < 1 || s > b) return false;
  const int64_t n_win = (int64_t(N - b) + s - 1) / s + 1;
  const int32_t m_l = (b - s) / 2;
  out->clear();
  out->reserve(size_t(n_win));
  for (int64_t w = 0; w < n_win; ++w) {
    Window g;
    g.a = int32_t(std::min<int64_t>(w * s, N - b));
    g.o = (w == 0) ? 0 : int32_t(w * s + m_l);
    g.o_next = (w == n_win - 1) ? N : int32_t((w + 1) * s + m_l);
    out->push_back(g);
  }
  return true;
}

// Tensor-core tiles hold at most 256 accumulator columns: a piece [o, o + len) of a window starting at a
// occupies MMA N = off + 2 len (rounded up to 16), off = 2 (o - a) mod 8 being the 8-row alignment of the
// filter-bank rows, so it fits iff off + 2 len <= 256.  Windows that fit stay whole (config 5: 126 outputs,
// off = 0); wider ones are split into the fewest output sub-windows over the same LS input range (same a_w,
// b), each as long as its alignment allows (125-128 outputs).  Reading the full b-wide input per
// sub-window re-reads y from L2; that is what makes b = N (the full LMMSE, NEXT-2) run on the tensor cores.
std::vector<Window> split_for_tensor_tiles(const std::vector<Window> &geo) {
  constexpr int32_t NMAX = 256;
  std::vector<Window> out;
  for (const Window &g : geo)
    for (int32_t o = g.o; o < g.o_next;) {
      const int32_t off = (2 * (o - g.a)) & 7;
      const int32_t len = std::min(g.o_next - o, (NMAX - off) / 2);
      out.push_back(Window{g.a, o, o + len});
      o += len;
    }
  return out;
}

}  // namespace ce

using ce::set_last_error;

struct ce_handle {
  int device = -1;
  int32_t N = 0, b = 0, stride = 0, n_sets = 0, n_win = 0, max_kept = 0;
  int32_t kernel = CE_KERNEL_AUTO;
  bool built = false;
  std::vector<ce::Window> geo;
  // device
  double2 *d_r = nullptr;       // [n_sets][b] first column of R_hh (only d < b is needed)
  double *d_sigma2 = nullptr;   // [n_sets]
  ce::Window *d_geo = nullptr;  // [n_win]
  std::vector<ce::Window> geo_tc;   // tensor-core window table (wide windows split into sub-windows)
  ce::Window *d_geo_tc = nullptr;   // [geo_tc.size()]
  double2 *d_ws = nullptr;      // [n_sets][4b + 1] K1 workspace: x = A^-1 e_0, recursion / refinement vectors (FP64)
  float2 *d_W = nullptr;        // [n_sets][b][b]
  float2 *d_Wt = nullptr;       // [n_sets][b][b] transposed
  float *d_bank = nullptr;      // K3 filter bank: hi plane then lo plane, [n_sets][nkc][NR][32] each
  size_t bank_plane = 0;        // floats per plane
  bool tf32_ok = false;         // the tensor-core filter banks fit (any b; wide windows are split)
  uint16_t *d_bank16 = nullptr; // K4 filter bank: bf16 hi plane then lo plane
  size_t bank16_plane = 0;      // elements per plane
  int32_t last_kernel = -1;     // kernel launched by the most recent ce_estimate
  bool even_starts = true;      // all window starts even (K4 TMA alignment)
  int32_t *d_flag = nullptr;    // [1] build error flag
  int32_t *h_flag = nullptr;    // pinned mirror
  // host-buffer path: two staging slots (grown on demand) so that two calls can be in flight; a call on slot s
  // waits for ev_slot_free[s], recorded after the last D2H copy of the previous call that used the slot
  void *d_stage[2] = {nullptr, nullptr};
  size_t stage_bytes[2] = {0, 0};
  int next_slot = 0;
  cudaEvent_t ev_slot_free[2] = {nullptr, nullptr};
  // host-buffer pipeline: streams[0] H2D copies, [1] kernels, [2] D2H copies; per-chunk events
  static constexpr int MAX_CHUNKS = 64;
  cudaStream_t streams[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev_start = nullptr, ev_done[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev_in[MAX_CHUNKS] = {}, ev_out[MAX_CHUNKS] = {};
  int64_t launches = 0;
};

namespace {

using ce::DeviceGuard;

int fail(int status, const std::string &msg) {
  set_last_error(msg);
  return status;
}

int cuda_fail(cudaError_t e, const char *what) {
  std::string m = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  set_last_error(m);
  return e == cudaErrorMemoryAllocation ? CE_ENOMEM : CE_ECUDA;
}

#define CE_CUDA(call, what)                    \
  do {                                         \
    cudaError_t _e = (call);                   \
    if (_e != cudaSuccess) return cuda_fail(_e, what); \
  } while (0)

void release(ce_handle *h) {
  cudaFree(h->d_r);
  cudaFree(h->d_sigma2);
  cudaFree(h->d_geo);
  cudaFree(h->d_geo_tc);
  cudaFree(h->d_ws);
  cudaFree(h->d_W);
  cudaFree(h->d_Wt);
  cudaFree(h->d_bank);
  cudaFree(h->d_bank16);
  cudaFree(h->d_flag);
  cudaFreeHost(h->h_flag);
  for (int i = 0; i < 2; ++i) {
    cudaFree(h->d_stage[i]);
    if (h->ev_slot_free[i]) cudaEventDestroy(h->ev_slot_free[i]);
  }
  for (auto &s : h->streams)
    if (s) cudaStreamDestroy(s);
  if (h->ev_start) cudaEventDestroy(h->ev_start);
  for (auto &e : h->ev_in)
    if (e) cudaEventDestroy(e);
  for (auto &e : h->ev_out)
    if (e) cudaEventDestroy(e);
  for (auto &e : h->ev_done)
    if (e) cudaEventDestroy(e);
}

bool overlaps(const void *a, size_t na, const void *b, size_t nb) {
  auto pa = reinterpret_cast<uintptr_t>(a), pb = reinterpret_cast<uintptr_t>(b);
  return pa < pb + nb && pb < pa + na;
}

int check_sizes(const ce_handle *h, int32_t T, int32_t M, int32_t K) {
  if (T < 1 || M < 1 || K < 1)
    return fail(CE_EINVAL, "T, M and K must be >= 1");
  // 64-bit element count; the kernels index elements with 64-bit offsets, but columns (T*M*K rows of N tones)
  // with 32-bit integers
  const long double elems = (long double)T * M * K * h->N;
  if (elems > 4.0e12L) return fail(CE_EINVAL, "problem too large");
  if ((long long)T * M * K >= (1LL << 31)) return fail(CE_EINVAL, "T*M*K must be < 2^31 (column index range)");
  return CE_OK;
}

}  // namespace

extern "C" {

const char *ce_version(void) {
  return "libce 0.4 sm_100a (K1 fp64 Levinson/Schur + refinement + Gohberg-Semencul/Trench, K2 fp32 simt, K3 tcgen05 "
         "tf32x3, K4 tcgen05 bf16x3 + TMA)";
}

const char *ce_status_string(int status) {
  switch (status) {
    case CE_OK: return "CE_OK: success";
    case CE_EINVAL: return "CE_EINVAL: invalid argument";
    case CE_ENOMEM: return "CE_ENOMEM: out of memory";
    case CE_ECUDA: return "CE_ECUDA: CUDA runtime error";
    case CE_ENOTPD: return "CE_ENOTPD: R_b + sigma^2 I is not positive definite";
    case CE_ESTATE: return "CE_ESTATE: filters not built";
    case CE_ENODEV: return "CE_ENODEV: no compute capability 10.x CUDA device";
    default: return "unknown ce_status";
  }
}

const char *ce_last_error(void) { return ce::g_last_error.c_str(); }

int ce_window_table(int32_t N, int32_t b, int32_t stride, int32_t *out, int32_t capacity) {
  std::vector<ce::Window> g;
  if (!ce::window_table(N, b, stride, &g))
    return fail(CE_EINVAL, "window table: need N >= 1, 1 <= b <= N, 1 <= stride <= b");
  const int32_t n = int32_t(g.size());
  if (out == nullptr && capacity == 0) return n;
  if (out == nullptr || capacity < n) return fail(CE_EINVAL, "window table: capacity too small");
  for (int32_t w = 0; w < n; ++w) {
    out[3 * w + 0] = g[w].a;
    out[3 * w + 1] = g[w].o;
    out[3 * w + 2] = g[w].o_next;
  }
  return n;
}

int ce_init(const ce_params *p, ce_handle **out) {
  if (p == nullptr || out == nullptr) return fail(CE_EINVAL, "ce_init: NULL params or out");
  if (p->N < 1) return fail(CE_EINVAL, "ce_init: N must be >= 1");
  if (p->b < 1 || p->b > p->N) return fail(CE_EINVAL, "ce_init: need 1 <= b <= N");
  if (p->stride < 1 || p->stride > p->b) return fail(CE_EINVAL, "ce_init: need 1 <= stride <= b");
  if (p->n_sets < 1) return fail(CE_EINVAL, "ce_init: n_sets must be >= 1");
  if (p->r_hh == nullptr || p->sigma2 == nullptr) return fail(CE_EINVAL, "ce_init: NULL r_hh or sigma2");
  const int32_t N = p->N, b = p->b, S = p->n_sets;
  for (int32_t s = 0; s < S; ++s) {
    const double s2 = p->sigma2[s];
    if (!std::isfinite(s2) || !(s2 > 0.0)) return fail(CE_EINVAL, "ce_init: sigma2 must be finite and > 0");
    const double *r = p->r_hh + size_t(s) * N * 2;
    for (int32_t d = 0; d < N; ++d)
      if (!std::isfinite(r[2 * d]) || !std::isfinite(r[2 * d + 1]))
        return fail(CE_EINVAL, "ce_init: r_hh must be finite");
    if (!(r[0] > 0.0) || std::fabs(r[1]) > 1e-9 * r[0])
      return fail(CE_EINVAL, "ce_init: r[0] must be real and > 0");
  }
  std::vector<ce::Window> geo;
  if (!ce::window_table(N, b, p->stride, &geo)) return fail(CE_EINVAL, "ce_init: bad geometry");

  int dev = -1, ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1 || cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return fail(CE_ENODEV, "ce_init: no CUDA device");
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess || prop.major != 10)
    return fail(CE_ENODEV, "ce_init: libce is built for sm_100a (compute capability 10.x)");

  ce_handle *h = new (std::nothrow) ce_handle();
  if (h == nullptr) return fail(CE_ENOMEM, "ce_init: host allocation");
  h->device = dev;
  h->N = N;
  h->b = b;
  h->stride = p->stride;
  h->n_sets = S;
  h->geo = geo;
  h->n_win = int32_t(geo.size());
  for (auto &g : geo) {
    h->max_kept = std::max(h->max_kept, g.o_next - g.o);
    if ((g.a & 1) || (N & 1)) h->even_starts = false;   // 16-byte TMA box starts and row pitch
  }

  std::vector<double2> r_b(size_t(S) * b);
  for (int32_t s = 0; s < S; ++s)
    for (int32_t d = 0; d < b; ++d)
      r_b[size_t(s) * b + d] = make_double2(p->r_hh[(size_t(s) * N + d) * 2], p->r_hh[(size_t(s) * N + d) * 2 + 1]);
  h->geo_tc = ce::split_for_tensor_tiles(geo);
  {
    int32_t nkc, NR;
    ce::tf32x3_bank_shape(b, &nkc, &NR);
    h->bank_plane = size_t(S) * nkc * NR * 32;
    ce::bf16x3_bank_shape(b, &nkc, &NR);
    h->bank16_plane = size_t(S) * nkc * NR * 32;
    // banks: 2 fp32 planes + 2 bf16 planes; keep them well inside HBM (b = 1200: 70 MB per set)
    const double bank_bytes = 2.0 * h->bank_plane * 4 + 2.0 * h->bank16_plane * 2;
    h->tf32_ok = ce::tf32x3_supported(b, h->geo_tc) && bank_bytes <= 8.0e9;
  }
  cudaError_t e = cudaSuccess;
  auto chk = [&](cudaError_t x) { if (e == cudaSuccess) e = x; };
  chk(cudaMalloc(&h->d_r, r_b.size() * sizeof(double2)));
  chk(cudaMalloc(&h->d_sigma2, size_t(S) * sizeof(double)));
  chk(cudaMalloc(&h->d_geo, geo.size() * sizeof(ce::Window)));
  chk(cudaMalloc(&h->d_geo_tc, h->geo_tc.size() * sizeof(ce::Window)));
  chk(cudaMalloc(&h->d_ws, size_t(S) * (4 * size_t(b) + 1) * sizeof(double2)));   // K1 Levinson workspace
  chk(cudaMalloc(&h->d_W, size_t(S) * b * b * sizeof(float2)));
  chk(cudaMalloc(&h->d_Wt, size_t(S) * b * b * sizeof(float2)));
  if (h->tf32_ok) chk(cudaMalloc(&h->d_bank, 2 * h->bank_plane * sizeof(float)));
  if (h->tf32_ok) chk(cudaMalloc(&h->d_bank16, 2 * h->bank16_plane * sizeof(uint16_t)));

  chk(cudaMalloc(&h->d_flag, sizeof(int32_t)));
  chk(cudaMallocHost(&h->h_flag, sizeof(int32_t)));
  if (e == cudaSuccess) {
    chk(cudaMemcpy(h->d_r, r_b.data(), r_b.size() * sizeof(double2), cudaMemcpyHostToDevice));
    chk(cudaMemcpy(h->d_sigma2, p->sigma2, size_t(S) * sizeof(double), cudaMemcpyHostToDevice));
    chk(cudaMemcpy(h->d_geo, geo.data(), geo.size() * sizeof(ce::Window), cudaMemcpyHostToDevice));
    chk(cudaMemcpy(h->d_geo_tc, h->geo_tc.data(), h->geo_tc.size() * sizeof(ce::Window), cudaMemcpyHostToDevice));
  }
  if (e != cudaSuccess) {
    int st = cuda_fail(e, "ce_init: device allocation/copy");
    release(h);
    delete h;
    return st;
  }
  *out = h;
  return CE_OK;
}

int ce_free(ce_handle *h) {
  if (h == nullptr) return CE_OK;
  {
    DeviceGuard g(h->device);
    release(h);
  }
  delete h;
  return CE_OK;
}

int ce_set_kernel(ce_handle *h, int32_t kernel) {
  if (h == nullptr) return fail(CE_EINVAL, "ce_set_kernel: NULL handle");
  if (kernel != CE_KERNEL_AUTO && kernel != CE_KERNEL_SIMT && kernel != CE_KERNEL_TF32X3 &&
      kernel != CE_KERNEL_BF16X3)
    return fail(CE_EINVAL, "ce_set_kernel: unknown kernel");
  if ((kernel == CE_KERNEL_TF32X3 || kernel == CE_KERNEL_BF16X3) && !h->tf32_ok)
    return fail(CE_EINVAL, "ce_set_kernel: tensor-core filter banks do not fit for this b");
  if (kernel == CE_KERNEL_BF16X3 && !h->even_starts)
    return fail(CE_EINVAL, "ce_set_kernel: BF16X3 needs every window start a_w even (16-byte TMA boxes)");
  h->kernel = kernel;
  return CE_OK;
}

int ce_selected_kernel(const ce_handle *h, int32_t *out) {
  if (h == nullptr || out == nullptr) return fail(CE_EINVAL, "ce_selected_kernel: NULL argument");
  if (h->last_kernel >= 0)
    *out = h->last_kernel;
  else if (h->kernel == CE_KERNEL_AUTO)
    *out = !h->tf32_ok ? CE_KERNEL_SIMT : (h->even_starts ? CE_KERNEL_BF16X3 : CE_KERNEL_TF32X3);
  else
    *out = h->kernel;
  return CE_OK;
}

int ce_launch_count(const ce_handle *h, int64_t *out) {
  if (h == nullptr || out == nullptr) return fail(CE_EINVAL, "ce_launch_count: NULL argument");
  *out = h->launches;
  return CE_OK;
}

int ce_build_filters(ce_handle *h, void *stream) {
  if (h == nullptr) return fail(CE_EINVAL, "ce_build_filters: NULL handle");
  DeviceGuard g(h->device);
  if (!g.ok) return fail(CE_ECUDA, "ce_build_filters: cannot select the handle's device");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  h->built = false;
  CE_CUDA(cudaMemsetAsync(h->d_flag, 0, sizeof(int32_t), st), "ce_build_filters: memset flag");
  CE_CUDA(ce::launch_filter_build(h->d_r, h->d_sigma2, h->N, h->b, h->n_sets, h->d_ws, h->d_W, h->d_Wt,
                                  h->d_flag, st, &h->launches),
          "ce_build_filters: launch");
  if (h->tf32_ok) {
    CE_CUDA(ce::launch_build_bank(h->d_W, h->b, h->n_sets, h->d_bank, h->d_bank + h->bank_plane, st, &h->launches),
            "ce_build_filters: bank launch");
    CE_CUDA(ce::launch_build_bank_bf16(h->d_W, h->b, h->n_sets, h->d_bank16, h->d_bank16 + h->bank16_plane, st,
                                       &h->launches),
            "ce_build_filters: bf16 bank launch");
  }
  CE_CUDA(cudaMemcpyAsync(h->h_flag, h->d_flag, sizeof(int32_t), cudaMemcpyDeviceToHost, st),
          "ce_build_filters: flag copy");
  CE_CUDA(cudaStreamSynchronize(st), "ce_build_filters: synchronize");
  if (*h->h_flag != 0)
    return fail(CE_ENOTPD, "ce_build_filters: a Levinson prediction-error power <= 0 or not finite (R_b + sigma^2 I not PD)");
  h->built = true;
  return CE_OK;
}

int ce_get_filters(ce_handle *h, void *host_W) {
  if (h == nullptr || host_W == nullptr) return fail(CE_EINVAL, "ce_get_filters: NULL argument");
  if (!h->built) return fail(CE_ESTATE, "ce_get_filters: filters not built");
  DeviceGuard g(h->device);
  CE_CUDA(cudaMemcpy(host_W, h->d_W, size_t(h->n_sets) * h->b * h->b * sizeof(float2), cudaMemcpyDeviceToHost),
          "ce_get_filters: copy");
  return CE_OK;
}

static int launch_contract(ce_handle *h, const float2 *y, const float2 *x, float2 *out, int32_t T, int32_t M,
                           int32_t K, const int32_t *soi, cudaStream_t st) {
  ce::ContractArgs a;
  a.y = y;
  a.x = x;
  a.h = out;
  a.Wt = h->d_Wt;
  a.geo = h->d_geo;
  a.geo_host = h->geo.data();
  a.soi = soi;
  a.T = T;
  a.M = M;
  a.K = K;
  a.N = h->N;
  a.b = h->b;
  a.n_win = h->n_win;
  a.n_sets = h->n_sets;
  a.max_kept = h->max_kept;
  a.even_starts = h->even_starts;
  int32_t k = h->kernel;
  if (k != CE_KERNEL_SIMT && h->tf32_ok) {   // tensor-core kernels run on the split window table
    a.geo = h->d_geo_tc;
    a.geo_host = h->geo_tc.data();
    a.n_win = int32_t(h->geo_tc.size());
  }
  if (k == CE_KERNEL_AUTO)
    k = !h->tf32_ok ? CE_KERNEL_SIMT : (ce::bf16x3_launchable(a) ? CE_KERNEL_BF16X3 : CE_KERNEL_TF32X3);
  if (k == CE_KERNEL_BF16X3 && !ce::bf16x3_launchable(a))
    return fail(CE_EINVAL, "ce_estimate: BF16X3 needs K <= 32, even N, even window starts, 16-byte aligned y/x");
  cudaError_t e;
  if (k == CE_KERNEL_BF16X3)
    e = ce::launch_contract_bf16x3(a, h->d_bank16, h->d_bank16 + h->bank16_plane, st, &h->launches);
  else if (k == CE_KERNEL_TF32X3)
    e = ce::launch_contract_tf32x3(a, h->d_bank, h->d_bank + h->bank_plane, st, &h->launches);
  else
    e = ce::launch_contract_simt(a, st, &h->launches);
  if (e != cudaSuccess) return cuda_fail(e, "ce_estimate: kernel launch");
  h->last_kernel = k;
  return CE_OK;
}

int ce_estimate(ce_handle *h, const void *d_y, const void *d_x, void *d_h, int32_t T, int32_t M, int32_t K,
                const int32_t *d_set_of_instance, void *stream) {
  if (h == nullptr) return fail(CE_EINVAL, "ce_estimate: NULL handle");
  if (!h->built) return fail(CE_ESTATE, "ce_estimate: call ce_build_filters first");
  if (d_y == nullptr || d_x == nullptr || d_h == nullptr) return fail(CE_EINVAL, "ce_estimate: NULL pointer");
  int st = check_sizes(h, T, M, K);
  if (st != CE_OK) return st;
  if ((reinterpret_cast<uintptr_t>(d_y) | reinterpret_cast<uintptr_t>(d_x) | reinterpret_cast<uintptr_t>(d_h)) & 7u)
    return fail(CE_EINVAL, "ce_estimate: pointers must be 8-byte aligned (complex64)");
  const size_t ny = size_t(T) * M * K * h->N * sizeof(float2);
  const size_t nx = size_t(T) * K * h->N * sizeof(float2);
  if (overlaps(d_h, ny, d_y, ny) || overlaps(d_h, ny, d_x, nx))
    return fail(CE_EINVAL, "ce_estimate: output aliases an input");
  DeviceGuard g(h->device);
  if (!g.ok) return fail(CE_ECUDA, "ce_estimate: cannot select the handle's device");
  return launch_contract(h, static_cast<const float2 *>(d_y), static_cast<const float2 *>(d_x),
                         static_cast<float2 *>(d_h), T, M, K, d_set_of_instance, static_cast<cudaStream_t>(stream));
}

static int estimate_host_impl(ce_handle *h, const void *y_host, const void *x_host, void *h_host, int32_t T,
                              int32_t M, int32_t K, const int32_t *set_of_instance, void *stream, bool sync) {
  const char *who = sync ? "ce_estimate_host" : "ce_estimate_host_async";
  if (h == nullptr) return fail(CE_EINVAL, std::string(who) + ": NULL handle");
  if (!h->built) return fail(CE_ESTATE, std::string(who) + ": call ce_build_filters first");
  if (y_host == nullptr || x_host == nullptr || h_host == nullptr)
    return fail(CE_EINVAL, std::string(who) + ": NULL pointer");
  int st = check_sizes(h, T, M, K);
  if (st != CE_OK) return st;
  const size_t N = size_t(h->N);
  const size_t ny = size_t(T) * M * K * N * sizeof(float2);
  const size_t nx = size_t(T) * K * N * sizeof(float2);
  if (overlaps(h_host, ny, y_host, ny) || overlaps(h_host, ny, x_host, nx))
    return fail(CE_EINVAL, std::string(who) + ": output aliases an input");
  if (set_of_instance)
    for (int32_t t = 0; t < T; ++t)
      if (set_of_instance[t] < 0 || set_of_instance[t] >= h->n_sets)
        return fail(CE_EINVAL, std::string(who) + ": set_of_instance out of range");
  DeviceGuard g(h->device);
  if (!g.ok) return fail(CE_ECUDA, std::string(who) + ": cannot select the handle's device");

  if (h->streams[0] == nullptr) {
    for (auto &s : h->streams) CE_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream create");
    CE_CUDA(cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming), "event create");
    for (auto &e : h->ev_done) CE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event create");
    for (auto &e : h->ev_in) CE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event create");
    for (auto &e : h->ev_out) CE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event create");
    for (auto &e : h->ev_slot_free) CE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event create");
  }
  // Device staging slot: [y | h | x | soi], each 256-byte aligned, grown on demand (after every call in flight on
  // the handle's streams has completed: the old buffer may still be read)
  const int slot = h->next_slot;
  h->next_slot ^= 1;
  auto al = [](size_t n) { return (n + 255) & ~size_t(255); };
  const size_t need = al(ny) * 2 + al(nx) + al(size_t(T) * sizeof(int32_t));
  if (need > h->stage_bytes[slot]) {
    for (auto s : h->streams) CE_CUDA(cudaStreamSynchronize(s), "ce_estimate_host: drain before staging growth");
    cudaFree(h->d_stage[slot]);
    h->d_stage[slot] = nullptr;
    h->stage_bytes[slot] = 0;
    CE_CUDA(cudaMalloc(&h->d_stage[slot], need), "ce_estimate_host: staging allocation");
    h->stage_bytes[slot] = need;
  }
  char *base = static_cast<char *>(h->d_stage[slot]);
  float2 *dy = reinterpret_cast<float2 *>(base);
  float2 *dh = reinterpret_cast<float2 *>(base + al(ny));
  float2 *dx = reinterpret_cast<float2 *>(base + 2 * al(ny));
  int32_t *dsoi = reinterpret_cast<int32_t *>(base + 2 * al(ny) + al(nx));
  cudaStream_t user = static_cast<cudaStream_t>(stream);
  cudaStream_t s_in = h->streams[0], s_k = h->streams[1], s_out = h->streams[2];
  // order after prior work on the user's stream, and after the previous call on this staging slot
  CE_CUDA(cudaEventRecord(h->ev_start, user), "event record");
  for (auto s : h->streams) CE_CUDA(cudaStreamWaitEvent(s, h->ev_start, 0), "stream wait");
  CE_CUDA(cudaStreamWaitEvent(s_in, h->ev_slot_free[slot], 0), "stream wait");
  CE_CUDA(cudaMemcpyAsync(dx, x_host, nx, cudaMemcpyHostToDevice, s_in), "x copy");
  if (set_of_instance)
    CE_CUDA(cudaMemcpyAsync(dsoi, set_of_instance, size_t(T) * sizeof(int32_t), cudaMemcpyHostToDevice, s_in),
            "soi copy");

  // Three-stage pipeline over chunks of (instances, antenna range): every H2D copy on one stream, every
  // kernel on a second, every D2H copy on a third, chained per chunk by events -- the host->device and
  // device->host DMA engines each stream back to back and run concurrently (measured 86 GB/s together,
  // 52 GB/s each alone); 4 MB chunks measured best for config 3 (2 MB: -10%,
  // 1 MB: -20%: per-copy overhead); large batches run at the PCIe duplex ceiling (config 4: 90 GB/s).  The
  // asynchronous call overlaps whole calls instead (call n's device->host copies with call n+1's host->device copies,
  // two staging slots), where fewer, larger copies win: config 3 with 32 MB chunks (one per call) 5.4-5.6e9
  // estimates/s against 4.1e9 with 4 MB chunks (same box; the synchronous call: 4 MB 3.8e9, 8 MB 3.6e9).
  const size_t ant_bytes = size_t(K) * N * sizeof(float2);
  static const long env_chunk_kb = getenv("CE_HOST_CHUNK_KB") ? atol(getenv("CE_HOST_CHUNK_KB")) : 0;   // experiments
  const long chunk_kb = env_chunk_kb > 0 ? env_chunk_kb : sync ? 4096 : 32768;
  int32_t m_chunk = int32_t(std::max<size_t>(1, size_t(chunk_kb) * 1024 / ant_bytes));
  m_chunk = std::min(m_chunk, M);
  // at most MAX_CHUNKS chunks: fall back to whole instances per chunk, several instances per chunk if needed
  int32_t t_chunk = 1;
  if (int64_t(T) * ((M + m_chunk - 1) / m_chunk) > ce_handle::MAX_CHUNKS) {
    m_chunk = M;
    t_chunk = int32_t((int64_t(T) + ce_handle::MAX_CHUNKS - 1) / ce_handle::MAX_CHUNKS);
  }
  int c = 0;
  for (int32_t t = 0; t < T; t += t_chunk) {
    const int32_t tc = std::min(t_chunk, T - t);
    for (int32_t m0 = 0; m0 < M; m0 += m_chunk, ++c) {
      const int32_t mc = std::min(m_chunk, M - m0);     // t_chunk > 1 only with m_chunk == M
      const size_t off = (size_t(t) * M + m0) * K * N;
      const size_t bytes = size_t(tc) * mc * ant_bytes;
      CE_CUDA(cudaMemcpyAsync(dy + off, static_cast<const float2 *>(y_host) + off, bytes, cudaMemcpyHostToDevice, s_in),
              "y copy");
      CE_CUDA(cudaEventRecord(h->ev_in[c], s_in), "event record");
      CE_CUDA(cudaStreamWaitEvent(s_k, h->ev_in[c], 0), "stream wait");
      int r = launch_contract(h, dy + off, dx + size_t(t) * K * N, dh + off, tc, mc, K,
                              set_of_instance ? dsoi + t : nullptr, s_k);
      if (r != CE_OK) return r;
      CE_CUDA(cudaEventRecord(h->ev_out[c], s_k), "event record");
      CE_CUDA(cudaStreamWaitEvent(s_out, h->ev_out[c], 0), "stream wait");
      CE_CUDA(cudaMemcpyAsync(static_cast<float2 *>(h_host) + off, dh + off, bytes, cudaMemcpyDeviceToHost, s_out),
              "h copy");
    }
  }
  CE_CUDA(cudaEventRecord(h->ev_slot_free[slot], s_out), "event record");   // the slot's last reader
  if (sync) {
    for (int i = 0; i < 3; ++i) CE_CUDA(cudaEventRecord(h->ev_done[i], h->streams[i]), "event record");
    for (int i = 0; i < 3; ++i) CE_CUDA(cudaStreamWaitEvent(user, h->ev_done[i], 0), "stream wait");
    CE_CUDA(cudaStreamSynchronize(user), "ce_estimate_host: synchronize");
  }
  return CE_OK;
}

int ce_estimate_host(ce_handle *h, const void *y_host, const void *x_host, void *h_host, int32_t T, int32_t M,
                     int32_t K, const int32_t *set_of_instance, void *stream) {
  return estimate_host_impl(h, y_host, x_host, h_host, T, M, K, set_of_instance, stream, true);
}

int ce_estimate_host_async(ce_handle *h, const void *y_host, const void *x_host, void *h_host, int32_t T, int32_t M,
                           int32_t K, const int32_t *set_of_instance, void *stream) {
  return estimate_host_impl(h, y_host, x_host, h_host, T, M, K, set_of_instance, stream, false);
}

int ce_estimate_host_wait(ce_handle *h, void *stream) {
  if (h == nullptr) return fail(CE_EINVAL, "ce_estimate_host_wait: NULL handle");
  if (h->streams[0] == nullptr) return CE_OK;              // no host-path call yet
  DeviceGuard g(h->device);
  if (!g.ok) return fail(CE_ECUDA, "ce_estimate_host_wait: cannot select the handle's device");
  cudaStream_t user = static_cast<cudaStream_t>(stream);
  for (int i = 0; i < 3; ++i) CE_CUDA(cudaEventRecord(h->ev_done[i], h->streams[i]), "event record");
  for (int i = 0; i < 3; ++i) CE_CUDA(cudaStreamWaitEvent(user, h->ev_done[i], 0), "stream wait");
  return CE_OK;
}

}  // extern "C"
