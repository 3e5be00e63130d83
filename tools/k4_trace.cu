// Per-CTA event trace of the K4 contraction (timing only; inputs are random, results unchecked).
// Build: tools/k4_trace.sh   Run: tools/k4_trace N b s M K T
// Prints, per event slot, the median / min / max over CTAs of (clock64 - CTA start) in ns.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../include/ce.h"

extern "C" int ce_k4_trace_set(void *dptr);
extern "C" int ce_k4p_trace_set(void *dptr);   // the pair variant (k4p_block_lmmse_pair.cu) keeps its own trace pointer

int main(int argc, char **argv) {
  int N = argc > 1 ? atoi(argv[1]) : 1200, b = argc > 2 ? atoi(argv[2]) : 100, s = argc > 3 ? atoi(argv[3]) : 100;
  int M = argc > 4 ? atoi(argv[4]) : 128, K = argc > 5 ? atoi(argv[5]) : 12, T = argc > 6 ? atoi(argv[6]) : 1;
  int kernel = argc > 7 ? atoi(argv[7]) : 3;
  std::vector<double> r(2 * size_t(N), 0.0);
  for (int d = 0; d < N; ++d) r[2 * d] = std::pow(0.97, d) * std::cos(0.01 * d), r[2 * d + 1] = -std::pow(0.97, d) * std::sin(0.01 * d);
  r[1] = 0;
  double s2 = 0.03;
  ce_params p{N, b, s, 1, r.data(), &s2};
  ce_handle *h = nullptr;
  int st = ce_init(&p, &h);
  if (st) { printf("init %d %s\n", st, ce_last_error()); return 1; }
  if ((st = ce_build_filters(h, nullptr))) { printf("build %d %s\n", st, ce_last_error()); return 1; }
  if ((st = ce_set_kernel(h, kernel))) { printf("set_kernel %d %s\n", st, ce_last_error()); return 1; }
  const size_t ny = size_t(T) * M * K * N, nx = size_t(T) * K * N;
  std::vector<float> hy(2 * ny), hx(2 * nx);
  srand(1);
  for (auto &v : hy) v = float(rand()) / RAND_MAX - 0.5f;
  for (size_t i = 0; i < nx; ++i) hx[2 * i] = 0.70710678f, hx[2 * i + 1] = (i & 1) ? 0.70710678f : -0.70710678f;
  const int NB = 8;   // rotate buffers so the traced launch is not L2-warm
  void *dy[NB], *dh[NB], *dx;
  for (int i = 0; i < NB; ++i) {
    cudaMalloc(&dy[i], ny * 8);
    cudaMalloc(&dh[i], ny * 8);
    cudaMemcpy(dy[i], hy.data(), ny * 8, cudaMemcpyHostToDevice);
  }
  cudaMalloc(&dx, nx * 8);
  cudaMemcpy(dx, hx.data(), nx * 8, cudaMemcpyHostToDevice);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *dtr;
  cudaMalloc(&dtr, size_t(nsm) * 256 * 8);
  cudaMemset(dtr, 0, size_t(nsm) * 256 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 20; ++i) ce_estimate(h, dy[i % NB], dx, dh[i % NB], T, M, K, nullptr, nullptr);
  cudaEventRecord(e0);
  const int reps = 200;
  for (int i = 0; i < reps; ++i) ce_estimate(h, dy[i % NB], dx, dh[i % NB], T, M, K, nullptr, nullptr);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  int32_t sel = -1;
  ce_selected_kernel(h, &sel);
  printf("kernel %d: %.2f us per call (untraced, back-to-back)\n", sel, 1e3 * ms / reps);
  ce_k4_trace_set(dtr);
  ce_k4p_trace_set(dtr);
  for (int i = 0; i < 3; ++i) {
    ce_estimate(h, dy[i % NB], dx, dh[i % NB], T, M, K, nullptr, nullptr);
    cudaDeviceSynchronize();
  }
  cudaEventRecord(e0);
  ce_estimate(h, dy[5], dx, dh[5], T, M, K, nullptr, nullptr);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("traced launch: %.2f us (event)\n", 1e3 * ms);
  std::vector<unsigned long long> tr(size_t(nsm) * 256);
  cudaMemcpy(tr.data(), dtr, tr.size() * 8, cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  // CTA start skew (globaltimer, ns)
  unsigned long long g0 = ~0ull, g1 = 0;
  int used = 0;
  for (int c = 0; c < nsm; ++c)
    if (tr[size_t(c) * 256]) { g0 = std::min(g0, tr[size_t(c) * 256]); g1 = std::max(g1, tr[size_t(c) * 256]); ++used; }
  printf("CTAs %d, start skew (globaltimer) %llu ns\n", used, g1 - g0);
  // effective SM clock: clock64 ticks over globaltimer ns, start (slots 1/0) to end (slots 4/5)
  std::vector<double> rates;
  for (int c = 0; c < nsm; ++c) {
    const unsigned long long *t = &tr[size_t(c) * 256];
    if (t[0] && t[5] && t[5] > t[0]) rates.push_back(double(t[4] - t[1]) / double(t[5] - t[0]));
  }
  std::sort(rates.begin(), rates.end());
  const double ghz = rates.empty() ? 1.965 : rates[rates.size() / 2];
  printf("effective clock %.3f GHz (median over CTAs; %zu CTAs)\n", ghz, rates.size());
  printf("grid: CTAs with a trace %s\n", kernel == 4 ? "(K5 pairs)" : "");
  const char *names[256] = {};
  names[2] = "setup done";
  names[3] = "epi warp done";
  names[4] = "all done";
  names[200] = "producer after pdl_wait";
  names[201] = "producer first decode";
  names[202] = "tmem alloc done";
  names[203] = "barrier init done";
  names[204] = "producer raw_empty passed";
  for (int slot = 2; slot < 205; ++slot) {
    if (slot == 5) continue;   // end globaltimer
    std::vector<double> v;
    for (int c = 0; c < nsm; ++c) {
      const unsigned long long *t = &tr[size_t(c) * 256];
      if (t[0] && t[slot]) v.push_back(double(t[slot] - t[1]) / ghz);
    }
    if (v.empty()) continue;
    std::sort(v.begin(), v.end());
    const char *nm = names[slot];
    char buf[64];
    if (!nm && kernel == 4) {
      if (slot >= 8 && slot < 32) snprintf(buf, 64, "raw TMA issue it=%d", slot - 8);
      else if (slot >= 32 && slot < 56) snprintf(buf, 64, "raw full seen it=%d", slot - 32);
      else if (slot >= 56 && slot < 80) snprintf(buf, 64, "B written it=%d", slot - 56);
      else if (slot >= 80 && slot < 104) snprintf(buf, 64, "W piece consumed pp=%d", slot - 80);
      else if (slot >= 104 && slot < 128) snprintf(buf, 64, "MMA b_full passed it=%d", slot - 104);
      else if (slot >= 128 && slot < 136) snprintf(buf, 64, "tile MMAs committed lt=%d", slot - 128);
      else if (slot >= 136 && slot < 144) snprintf(buf, 64, "epi start lt=%d", slot - 136);
      else if (slot < 152) snprintf(buf, 64, "epi done lt=%d", slot - 144);
      else if (slot < 160) snprintf(buf, 64, "MMA w_full passed e=%d", slot - 152);
      else if (slot < 168) snprintf(buf, 64, "W load start e=%d", slot - 160);
      else snprintf(buf, 64, "W load done e=%d", slot - 168);
      nm = buf;
    }
    if (!nm) {
      if (slot >= 8 && slot < 32) snprintf(buf, 64, "raw TMA issue it=%d", slot - 8);
      else if (slot >= 32 && slot < 56) snprintf(buf, 64, "raw full seen it=%d", slot - 32);
      else if (slot >= 56 && slot < 80) snprintf(buf, 64, "A written it=%d", slot - 56);
      else if (slot >= 80 && slot < 104) snprintf(buf, 64, "B issue/fwd it=%d", slot - 80);
      else if (slot >= 104 && slot < 128) snprintf(buf, 64, "MMA issue it=%d", slot - 104);
      else if (slot >= 128 && slot < 136) snprintf(buf, 64, "tile MMAs committed lt=%d", slot - 128);
      else if (slot >= 136 && slot < 144) snprintf(buf, 64, "epi start lt=%d", slot - 136);
      else if (slot < 152) snprintf(buf, 64, "epi done lt=%d", slot - 144);
      else if (slot < 176) snprintf(buf, 64, "K5 a_full passed it=%d / K4 tile commit lt=%d", slot - 152, slot - 144);
      else snprintf(buf, 64, "K5 b_full passed it=%d", slot - 176);
      nm = buf;
    }
    printf("%-28s median %8.0f  min %8.0f  max %8.0f ns  (n=%zu)\n", nm, v[v.size() / 2], v.front(), v.back(), v.size());
  }
  ce_free(h);
  return 0;
}
