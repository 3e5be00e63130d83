// Per-SM throughput of the copy engines that feed K4/K5, from an L2-resident source (the filter bank's situation:
// every SM reads the same few hundred KB), grid = 1 and grid = 148:
//   bulk  : cp.async.bulk (1-D TMA) of `sz` bytes per op
//   box   : cp.async.bulk.tensor.2d box of `rows` x `rowbytes`
//   ldgsts: cp.async.cg.shared.global 16 B per thread (LSU path), 4 warps
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1802_05427_b200/csrc -o tools/tma_unit_bench tools/tma_unit_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

#include "tc_ptx.cuh"
#include "tmap.cuh"

using namespace ce;

constexpr int STAGES = 8;
constexpr int STAGE_BYTES = 16384;

__global__ void bulk_kernel(const uint8_t *src, size_t span, int sz, int iters, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[STAGES];
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int s = it % STAGES;
      if (it >= STAGES) mbar_wait(&full[s], ((it / STAGES) - 1) & 1);
      mbar_arrive_expect_tx(&full[s], sz);
      bulk_g2s(sm + s * STAGE_BYTES, src + (size_t(it) * sz) % span, sz, &full[s]);
    }
    for (int it = iters; it < iters + STAGES; ++it) mbar_wait(&full[it % STAGES], ((it / STAGES) - 1) & 1);
    out[blockIdx.x] = clock64() - t0;
  }
}

__global__ void box_kernel(const __grid_constant__ CUtensorMap tm, int rows_total, int box_rows, int box_bytes,
                           int iters, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[STAGES];
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int s = it % STAGES;
      if (it >= STAGES) mbar_wait(&full[s], ((it / STAGES) - 1) & 1);
      mbar_arrive_expect_tx(&full[s], box_rows * box_bytes);
      tma_load_2d(sm + s * STAGE_BYTES, &tm, 0, (it * box_rows) % (rows_total - box_rows), &full[s]);
    }
    for (int it = iters; it < iters + STAGES; ++it) mbar_wait(&full[it % STAGES], ((it / STAGES) - 1) & 1);
    out[blockIdx.x] = clock64() - t0;
  }
}

__global__ void ldgsts_kernel(const uint8_t *src, size_t span, int iters, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  // 4 warps, each op = 128 threads x 16 B = 2 KB; STAGES groups in flight
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int s = it % STAGES;
    const uint32_t dst = smem_u32(sm + s * STAGE_BYTES + threadIdx.x * 16);
    const uint8_t *g = src + (size_t(it) * 2048 + threadIdx.x * 16) % span;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(g) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 7;" ::: "memory");
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t span = 256 * 1024;              // L2-resident source shared by every SM
  uint8_t *src;
  cudaMalloc(&src, 64 << 20);
  cudaMemset(src, 1, 64 << 20);
  unsigned long long *dout, h[256];
  cudaMalloc(&dout, 256 * 8);
  const int smem = STAGES * STAGE_BYTES;
  cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(box_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(ldgsts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const double ghz = 1.965;
  for (int grid : {1, nsm}) {
    for (int sz : {2048, 4096, 8192, 16384}) {
      const int iters = 2048;
      bulk_kernel<<<grid, 32, smem>>>(src, span, sz, iters, dout);
      cudaDeviceSynchronize();
      cudaMemcpy(h, dout, 8 * grid, cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("grid %3d bulk %5d B: %.1f cyc/op  %.1f B/clk/SM  %.1f GB/s/SM  %s\n", grid, sz, mx / iters,
             double(sz) * iters / mx, double(sz) * iters / mx * ghz, cudaGetErrorString(cudaGetLastError()));
    }
    for (int rb : {128, 256}) {
      for (int rows : {64, 128}) {
        if (rows * rb > STAGE_BYTES) continue;
        CUtensorMap tm;
        const long long rows_total = (64 << 20) / (2 * rb) > 4096 ? 4096 : (64 << 20) / (2 * rb);
        if (!make_map(&tm, src, rb / 8 /*N complex: 2N floats = rb/4*/, rows_total, rows, rb / 4)) {
          printf("encode failed\n");
          continue;
        }
        const int iters = 2048;
        box_kernel<<<grid, 32, smem>>>(tm, int(rows_total), rows, rb, iters, dout);
        cudaDeviceSynchronize();
        cudaMemcpy(h, dout, 8 * grid, cudaMemcpyDeviceToHost);
        double mx = 0;
        for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
        const double bytes = double(rows) * rb * iters;
        printf("grid %3d box %3d rows x %3d B: %.1f cyc/op  %.2f cyc/row  %.1f GB/s/SM  %s\n", grid, rows, rb,
               mx / iters, mx / iters / rows, bytes / mx * ghz, cudaGetErrorString(cudaGetLastError()));
      }
    }
    {
      const int iters = 4096;
      ldgsts_kernel<<<grid, 128, smem>>>(src, span, iters, dout);
      cudaDeviceSynchronize();
      cudaMemcpy(h, dout, 8 * grid, cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("grid %3d ldgsts 4 warps x 16 B: %.1f GB/s/SM  %s\n", grid, 2048.0 * iters / mx * ghz,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
