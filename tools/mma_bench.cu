// tcgen05 kind::f16 MMA throughput microbenchmark: back-to-back 128 x N x 16 BF16 MMAs from shared-memory
// operands with SWIZZLE_64B (64-byte K-major rows, as K4) or SWIZZLE_128B descriptors.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1802_05427_b200/csrc -o tools/mma_bench tools/mma_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

#include "tc_ptx.cuh"

using namespace ce;

__device__ __forceinline__ uint64_t sw128(uint32_t saddr) { return sw128_desc(saddr); }

template <int SW>
__global__ void bench(int iters, int N, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t *smem = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 256);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    // A: 128 rows, B: N rows; SW64: rows of 64 B; SW128: rows of 128 B
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 32 * 1024);
    const uint64_t ad = SW == 64 ? sw64_desc(a0) : sw128(a0);
    const uint64_t bd = SW == 64 ? sw64_desc(b0) : sw128(b0);
    const int ksteps = SW == 64 ? 2 : 4;            // 16-element K steps per swizzle row
    unsigned long long t0 = clock64();
    int ph = 0;
    for (int it = 0; it < iters; ++it) {
      for (int ks = 0; ks < ksteps; ++ks) {
        const uint64_t adv = uint64_t(2 * ks);
        mma_bf16(d, ad + adv, bd + adv, idesc, (it | ks) != 0);
      }
      if ((it & 15) == 15) {
        mma_commit(&bar);
        mbar_wait(&bar, ph);
        ph ^= 1;
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, ph);
    unsigned long long t1 = clock64();
    out[blockIdx.x] = (t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(d, 256);
  }
}

// CTA pair: cta_group::2, M = 256 (128 rows per CTA), N columns with N/2 B rows staged in each CTA.
__global__ void __cluster_dims__(2, 1, 1) bench_pair(int iters, int N, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t *smem = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) tmem_alloc2(&slot, 256);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t d = slot;
  if (threadIdx.x == 0 && cluster_ctarank() == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(256 >> 4) << 24);
    const uint64_t ad = sw64_desc(smem_u32(smem)), bd = sw64_desc(smem_u32(smem + 32 * 1024));
    unsigned long long t0 = clock64();
    int ph = 0;
    for (int it = 0; it < iters; ++it) {
      for (int ks = 0; ks < 2; ++ks) mma_bf16_pair(d, ad + uint64_t(2 * ks), bd + uint64_t(2 * ks), idesc, (it | ks) != 0);
      if ((it & 15) == 15) {
        mma_commit_pair(&bar);
        mbar_wait(&bar, ph);
        ph ^= 1;
      }
    }
    mma_commit_pair(&bar);
    mbar_wait(&bar, ph);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc2(d, 256);
  }
}

__device__ __forceinline__ void mma2_ts_b(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

// CTA pair, A from TMEM (K5's form): M = 256, N columns, N/2 B rows per CTA in SW64 smem; commit every `cevery` MMAs
__global__ void __cluster_dims__(2, 1, 1) bench_pair_ts(int iters, int N, int cevery, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t *smem = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) tmem_alloc2(&slot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t d = slot;
  if (threadIdx.x == 0 && cluster_ctarank() == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(256 >> 4) << 24);
    const uint64_t bd = sw64_desc(smem_u32(smem + 32 * 1024));
    unsigned long long t0 = clock64();
    int ph = 0, n = 0;
    for (int it = 0; it < iters; ++it) {
      for (int ks = 0; ks < 2; ++ks) {
        mma2_ts_b(d, d + 256 + 8 * ks, bd + uint64_t(2 * ks), idesc, (it | ks) != 0);
        if (++n == cevery) {
          n = 0;
          mma_commit_pair(&bar);
        }
      }
      if ((it & 15) == 15) {
        mma_commit_pair(&bar);
        mbar_wait(&bar, ph);
        ph ^= 1;
        if (cevery < 1000) {   // the per-chunk commits also arrived: drain by waiting the phase parity again
        }
      }
    }
    mma_commit_pair(&bar);
    mbar_wait(&bar, ph);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc2(d, 512);
  }
}

// single CTA, A from TMEM: M = 128, N columns (D at columns 0.., A at columns 256..)
__global__ void bench_ts1(int iters, int N, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t *smem = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint64_t bd = sw64_desc(smem_u32(smem + 32 * 1024));
    unsigned long long t0 = clock64();
    int ph = 0;
    for (int it = 0; it < iters; ++it) {
      for (int ks = 0; ks < 2; ++ks) {
        const uint32_t a = d + 256 + 8 * ks;
        const uint32_t acc = (it | ks) != 0;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
            "r"(a), "l"(bd + uint64_t(2 * ks)), "r"(idesc), "r"(acc)
            : "memory");
      }
      if ((it & 15) == 15) {
        mma_commit(&bar);
        mbar_wait(&bar, ph);
        ph ^= 1;
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, ph);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(d, 512);
  }
}

// K10 / K4 issue pattern: units of 2 K-steps x 3 products (A_hi B_hi, A_hi B_lo, A_lo B_hi) into one of NACC
// accumulators, one commit per unit to that accumulator's mbarrier; before unit u the issuer waits for unit u - NACC
// (the accumulator is free again).  mode 1: additionally wait on unit u - 1's barrier (fully serialised units)
__global__ void bench_units(int iters, int N, int nacc, int mode, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bars[8];
  __shared__ uint32_t slot;
  uint8_t *smem = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d0 = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint64_t ah = sw64_desc(smem_u32(smem)), al = sw64_desc(smem_u32(smem + 16 * 1024));
    const uint64_t bh = sw64_desc(smem_u32(smem + 32 * 1024)), bl = sw64_desc(smem_u32(smem + 48 * 1024));
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int acc = it % nacc;
      if (it >= nacc) mbar_wait(&bars[acc], ((it - nacc) / nacc) & 1);
      if (mode == 1 && it >= 1) mbar_wait(&bars[(it - 1) % nacc], ((it - 1) / nacc) & 1);
      tc_fence_after();
      const uint32_t d = d0 + uint32_t(acc * N);
      for (int ks = 0; ks < 2; ++ks) {
        const uint64_t adv = uint64_t(2 * ks);
        mma_bf16(d, ah + adv, bh + adv, idesc, ks != 0);
        mma_bf16(d, ah + adv, bl + adv, idesc, 1u);
        mma_bf16(d, al + adv, bh + adv, idesc, 1u);
      }
      mma_commit(&bars[acc]);
    }
    for (int it = iters - nacc; it < iters; ++it) if (it >= 0) mbar_wait(&bars[it % nacc], (it / nacc) & 1);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(d0, 512);
  }
}

int main() {
  unsigned long long *dout, h[148];
  cudaMalloc(&dout, 148 * 8);
  cudaFuncSetAttribute(bench<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(bench<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int N : {256, 208, 128}) {
    for (int grid : {1, 148}) {
      const int iters = 4096;
      bench<64><<<grid, 128, 100 * 1024>>>(iters, N, dout);
      cudaDeviceSynchronize();
      cudaMemcpy(h, dout, 8 * grid, cudaMemcpyDeviceToHost);
      double c64 = double(h[0]) / (iters * 2);
      bench<128><<<grid, 128, 100 * 1024>>>(iters, N, dout);
      cudaDeviceSynchronize();
      cudaMemcpy(h, dout, 8 * grid, cudaMemcpyDeviceToHost);
      double c128 = double(h[0]) / (iters * 4);
      const double flop = 2.0 * 128 * N * 16;
      printf("N=%3d grid %3d: SW64 %.1f cyc/MMA (%.0f flop/clk)  SW128 %.1f cyc/MMA (%.0f flop/clk)  %s\n", N, grid, c64,
             flop / c64, c128, flop / c128, cudaGetErrorString(cudaGetLastError()));
    }
  }
  cudaFuncSetAttribute(bench_units, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int N : {128, 256}) {
    for (int nacc : {1, 2, 4}) {
      if (nacc * N > 512) continue;
      for (int mode : {0, 1}) {
        const int iters = 2048;
        bench_units<<<148, 128, 100 * 1024>>>(iters, N, nacc, mode, dout);
        cudaDeviceSynchronize();
        cudaMemcpy(h, dout, 8, cudaMemcpyDeviceToHost);
        const double c = double(h[0]) / (iters * 6);
        printf("UNITS N=%3d nacc %d mode %d: %.1f cyc/MMA  %s\n", N, nacc, mode, c, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  cudaFuncSetAttribute(bench_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int N : {256, 208}) {
    const int iters = 4096;
    bench_pair<<<2, 128, 100 * 1024>>>(iters, N, dout);
    cudaDeviceSynchronize();
    cudaMemcpy(h, dout, 8, cudaMemcpyDeviceToHost);
    const double c = double(h[0]) / (iters * 2);
    printf("PAIR M=256 N=%3d: %.1f cyc/MMA (%.0f flop/clk per SM)  %s\n", N, c, 2.0 * 128 * N * 16 / c,
           cudaGetErrorString(cudaGetLastError()));
  }
  cudaFuncSetAttribute(bench_ts1, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int N : {256, 208, 128, 64}) {
    const int iters = 4096;
    bench_ts1<<<148, 128, 100 * 1024>>>(iters, N, dout);
    cudaDeviceSynchronize();
    cudaMemcpy(h, dout, 8, cudaMemcpyDeviceToHost);
    const double c = double(h[0]) / (iters * 2);
    printf("TS1 (A in TMEM) M=128 N=%3d: %.1f cyc/MMA (%.0f flop/clk)  %s\n", N, c, 2.0 * 128 * N * 16 / c,
           cudaGetErrorString(cudaGetLastError()));
  }
  cudaFuncSetAttribute(bench_pair_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int N : {256, 128, 96, 64}) {
    for (int grid : {2, 148}) {
      const int iters = 4096;
      bench_pair_ts<<<grid, 128, 100 * 1024>>>(iters, N, 1 << 30, dout);
      cudaDeviceSynchronize();
      cudaMemcpy(h, dout, 8, cudaMemcpyDeviceToHost);
      const double c = double(h[0]) / (iters * 2);
      printf("PAIR TS (A in TMEM) M=256 N=%3d grid %3d: %.1f cyc/MMA (%.0f flop/clk per SM)  %s\n", N, grid, c,
             2.0 * 128 * N * 16 / c, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
