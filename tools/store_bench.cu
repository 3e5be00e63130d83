// TMA-store pattern microbenchmark: persistent CTAs write a [rows][pitch floats] fp32 tensor as tiles of
// [tile_rows][tile_floats] (K4 / K10 output tiles), each tile as TMA stores of boxes [box_rows][32 floats] (SW128) from a
// staging buffer, tiles dealt grid-stride with the column tile fastest (K4's order).  Prints TB/s per shape.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1802_05427_b200/csrc -o tools/store_bench tools/store_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>

#include "tc_ptx.cuh"
#include "tmap.cuh"

using namespace ce;

struct SP {
  int rows, pitch, tile_rows, tile_floats, box_rows, n_ct, n_tiles, warps, contiguous;
};

__global__ void __launch_bounds__(512, 1) store_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ SP p) {
  extern __shared__ uint8_t sm[];
  uint8_t *stg = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= p.warps) return;
  // staging: one [box_rows][128 B] box per warp, filled once (contents do not matter)
  uint8_t *buf = stg + warp * p.box_rows * 128;
  for (int i = lane; i < p.box_rows * 32; i += 32) reinterpret_cast<float *>(buf)[i] = float(i);
  fence_proxy_async();
  __syncwarp();
  const int nb_r = p.tile_rows / p.box_rows, nb_c = p.tile_floats / 32;
  const int g0 = p.contiguous ? int((long long)blockIdx.x * p.n_tiles / gridDim.x) : int(blockIdx.x);
  const int g1 = p.contiguous ? int((long long)(blockIdx.x + 1) * p.n_tiles / gridDim.x) : p.n_tiles;
  const int gs = p.contiguous ? 1 : int(gridDim.x);
  for (int g = g0; g < g1; g += gs) {
    const int ct = g % p.n_ct, rt = g / p.n_ct;
    // the tile's boxes split over the warps: box index b = warp, warp + warps, ... (row blocks outer, columns inner)
    for (int b = warp; b < nb_r * nb_c; b += p.warps) {
      const int br = b / nb_c, bc = b % nb_c;
      if (lane == 0) {
        bulk_wait_read0();
        tma_store_2d(&tm, buf, ct * p.tile_floats + bc * 32, rt * p.tile_rows + br * p.box_rows);
        bulk_commit();
      }
      __syncwarp();
    }
  }
  if (lane == 0) bulk_wait0();
}

int main(int argc, char **argv) {
  const int rows = argc > 1 ? atoi(argv[1]) : 6144 * 20, pitch = argc > 2 ? atoi(argv[2]) : 6144;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float *d;
  const size_t bytes = size_t(rows) * pitch * 4;
  cudaMalloc(&d, bytes);
  cudaFuncSetAttribute(store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int contiguous = argc > 3 ? atoi(argv[3]) : 0;
  struct Shape { int tile_rows, tile_floats, box_rows, warps; } shapes[] = {
      {128, 256, 32, 4}, {128, 256, 32, 8}, {128, 256, 32, 16}, {128, 256, 16, 16}, {128, 256, 8, 16},
      {128, 256, 64, 8}, {128, 256, 128, 4}, {64, 512, 32, 8}, {32, 1024, 32, 8}, {32, 1024, 8, 16},
      {128, 128, 32, 8}, {16, 2048, 16, 16}, {8, 4096, 8, 16}, {128, 96, 32, 8}, {128, 96, 32, 16},
      {128, 96, 32, 4}, {128, 192, 32, 8}, {128, 480, 32, 8}, {128, 480, 32, 16}, {128, 32, 32, 4},
      {128, 64, 32, 4}, {128, 64, 32, 8}, {128, 160, 32, 8}, {128, 224, 32, 8}, {128, 256, 32, 8}, {128, 320, 32, 8},
      {128, 384, 32, 8}, {128, 576, 32, 8}, {128, 768, 32, 8}};
  for (auto sh : shapes) {
    if (pitch % sh.tile_floats || rows % sh.tile_rows || sh.tile_floats % 32) continue;
    CUtensorMap tm;
    cuuint64_t dims[2] = {cuuint64_t(pitch), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(pitch) * 4};
    cuuint32_t box[2] = {32, cuuint32_t(sh.box_rows)};
    cuuint32_t estr[2] = {1, 1};
    if (encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS) {
      printf("encode failed\n");
      continue;
    }
    SP p{rows, pitch, sh.tile_rows, sh.tile_floats, sh.box_rows, pitch / sh.tile_floats,
         (rows / sh.tile_rows) * (pitch / sh.tile_floats), sh.warps, contiguous};
    const size_t smem = size_t(sh.warps) * sh.box_rows * 128 + 1024;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    store_kernel<<<nsm, 512, smem>>>(tm, p);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int i = 0; i < reps; ++i) store_kernel<<<nsm, 512, smem>>>(tm, p);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double t = ms / reps * 1e-3;
    printf("%s tile %3d x %4d floats, box %3d rows x 128 B, %2d warps: %.1f us  %.2f TB/s  %s\n",
           contiguous ? "contig" : "strided", sh.tile_rows, sh.tile_floats, sh.box_rows, sh.warps, t * 1e6, bytes / t / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  // linear reference: cudaMemset
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaMemset(d, 0, bytes);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) cudaMemset(d, 0, bytes);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("cudaMemset: %.1f us  %.2f TB/s\n", ms / 5 * 1e3, bytes / (ms / 5 * 1e-3) / 1e12);
  return 0;
}
