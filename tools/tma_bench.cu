// TMA read-stream microbenchmark: per-SM throughput of 2-D tensor loads vs box shape and ring depth.
// Each persistent CTA streams boxes [box_rows][box_floats] of a [rows][2N] float tensor into an S-deep
// smem ring (one elected thread issues; the same thread waits and re-issues).  Reports GB/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tma_bench tools/tma_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void stream(const __grid_constant__ CUtensorMap tm, int box_rows, int box_floats, int n_row_blocks,
                       int n_col_blocks, int stages, uint32_t stage_bytes, unsigned long long *sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bars[16];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int total = n_row_blocks * n_col_blocks;
  int it = 0;
  unsigned long long acc = 0;
  auto issue = [&](int u, int s) {
    const int rb = u / n_col_blocks, cb = u % n_col_blocks;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[s])), "r"(stage_bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(sm + size_t(s) * stage_bytes)),
        "l"(reinterpret_cast<uint64_t>(&tm)), "r"(cb * box_floats), "r"(rb * box_rows), "r"(smem_u32(&bars[s]))
        : "memory");
  };
  int next = blockIdx.x;
  for (int s = 0; s < stages && next < total; ++s, next += gridDim.x) issue(next, s);
  for (int u = blockIdx.x; u < total; u += gridDim.x, ++it) {
    const int s = it % stages;
    const uint32_t ph = (it / stages) & 1;
    asm volatile(
        "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(
            smem_u32(&bars[s])),
        "r"(ph)
        : "memory");
    acc += sm[size_t(s) * stage_bytes + 5];
    if (next < total) {
      issue(next, s);
      next += gridDim.x;
    }
  }
  sink[blockIdx.x] = acc;
}

// copy: warp 0 lane 0 streams boxes into an S-deep ring; warps 1..4 copy each landed box to dst with
// 16-byte coalesced stores (same rows/cols as the source), then release the slot.
__global__ void copyk(const __grid_constant__ CUtensorMap tm, float *dst, long long pitch_f, int box_rows,
                      int box_floats, int n_row_blocks, int n_col_blocks, int stages, uint32_t stage_bytes) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[16], empty[16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 128;" ::"r"(smem_u32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int total = n_row_blocks * n_col_blocks;
  auto wait = [](uint64_t *b, uint32_t ph) {
    asm volatile(
        "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(
            smem_u32(b)),
        "r"(ph)
        : "memory");
  };
  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int u = blockIdx.x; u < total; u += gridDim.x, ++it) {
        const int s = it % stages;
        wait(&empty[s], ((it / stages) & 1) ^ 1);
        const int rb = u / n_col_blocks, cb = u % n_col_blocks;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(stage_bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                smem_u32(sm + size_t(s) * stage_bytes)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(cb * box_floats), "r"(rb * box_rows), "r"(smem_u32(&full[s]))
            : "memory");
      }
    }
  } else if (warp <= 4) {
    const int t = threadIdx.x - 32;    // 0..127
    int it = 0;
    const int v_per_row = box_floats / 4;
    for (int u = blockIdx.x; u < total; u += gridDim.x, ++it) {
      const int s = it % stages;
      wait(&full[s], (it / stages) & 1);
      const int rb = u / n_col_blocks, cb = u % n_col_blocks;
      const float4 *src = reinterpret_cast<const float4 *>(sm + size_t(s) * stage_bytes);
      for (int e = t; e < box_rows * v_per_row; e += 128) {
        const int r = e / v_per_row, v = e % v_per_row;
        float4 val = src[e];
        *reinterpret_cast<float4 *>(dst + (size_t(rb) * box_rows + r) * pitch_f + size_t(cb) * box_floats + 4 * v) = val;
      }
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
    }
  }
}

// K4 read pattern: tile g -> (t, w, ct) by `order`; each tile reads nkc boxes [128 rows][16 complex] at
// columns 2(a_w + 16 kc) of rows t*cols + ct*128.  order 0: ct fastest; 1: w fastest; 2: kc-outer
// (all tiles of a CTA interleaved per chunk is not modelled).
__global__ void k4pat(const __grid_constant__ CUtensorMap tm, int T, int n_win, int n_ct, int b, int s_stride,
                      int cols, int nkc, int stages, int order, unsigned long long *sink, int bw = 32) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bars[16];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int n_tiles = T * n_win * n_ct;
  const int total = ((n_tiles - int(blockIdx.x) + int(gridDim.x) - 1) / int(gridDim.x)) * nkc;
  auto coords = [&](int j, int *c0, int *c1) {
    const int tile = blockIdx.x + (j / nkc) * gridDim.x, kc = j % nkc;
    int t, w, ct;
    if (order == 0) { ct = tile % n_ct; w = (tile / n_ct) % n_win; t = tile / (n_ct * n_win); }
    else { w = tile % n_win; ct = (tile / n_win) % n_ct; t = tile / (n_ct * n_win); }
    const int a = min(w * s_stride, 2 * 1638 - b);   // N = 3276 for this bench tensor
    *c0 = 2 * a + bw * kc;
    *c1 = t * cols + ct * 128;
  };
  auto issue = [&](int j, int s) {
    int c0, c1;
    coords(j, &c0, &c1);
    const uint32_t sbytes = 128u * uint32_t(bw) * 4u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[s])), "r"(sbytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(sm + size_t(s) * sbytes)),
        "l"(reinterpret_cast<uint64_t>(&tm)), "r"(c0), "r"(c1), "r"(smem_u32(&bars[s]))
        : "memory");
  };
  unsigned long long acc = 0;
  int next = 0;
  for (int s = 0; s < stages && next < total; ++s, ++next) issue(next, s);
  for (int j = 0; j < total; ++j) {
    const int s = j % stages;
    asm volatile(
        "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(
            smem_u32(&bars[s])),
        "r"((j / stages) & 1)
        : "memory");
    acc += sm[size_t(s) * 128u * bw * 4u + 7];
    if (next < total) issue(next++, s);
  }
  sink[blockIdx.x] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char **argv) {
  const long long rows = 20LL * 6144;   // config 5: T*M*K rows of N = 3276 complex
  const int N = 3276;
  const size_t bytes = size_t(rows) * N * 8;
  void *d;
  cudaMalloc(&d, bytes);
  cudaMemset(d, 1, bytes);
  void *fp;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(fp);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *sink;
  cudaMalloc(&sink, 4096 * 8);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  {
    // K4 config-5 read pattern on the first T=2 instances (rows = T * 6144)
    CUtensorMap tm;
    cuuint64_t dims[2] = {cuuint64_t(2) * N, cuuint64_t(rows)};
    cuuint64_t str[1] = {cuuint64_t(2) * N * 4};
    cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(k4pat, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaEvent_t c0, c1;
    cudaEventCreate(&c0);
    cudaEventCreate(&c1);
    for (int Tn : {2, 20})
      for (int order : {0, 1})
        for (int st : {3, 4, 8}) {
          k4pat<<<nsm, 32, st * 16384>>>(tm, Tn, 26, 48, 126, 126, 6144, 8, st, order, sink);
          cudaEventRecord(c0);
          k4pat<<<nsm, 32, st * 16384>>>(tm, Tn, 26, 48, 126, 126, 6144, 8, st, order, sink);
          cudaEventRecord(c1);
          cudaEventSynchronize(c1);
          float ms;
          cudaEventElapsedTime(&ms, c0, c1);
          const double moved = double(Tn) * 26 * 48 * 8 * 16384;
          printf("K4PAT T=%d order %d stages %d: %.1f us  %.1f GB/s  %s\n", Tn, order, st, ms * 1e3, moved / ms / 1e6,
                 cudaGetErrorString(cudaGetLastError()));
        }
  }
  {
    // K4 read pattern with wider boxes: 128 rows x {128, 256, 512} B, the same bytes in flight (~64-128 KB)
    cudaEvent_t c0, c1;
    cudaEventCreate(&c0);
    cudaEventCreate(&c1);
    for (int bw : {32, 64, 128}) {
      CUtensorMap tm;
      cuuint64_t dims[2] = {cuuint64_t(2) * N, cuuint64_t(rows)};
      cuuint64_t str[1] = {cuuint64_t(2) * N * 4};
      cuuint32_t box[2] = {cuuint32_t(bw), 128}, es[2] = {1, 1};
      enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      const int nkc = (2 * 126 + bw - 1) / bw;
      for (int kb : {64, 128, 192}) {
        const int st = std::max(1, std::min(16, kb * 1024 / (128 * bw * 4)));
        k4pat<<<nsm, 32, st * 128 * bw * 4>>>(tm, 20, 26, 48, 126, 126, 6144, nkc, st, 0, sink, bw);
        cudaEventRecord(c0);
        k4pat<<<nsm, 32, st * 128 * bw * 4>>>(tm, 20, 26, 48, 126, 126, 6144, nkc, st, 0, sink, bw);
        cudaEventRecord(c1);
        cudaEventSynchronize(c1);
        float ms;
        cudaEventElapsedTime(&ms, c0, c1);
        const double moved = 20.0 * 26 * 48 * nkc * 128.0 * bw * 4;
        printf("K4PAT-W box 128 x %3d B stages %2d (%3d KB): %.1f us  %.1f GB/s  %s\n", bw * 4, st, st * bw / 2, ms * 1e3,
               moved / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  float *dcopy;
  cudaMalloc(&dcopy, bytes);
  cudaFuncSetAttribute(copyk, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  {
    const int cshapes[][2] = {{128, 32}, {64, 64}, {32, 128}, {16, 256}, {128, 64}, {64, 128}, {32, 256}};
    cudaEvent_t c0, c1;
    cudaEventCreate(&c0);
    cudaEventCreate(&c1);
    for (auto &sh : cshapes) {
      const int br = sh[0], bf = sh[1];
      const uint32_t sb = uint32_t(br) * bf * 4;
      CUtensorMap tm;
      cuuint64_t dims[2] = {cuuint64_t(2) * N, cuuint64_t(rows)};
      cuuint64_t str[1] = {cuuint64_t(2) * N * 4};
      cuuint32_t box[2] = {cuuint32_t(bf), cuuint32_t(br)}, es[2] = {1, 1};
      enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      const int nrb = int(rows / br), ncb = (2 * N) / bf;
      for (int rk : {48, 96, 160}) {
        int stages = int((rk * 1024) / sb);
        if (stages < 2) continue;
        if (stages > 16) stages = 16;
        copyk<<<nsm, 160, stages * sb>>>(tm, dcopy, 2LL * N, br, bf, nrb, ncb, stages, sb);
        cudaEventRecord(c0);
        copyk<<<nsm, 160, stages * sb>>>(tm, dcopy, 2LL * N, br, bf, nrb, ncb, stages, sb);
        cudaEventRecord(c1);
        cudaEventSynchronize(c1);
        float ms;
        cudaEventElapsedTime(&ms, c0, c1);
        const double moved = 2.0 * double(nrb) * ncb * sb;
        printf("COPY box %3d rows x %4d B  stages %2d  %7.1f GB/s (read+write)  %s\n", br, bf * 4, stages,
               moved / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  const int shapes[][2] = {{128, 32}, {128, 64}, {128, 128}, {128, 256}, {64, 64}, {64, 128}, {64, 256},
                           {32, 256}, {16, 256}, {256, 32}, {256, 64}};
  const int ring_kb[] = {48, 96, 192};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (auto &sh : shapes) {
    const int br = sh[0], bf = sh[1];
    const uint32_t sb = uint32_t(br) * bf * 4;
    CUtensorMap tm;
    cuuint64_t dims[2] = {cuuint64_t(2) * N, cuuint64_t(rows)};
    cuuint64_t str[1] = {cuuint64_t(2) * N * 4};
    cuuint32_t box[2] = {cuuint32_t(bf), cuuint32_t(br)}, es[2] = {1, 1};
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS) {
      printf("encode failed %d %d\n", br, bf);
      continue;
    }
    const int nrb = int(rows / br), ncb = (2 * N) / bf;
    for (int rk : ring_kb) {
      int stages = int((rk * 1024) / sb);
      if (stages < 1) stages = 1;
      if (stages > 16) stages = 16;
      if (size_t(stages) * sb > 220 * 1024) continue;
      // ~1.6 GB read per run
      const int use_rb = nrb;
      const int grid = getenv("TMA_GRID") ? atoi(getenv("TMA_GRID")) : nsm;
      const int use_rb2 = grid < nsm ? (use_rb * grid) / nsm + 1 : use_rb;
      stream<<<grid, 32, stages * sb>>>(tm, br, bf, use_rb2, ncb, stages, sb, sink);
      cudaEventRecord(e0);
      stream<<<grid, 32, stages * sb>>>(tm, br, bf, use_rb2, ncb, stages, sb, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double moved = double(use_rb2) * ncb * sb;
      printf("grid %3d box %3d rows x %4d B  stages %2d (%3d KB)  %7.1f GB/s  (%.2f GB/s/SM)  %s\n", grid, br, bf * 4,
             stages, stages * sb / 1024, moved / ms / 1e6, moved / ms / 1e6 / grid, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
