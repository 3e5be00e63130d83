// Host-side TMA tensor-map helpers shared by the tcgen05 contraction kernels (K4, K8).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

namespace ce {
namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// L2 promotion of the TMA load maps: 64 B measured best for K4 (config 3 10.48 -> 10.31-10.33 us same box, two
// repetitions; configs 4-6 and the statistics kernels equal; 256 B was 2% slower).  CE_TMA_L2PROMO (experiments):
// 0 none, 1 64B (default), 2 128B, 3 256B.
CUtensorMapL2promotion load_promotion() {
  static const int v = getenv("CE_TMA_L2PROMO") ? atoi(getenv("CE_TMA_L2PROMO")) : 1;
  return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                : v == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                         : v == 3 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
}

bool make_map(CUtensorMap *m, const void *ptr, int N, long long rows, int box_rows, int box_floats = 32) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cuuint64_t(2) * N, cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(2) * N * 4};
  cuuint32_t box[2] = {cuuint32_t(box_floats), cuuint32_t(box_rows)};   // 16 complex per box row by default
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, load_promotion(),
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// y [T][M][K][2N floats] as a 4-D tensor (2N, K, M, T): box {box_floats, 1, box_rows, 1} = box_rows antennas of
// one user (K8: a chunk's columns share their LS factors); antennas beyond M are zero-filled.
bool make_map_kmajor(CUtensorMap *m, const void *ptr, int N, int K, int M, int T, int box_rows, int box_floats) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {cuuint64_t(2) * N, cuuint64_t(K), cuuint64_t(M), cuuint64_t(T)};
  const cuuint64_t row = cuuint64_t(2) * N * 4;
  cuuint64_t strides[3] = {row, row * K, row * K * M};
  cuuint32_t box[4] = {cuuint32_t(box_floats), 1, cuuint32_t(box_rows), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void *>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// [rows][2N] float tensor, box [box_rows][box_floats], SWIZZLE_128B (box_floats * 4 == 128): store maps.
bool make_map_sw128(CUtensorMap *m, const void *ptr, int N, long long rows, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cuuint64_t(2) * N, cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(2) * N * 4};
  cuuint32_t box[2] = {cuuint32_t(32), cuuint32_t(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Tensor maps are a pure function of (pointer, N, rows, box rows): cache the last few per host thread so
// back-to-back calls on the same buffers skip the driver encode.
struct MapCacheEntry {
  const void *ptr;
  int N, box_rows, box_floats;
  long long rows;
  bool sw128;
  CUtensorMap map;
};
bool cached_map(CUtensorMap *m, const void *ptr, int N, long long rows, int box_rows, bool sw128 = false,
                int box_floats = 32) {
  constexpr int NC = 32;
  static thread_local MapCacheEntry cache[NC];
  static thread_local int used = 0, next = 0;
  for (int i = 0; i < used; ++i)
    if (cache[i].ptr == ptr && cache[i].N == N && cache[i].rows == rows && cache[i].box_rows == box_rows &&
        cache[i].sw128 == sw128 && cache[i].box_floats == box_floats) {
      *m = cache[i].map;
      return true;
    }
  if (!(sw128 ? make_map_sw128(m, ptr, N, rows, box_rows) : make_map(m, ptr, N, rows, box_rows, box_floats)))
    return false;
  MapCacheEntry &e = cache[next];
  e = MapCacheEntry{ptr, N, box_rows, box_floats, rows, sw128, *m};
  next = (next + 1) % NC;
  if (used < NC) ++used;
  return true;
}

}  // namespace
}  // namespace ce
