// K4 -- fused LS + block-LMMSE contraction on tcgen05 (kind::f16, BF16 operands), error-compensated
// "BF16x3":  D = A_hi B_hi + A_hi B_lo + A_lo B_hi,  X_hi = bf16_rn(X), X_lo = bf16_rn(X - X_hi),
// FP32 accumulation in TMEM.  Per-product error <= ~3 * 2^-18 (the dropped A_lo B_lo term and the
// rounding of the lo parts); DESIGN.md §5 derives the bound and the emulation that measured
// 1.4e-6 relative Frobenius error on configs 2-5 against the 1e-4 bar.
//
// Same operation as K2/K3 (Eq. 12 per block, LS of Eq. 9 fused into the load) and
// the same complex -> real embedding as K3 (A = interleaved LS row, D = interleaved output row,
// B_r^T rows 2i / 2i+1 = (Re W_ij, -Im W_ij) / (Im W_ij, Re W_ij)).  BF16 runs the tensor core at
// twice the TF32 rate and halves the operand bytes in shared memory and L2.
//
// Pipeline (persistent CTAs, one per SM, 480 threads):
//   warp 12   : raw producer -- 2D TMA (cp.async.bulk.tensor) of the raw y box [128 rows x 16
//               complex] and the pilot box [K rows x 16 complex] of each K chunk into a 3-deep
//               raw ring (no registers held, ~48 KB of HBM reads in flight per SM)
//   warps 0-7 : transform -- per chunk: LS factors f = conj(x)/|x|^2 computed once per (k, j) in
//               place in the raw pilot slot (named barrier), then LS = y f -> bf16 hi/lo ->
//               SWIZZLE_64B K-major A tiles of the 3-deep AB ring; fence.proxy.async; arrive a_full
//   warp 14   : B producer -- cp.async.bulk of the bf16 hi/lo bank chunk (pre-swizzled SW64 image)
//   warp 13   : TMEM allocator + MMA issuer: 2 K-steps x 3 MMAs per chunk, commit -> ab_empty;
//               per tile commit -> tmem_full[acc] (two 256-column accumulators)
//   warps 8-11: epilogue -- tcgen05.ld 32 columns, transpose through smem, coalesced stores
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ce_internal.h"
#include "tc_ptx.cuh"

namespace ce {
namespace {

constexpr int K4_THREADS = 480;            // 15 warps: 8 transform, 4 epilogue, 3 single-thread roles
constexpr int NTR = 256;                   // transform threads
constexpr int CK = 16;                     // complex per K chunk = 32 bf16 = 64-byte rows
constexpr int S_AB = 3;                    // A/B stages
constexpr int S_RAW = 3;                   // raw y/x stages
constexpr int TM = 128;                    // MMA M (columns c per tile)
constexpr int NMAXW = 256;                 // MMA N max (2*kept + row alignment)
constexpr int KMAX = 32;                   // pilot rows per raw stage (K <= 32)
constexpr int A_PLANE = TM * 64;           // 8 KB
constexpr int B_PLANE = NMAXW * 64;        // 16 KB
constexpr int AB_STAGE = 2 * A_PLANE + 2 * B_PLANE;      // 48 KB
constexpr int RAWY = TM * CK * 8;          // 16 KB
constexpr int RAWX = KMAX * CK * 8;        // 4 KB
constexpr int RAW_STAGE = RAWY + RAWX;     // 20 KB
constexpr int EPI_STRIDE = 34;
constexpr int EPI_BYTES = 4 * 32 * EPI_STRIDE * 4;
constexpr int BAR_BYTES = 256;
constexpr int K4_SMEM = S_AB * AB_STAGE + S_RAW * RAW_STAGE + EPI_BYTES + BAR_BYTES + 1024;

struct K4Params {
  float2 *h;
  const uint16_t *bank_hi;   // bf16 [n_sets][nkc][NR][32] swizzled SW64 rows
  const uint16_t *bank_lo;
  const Window *geo;
  const int32_t *soi;
  int T, K, N, b, n_win, n_sets, nkc, NR, cols, n_ct, n_tiles;
};

struct Tile4 {
  int t, ct, a, o, kept, n0, off, nw, set;
  bool set_ok;
};

__device__ __forceinline__ Tile4 decode4(const K4Params &p, int tile) {
  Tile4 ti;
  ti.ct = tile % p.n_ct;
  const int rest = tile / p.n_ct;
  const int w = rest % p.n_win;
  ti.t = rest / p.n_win;
  const Window g = p.geo[w];
  ti.a = g.a;
  ti.o = g.o;
  ti.kept = g.o_next - g.o;
  const int row2 = 2 * (g.o - g.a);
  ti.n0 = row2 & ~7;
  ti.off = row2 - ti.n0;
  ti.nw = (ti.off + 2 * ti.kept + 15) & ~15;
  const int s = p.soi ? p.soi[ti.t] : 0;
  ti.set_ok = s >= 0 && s < p.n_sets;
  ti.set = ti.set_ok ? s : 0;
  return ti;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo_addr, float hi_addr) {
  // memory order: first float at the lower address = lower 16 bits
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi_addr), "f"(lo_addr));
  return r;
}
__device__ __forceinline__ float bf16_lo_f(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi_f(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }
__device__ __forceinline__ float rcp_approx(float v) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

__global__ void __launch_bounds__(K4_THREADS, 1)
    k4_bf16x3(const __grid_constant__ CUtensorMap tmy, const __grid_constant__ CUtensorMap tmx, K4Params p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment by pointer arithmetic on the __shared__ array (keeps the shared address space
  // visible to the compiler: LDS/STS instead of generic LD/ST)
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *ab = smem;                                   // [S_AB][A_hi | A_lo | B_hi | B_lo]
  uint8_t *raw = smem + S_AB * AB_STAGE;                // [S_RAW][y 16 KB | x 4 KB]
  float *epi = reinterpret_cast<float *>(raw + S_RAW * RAW_STAGE);
  uint64_t *bars = reinterpret_cast<uint64_t *>(reinterpret_cast<uint8_t *>(epi) + EPI_BYTES);
  uint64_t *raw_full = bars;                            // [S_RAW]
  uint64_t *raw_empty = bars + S_RAW;                   // [S_RAW]
  uint64_t *a_full = bars + 2 * S_RAW;                  // [S_AB]
  uint64_t *b_full = a_full + S_AB;                     // [S_AB]
  uint64_t *ab_empty = b_full + S_AB;                   // [S_AB]
  uint64_t *tmem_full = ab_empty + S_AB;                // [2]
  uint64_t *tmem_empty = tmem_full + 2;                 // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_empty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < S_RAW; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_empty[s], NTR);
    }
    for (int s = 0; s < S_AB; ++s) {
      mbar_init(&a_full[s], NTR);
      mbar_init(&b_full[s], 1);
      mbar_init(&ab_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&tmem_empty[i], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 12 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmy)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmx)) : "memory");
  }
  if (warp == 13) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int nks_total = (2 * p.b + 15) / 16;   // 16-element (bf16) MMA K steps over 2b

  if (warp == 12) {
    // ---------------------------------------------------------------- raw producer (TMA)
    if (lane == 0) {
      const uint32_t xbytes = uint32_t(p.K) * CK * 8;
      int it = 0;
      for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
        const Tile4 ti = decode4(p, tile);
        const int row0 = ti.t * p.cols + ti.ct * TM;
        for (int kc = 0; kc < p.nkc; ++kc, ++it) {
          const int s = it % S_RAW;
          mbar_wait(&raw_empty[s], ((it / S_RAW) & 1) ^ 1);
          mbar_arrive_expect_tx(&raw_full[s], RAWY + xbytes);
          const int f0 = 2 * (ti.a + kc * CK);        // first float of the chunk in the row
          tma_load_2d(raw + s * RAW_STAGE, &tmy, f0, row0, &raw_full[s]);
          tma_load_2d(raw + s * RAW_STAGE + RAWY, &tmx, f0, ti.t * p.K, &raw_full[s]);
        }
      }
    }
  } else if (warp < 8) {
    // ---------------------------------------------------------------- transform
    const int jp = tid & 7;            // complex pair 2jp, 2jp+1 of the 16-complex chunk
    const int rb = tid >> 3;           // rows rb + 32 i, i < 4
    int it = 0;
    for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
      const Tile4 ti = decode4(p, tile);
      const int c_first = ti.ct * TM + rb;
      const int x_first = c_first % p.K;
      const int x_step = 32 % p.K;
      for (int kc = 0; kc < p.nkc; ++kc, ++it) {
        const int sr = it % S_RAW, sa = it % S_AB;
        mbar_wait(&raw_full[sr], (it / S_RAW) & 1);
        const float4 *ry = reinterpret_cast<const float4 *>(raw + sr * RAW_STAGE);
        float4 *rx = reinterpret_cast<float4 *>(raw + sr * RAW_STAGE + RAWY);
        // LS factors in place: f = conj(x) / |x|^2 for the K x 16 pilots of this chunk
        const int j0 = kc * CK + 2 * jp;                // window-relative complex index
        if (tid < p.K * 8) {
          const float4 xv = rx[tid];
          const float i0 = rcp_approx(xv.x * xv.x + xv.y * xv.y);
          const float i1 = rcp_approx(xv.z * xv.z + xv.w * xv.w);
          const bool ok0 = kc * CK + 2 * (tid & 7) < p.b, ok1 = kc * CK + 2 * (tid & 7) + 1 < p.b;
          rx[tid] = make_float4(ok0 ? xv.x * i0 : 0.f, ok0 ? -xv.y * i0 : 0.f, ok1 ? xv.z * i1 : 0.f,
                                ok1 ? -xv.w * i1 : 0.f);   // zero factor masks the K tail (j >= b)
        }
        named_bar_sync(1, NTR);
        mbar_wait(&ab_empty[sa], ((it / S_AB) & 1) ^ 1);
        uint8_t *ah = ab + sa * AB_STAGE;
        uint8_t *al = ah + A_PLANE;
        (void)j0;
        int xr = x_first;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = rb + 32 * i;
          const float4 yv = ry[r * 8 + jp];
          const float4 fv = rx[xr * 8 + jp];
          const float l0r = yv.x * fv.x - yv.y * fv.y, l0i = yv.x * fv.y + yv.y * fv.x;
          const float l1r = yv.z * fv.z - yv.w * fv.w, l1i = yv.z * fv.w + yv.w * fv.z;
          const uint32_t h0 = pack_bf16(l0r, l0i), h1 = pack_bf16(l1r, l1i);
          const uint32_t g0 = pack_bf16(l0r - bf16_lo_f(h0), l0i - bf16_hi_f(h0));
          const uint32_t g1 = pack_bf16(l1r - bf16_lo_f(h1), l1i - bf16_hi_f(h1));
          // SW64 K-major: row r at r*64 bytes, 16-byte chunk (jp>>1) ^ ((r>>1)&3), 8-byte half (jp&1)
          const int off = r * 64 + ((((jp >> 1) ^ ((r >> 1) & 3))) << 4) + ((jp & 1) << 3);
          *reinterpret_cast<uint2 *>(ah + off) = make_uint2(h0, h1);
          *reinterpret_cast<uint2 *>(al + off) = make_uint2(g0, g1);
          xr += x_step;
          if (xr >= p.K) xr -= p.K;
        }
        fence_proxy_async();
        mbar_arrive(&a_full[sa]);
        mbar_arrive(&raw_empty[sr]);
      }
    }
  } else if (warp < 12) {
    // ---------------------------------------------------------------- epilogue
    const int q = warp & 3;
    float *stage = epi + q * 32 * EPI_STRIDE;
    int lt = 0;
    for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++lt) {
      const Tile4 ti = decode4(p, tile);
      const int acc = lt & 1;
      mbar_wait(&tmem_full[acc], (lt >> 1) & 1);
      tc_fence_after();
      const int nf = 2 * ti.kept;
      const int ncb = (ti.off + nf + 31) / 32;
      const int row_base = ti.ct * TM + q * 32;
      const float qnan = __int_as_float(0x7fc00000);
      for (int cb = 0; cb < ncb; ++cb) {
        float v[32];
        tmem_ld32(tmem_base + uint32_t(acc * NMAXW + cb * 32) + (uint32_t(q * 32) << 16), v);
#pragma unroll
        for (int u = 0; u < 32; u += 2)
          *reinterpret_cast<float2 *>(stage + lane * EPI_STRIDE + u) = make_float2(v[u], v[u + 1]);
        __syncwarp();
        const int f = cb * 32 - ti.off + 2 * (lane & 15);
        const bool fok = f >= 0 && f < nf;
#pragma unroll 4
        for (int rr = 0; rr < 32; rr += 2) {
          const int r = rr + (lane >> 4);
          const int c = row_base + r;
          if (fok && c < p.cols) {
            float2 val = *reinterpret_cast<const float2 *>(stage + r * EPI_STRIDE + 2 * (lane & 15));
            if (!ti.set_ok) val = make_float2(qnan, qnan);
            p.h[(size_t(ti.t) * p.cols + c) * p.N + ti.o + (f >> 1)] = val;
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      mbar_arrive(&tmem_empty[acc]);
    }
  } else if (warp == 14) {
    // ---------------------------------------------------------------- B producer
    if (lane == 0) {
      int it = 0;
      for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
        const Tile4 ti = decode4(p, tile);
        const uint32_t bytes = uint32_t(ti.nw) * 64;
        for (int kc = 0; kc < p.nkc; ++kc, ++it) {
          const int s = it % S_AB;
          mbar_wait(&ab_empty[s], ((it / S_AB) & 1) ^ 1);
          mbar_arrive_expect_tx(&b_full[s], 2 * bytes);
          const size_t src = ((size_t(ti.set) * p.nkc + kc) * p.NR + ti.n0) * 32;   // bf16 elements
          uint8_t *bh = ab + s * AB_STAGE + 2 * A_PLANE;
          bulk_g2s(bh, p.bank_hi + src, bytes, &b_full[s]);
          bulk_g2s(bh + B_PLANE, p.bank_lo + src, bytes, &b_full[s]);
        }
      }
    }
  } else {
    // ---------------------------------------------------------------- MMA issuer (warp 13)
    if (lane == 0) {
      int it = 0, lt = 0;
      for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++lt) {
        const Tile4 ti = decode4(p, tile);
        const int acc = lt & 1;
        // F32 accumulate, BF16 A/B, K-major A/B, N = nw, M = 128
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(ti.nw >> 3) << 17) |
                               (uint32_t(TM >> 4) << 24);
        mbar_wait(&tmem_empty[acc], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + uint32_t(acc * NMAXW);
        for (int kc = 0; kc < p.nkc; ++kc, ++it) {
          const int s = it % S_AB;
          const uint32_t ph = (it / S_AB) & 1;
          mbar_wait(&a_full[s], ph);
          mbar_wait(&b_full[s], ph);
          tc_fence_after();
          uint8_t *st = ab + s * AB_STAGE;
          const uint64_t ah = sw64_desc(smem_u32(st));
          const uint64_t al = sw64_desc(smem_u32(st + A_PLANE));
          const uint64_t bh = sw64_desc(smem_u32(st + 2 * A_PLANE));
          const uint64_t bl = sw64_desc(smem_u32(st + 2 * A_PLANE + B_PLANE));
          const int nks = min(2, nks_total - 2 * kc);
          for (int ks = 0; ks < nks; ++ks) {
            const uint64_t adv = uint64_t(2 * ks);      // +32 bytes along K
            mma_bf16(d, ah + adv, bh + adv, idesc, (kc | ks) != 0);
            mma_bf16(d, ah + adv, bl + adv, idesc, 1u);
            mma_bf16(d, al + adv, bh + adv, idesc, 1u);
          }
          mma_commit(&ab_empty[s]);
        }
        mma_commit(&tmem_full[acc]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 13) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

// bank[set][kc][n][32] bf16 hi/lo planes of B_r^T[n][32 kc + kk] in the SW64 shared-memory image:
// row n at n*64 bytes, 16-byte chunk (kk/8) ^ ((n>>1)&3).
__global__ void k4_build_bank(const float2 *__restrict__ W, int b, int nkc, int NR, uint16_t *__restrict__ bank_hi,
                              uint16_t *__restrict__ bank_lo) {
  const int set = blockIdx.x, kc = blockIdx.y;
  const float2 *Ws = W + size_t(set) * b * b;
  uint16_t *bh = bank_hi + (size_t(set) * nkc + kc) * NR * 32;
  uint16_t *bl = bank_lo + (size_t(set) * nkc + kc) * NR * 32;
  for (int e = threadIdx.x; e < NR * 32; e += blockDim.x) {
    const int n = e / 32, kk = e % 32;
    const int k = kc * 32 + kk;
    const int i = n >> 1, jw = k >> 1;
    float v = 0.f;
    if (i < b && jw < b) {
      const float2 w = Ws[size_t(i) * b + jw];
      const int sel = ((n & 1) << 1) | (k & 1);
      v = sel == 0 ? w.x : sel == 1 ? -w.y : sel == 2 ? w.y : w.x;
    }
    const uint32_t hi2 = pack_bf16(v, 0.f);          // low half = bf16(v)
    const float hi = bf16_lo_f(hi2);
    const uint32_t lo2 = pack_bf16(v - hi, 0.f);
    const int dst = n * 32 + ((((kk >> 3) ^ ((n >> 1) & 3))) << 3) + (kk & 7);
    bh[dst] = uint16_t(hi2 & 0xFFFFu);
    bl[dst] = uint16_t(lo2 & 0xFFFFu);
  }
}

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

bool make_map(CUtensorMap *m, const void *ptr, int N, long long rows, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cuuint64_t(2) * N, cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(2) * N * 4};
  cuuint32_t box[2] = {cuuint32_t(2 * CK), cuuint32_t(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

void bf16x3_bank_shape(int32_t b, int32_t *nkc, int32_t *NR) {
  *nkc = (2 * b + 31) / 32;
  *NR = ((2 * b + 16) + 7) & ~7;
}

bool bf16x3_launchable(const ContractArgs &a) {
  const long long rows = (long long)a.T * a.M * a.K;
  // TMA box starts must be 16-byte aligned: even window starts, even N (row pitch), aligned bases.
  return a.even_starts && a.K <= KMAX && (a.N % 2) == 0 && (reinterpret_cast<uintptr_t>(a.y) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(a.x) & 15) == 0 && rows < (1LL << 31) && encode_fn() != nullptr;
}

cudaError_t launch_build_bank_bf16(const float2 *d_W, int32_t b, int32_t n_sets, uint16_t *bank_hi,
                                   uint16_t *bank_lo, cudaStream_t stream, int64_t *launches) {
  int32_t nkc, NR;
  bf16x3_bank_shape(b, &nkc, &NR);
  k4_build_bank<<<dim3(n_sets, nkc), 256, 0, stream>>>(d_W, b, nkc, NR, bank_hi, bank_lo);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) ++*launches;
  return e;
}

cudaError_t launch_contract_bf16x3(const ContractArgs &a, const uint16_t *bank_hi, const uint16_t *bank_lo,
                                   cudaStream_t stream, int64_t *launches) {
  if (!bf16x3_launchable(a)) return cudaErrorNotSupported;
  K4Params p;
  p.h = a.h;
  p.bank_hi = bank_hi;
  p.bank_lo = bank_lo;
  p.geo = a.geo;
  p.soi = a.soi;
  p.T = a.T;
  p.K = a.K;
  p.N = a.N;
  p.b = a.b;
  p.n_win = a.n_win;
  p.n_sets = a.n_sets;
  bf16x3_bank_shape(a.b, &p.nkc, &p.NR);
  p.cols = a.M * a.K;
  p.n_ct = (p.cols + TM - 1) / TM;
  const long long tiles = (long long)a.T * a.n_win * p.n_ct;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  p.n_tiles = int(tiles);
  CUtensorMap tmy, tmx;
  if (!make_map(&tmy, a.y, a.N, (long long)a.T * p.cols, TM) || !make_map(&tmx, a.x, a.N, (long long)a.T * a.K, a.K))
    return cudaErrorInvalidValue;
  static int num_sms = 0;
  if (num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  cudaError_t e = cudaFuncSetAttribute(k4_bf16x3, cudaFuncAttributeMaxDynamicSharedMemorySize, K4_SMEM);
  if (e != cudaSuccess) return e;
  const int grid = int(tiles < num_sms ? tiles : num_sms);
  k4_bf16x3<<<grid, K4_THREADS, K4_SMEM, stream>>>(tmy, tmx, p);
  e = cudaGetLastError();
  if (e == cudaSuccess) ++*launches;
  return e;
}

}  // namespace ce
