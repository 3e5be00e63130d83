"""Writes single-change variants of K4's source (csrc/k4_block_lmmse_bf16x3.cu) into tools/ab_variants/ for
tools/ab_bisect.sh: which source change moves the kernel out of its fast code-generation state (DESIGN.md section 6,
"How the tile loop is written")?  Each variant is K4's file with one textual edit; nothing here is built into libce.

v1_template   the kernel wrapped in template <bool PAIR> (instantiated for false)
v2_gfirst     first tile index / tile stride held in registers from the kernel top (g_first, g_step)
v3_decode     a K4Params::pair field and the pair branch in the tile decode
v4_bars       six raw-ring barrier slots and b_peer slots
v6_gridparam  the grid size from the kernel parameters instead of gridDim.x
v8_gfirst_param  v2 with the stride from the kernel parameters
v9_sraw       p.s_raw re-read at each use
v10_nks       the MMA K-step count computed inside the MMA role instead of at the kernel top
v12_srstep    the transform's raw-ring slot and phase stepped instead of divided out of the chunk counter
v13_prodstep  the same in the raw producer (two integer divisions less before the first TMA issue)
"""
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_1802_05427_b200", "csrc", "k4_block_lmmse_bf16x3.cu")
OUT = os.path.join(ROOT, "tools", "ab_variants")


def must(s, a, b, cnt=1):
    assert s.count(a) == cnt, (a[:60], s.count(a))
    return s.replace(a, b)


def main():
    base = open(SRC).read()
    os.makedirs(OUT, exist_ok=True)
    launch = "  e = cudaLaunchKernelEx(&cfg, k4_bf16x3, tmy, tmx, tmh, p);"
    ntiles = "  int n_tiles;               // T * n_win * n_ct\n"
    v = {}
    s = must(base, "__global__ void __launch_bounds__(K4_THREADS, 1)\n    k4_bf16x3(",
             "template <bool PAIR>\n__global__ void __launch_bounds__(K4_THREADS, 1)\n    k4_bf16x3(")
    s = must(s, "cudaFuncSetAttribute(k4_bf16x3,", "cudaFuncSetAttribute(k4_bf16x3<false>,")
    v["v1_template"] = must(s, "cudaLaunchKernelEx(&cfg, k4_bf16x3,", "cudaLaunchKernelEx(&cfg, k4_bf16x3<false>,")

    top = ("  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;\n#ifdef CE_K4_TRACE\n"
           "  if (tid == 0 && g_k4_trace) {\n    unsigned long long gt;")
    s = must(base, top, top.replace("lane = tid & 31;\n", "lane = tid & 31;\n  const int g_first = int(blockIdx.x), "
                                                          "g_step = int(gridDim.x);\n", 1))
    s = s.replace("for (int g = blockIdx.x; g < p.n_tiles; g += gridDim.x", "for (int g = g_first; g < p.n_tiles; g += g_step")
    s = s.replace("g == int(blockIdx.x)", "g == g_first")
    s = must(s, "if (int(blockIdx.x) < p.n_tiles) ti0 = decode4(p, blockIdx.x);",
             "if (g_first < p.n_tiles) ti0 = decode4(p, g_first);")
    v["v2_gfirst"] = must(s, "g + int(gridDim.x) >= p.n_tiles", "g + g_step >= p.n_tiles")

    s = must(base, ntiles, ntiles + "  int pair;\n")
    s = must(s, "__device__ __forceinline__ Tile4 decode4(const K4Params &p, int g) {",
             "__device__ __forceinline__ Tile4 decode4(const K4Params &p, int g, int rank = 0) {")
    s = must(s, "  ti.ct = g % p.n_ct;", "  ti.ct = p.pair ? 2 * (g % p.n_ct) + rank : g % p.n_ct;")
    v["v3_decode"] = must(s, "  p.n_ct = (p.cols + TM - 1) / TM;\n", "  p.n_ct = (p.cols + TM - 1) / TM;\n  p.pair = 0;\n")

    s = must(base, "constexpr int BAR_BYTES = 256;", "constexpr int BAR_BYTES = 320;\nconstexpr int S_RAW_BARS = 6;")
    s = must(s, "  uint64_t *raw_empty = bars + S_RAW_MAX;               // [S_RAW_MAX]\n"
                "  uint64_t *a_full = bars + 2 * S_RAW_MAX;",
             "  uint64_t *raw_empty = bars + S_RAW_BARS;\n  uint64_t *a_full = bars + 2 * S_RAW_BARS;")
    s = must(s, "  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_empty + 2);",
             "  uint64_t *b_peer = tmem_empty + 2;\n  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(b_peer + S_AB);")
    s = must(s, "    for (int s = 0; s < S_RAW_MAX; ++s) {\n      mbar_init(&raw_full[s], 1);",
             "    for (int s = 0; s < S_RAW_BARS; ++s) {\n      mbar_init(&raw_full[s], 1);")
    v["v4_bars"] = must(s, "      mbar_init(&st_empty[s], 1);\n", "      mbar_init(&st_empty[s], 1);\n      mbar_init(&b_peer[s], 1);\n")

    s = must(base, ntiles, ntiles + "  int grid;\n")
    s = s.replace("int(gridDim.x)", "p.grid").replace("gridDim.x", "p.grid")
    s = s.replace("cfg.p.grid", "cfg.gridDim.x")
    v["v6_gridparam"] = must(s, launch, "  p.grid = int(cfg.gridDim.x);\n" + launch)

    s = must(v["v2_gfirst"], ntiles, ntiles + "  int grid;\n")
    s = must(s, "g_step = int(gridDim.x);", "g_step = p.grid;")
    v["v8_gfirst_param"] = must(s, launch, "  p.grid = int(cfg.gridDim.x);\n" + launch)

    v["v9_sraw"] = must(base, "  const int S_RAW = p.s_raw;\n", "#define S_RAW p.s_raw\n")

    nks = "  const int nks_total = (2 * p.b + 15) / 16;   // 16-element (bf16) MMA K steps over 2b\n"
    s = must(base, nks, "")
    v["v10_nks"] = must(s, "    if (lane == 0) {\n      int it = 0, lt = 0;\n",
                        "    if (lane == 0) {\n    " + nks + "      int it = 0, lt = 0;\n")

    s = must(base, "    int it = 0;\n    for (int g = blockIdx.x; g < p.n_tiles; g += gridDim.x) {\n"
                   "      const Tile4 ti = decode4(p, g);\n      const int c_first = ti.ct * TM + rb;",
             "    int it = 0, sr = 0;\n    uint32_t phr = 0;\n    for (int g = blockIdx.x; g < p.n_tiles; g += gridDim.x) {\n"
             "      const Tile4 ti = decode4(p, g);\n      const int c_first = ti.ct * TM + rb;")
    s = must(s, "        const int sr = it % S_RAW, sa = it % S_AB;\n        mbar_wait(&raw_full[sr], (it / S_RAW) & 1);",
             "        const int sa = it % S_AB;\n        mbar_wait(&raw_full[sr], phr);")
    v["v12_srstep"] = must(s, "        if (tid == 0 && it < 24) K4TR(56 + it);\n        mbar_arrive(&a_full[sa]);\n      }",
                           "        if (tid == 0 && it < 24) K4TR(56 + it);\n        mbar_arrive(&a_full[sa]);\n"
                           "        if (++sr == S_RAW) {\n          sr = 0;\n          phr ^= 1u;\n        }\n      }")
    s = must(base, "      const uint32_t xbytes = uint32_t(xbytes0);\n      int it = 0;\n",
             "      const uint32_t xbytes = uint32_t(xbytes0);\n      int it = 0, s = 0;\n      uint32_t phe = 1;\n")
    s = must(s, "          const int s = it % S_RAW;\n          mbar_wait(&raw_empty[s], ((it / S_RAW) & 1) ^ 1);\n#ifdef CE_K4_TRACE\n          if (it == 0) c_w0",
             "          mbar_wait(&raw_empty[s], phe);\n#ifdef CE_K4_TRACE\n          if (it == 0) c_w0")
    v["v13_prodstep"] = must(s, "            tma_load_2d(raw + s * RAW_STAGE + RAWY, &tmx, f0, ti.t * K0, &raw_full[s]);\n        }",
                             "            tma_load_2d(raw + s * RAW_STAGE + RAWY, &tmx, f0, ti.t * K0, &raw_full[s]);\n"
                             "          if (++s == S_RAW) {\n            s = 0;\n            phe ^= 1u;\n          }\n        }")
    for name, text in v.items():
        with open(os.path.join(OUT, name + ".cu"), "w") as f:
            f.write(text)
    print("wrote", ", ".join(sorted(v)), "to", OUT)


if __name__ == "__main__":
    main()
