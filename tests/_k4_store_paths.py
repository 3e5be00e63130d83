"""Run by tests/test_gpu_parity.py::test_k4_store_paths and ::test_k4_pair_paths in a subprocess (CE_K4_TMA_STORE
and CE_K4_PAIR are read once per process): K4 (CE_KERNEL_BF16X3) against the oracle on shapes that mix the epilogue's TMA-store column blocks
(interior, 16-byte aligned, full 32-row warp groups) with its direct-store blocks (window edges, odd output
starts, ragged column tiles, tails).  Exit status 0 = every instance within 1e-4."""
import sys

import numpy as np
import torch

import oracle
import paper_1802_05427_b200 as ce

SHAPES = [  # N, b, s, M, K, T
    (1200, 100, 100, 128, 12, 1),   # config-3 geometry: 6 staged blocks + an 8-float direct tail per window
    (3276, 126, 126, 8, 24, 2),     # config-5 geometry, ragged second column tile (192 columns)
    (300, 50, 24, 16, 16, 3),       # overlapping windows: off = 2, odd output starts
    (130, 64, 64, 5, 7, 2),         # 35 columns: no warp group is complete -> direct stores only
    (512, 96, 64, 32, 8, 2),        # 256 columns = two full tiles, clamped last window
    (1200, 100, 100, 32, 12, 2),    # 384 columns = three tiles: in pair mode the last pair's second CTA has no tile
]


def main():
    bad = 0
    for N, b, s, M, K, T in SHAPES:
        rng = np.random.default_rng(N + 3 * b + M)
        L = 6
        p = np.exp(-np.arange(L) / 2.5)
        p /= p.sum()
        tau = np.array([0.0, 0.7, 1.9, 3.2, 5.5, 7.0])
        d = np.arange(N)
        r = (p[None] * np.exp(-2j * np.pi * np.outer(d, tau) / (2 * N))).sum(1)[None]
        s2 = np.array([0.03])
        y = (rng.standard_normal((T, M, K, N)) + 1j * rng.standard_normal((T, M, K, N))).astype(np.complex64)
        x = np.exp(2j * np.pi * rng.random((T, K, N))).astype(np.complex64)
        est = ce.ChannelEstimator(N, b, s, r, s2)
        ce.ce_set_kernel(est.handle, ce.CE_KERNEL_BF16X3)
        est.build()
        h = est.estimate(torch.from_numpy(y).cuda(), torch.from_numpy(x).cuda())
        torch.cuda.synchronize()
        got = h.cpu().numpy()
        est.close()
        ref = oracle.block_lmmse(y, x, r, s2, None, b, s)
        err = oracle.rel_fro_error_per_instance(got, ref)
        ok = bool(np.all(err <= 1e-4)) and bool(np.isfinite(got).all())
        print(f"N={N} b={b} s={s} M={M} K={K} T={T}: max rel err {err.max():.2e} {'ok' if ok else 'FAIL'}")
        bad += not ok
        if T >= 2:
            # an out-of-range statistic set makes that instance NaN through either store path; the others exact
            est = ce.ChannelEstimator(N, b, s, r, s2)
            ce.ce_set_kernel(est.handle, ce.CE_KERNEL_BF16X3)
            est.build()
            soi = torch.tensor([0] + [7] * (T - 1), dtype=torch.int32, device="cuda")
            hb = est.estimate(torch.from_numpy(y).cuda(), torch.from_numpy(x).cuda(), set_of_instance=soi)
            torch.cuda.synchronize()
            hb = hb.cpu().numpy()
            est.close()
            ok2 = bool(np.isnan(hb[1:]).all()) and bool(np.all(oracle.rel_fro_error_per_instance(hb[:1], ref[:1]) <= 1e-4))
            print(f"  bad set index on instances 1..{T - 1}: {'ok' if ok2 else 'FAIL'}")
            bad += not ok2
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
