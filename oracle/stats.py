"""CPU oracle for the statistics that feed the filter build (NEXT-3).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain NumPy in complex128; shares no code with the
CUDA path.

The paper designs its weights offline from an ASSUMED path count L and SNR_fixed (PAPER.md:306,
423, 442) and runs its detector with a fixed sigma^2 "for the lack of SNR estimation module"
(PAPER.md:519); it studies the sensitivity to both (Fig. fig7 c/d).  This module
(a) estimates the statistics from the received pilots themselves and (b) evaluates, in closed form, the
MSE of a filter designed for one set of statistics and used on a channel with another (the robustness
sweep of Fig. fig7 c/d).

Estimators (readings D1-D3 in DESIGN.md), from the LS estimates H_LS = y / x (Eq. 9) of every column c
(antenna x user) of a statistic set:
  R_hat[d]  = sum_c sum_{n < N-d} H_LS[c, n+d] conj(H_LS[c, n]) / (C (N - d)),   d < D
              (= r[d] + sigma^2 delta[d] in expectation: the noise is white across tones)
  sigma2_hat = mean over c and over the delay bins kappa in the noise window of |IDFT_N(H_LS[c])[kappa]|^2
              with the unitary N-point IDFT; the window is the B bins centred on N/2, far from the channel's
              delay support at the start (and wrap-around end) of the N-bin delay axis.
  r_hat[d]  = R_hat[d] - sigma2_hat delta[d]
"""
from __future__ import annotations

import numpy as np

from .lmmse import lmmse_filter, toeplitz_hermitian


def ls_rows(y, x):
    """H_LS [C][N] complex128 of every (t, m, k) column: y [T][M][K][N] / x [T][K][N]."""
    y = np.asarray(y).astype(np.complex128)
    x = np.asarray(x).astype(np.complex128)
    return (y / x[:, None, :, :]).reshape(-1, y.shape[-1])


def correlation_estimate(H: np.ndarray, D: int) -> np.ndarray:
    """R_hat[d], d < D, averaged over rows and over the N - d tone pairs of each row."""
    H = np.asarray(H, np.complex128)
    C, N = H.shape
    out = np.empty(D, np.complex128)
    for d in range(D):
        out[d] = np.sum(H[:, d:] * np.conj(H[:, :N - d])) / (C * (N - d))
    return out


def noise_bins(N: int, B: int):
    """The B delay bins centred on N/2 (the noise window)."""
    lo = N // 2 - B // 2
    return np.arange(lo, lo + B)


def noise_variance_estimate(H: np.ndarray, B: int) -> float:
    """Mean power of the unitary N-point IDFT of every LS row over the noise window."""
    H = np.asarray(H, np.complex128)
    N = H.shape[1]
    h = np.fft.ifft(H, axis=1) * np.sqrt(N)          # unitary: white noise keeps its per-bin variance
    return float(np.mean(np.abs(h[:, noise_bins(N, B)]) ** 2))


def estimate_stats(y, x, D: int, B: int):
    """(r_hat [D] complex128, sigma2_hat float) from one statistic set's instances."""
    H = ls_rows(y, x)
    s2 = noise_variance_estimate(H, B)
    r = correlation_estimate(H, D)
    r[0] -= s2
    return r, s2


def mismatched_block_mse(r_true, sigma2_true: float, r_design, sigma2_design: float, b: int) -> float:
    """Per-tone MSE of the b x b block filter designed for (r_design, sigma2_design) applied to a channel
    with (r_true, sigma2_true):  tr[(I - W) R (I - W)^H + sigma2 W W^H] / b,  W = lmmse_filter(R_d, s2_d)."""
    R = toeplitz_hermitian(r_true, b)
    W = lmmse_filter(toeplitz_hermitian(r_design, b), sigma2_design)
    E = np.eye(b) - W
    return float(np.real(np.trace(E @ R @ E.conj().T + sigma2_true * W @ W.conj().T))) / b
