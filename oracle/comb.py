"""CPU oracle for the paper's comb-pilot grouped LMMSE estimators (3W-LMMSE, 12W-LMMSE) -- NEXT-1.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain NumPy/LAPACK in complex128; shares no
code with the CUDA path.

Paper (line numbers in /root/reference/PAPER.md):
  * comb pilots: UE s (1-based) owns tones s, s+S, s+2S, ... (Fig. fig1; Eq. 6, 102)
  * LS at its pilots, Eq. 9
  * per-group weights W = R_{H,H_LS} (R_{H_LS,H_LS} + sigma^2/sigma_s^2 I)^-1, Eq. 17,
    with R built from r_d (Eq. eqrd): element (k_a, k_b) = r[k_a - k_b]
  * 3W-LMMSE (Table I): K groups, each 3 outputs spaced S/3 apart starting at the UE's
    pilot tone, from 3 consecutive pilots; W(1), W(2), W(3) shared by all UEs (Eq. W1-W3, P)
  * 12W-LMMSE (Table II): K groups of S consecutive output tones from 12 consecutive
    pilots; 12 weight matrices per UE (W_s^(1..12))
  * zero-order hold for the tones 3W does not estimate: "the following subcarrier blanks are padded with
    the last channel estimation value"

Index conventions (0-based; readings C1-C4 in DESIGN.md):
  UE s in [0, S) owns tones S*j + s, j in [0, K), K = N / S (N % S == 0, reading C1).
  Group g in [0, K) uses pilot window [a_g, a_g + G) from the window rule of the main path applied to
  pilot positions, window_table(K, G, 1) (pinned against Tables I-II in tests/test_geometry.py); its
  weight type is g - a_g (Table I/II "W" column minus 1).
  Output tones of group g for UE s:
    mode "full" (12W): S*g + q, q in [0, S)                        (every tone; Table II)
    mode "sub"  (3W):  S*g + s + (S/G)*q, q in [0, G), S % G == 0  (Table I: 1,5,9 / 13,17,21 ...)
  ZOH (sub mode): tone k takes the estimate of the last estimated tone <= k; tones before the UE's
  first pilot take the first estimate (reading C3).
"""
from __future__ import annotations

import numpy as np

from .lmmse import window_table


def comb_geometry(N: int, S: int, G: int):
    """(K, windows): K = N/S pilots per UE, windows = [(a_g, type_g)] for g in [0, K)."""
    if N % S:
        raise ValueError("N must be a multiple of S (reading C1)")
    K = N // S
    if not 1 <= G <= K:
        raise ValueError("need 1 <= G <= K")
    wins = []
    for a, o, o_next in window_table(K, G, 1):
        for g in range(o, o_next):
            wins.append((a, g - a))
    return K, wins


def comb_out_tones(g: int, s: int, S: int, G: int, mode: str, N: int):
    if mode == "full":
        return [S * g + q for q in range(S) if S * g + q < N]
    if S % G:
        raise ValueError("sub mode needs S % G == 0")
    return [S * g + s + (S // G) * q for q in range(G)]


def rect_filter(r: np.ndarray, sigma2: float, out_tones, in_tones) -> np.ndarray:
    """W = R[out, in] (R[in, in] + sigma2 I)^-1, R[p, q] = r[p - q] (conj for p < q), Eq. 17."""
    r = np.asarray(r, np.complex128)

    def R(p, q):
        d = np.subtract.outer(np.asarray(p), np.asarray(q))
        return np.where(d >= 0, r[np.abs(d)], np.conj(r[np.abs(d)]))

    A = R(in_tones, in_tones) + sigma2 * np.eye(len(in_tones))
    C = R(out_tones, in_tones)
    # W A = C  <=>  A^H W^H = C^H (LU solve, not Cholesky)
    return np.linalg.solve(A.conj().T, C.conj().T).conj().T


def comb_filters(r: np.ndarray, sigma2: float, N: int, S: int, G: int, mode: str, n_ue: int):
    """{(s, type): W} for every UE s < n_ue and window type (12 per UE for 12W; 3W's are UE-independent)."""
    K, wins = comb_geometry(N, S, G)
    out = {}
    for g, (a, typ) in enumerate(wins):
        for s in range(n_ue):
            if (s, typ) in out:
                continue
            ins = [S * (a + j) + s for j in range(G)]
            out[(s, typ)] = rect_filter(r, sigma2, comb_out_tones(g, s, S, G, mode, N), ins)
    return out


def comb_ls(y: np.ndarray, x: np.ndarray, S: int, s: int) -> np.ndarray:
    """LS at UE s's pilots, Eq. 9: y[..., S j + s] / x[..., S j + s] (true division)."""
    y = np.asarray(y).astype(np.complex128)
    x = np.asarray(x).astype(np.complex128)
    return y[..., s::S] / x[..., s::S]


def zoh_fill(est: dict, N: int) -> np.ndarray:
    """Zero-order hold over tones: est = {tone: value[...]} -> [..., N]."""
    tones = sorted(est)
    first = est[tones[0]]
    out = np.empty(first.shape + (N,), np.complex128)
    cur = first
    ti = 0
    for k in range(N):
        while ti < len(tones) and tones[ti] <= k:
            cur = est[tones[ti]]
            ti += 1
        out[..., k] = cur
    return out


def comb_estimate(y, x, r, sigma2, N: int, S: int, G: int, mode: str, n_ue: int) -> np.ndarray:
    """Grouped comb LMMSE for every UE s < n_ue.

    y: [T][M][N] received pilot symbol (all UEs on their combs), x: [T][N] comb pilot symbol
    (tone k carries UE k % S's pilot).  Returns complex128 [T][M][n_ue][N].
    """
    y = np.asarray(y)
    T, M, _ = y.shape
    K, wins = comb_geometry(N, S, G)
    filt = comb_filters(r, sigma2, N, S, G, mode, n_ue)
    out = np.empty((T, M, n_ue, N), np.complex128)
    for s in range(n_ue):
        ls = comb_ls(y, x[:, None, :], S, s)                    # [T][M][K]
        est = {}
        for g, (a, typ) in enumerate(wins):
            W = filt[(s, typ)]
            vals = ls[..., a:a + G] @ W.T                        # [T][M][n_out]
            for q, k in enumerate(comb_out_tones(g, s, S, G, mode, N)):
                est[k] = vals[..., q]
        if mode == "full":
            for k in range(N):
                out[:, :, s, k] = est[k]
        else:
            out[:, :, s, :] = zoh_fill(est, N)
    return out


def comb_full_lmmse(y, x, r, sigma2, N: int, S: int, n_ue: int) -> np.ndarray:
    """Un-windowed comb LMMSE: every tone from ALL K pilots of the UE (Eq. 12-15 with the comb
    R_{H,H_LS}); the reference the grouped estimators approximate."""
    y = np.asarray(y)
    T, M, _ = y.shape
    K = N // S
    out = np.empty((T, M, n_ue, N), np.complex128)
    for s in range(n_ue):
        ins = [S * j + s for j in range(K)]
        W = rect_filter(r, sigma2, list(range(N)), ins)
        out[:, :, s, :] = comb_ls(y, x[:, None, :], S, s) @ W.T
    return out


def comb_mse_per_tone(r, sigma2, N: int, S: int, G: int, mode: str, s: int) -> np.ndarray:
    """Closed-form MSE per tone of the grouped estimator for UE s (before ZOH for 'sub' tones that are
    not estimated: those get the hold error E|H_k - Hhat_e|^2, also closed form)."""
    r = np.asarray(r, np.complex128)

    def R(p, q):
        d = np.subtract.outer(np.asarray(p), np.asarray(q))
        return np.where(d >= 0, r[np.abs(d)], np.conj(r[np.abs(d)]))

    K, wins = comb_geometry(N, S, G)
    mse = np.full(N, np.nan)
    coef = {}
    for g, (a, typ) in enumerate(wins):
        ins = [S * (a + j) + s for j in range(G)]
        outs = comb_out_tones(g, s, S, G, mode, N)
        W = rect_filter(r, sigma2, outs, ins)
        for q, k in enumerate(outs):
            coef[k] = (ins, W[q])
    for k in range(N):
        e = k if mode == "full" else max([t for t in coef if t <= k], default=min(coef))
        ins, w = coef[e]
        # Hhat = w . (H_in + n), error H_k - Hhat
        Rkk = r[0].real
        Rki = R([k], ins)[0]
        Rii = R(ins, ins) + sigma2 * np.eye(len(ins))
        # Hhat = w . LS, E{H_k conj(Hhat)} = conj(w) . R[k, in], E|Hhat|^2 = w (R_ii + s2 I) conj(w)
        mse[k] = Rkk - 2 * np.real(np.conj(w) @ Rki) + np.real(w @ Rii @ np.conj(w))
    return mse
