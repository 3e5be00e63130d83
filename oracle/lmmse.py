"""CPU oracle for the block-LMMSE pilot channel estimator of arXiv 1802.05427.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  It shares no code with the CUDA path (``paper_1802_05427_b200``):
window geometry, Toeplitz expansion, LS and the filter are all re-derived here,
with an LU ``solve`` of the window system (the GPU inverts the Toeplitz matrix by
Levinson-Durbin + Gohberg-Semencul/Trench; the paper's own solver is ``cposv``).

Everything is plain NumPy/LAPACK in complex128.  Each function cites the
passage of PAPER.md it follows (line numbers in /root/reference/PAPER.md) and,
where the paper is silent, the reading of SURVEY.md §8(c) adopted in DESIGN.md.

Pinning status: every function below is pinned by a
``-m "not gpu"`` test in tests/test_oracle_pins.py or tests/test_geometry.py;
none is "parity unpinned".
"""
from __future__ import annotations

import numpy as np


# --------------------------------------------------------------------------------------
# a1: window geometry (reading A7; generalises the edge clamping of PAPER.md Tables I-II,
#     lines 203-260, and the overlapping partition credited to [5])
# --------------------------------------------------------------------------------------
def window_table(N: int, b: int, s: int):
    """List of windows (a_w, o_w, o_next) over tones 0..N-1.

    Window w reads LS tones [a_w, a_w + b) and keeps outputs [o_w, o_next).
    Windows start on the stride grid w*s, the last one clamped to N-b
    (groups 95-100 of 12W reuse the last input group).
    Kept outputs are the centre s tones, m_l = floor((b-s)/2) tones from the
    window start; the first window also keeps [0, m_l) and the last keeps
    everything up to N, so the kept ranges partition [0, N).
    """
    if not (1 <= b <= N and 1 <= s <= b):
        raise ValueError("need 1 <= b <= N and 1 <= s <= b")
    n_win = -(-(N - b) // s) + 1          # ceil((N-b)/s) + 1
    m_l = (b - s) // 2
    out = []
    for w in range(n_win):
        a = min(w * s, N - b)
        o = 0 if w == 0 else w * s + m_l
        o_next = N if w == n_win - 1 else (w + 1) * s + m_l
        out.append((a, o, o_next))
    return out


# --------------------------------------------------------------------------------------
# R_hh (each element "only depends on the difference between k_a and k_b")
# --------------------------------------------------------------------------------------
def toeplitz_hermitian(r: np.ndarray, n: int) -> np.ndarray:
    """R[p, q] = r[p-q] for p >= q and conj(r[q-p]) otherwise (n x n, complex128)."""
    r = np.asarray(r, np.complex128)
    p = np.arange(n)[:, None]
    q = np.arange(n)[None, :]
    d = p - q
    return np.where(d >= 0, r[np.abs(d)], np.conj(r[np.abs(d)]))


def rd_uniform(L: float, N: float, d) -> np.ndarray:
    """Closed-form subcarrier correlation, PAPER.md:288-305 (Eq. ``eqrd``).

    r_d = 1 for d = 0, else (1 - exp(-j 2 pi L d / N)) / (j 2 pi L d / N).
    (Reading A5: N here is the normalising FFT length of the delay grid.)
    """
    d = np.atleast_1d(np.asarray(d, np.float64))
    out = np.ones(d.shape, np.complex128)
    nz = d != 0
    z = 2j * np.pi * L * d[nz] / N
    out[nz] = (1.0 - np.exp(-z)) / z
    return out


# --------------------------------------------------------------------------------------
# a3: LS at the pilots, PAPER.md:173-180 (Eq. 8-9): H_LS = Y / X, true complex division
# --------------------------------------------------------------------------------------
def ls_estimate(y: np.ndarray, x: np.ndarray) -> np.ndarray:
    """y [T][M][K][N], x [T][K][N] (pilot shared by all antennas) -> H_LS complex128."""
    y = np.asarray(y).astype(np.complex128)
    x = np.asarray(x).astype(np.complex128)
    return y / x[:, None, :, :]


# --------------------------------------------------------------------------------------
# a2: filter, PAPER.md:306-309 (Eq. 17) on a b x b block of R_hh (square case, reading A2)
# --------------------------------------------------------------------------------------
def lmmse_filter(R: np.ndarray, sigma2: float) -> np.ndarray:
    """W = R (R + sigma2 I)^-1 (Eq. 13/17 with R_HH_LS = R_HH for full-tone pilots).

    Computed as W = solve((R + sigma2 I)^H, R^H)^H (LU, not Cholesky).
    """
    R = np.asarray(R, np.complex128)
    A = R + sigma2 * np.eye(R.shape[0])
    return np.linalg.solve(A.conj().T, R.conj().T).conj().T


def block_filter(r: np.ndarray, sigma2: float, b: int) -> np.ndarray:
    """W_b for one statistic set: the b x b leading block of Toeplitz R_hh.

    Every window's R_w = R[a:a+b, a:a+b] equals this block because R is Toeplitz
    (equal tone differences give the same correlation matrix).
    """
    return lmmse_filter(toeplitz_hermitian(r, b), sigma2)


# --------------------------------------------------------------------------------------
# a4/a5: block application, PAPER.md:186-190 (Eq. 12) per window
# --------------------------------------------------------------------------------------
def block_apply(H_ls_t: np.ndarray, filters, b: int, s: int) -> np.ndarray:
    """Apply per-window filters to one instance's LS estimates H_ls_t [..., N].

    For every window (a, o, o_next) of window_table(N, b, s):
        out[..., o:o_next] = W_w[o-a : o_next-a, :] @ H_ls_t[..., a:a+b]
    i.e. output tone o + i is sum_j W_w[o-a+i, j] * H_LS[a+j] (Eq. 12 on the block).
    """
    N = H_ls_t.shape[-1]
    out = np.empty(H_ls_t.shape, np.complex128)
    for (a, o, o_next), W in zip(window_table(N, b, s), filters):
        out[..., o:o_next] = H_ls_t[..., a:a + b] @ W[o - a:o_next - a, :].T
    return out


def block_lmmse_general(H_ls_t: np.ndarray, R: np.ndarray, sigma2: float, b: int, s: int):
    """Block LMMSE for an arbitrary N x N correlation R (the definition):
    W_w = R_w (R_w + sigma2 I)^-1 with R_w = R[a:a+b, a:a+b] for each window."""
    N = R.shape[0]
    filters = [lmmse_filter(R[a:a + b, a:a + b], sigma2) for (a, _, _) in window_table(N, b, s)]
    return block_apply(H_ls_t, filters, b, s)


def block_lmmse(y, x, r_sets, sigma2_sets, set_of_instance, b: int, s: int,
                toeplitz_shortcut: bool = True) -> np.ndarray:
    """Block / overlapping-window LMMSE estimate, complex128 [T][M][K][N].

    H_LS = y / x (Eq. 9), then block_apply with the set's filters.  With Toeplitz
    R_hh every window's R_w is the same leading b x b block, so one W_b serves all
    windows (``toeplitz_shortcut``); without it each W_w is rebuilt from its own
    slice of the full N x N R_hh (a pin checks the two agree).
    """
    H_ls = ls_estimate(y, x)
    T, M, K, N = H_ls.shape
    out = np.empty_like(H_ls)
    n_win = len(window_table(N, b, s))
    cache = {}
    for t in range(T):
        st = int(set_of_instance[t]) if set_of_instance is not None else 0
        if st not in cache:
            if toeplitz_shortcut:
                cache[st] = [block_filter(r_sets[st], float(sigma2_sets[st]), b)] * n_win
            else:
                R = toeplitz_hermitian(r_sets[st], N)
                cache[st] = [lmmse_filter(R[a:a + b, a:a + b], float(sigma2_sets[st]))
                             for (a, _, _) in window_table(N, b, s)]
        out[t] = block_apply(H_ls[t], cache[st], b, s)
    return out


def full_lmmse_general(H_ls_t: np.ndarray, R: np.ndarray, sigma2: float) -> np.ndarray:
    """Full LMMSE for one instance with an arbitrary N x N R (Eq. 12-13)."""
    return H_ls_t @ lmmse_filter(R, sigma2).T


def full_lmmse(y, x, r_sets, sigma2_sets, set_of_instance) -> np.ndarray:
    """Full N x N LMMSE, PAPER.md:186-200 (Eq. 12-15): W = R_hh (R_hh + sigma2 I)^-1."""
    H_ls = ls_estimate(y, x)
    T = H_ls.shape[0]
    N = H_ls.shape[-1]
    out = np.empty_like(H_ls)
    cache = {}
    for t in range(T):
        st = int(set_of_instance[t]) if set_of_instance is not None else 0
        if st not in cache:
            cache[st] = lmmse_filter(toeplitz_hermitian(r_sets[st], N), float(sigma2_sets[st]))
        out[t] = H_ls[t] @ cache[st].T
    return out


# --------------------------------------------------------------------------------------
# closed-form error covariance (north_star: per-block MSE = tr(R_b - R_b (R_b+s2 I)^-1 R_b)/b)
# --------------------------------------------------------------------------------------
def error_cov(R: np.ndarray, sigma2: float) -> np.ndarray:
    """E = R - R (R + sigma2 I)^-1 R  (LMMSE error covariance for H_LS = H + noise)."""
    R = np.asarray(R, np.complex128)
    A = R + sigma2 * np.eye(R.shape[0])
    return R - R @ np.linalg.solve(A, R)


def block_mse_per_tone(r: np.ndarray, sigma2: float, N: int, b: int, s: int) -> np.ndarray:
    """Per-tone MSE of the block estimator: diag(E_w) on each window's kept rows."""
    E = np.real(np.diag(error_cov(toeplitz_hermitian(r, b), sigma2)))
    mse = np.empty(N, np.float64)
    for a, o, o_next in window_table(N, b, s):
        mse[o:o_next] = E[o - a:o_next - a]
    return mse


def block_mse(r: np.ndarray, sigma2: float, b: int) -> float:
    """Per-block MSE tr(E_b)/b (north_star closed form, non-overlapping blocks)."""
    return float(np.real(np.trace(error_cov(toeplitz_hermitian(r, b), sigma2)))) / b


def full_mse_per_tone(r: np.ndarray, sigma2: float, N: int) -> np.ndarray:
    return np.real(np.diag(error_cov(toeplitz_hermitian(r, N), sigma2)))


# --------------------------------------------------------------------------------------
# parity metric (SURVEY.md §8(c) "GPU vs oracle")
# --------------------------------------------------------------------------------------
def rel_fro_error_per_instance(h_test: np.ndarray, h_ref: np.ndarray) -> np.ndarray:
    """||h_test[t] - h_ref[t]||_F / ||h_ref[t]||_F for every instance t."""
    d = (np.asarray(h_test).astype(np.complex128) - h_ref).reshape(h_ref.shape[0], -1)
    n = np.asarray(h_ref).reshape(h_ref.shape[0], -1)
    return np.linalg.norm(d, axis=1) / np.linalg.norm(n, axis=1)
