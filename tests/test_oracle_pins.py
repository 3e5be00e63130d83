"""Pins for the CPU oracle (oracle/lmmse.py) against what the paper and mathematics fix.

None of these re-types the oracle's own formula: each check reaches the same
quantity by a different route (quadrature, eigendecomposition, Monte Carlo over
the signal model, special cases with textbook answers, structural identities).
Chosen so that a dropped term, a wrong sign/index, a transposed or conjugated
operand in the oracle fails at least one of them.
"""
import dataclasses

import numpy as np
import pytest
from scipy import integrate, linalg

import oracle
import workload
from workload import CONFIGS


def _rand_psd(rng, n, rank=None):
    rank = n if rank is None else rank
    G = rng.standard_normal((n, rank)) + 1j * rng.standard_normal((n, rank))
    return G @ G.conj().T / rank


# ------------------------------------------------------------------ r_d
@pytest.mark.parametrize("L,N", [(8, 1200), (7, 2048), (3.5, 128)])
def test_rd_equals_uniform_delay_expectation(L, N):
    """Eq. eqrd is E{exp(-j 2 pi d tau / N)} for tau ~ U[0, L):
    evaluate the expectation by numerical quadrature."""
    for d in [-37, -5, -1, 0, 1, 2, 11, 100, 600]:
        re = integrate.quad(lambda tau: np.cos(2 * np.pi * d * tau / N), 0, L)[0] / L
        im = integrate.quad(lambda tau: -np.sin(2 * np.pi * d * tau / N), 0, L)[0] / L
        assert abs(oracle.rd_uniform(L, N, d)[0] - (re + 1j * im)) < 1e-12


def test_rd_properties_and_monte_carlo():
    d = np.arange(-50, 51)
    r = oracle.rd_uniform(8, 1200, d)
    assert r[50] == 1
    assert np.allclose(r[::-1], np.conj(r), atol=1e-15)        # r_{-d} = conj(r_d)
    assert (np.abs(r) <= 1 + 1e-15).all()
    rng = np.random.default_rng(1)                               # SPEC.md:135 example
    tau = rng.uniform(0, 8, size=200_000)
    for dd in (1, 7, 30):
        mc = np.exp(-2j * np.pi * dd * tau / 1200).mean()
        assert abs(mc - oracle.rd_uniform(8, 1200, dd)[0]) < 0.01


# ------------------------------------------------------------------ Toeplitz R_hh
def test_toeplitz_matches_scipy():
    rng = np.random.default_rng(2)
    r = rng.standard_normal(9) + 1j * rng.standard_normal(9)
    r[0] = 3.0
    R = oracle.toeplitz_hermitian(r, 9)
    assert np.array_equal(R, linalg.toeplitz(r, np.conj(r)))
    assert np.allclose(R, R.conj().T)


def test_generated_channel_correlation_matches_r():
    """Sample E{H(p) H*(q)} of the signal model equals toeplitz_hermitian(r)[p, q]
    (pins the sign of d: R[p,q] = r[p-q] for p >= q)."""
    cfg = dataclasses.replace(CONFIGS[3], M=400, K=10, N=40)
    r, _ = workload.channel_stats(cfg)
    _, H = workload.gen_instances(cfg, 0, return_channel=True, noiseless=True)
    H = H.reshape(-1, cfg.N)
    R_mc = H.T @ H.conj() / H.shape[0]
    R = oracle.toeplitz_hermitian(r[0], cfg.N)
    assert np.abs(R_mc - R).max() < 0.05
    assert abs(np.angle(R_mc[5, 0]) - np.angle(r[0][5])) < 0.1  # lower triangle = r[d]


# ------------------------------------------------------------------ LS
def test_ls_noiseless_is_exact():
    cfg = CONFIGS[1]
    y, H = workload.gen_instances(cfg, 0, return_channel=True, noiseless=True)
    x = workload.gen_pilots(cfg, 0)
    H_ls = oracle.ls_estimate(y, x)
    assert np.abs(H_ls - H).max() <= 4e-7 * np.abs(H).max()   # complex64 rounding of y only


def test_ls_noise_variance_is_sigma2():
    cfg = dataclasses.replace(CONFIGS[3], M=64, K=4)
    y, H = workload.gen_instances(cfg, 0, return_channel=True)
    x = workload.gen_pilots(cfg, 0)
    _, s2 = workload.channel_stats(cfg)
    mse = np.mean(np.abs(oracle.ls_estimate(y, x) - H) ** 2)
    assert abs(mse / s2[0] - 1) < 0.02


# ------------------------------------------------------------------ filter (Eq. 17)
def test_filter_eigen_form_and_hermitian():
    """W = U diag(lam/(lam+s2)) U^H from eigh(R) -- a different LAPACK route than solve."""
    rng = np.random.default_rng(3)
    cases = [(_rand_psd(rng, 20), 0.3), (_rand_psd(rng, 30, rank=4), 0.05)]
    for c in (1, 3, 4):
        r, s2 = workload.channel_stats(CONFIGS[c])
        cases.append((oracle.toeplitz_hermitian(r[0], CONFIGS[c].b), s2[0]))
    for R, s2 in cases:
        W = oracle.lmmse_filter(R, s2)
        lam, U = np.linalg.eigh(R)
        W_eig = (U * (lam / (lam + s2))) @ U.conj().T
        assert np.abs(W - W_eig).max() < 1e-9 * max(1, np.abs(W).max())
        assert np.abs(W - W.conj().T).max() < 1e-9
        ev = np.linalg.eigvalsh((W + W.conj().T) / 2)
        assert ev.min() > -1e-9 and ev.max() < 1


def test_filter_special_cases():
    s2 = 0.37
    # R = I -> scalar Wiener filter I/(1+s2) (textbook)
    assert np.allclose(oracle.lmmse_filter(np.eye(6), s2), np.eye(6) / (1 + s2), atol=1e-15)
    # b = 1 -> r0/(r0+s2)
    assert np.isclose(oracle.block_filter(np.array([2.5 + 0j]), s2, 1)[0, 0], 2.5 / (2.5 + s2))
    # s2 -> infinity: W = R/s2 + O(1/s2^2) -> 0
    R = oracle.toeplitz_hermitian(workload.channel_stats(CONFIGS[3])[0][0], 50)
    big = 1e8
    assert np.abs(big * oracle.lmmse_filter(R, big) - R).max() < 1e-6
    # exact identity (reading A9): ||W - I||_2 = s2/(lam_min + s2); KMS r_d = rho^|d| is nonsingular
    rho = 0.8
    Rk = oracle.toeplitz_hermitian(rho ** np.arange(40) + 0j, 40)
    lam_min = np.linalg.eigvalsh(Rk).min()
    for s in (1.0, 1e-2, 1e-6):
        W = oracle.lmmse_filter(Rk, s)
        assert np.isclose(np.linalg.norm(W - np.eye(40), 2), s / (lam_min + s), rtol=1e-8)
    # W -> I as s2 -> 0 for nonsingular R (north_star)
    assert np.linalg.norm(oracle.lmmse_filter(Rk, 1e-12) - np.eye(40), 2) < 1e-9


# ------------------------------------------------------------------ block vs full
def test_block_equals_full_for_block_diagonal_R():
    """north_star: block == full LMMSE when R_hh is block-diagonal aligned to b."""
    rng = np.random.default_rng(4)
    N, b = 60, 12
    R = linalg.block_diag(*[_rand_psd(rng, b) for _ in range(N // b)])
    H_ls = rng.standard_normal((3, 5, N)) + 1j * rng.standard_normal((3, 5, N))
    blk = oracle.block_lmmse_general(H_ls, R, 0.2, b, b)
    full = oracle.full_lmmse_general(H_ls, R, 0.2)
    assert np.abs(blk - full).max() < 1e-10


def test_b_equals_N_block_equals_full():
    cfg = dataclasses.replace(CONFIGS[1], b=72, stride=72)
    y = workload.gen_instances(cfg, 0)
    x = workload.gen_pilots(cfg, 0)
    r, s2 = workload.channel_stats(cfg)
    soi = workload.set_of_instance(cfg)
    blk = oracle.block_lmmse(y, x, r, s2, soi, 72, 72)
    full = oracle.full_lmmse(y, x, r, s2, soi)
    assert np.abs(blk - full).max() < 1e-10 * np.abs(full).max()


def test_toeplitz_shortcut_equals_per_window_slices():
    for c in (1, 2):
        cfg = CONFIGS[c]
        y = workload.gen_instances(cfg, 0)
        x = workload.gen_pilots(cfg, 0)
        r, s2 = workload.channel_stats(cfg)
        soi = workload.set_of_instance(cfg)
        a = oracle.block_lmmse(y, x, r, s2, soi, cfg.b, cfg.stride, toeplitz_shortcut=True)
        b = oracle.block_lmmse(y, x, r, s2, soi, cfg.b, cfg.stride, toeplitz_shortcut=False)
        assert np.abs(a - b).max() < 1e-12 * np.abs(a).max()


def test_brute_force_tiny():
    """Element-by-element loops on a tiny case: out[o] = sum_j W[o-a, j] * y[a+j]/x[a+j]."""
    rng = np.random.default_rng(5)
    N, b, s = 11, 4, 3
    r = np.array([1.0, 0.6 - 0.2j, 0.3 + 0.1j, 0.1j])
    r = np.concatenate([r, np.zeros(N - 4)])
    y = (rng.standard_normal((1, 2, 1, N)) + 1j * rng.standard_normal((1, 2, 1, N))).astype(np.complex64)
    x = np.exp(2j * np.pi * rng.random((1, 1, N))).astype(np.complex64)
    out = oracle.block_lmmse(y, x, r[None], np.array([0.5]), np.zeros(1, int), b, s)
    lam, U = np.linalg.eigh(linalg.toeplitz(r[:b], np.conj(r[:b])))
    W = (U * (lam / (lam + 0.5))) @ U.conj().T
    # windows for (11, 4, 3): starts 0,3,6,7 ; m_l = 0 ; kept [0,3),[3,6),[6,9),[9,11)
    owner = {o: (min(3 * (o // 3), N - b) if o < 9 else 7) for o in range(N)}
    for m in range(2):
        for o in range(N):
            a = owner[o]
            v = sum(W[o - a, j] * complex(y[0, m, 0, a + j]) / complex(x[0, 0, a + j]) for j in range(b))
            assert abs(out[0, m, 0, o] - v) < 1e-12


# ------------------------------------------------------------------ MSE (north_star closed form)
@pytest.mark.slow
def test_closed_form_mse_matches_monte_carlo_and_ordering():
    """Per-block MSE tr(R_b - R_b(R_b+s2 I)^-1 R_b)/b vs the oracle's Monte-Carlo MSE on
    the signal model (>= 2e4 independent (m,k) draws), within 5 standard errors."""
    cfg = dataclasses.replace(CONFIGS[3], M=1000, K=20, N=300)
    r, s2 = workload.channel_stats(cfg)
    x = workload.gen_pilots(cfg, 0)
    errs_b, errs_ls = [], []
    for m0 in range(0, cfg.M, 250):
        y, H = workload.gen_instances(cfg, 0, m_lo=m0, m_hi=m0 + 250, x=x, return_channel=True)
        est = oracle.block_lmmse(y, x, r, s2, None, cfg.b, cfg.stride)
        errs_b.append((np.abs(est - H) ** 2).reshape(-1, cfg.N))
        errs_ls.append((np.abs(oracle.ls_estimate(y, x) - H) ** 2).reshape(-1, cfg.N))
    eb = np.concatenate(errs_b)
    el = np.concatenate(errs_ls)
    cf_tone = oracle.block_mse_per_tone(r[0], s2[0], cfg.N, cfg.b, cfg.stride)
    for blk in range(cfg.N // cfg.b):
        sl = slice(blk * cfg.b, (blk + 1) * cfg.b)
        per_draw = eb[:, sl].mean(axis=1)
        se = per_draw.std(ddof=1) / np.sqrt(len(per_draw))
        assert abs(per_draw.mean() - cf_tone[sl].mean()) < 5 * se
        assert np.isclose(cf_tone[sl].mean(), oracle.block_mse(r[0], s2[0], cfg.b))
    assert abs(el.mean() / s2[0] - 1) < 0.01
    # LMMSE optimality: full <= block <= LS per tone (closed forms)
    full_tone = oracle.full_mse_per_tone(r[0], s2[0], cfg.N)
    assert (full_tone <= cf_tone + 1e-12).all() and (cf_tone < s2[0]).all()


def test_orthogonality_principle_monte_carlo():
    """LMMSE error is uncorrelated with the observations in its window:
    E{(H_o - H_hat_o) conj(H_LS_j)} = 0.  A conjugated/transposed W fails this."""
    cfg = dataclasses.replace(CONFIGS[1], M=2000, K=10)
    r, s2 = workload.channel_stats(cfg)
    x = workload.gen_pilots(cfg, 0)
    y, H = workload.gen_instances(cfg, 0, x=x, return_channel=True)
    H_ls = oracle.ls_estimate(y, x).reshape(-1, cfg.N)
    est = oracle.block_lmmse(y, x, r, s2, None, cfg.b, cfg.stride).reshape(-1, cfg.N)
    e = H.reshape(-1, cfg.N) - est
    W = oracle.block_filter(r[0], s2[0], cfg.b)
    bad = H.reshape(-1, cfg.N)[:, :12] - H_ls[:, :12] @ W.T.conj()       # wrong: conj(W)
    worst_good, worst_bad = 0.0, 0.0
    for o in range(0, 12, 3):
        for j in range(12):
            prod = e[:, o] * np.conj(H_ls[:, j])
            z = abs(prod.mean()) / (prod.std() / np.sqrt(len(prod)))
            worst_good = max(worst_good, z)
            pb = bad[:, o] * np.conj(H_ls[:, j])
            worst_bad = max(worst_bad, abs(pb.mean()) / (pb.std() / np.sqrt(len(pb))))
    assert worst_good < 5.0
    assert worst_bad > 10.0


def test_survey_closed_form_values():
    """Cross-check of the A6 PDP reading against the closed-form MSEs quoted in
    SURVEY.md §8(c) ("A builder who reproduces these has followed A6")."""
    r3, s3 = workload.channel_stats(CONFIGS[3])
    assert np.isclose(oracle.block_mse(r3[0], s3[0], 100), 3.5072e-3, rtol=1e-4)
    assert np.isclose(oracle.full_mse_per_tone(r3[0], s3[0], 1200).mean(), 3.7554e-4, rtol=1e-4)
    r1, s1 = workload.channel_stats(CONFIGS[1])
    assert np.isclose(oracle.block_mse(r1[0], s1[0], 12), 1.4550e-2, rtol=1e-4)
    r5, s5 = workload.channel_stats(CONFIGS[5])
    assert np.isclose(oracle.block_mse(r5[0], s5[0], 126), 1.0382e-3, rtol=1e-4)
    assert np.isclose(workload.rms_spread_taps(16), 1.417831, rtol=1e-6)
    assert np.isclose(workload.rms_spread_taps(24), 1.419249, rtol=1e-6)


def test_linearity_and_zero():
    cfg = CONFIGS[2]
    y = workload.gen_instances(cfg, 0)
    x = workload.gen_pilots(cfg, 0)
    r, s2 = workload.channel_stats(cfg)
    soi = workload.set_of_instance(cfg)
    f = lambda yy: oracle.block_lmmse(yy, x, r, s2, soi, cfg.b, cfg.stride)  # noqa: E731
    assert not f(np.zeros_like(y)).any()
    a = (0.3 - 1.1j)
    assert np.abs(f(y * np.complex64(a)) - a * f(y)).max() < 1e-6 * np.abs(f(y)).max()
    perm = np.random.default_rng(0).permutation(cfg.M)      # antenna-permutation equivariance
    assert np.abs(f(y[:, perm]) - f(y)[:, perm]).max() == 0


def test_rel_fro_metric():
    ref = np.ones((2, 3, 4), np.complex128)
    t = ref.copy()
    t[1] *= 1 + 1e-3
    err = oracle.rel_fro_error_per_instance(t, ref)
    assert err[0] == 0 and np.isclose(err[1], 1e-3)
