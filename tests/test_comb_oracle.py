"""Pins of the comb-pilot oracle (NEXT-1: the paper's 3W / 12W-LMMSE mapping rules) -- CPU only."""
import numpy as np
import pytest

import oracle
import workload


def _r(L=8.0, Nfft=2048, N=1200):
    return oracle.rd_uniform(L, Nfft, np.arange(N))


def _rm(r, d):
    """r_d for any integer d (r_{-d} = conj(r_d))."""
    return r[d] if d >= 0 else np.conj(r[-d])


def test_3w_weights_match_printed_equations():
    """PAPER.md:354-385 (Eq. W1-W3, P): the three 3W weights, shared by all UEs.  The printed index
    patterns are typed here; the oracle derives them from tone positions.  P is inverted with inv()
    (a different LAPACK route than the oracle's solve)."""
    r = _r()
    s2 = 1e-3
    P = np.array([[_rm(r, 0), _rm(r, -12), _rm(r, -24)],
                  [_rm(r, 12), _rm(r, 0), _rm(r, -12)],
                  [_rm(r, 24), _rm(r, 12), _rm(r, 0)]]) + s2 * np.eye(3)
    printed = {
        0: [[0, -12, -24], [4, -8, -20], [8, -4, -16]],      # W(1)
        1: [[12, 0, -12], [16, 4, -8], [20, 8, -4]],         # W(2)
        2: [[24, 12, 0], [28, 16, 4], [32, 20, 8]],          # W(3)
    }
    F = oracle.comb_filters(r, s2, 1200, 12, 3, "sub", 4)
    for typ, idx in printed.items():
        Wp = np.array([[_rm(r, d) for d in row] for row in idx]) @ np.linalg.inv(P)
        for s in range(4):                                   # "correspond to weight matrices for all UEs"
            np.testing.assert_allclose(F[(s, typ)], Wp, rtol=0, atol=1e-10)


def test_3w_groups_and_output_tones_table1():
    """Table I rows: group -> output tones, weight id, input tones (UE 1)."""
    K, wins = oracle.comb_geometry(1200, 12, 3)
    rows = {1: ((1, 5, 9), 1, (1, 13, 25)), 2: ((13, 17, 21), 2, (1, 13, 25)), 3: ((25, 29, 33), 2, (13, 25, 37)),
            4: ((37, 41, 45), 2, (25, 37, 49)), 99: ((1177, 1181, 1185), 2, (1165, 1177, 1189)),
            100: ((1189, 1193, 1197), 3, (1165, 1177, 1189))}
    for g1, (outs, wid, ins) in rows.items():
        a, typ = wins[g1 - 1]
        assert typ + 1 == wid
        assert tuple(t + 1 for t in oracle.comb_out_tones(g1 - 1, 0, 12, 3, "sub", 1200)) == outs
        assert tuple(12 * (a + j) + 1 for j in range(3)) == ins


def test_12w_per_ue_weights_and_table2():
    """Table II + PAPER.md:403: 12 weight matrices per UE, different across UEs."""
    r = _r()
    K, wins = oracle.comb_geometry(1200, 12, 12)
    assert [t for _, t in wins[:8]] == [0, 1, 2, 3, 4, 5, 5, 5]
    assert [t for _, t in wins[-6:]] == [6, 7, 8, 9, 10, 11]
    assert wins[6][0] == 1 and wins[93][0] == 88            # group 7 -> pilots 13:12:145, 94 -> 1057:12:1189
    assert oracle.comb_out_tones(6, 0, 12, 12, "full", 1200) == list(range(72, 84))
    F = oracle.comb_filters(r, 1e-4, 1200, 12, 12, "full", 4)
    assert len(F) == 4 * 12
    assert F[(0, 5)].shape == (12, 12)
    assert np.abs(F[(0, 5)] - F[(1, 5)]).max() > 1e-3      # UE-dependent


def test_full_window_equals_full_lmmse():
    """G = K: one window covering all pilots == the un-windowed comb LMMSE (Eq. 12-15)."""
    cfg = workload.get_comb_config("comb_tiny12")
    r, s2 = workload.comb_stats(cfg)
    x = workload.comb_pilots(cfg)
    y = workload.comb_instances(cfg, x=x)
    K = cfg.N // cfg.S
    got = oracle.comb_estimate(y, x, r, s2, cfg.N, cfg.S, K, "full", cfg.n_ue)
    ref = oracle.comb_full_lmmse(y, x, r, s2, cfg.N, cfg.S, cfg.n_ue)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-10)


def test_brute_force_tiny_and_zoh():
    """Element loops on a tiny case: out[k] = sum_j W[q][j] y[S(a+j)+s]/x[...]; 3W tones ZOH-filled."""
    rng = np.random.default_rng(3)
    N, S, G, n_ue = 24, 6, 3, 2
    r = oracle.rd_uniform(3.0, 64, np.arange(N))
    s2 = 0.05
    y = (rng.standard_normal((1, 2, N)) + 1j * rng.standard_normal((1, 2, N))).astype(np.complex64)
    x = np.exp(2j * np.pi * rng.random((1, N))).astype(np.complex64)
    got = oracle.comb_estimate(y, x, r, s2, N, S, G, "sub", n_ue)
    F = oracle.comb_filters(r, s2, N, S, G, "sub", n_ue)
    K, wins = oracle.comb_geometry(N, S, G)
    for m in range(2):
        for s in range(n_ue):
            est = {}
            for g, (a, typ) in enumerate(wins):
                for q in range(G):
                    acc = 0
                    for j in range(G):
                        k_in = S * (a + j) + s
                        acc += F[(s, typ)][q, j] * complex(y[0, m, k_in]) / complex(x[0, k_in])
                    est[S * g + s + (S // G) * q] = acc
            for k in range(N):
                prev = [t for t in est if t <= k]
                e = max(prev) if prev else min(est)
                assert abs(got[0, m, s, k] - est[e]) < 1e-12


def test_ls_error_is_the_noise():
    cfg = workload.get_comb_config("comb_tiny12")
    x = workload.comb_pilots(cfg)
    y, H = workload.comb_instances(cfg, x=x, return_channel=True)
    y0 = np.asarray(y, np.complex128)      # the float32 rounding of y is the only error left
    for s in range(cfg.S):
        ls = oracle.comb_ls(y0, x[:, None, :], cfg.S, s)
        tones = np.arange(s, cfg.N, cfg.S)
        noise = ls - H[:, :, s, tones]
        sigma2 = workload.comb_true_stats(cfg)[1]
        assert abs(np.mean(np.abs(noise) ** 2) / sigma2 - 1) < 0.35      # LS error = noise (|x| = 1)


@pytest.mark.parametrize("name", ["comb_tiny12", "comb_tiny3"])
def test_closed_form_mse_matches_monte_carlo(name):
    """Per-tone closed form (incl. the ZOH hold error) vs Monte-Carlo on the synthetic channel with the
    TRUE statistics, within 5 standard errors."""
    import dataclasses
    cfg = dataclasses.replace(workload.get_comb_config(name), M=400, T=8)
    r, s2 = workload.comb_true_stats(cfg)
    x = workload.comb_pilots(cfg)
    y, H = workload.comb_instances(cfg, x=x, return_channel=True)
    h = oracle.comb_estimate(y, x, r, s2, cfg.N, cfg.S, cfg.G, cfg.mode, cfg.n_ue)
    for s in range(cfg.n_ue):
        err = np.abs(h[:, :, s, :] - H[:, :, s, :]) ** 2           # [T][M][N]
        e = err.reshape(-1, cfg.N)
        mc, se = e.mean(0), e.std(0) / np.sqrt(e.shape[0])
        cf = oracle.comb_mse_per_tone(r, s2, cfg.N, cfg.S, cfg.G, cfg.mode, s)
        assert np.all(np.abs(mc - cf) <= 5 * se + 1e-12), (s, np.max(np.abs(mc - cf) / se))


def test_mse_ordering_paper_fig7a():
    """full LMMSE <= 12W <= 3W (+ZOH) in MSE at matched statistics (closed forms)."""
    cfg = workload.get_comb_config("paper_12w")
    r, s2 = workload.comb_true_stats(cfg)
    m12 = oracle.comb_mse_per_tone(r, s2, cfg.N, cfg.S, 12, "full", 0).mean()
    m3 = oracle.comb_mse_per_tone(r, s2, cfg.N, cfg.S, 3, "sub", 0).mean()
    mfull = oracle.comb_mse_per_tone(r, s2, cfg.N, cfg.S, cfg.N // cfg.S, "full", 0).mean()
    assert mfull <= m12 <= m3
