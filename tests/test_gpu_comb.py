"""GPU parity of the comb-pilot 3W / 12W-LMMSE path (NEXT-1, K6) against the CPU oracle, via the C-ABI."""
import dataclasses

import numpy as np
import pytest

import oracle
import workload

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-4


def _run(cfg, y, x, r, s2):
    import paper_1802_05427_b200 as ce
    est = ce.CombEstimator(cfg.N, cfg.S, cfg.n_ue, cfg.G, cfg.mode, r, s2).build()
    h = est.estimate(torch.from_numpy(y).cuda(), torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    W = est.filters()
    est.close()
    return h.cpu().numpy(), W


def _rel(h, ref):
    d = (h.astype(np.complex128) - ref).reshape(ref.shape[0], -1)
    return np.linalg.norm(d, axis=1) / np.linalg.norm(ref.reshape(ref.shape[0], -1), axis=1)


@pytest.mark.parametrize("name", ["comb_tiny12", "comb_tiny3", "comb_small12", "comb_small3", "paper_12w",
                                  "paper_3w"])
def test_comb_parity_full(name):
    cfg = workload.get_comb_config(name)
    r, s2 = workload.comb_stats(cfg)
    x = workload.comb_pilots(cfg)
    y = workload.comb_instances(cfg, x=x)
    h, W = _run(cfg, y, x, r, s2)
    ref = oracle.comb_estimate(y, x, r, s2, cfg.N, cfg.S, cfg.G, cfg.mode, cfg.n_ue)
    assert np.all(_rel(h, ref) <= TOL), _rel(h, ref)
    # weights: FP64 build, complex64 rounding only
    F = oracle.comb_filters(r, s2, cfg.N, cfg.S, cfg.G, cfg.mode, cfg.n_ue)
    for (s, typ), Wo in F.items():
        Wg = W[s if cfg.mode == "full" else 0, typ]
        assert np.linalg.norm(Wg - Wo) / np.linalg.norm(Wo) < 1e-6, (s, typ)


def test_comb_massive_sampled():
    """massive_12w (the comb bench workload) at full size in one launch; sampled antennas vs the oracle."""
    cfg = workload.get_comb_config("massive_12w")
    r, s2 = workload.comb_stats(cfg)
    x = workload.comb_pilots(cfg)
    y = workload.comb_instances(cfg, x=x)
    h, _ = _run(cfg, y, x, r, s2)
    rng = np.random.default_rng(11)
    for m in rng.choice(cfg.M, size=3, replace=False):
        ref = oracle.comb_estimate(y[:, m:m + 1], x, r, s2, cfg.N, cfg.S, cfg.G, cfg.mode, cfg.n_ue)
        assert np.all(_rel(h[:, m:m + 1], ref) <= TOL)
    assert np.isfinite(h).all()


@pytest.mark.parametrize("N,S,n_ue,G,mode", [(60, 6, 6, 10, "full"),     # G = K: one window, full LMMSE
                                             (60, 6, 2, 1, "full"),      # G = 1: scalar Wiener per group
                                             (48, 6, 3, 6, "sub"),       # 3W-like with G = S (1 tone step)
                                             (64, 8, 5, 2, "sub")])      # ragged n_ue, ZOH step 4
def test_comb_edge_shapes(N, S, n_ue, G, mode):
    cfg = workload.CombConfig("edge", M=3, S=S, n_ue=n_ue, N=N, Nfft=128, T=2, G=G, mode=mode,
                              tap_delays=(0, 1.5, 3), tap_db=(-1, -5, -9), snr_db=12.0, L_assumed=5.0,
                              snr_fixed_db=25.0)
    r, s2 = workload.comb_stats(cfg)
    rng = np.random.default_rng(N + G)
    x = (np.exp(2j * np.pi * rng.random((2, N))) * 1.3).astype(np.complex64)      # non-unit pilots
    y = workload.comb_instances(cfg, x=x)
    h, _ = _run(cfg, y, x, r, s2)
    ref = oracle.comb_estimate(y, x, r, s2, N, S, G, mode, n_ue)
    assert np.all(_rel(h, ref) <= TOL)
    if G == N // S and mode == "full":
        assert np.all(_rel(h, oracle.comb_full_lmmse(y, x, r, s2, N, S, n_ue)) <= TOL)


def test_comb_errors_zero_and_not_pd():
    import paper_1802_05427_b200 as ce
    cfg = workload.get_comb_config("comb_tiny12")
    r, s2 = workload.comb_stats(cfg)
    est = ce.CombEstimator(cfg.N, cfg.S, cfg.n_ue, cfg.G, cfg.mode, r, s2)
    y = torch.zeros((cfg.T, cfg.M, cfg.N), dtype=torch.complex64, device="cuda")
    x = torch.ones((cfg.T, cfg.N), dtype=torch.complex64, device="cuda")
    with pytest.raises(ce.CEError) as e:
        est.estimate(y, x)
    assert e.value.status == ce.CE_ESTATE
    est.build()
    assert not torch.view_as_real(est.estimate(y, x)).any()                       # zero in -> zero out
    st = ce.ce.lib.ce_comb_estimate(est.handle, y.data_ptr(), x.data_ptr(), y.data_ptr(), cfg.T, cfg.M, None)
    assert st == ce.CE_EINVAL                                                     # output aliases y
    assert est.launch_count() >= 2
    est.close()
    bad = np.zeros(cfg.N, np.complex128)
    bad[0], bad[cfg.S] = 1.0, 2.0                                                 # |r_S| > r_0: R_pp indefinite
    est = ce.CombEstimator(cfg.N, cfg.S, cfg.n_ue, 2, "full", bad, 1e-3)
    with pytest.raises(ce.CEError) as e:
        est.build()
    assert e.value.status == ce.CE_ENOTPD
    est.close()
