"""GPU parity of the comb-pilot 3W / 12W-LMMSE path (NEXT-1, K6) against the CPU oracle, via the C-ABI."""
import dataclasses

import numpy as np
import pytest

import oracle
import workload

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-4


def _run(cfg, y, x, r, s2, kernel="auto"):
    import paper_1802_05427_b200 as ce
    est = ce.CombEstimator(cfg.N, cfg.S, cfg.n_ue, cfg.G, cfg.mode, r, s2).build()
    # K10 (tcgen05) serves every 12W-style shape (full mode, G <= 13, N even): "tc" forces it there, "simt" forces K6b;
    # AUTO takes K10 only for calls with >= 4 units per SM (checked in test_comb_auto_policy)
    tc_shape = cfg.mode == "full" and cfg.G <= 13 and cfg.N % 2 == 0
    if kernel == "tc" and not tc_shape:
        kernel = "auto"
    est.set_kernel(kernel)
    want = ce.CE_COMB_KERNEL_TC if kernel == "tc" else ce.CE_COMB_KERNEL_SIMT if kernel == "simt" else None
    if want is not None:
        assert est.selected_kernel(cfg.T, cfg.M) == want
    h = est.estimate(torch.from_numpy(y).cuda(), torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    W = est.filters()
    est.close()
    return h.cpu().numpy(), W


def _rel(h, ref):
    d = (h.astype(np.complex128) - ref).reshape(ref.shape[0], -1)
    return np.linalg.norm(d, axis=1) / np.linalg.norm(ref.reshape(ref.shape[0], -1), axis=1)


@pytest.mark.parametrize("kernel", ["tc", "simt"])
@pytest.mark.parametrize("name", ["comb_tiny12", "comb_tiny3", "comb_small12", "comb_small3", "paper_12w",
                                  "paper_3w"])
def test_comb_parity_full(name, kernel):
    cfg = workload.get_comb_config(name)
    r, s2 = workload.comb_stats(cfg)
    x = workload.comb_pilots(cfg)
    y = workload.comb_instances(cfg, x=x)
    h, W = _run(cfg, y, x, r, s2, kernel)
    ref = oracle.comb_estimate(y, x, r, s2, cfg.N, cfg.S, cfg.G, cfg.mode, cfg.n_ue)
    assert np.all(_rel(h, ref) <= TOL), _rel(h, ref)
    # weights: FP64 build, complex64 rounding only
    F = oracle.comb_filters(r, s2, cfg.N, cfg.S, cfg.G, cfg.mode, cfg.n_ue)
    for (s, typ), Wo in F.items():
        Wg = W[s if cfg.mode == "full" else 0, typ]
        assert np.linalg.norm(Wg - Wo) / np.linalg.norm(Wo) < 1e-6, (s, typ)


@pytest.mark.parametrize("kernel", ["auto", "simt"])
def test_comb_massive_sampled(kernel):
    """massive_12w (the comb bench workload) at full size in one launch; sampled antennas vs the oracle."""
    cfg = workload.get_comb_config("massive_12w")
    r, s2 = workload.comb_stats(cfg)
    x = workload.comb_pilots(cfg)
    y = workload.comb_instances(cfg, x=x)
    h, _ = _run(cfg, y, x, r, s2, kernel)
    rng = np.random.default_rng(11)
    for m in rng.choice(cfg.M, size=3, replace=False):
        ref = oracle.comb_estimate(y[:, m:m + 1], x, r, s2, cfg.N, cfg.S, cfg.G, cfg.mode, cfg.n_ue)
        assert np.all(_rel(h[:, m:m + 1], ref) <= TOL)
    assert np.isfinite(h).all()


@pytest.mark.parametrize("N,S,n_ue,G,mode", [(60, 6, 6, 10, "full"),     # G = K: one window, full LMMSE
                                             (60, 6, 2, 1, "full"),      # G = 1: scalar Wiener per group
                                             (48, 6, 3, 6, "sub"),       # 3W-like with G = S (1 tone step)
                                             (64, 8, 5, 2, "sub"),       # ragged n_ue, ZOH step 4
                                             (640, 64, 3, 10, "full"),   # S = 64: one group per K10 block
                                             (390, 3, 2, 13, "full"),    # G = 13: the widest K10 window
                                             (520, 4, 4, 14, "full")])   # G = 14: AUTO falls back to K6b
@pytest.mark.parametrize("kernel", ["tc", "simt"])
def test_comb_edge_shapes(N, S, n_ue, G, mode, kernel):
    cfg = workload.CombConfig("edge", M=3, S=S, n_ue=n_ue, N=N, Nfft=128, T=2, G=G, mode=mode,
                              tap_delays=(0, 1.5, 3), tap_db=(-1, -5, -9), snr_db=12.0, L_assumed=5.0,
                              snr_fixed_db=25.0)
    r, s2 = workload.comb_stats(cfg)
    rng = np.random.default_rng(N + G)
    x = (np.exp(2j * np.pi * rng.random((2, N))) * 1.3).astype(np.complex64)      # non-unit pilots
    y = workload.comb_instances(cfg, x=x)
    h, _ = _run(cfg, y, x, r, s2, kernel)
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


def _row_rel(h, ref):
    """max over (instance, antenna, UE) of the relative error of one estimated row (N tones)."""
    d = np.linalg.norm((h.astype(np.complex128) - ref), axis=-1)
    return np.max(d / np.maximum(np.linalg.norm(ref, axis=-1), 1e-30))


@pytest.mark.parametrize("T,M", [(3, 50), (1, 1), (2, 129), (5, 64)])
def test_comb_tc_ragged_rows(T, M):
    """K10 with T*M not a multiple of its 128-row tile (ragged last tile, rows of the next UE inside the TMA box),
    one row, and exactly two tiles: equal to the oracle per instance (1e-4) and per row (1e-3), and to K6b."""
    cfg = dataclasses.replace(workload.get_comb_config("comb_small12"), T=T, M=M)
    r, s2 = workload.comb_stats(cfg)
    x = workload.comb_pilots(cfg)
    y = workload.comb_instances(cfg, x=x)
    h_tc, _ = _run(cfg, y, x, r, s2, "tc")
    h_simt, _ = _run(cfg, y, x, r, s2, "simt")
    ref = oracle.comb_estimate(y, x, r, s2, cfg.N, cfg.S, cfg.G, cfg.mode, cfg.n_ue)
    assert np.all(_rel(h_tc, ref) <= TOL)
    assert _row_rel(h_tc, ref) <= 1e-3
    assert np.all(_rel(h_tc, h_simt.astype(np.complex128)) <= TOL)


def test_comb_tc_deterministic_and_rejects():
    """K10 is bitwise repeatable across calls and workspace growth; forcing it on a 3W shape is CE_EINVAL."""
    import paper_1802_05427_b200 as ce
    cfg = workload.get_comb_config("paper_12w")
    r, s2 = workload.comb_stats(cfg)
    x = torch.from_numpy(workload.comb_pilots(cfg)).cuda()
    y = torch.from_numpy(workload.comb_instances(cfg, x=x.cpu().numpy())).cuda()
    est = ce.CombEstimator(cfg.N, cfg.S, cfg.n_ue, cfg.G, cfg.mode, r, s2).build().set_kernel("tc")
    h1 = est.estimate(y[:2], x[:2]).clone()            # small workspace first, then a larger call
    h2 = est.estimate(y, x)
    h3 = est.estimate(y, x)
    torch.cuda.synchronize()
    assert torch.equal(h2, h3)
    assert torch.equal(h1, h2[:2])
    n0 = est.launch_count()
    est.estimate(y, x)
    assert est.launch_count() == n0 + 2                # k10_ls + k10_comb_tc
    est.close()
    cfg3 = workload.get_comb_config("paper_3w")
    est = ce.CombEstimator(cfg3.N, cfg3.S, cfg3.n_ue, cfg3.G, cfg3.mode, r, s2)
    with pytest.raises(ce.CEError) as e:
        est.set_kernel("tc")
    assert e.value.status == ce.CE_EINVAL
    assert est.selected_kernel(cfg3.T, cfg3.M) == ce.CE_COMB_KERNEL_SIMT
    est.close()


def test_comb_auto_policy():
    """AUTO: K10 for massive_12w-sized calls (>= 4 units of (128 rows, UE, block) per SM), K6b for small calls and for
    the 3W; the massive call itself goes through K10 (two launches) and the small one through K6b (one)."""
    import paper_1802_05427_b200 as ce
    cfg = workload.get_comb_config("massive_12w")
    r, s2 = workload.comb_stats(cfg)
    est = ce.CombEstimator(cfg.N, cfg.S, cfg.n_ue, cfg.G, cfg.mode, r, s2).build()
    assert est.selected_kernel(cfg.T, cfg.M) == ce.CE_COMB_KERNEL_TC
    assert est.selected_kernel(1, 16) == ce.CE_COMB_KERNEL_SIMT
    x = torch.from_numpy(workload.comb_pilots(cfg)).cuda()
    y = torch.zeros((1, 16, cfg.N), dtype=torch.complex64, device="cuda")
    n0 = est.launch_count()
    est.estimate(y, x[:1])
    assert est.launch_count() == n0 + 1
    with pytest.raises(ce.CEError):
        est.selected_kernel(0, 4)
    est.close()
