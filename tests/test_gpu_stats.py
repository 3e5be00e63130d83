"""GPU parity of the NEXT-3 statistics estimator (K7) against the oracle, and the estimate -> build ->
estimate loop it enables."""
import dataclasses

import numpy as np
import pytest

import oracle
import workload
from workload import CONFIGS

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _gpu_stats(y, x, D, B, soi=None, n_sets=1):
    import paper_1802_05427_b200 as ce
    soi_t = None if soi is None else torch.from_numpy(np.ascontiguousarray(soi, np.int32)).cuda()
    r, s2 = ce.ce_stats_estimate(torch.from_numpy(y).cuda(), torch.from_numpy(x).cuda(), D, B, soi_t, n_sets)
    torch.cuda.synchronize()
    return r.cpu().numpy(), s2.cpu().numpy()


@pytest.mark.parametrize("cfg_id,m_hi", [(3, 64), (2, None), (4, 8), (5, 4)])
def test_stats_parity(cfg_id, m_hi):
    cfg = CONFIGS[cfg_id]
    x = workload.gen_pilots(cfg, 0)
    y = workload.gen_instances(cfg, 0, x=x, m_hi=m_hi)
    soi = workload.set_of_instance(cfg)
    D, B = cfg.b, cfg.N // 8
    r_g, s2_g = _gpu_stats(y, x, D, B, soi, cfg.n_sets)
    for s in range(cfg.n_sets):
        sel = soi == s
        r_o, s2_o = oracle.estimate_stats(y[sel], x[sel], D, B)
        assert abs(s2_g[s] / s2_o - 1) < 1e-4, (s, s2_g[s], s2_o)
        assert np.max(np.abs(r_g[s] - r_o)) < 1e-4 * abs(r_o[0]), (s, np.max(np.abs(r_g[s] - r_o)))


@pytest.mark.parametrize("cfg_id,m_hi,B", [(3, 16, 32), (3, 16, 100), (2, None, 64), (4, 8, 32), (5, 4, 32),
                                           (5, 4, 300)])
def test_stats_parity_noise_windows(cfg_id, m_hi, B):
    """The bench's noise window (B = 32) and windows of 2-10 groups of 32 bins (K7c runs up to 128 bins per pass
    over the columns, masking the last group)."""
    cfg = CONFIGS[cfg_id]
    x = workload.gen_pilots(cfg, 0)
    y = workload.gen_instances(cfg, 0, x=x, m_hi=m_hi)
    soi = workload.set_of_instance(cfg)
    D = min(cfg.b, 64)
    r_g, s2_g = _gpu_stats(y, x, D, B, soi, cfg.n_sets)
    for s in range(cfg.n_sets):
        sel = soi == s
        r_o, s2_o = oracle.estimate_stats(y[sel], x[sel], D, B)
        assert abs(s2_g[s] / s2_o - 1) < 1e-4, (s, s2_g[s], s2_o)
        assert np.max(np.abs(r_g[s] - r_o)) < 1e-4 * abs(r_o[0]), (s, np.max(np.abs(r_g[s] - r_o)))


def test_stats_parity_odd_tone_count():
    """N odd: no 16-byte bulk copies, the noise window runs inside K7a."""
    cfg = dataclasses.replace(CONFIGS[2], N=299, b=40, stride=20)
    x = workload.gen_pilots(cfg, 0)
    y = workload.gen_instances(cfg, 0, x=x)
    r_g, s2_g = _gpu_stats(y, x, 40, 32)
    r_o, s2_o = oracle.estimate_stats(y, x, 40, 32)
    assert abs(s2_g[0] / s2_o - 1) < 1e-4
    assert np.max(np.abs(r_g[0] - r_o)) < 1e-4 * abs(r_o[0])


def test_stats_parity_ragged_shape():
    """M = 5 antennas (a partial 4-column group in K7c, a partial 16-column chunk in K8), K = 3 users, N = 302
    tones (a partial 128-tone chunk and a partial 32-tone block), D = 37 lags, B = 40 bins (a masked second bin
    group); run under every kernel policy by test_stats_parity_other_kernel_paths."""
    cfg = dataclasses.replace(CONFIGS[2], M=5, K=3, N=302, b=40, stride=20)
    x = workload.gen_pilots(cfg, 1)
    y = workload.gen_instances(cfg, 1, x=x)
    r_g, s2_g = _gpu_stats(y, x, 37, 40)
    r_o, s2_o = oracle.estimate_stats(y, x, 37, 40)
    assert abs(s2_g[0] / s2_o - 1) < 1e-4
    assert np.max(np.abs(r_g[0] - r_o)) < 1e-4 * abs(r_o[0])


def test_stats_parity_wide_band():
    """N = 2400 tones on the FP32 path (K7a: 16 KB static + 39 KB dynamic shared memory, past the 48 KB default
    without an opt-in)."""
    cfg = dataclasses.replace(CONFIGS[2], M=4, K=2, N=2400, b=50, stride=25)
    x = workload.gen_pilots(cfg, 2)
    y = workload.gen_instances(cfg, 2, x=x)[:1]
    r_g, s2_g = _gpu_stats(y, x[:1], 50, 32)
    r_o, s2_o = oracle.estimate_stats(y, x[:1], 50, 32)
    assert abs(s2_g[0] / s2_o - 1) < 1e-4
    assert np.max(np.abs(r_g[0] - r_o)) < 1e-4 * abs(r_o[0])


def test_stats_skipped_and_empty_sets():
    cfg = CONFIGS[2]
    x = workload.gen_pilots(cfg, 0)
    y = workload.gen_instances(cfg, 0, x=x)
    r_g, s2_g = _gpu_stats(y, x, 10, 16, np.array([0, 7], np.int32), 3)     # instance 1: out of range
    r_o, s2_o = oracle.estimate_stats(y[:1], x[:1], 10, 16)
    assert abs(s2_g[0] / s2_o - 1) < 1e-4
    assert np.isnan(s2_g[1]) and np.isnan(r_g[2]).all()                     # sets with no instance


@pytest.mark.parametrize("N,D,B", [(40, 25, 8), (100, 20, 16), (200, 50, 24), (400, 100, 32), (700, 200, 32),
                                   (1200, 150, 32), (3276, 126, 32), (5000, 200, 64), (1201, 64, 31)])
def test_stats_spectrum_lengths(N, D, B):
    """The power-spectrum lag path (K9) at every FFT length it instantiates: L = 64 .. 8192, i.e. every final-pass
    radix (16 x 4, 16 x 8, 16 x 16, 16 x 16 x 2, ... 16 x 16 x 16 x 2); an odd N takes the K7a noise window."""
    rng = np.random.default_rng(N + D)
    T, M, K = 2, 5, 3
    x = np.exp(1j * np.pi / 2 * rng.integers(0, 4, (T, K, N)) + 1j * np.pi / 4).astype(np.complex64)
    # a smooth channel (few delay taps) plus white noise, so that the lags decay as in the workloads
    taps = rng.standard_normal((T, M, K, 4)) + 1j * rng.standard_normal((T, M, K, 4))
    n = np.arange(N)
    Hc = sum(taps[..., i:i + 1] * np.exp(-2j * np.pi * 3 * i * n / N) for i in range(4))
    noise = 0.1 * (rng.standard_normal((T, M, K, N)) + 1j * rng.standard_normal((T, M, K, N)))
    y = ((Hc + noise) * x[:, None, :, :]).astype(np.complex64)
    r_g, s2_g = _gpu_stats(y, x, D, B)
    r_o, s2_o = oracle.estimate_stats(y, x, D, B)
    assert abs(s2_g[0] / s2_o - 1) < 1e-4, (s2_g[0], s2_o)
    assert np.max(np.abs(r_g[0] - r_o)) < 1e-4 * abs(r_o[0]), np.max(np.abs(r_g[0] - r_o)) / abs(r_o[0])


def test_estimated_statistics_drive_the_filters():
    """Data-driven design: K7 statistics -> ce_init/ce_build_filters -> K4 estimate.  The MSE vs the true
    channel is close to the matched closed form (the paper's fixed design is not needed)."""
    import paper_1802_05427_b200 as ce
    cfg = dataclasses.replace(CONFIGS[3], M=64)
    x = workload.gen_pilots(cfg, 0)
    y, H = workload.gen_instances(cfg, 0, x=x, return_channel=True)
    r_true, s2_true = workload.channel_stats(cfg, 0)
    r_g, s2_g = _gpu_stats(y, x, cfg.b, cfg.N // 8)
    r_full = np.zeros((1, cfg.N), np.complex128)
    r_full[0, :cfg.b] = r_g[0]
    r_full[0, 0] = r_full[0, 0].real                                         # ce_init wants r[0] real
    est = ce.ChannelEstimator(cfg.N, cfg.b, cfg.stride, r_full, s2_g).build()
    h = est.estimate(torch.from_numpy(y).cuda(), torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    est.close()
    mse = np.mean(np.abs(h.cpu().numpy() - H) ** 2)
    cf = oracle.block_mse(r_true[0], s2_true[0], cfg.b)
    assert mse < 1.10 * cf, (mse, cf)


@pytest.mark.parametrize("env", [{"CE_K9": "0", "CE_K8_GRAM": "1", "CE_K4_NOISE": "0"},
                                 {"CE_K9": "0", "CE_K8_GRAM": "0", "CE_K7_NOISE": "0"},
                                 {"CE_K9": "0", "CE_K8_GRAM": "0", "CE_K7_NOISE": "1"},
                                 {"CE_K4_NOISE": "0", "CE_K7_NOISE": "0"},
                                 {"CE_K4_NOISE": "0"}],
                         ids=["k8_k7c", "k7a_only", "k7a_k7c", "k9_k7a_noise", "k9_k7c"])
def test_stats_parity_other_kernel_paths(env):
    """The statistics parity tests again with the other kernel paths (by default the lags go through the power
    spectrum, K9, and the noise window through K4 in power mode): (i) the tensor-core lag correlation (K8) forced on
    every shape with K7c streaming the noise window, (ii) K7a alone (lags and noise window in one pass), (iii) K7a
    lags + K7c, (iv) K9 lags + the noise window in K7a, (v) K9 + K7c; in a subprocess: the variables are read once
    per process."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PYTHONPATH=root, **env)
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k", "not other_kernel_paths",
                          os.path.join(root, "tests", "test_gpu_stats.py")], env=env, capture_output=True, text=True,
                         timeout=900, cwd=root)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]
