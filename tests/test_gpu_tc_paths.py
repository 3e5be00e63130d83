"""Every path the tensor-core kernels serve, on geometries where they are the launched kernel.

K4 (CE_KERNEL_BF16X3, the AUTO kernel) needs even window starts, so the config-2 checks of test_gpu_parity.py
(odd starts) never reach it.  Here, on the config-3 and config-4 geometries (the paper-scale
slot and the batched frame, Eq. 12 per block with the Table II edge clamping):
- shard invariance through offset device pointers (the multi-GPU design rests on it: the filters
  "bear no relation with the receiving antennas"), G = 2 / 4 / 8 antenna shards bitwise equal to the full call;
- ce_estimate_host (the end-to-end entry point bench.py times) bitwise equal to ce_estimate and within the bar;
- determinism across repeated calls;
- zero input, exact scaling by 2, an out-of-range statistic set, argument validation;
- window tables longer than the 32 entries carried in K4's kernel parameters (the paper's 12-tone groups:
  N = 1200, b = 12 -> 100 windows; N = 3276, b = 50 -> 66 windows) and an even-start b = 2;
and each asserts that the requested kernel is the one that ran (ce_selected_kernel).
"""
import numpy as np
import pytest

import oracle
import workload
from _parity import assert_parity
from workload import CONFIGS

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TC_KERNELS = [3]        # CE_KERNEL_BF16X3 (K4); AUTO selects it on every geometry below


def _ce():
    import paper_1802_05427_b200 as ce
    return ce


def _est(N, b, s, r, s2, kernel):
    ce = _ce()
    est = ce.ChannelEstimator(N, b, s, r, s2)
    try:
        ce.ce_set_kernel(est.handle, kernel)
    except ce.CEError as e:
        est.close()
        if e.status == ce.CE_EINVAL:
            pytest.skip(f"kernel {kernel} not applicable to N={N} b={b} s={s}: {e}")
        raise
    return est.build()


def _geometry(cfg_id, m_hi):
    cfg = CONFIGS[cfg_id]
    r, s2 = workload.channel_stats(cfg, 0)
    x = workload.gen_pilots(cfg, 0)
    y = workload.gen_instances(cfg, 0, x=x, m_hi=m_hi)
    return cfg, r, s2, x, y, workload.set_of_instance(cfg)


def _stream():
    return torch.cuda.current_stream().cuda_stream


@pytest.mark.parametrize("kernel", TC_KERNELS)
@pytest.mark.parametrize("cfg_id", [3, 4])
def test_shard_invariance_host_path_determinism(cfg_id, kernel):
    ce = _ce()
    cfg, r, s2, x, y, soi = _geometry(cfg_id, 16)
    T, M, K, N = y.shape
    est = _est(cfg.N, cfg.b, cfg.stride, r, s2, kernel)
    y_d, x_d, soi_d = torch.from_numpy(y).cuda(), torch.from_numpy(x).cuda(), torch.from_numpy(soi).cuda()
    full = est.estimate(y_d, x_d, set_of_instance=soi_d)
    torch.cuda.synchronize()
    assert est.selected_kernel() == kernel
    ref = oracle.block_lmmse(y, x, r, s2, soi, cfg.b, cfg.stride)
    assert_parity(full.cpu().numpy(), ref, N, cfg.b, cfg.stride)
    for _ in range(2):                                  # deterministic across calls
        again = est.estimate(y_d, x_d, set_of_instance=soi_d)
        torch.cuda.synchronize()
        assert torch.equal(torch.view_as_real(full), torch.view_as_real(again))
    for G in (2, 4, 8):                                 # antenna shards through offset device pointers
        out = torch.full_like(y_d, complex("nan+nanj"))
        Mg = M // G
        for g in range(G):         # [T][M][K][N]: an antenna shard is strided over t -> one call per instance
            for t in range(T):
                ce.ce_estimate(est.handle, y_d[t, g * Mg].data_ptr(), x_d[t].data_ptr(), out[t, g * Mg].data_ptr(),
                               1, Mg, K, soi_d[t:].data_ptr(), _stream())
        torch.cuda.synchronize()
        assert est.selected_kernel() == kernel
        assert torch.equal(torch.view_as_real(out), torch.view_as_real(full)), G
    # end-to-end host-buffer entry point: same bits as the device call
    h_host = est.estimate_host(y, x, set_of_instance=soi)
    assert est.selected_kernel() == kernel
    assert np.array_equal(h_host.view(np.float32), full.cpu().numpy().view(np.float32))
    pin_y, pin_x = torch.from_numpy(y).pin_memory(), torch.from_numpy(x).pin_memory()
    pin_out = torch.empty(y.shape, dtype=torch.complex64).pin_memory()
    est.estimate_host(pin_y, pin_x, out=pin_out, set_of_instance=soi)
    assert torch.equal(torch.view_as_real(pin_out), torch.view_as_real(full.cpu()))
    est.close()


@pytest.mark.parametrize("kernel", TC_KERNELS)
def test_zero_scaling_bad_set_validation(kernel):
    ce = _ce()
    cfg, r, s2, x, y, soi = _geometry(4, 8)
    y, x, soi = y[:3], x[:3], soi[:3]                 # 3 instances, sets 0, 0, 1
    T, M, K, N = y.shape
    est = _est(cfg.N, cfg.b, cfg.stride, r, s2, kernel)
    x_d, soi_d = torch.from_numpy(x).cuda(), torch.from_numpy(np.ascontiguousarray(soi)).cuda()
    y_d = torch.from_numpy(np.ascontiguousarray(y)).cuda()
    z = est.estimate(torch.zeros_like(y_d), x_d, set_of_instance=soi_d)
    torch.cuda.synchronize()
    assert est.selected_kernel() == kernel
    assert not torch.view_as_real(z).any()
    h1 = est.estimate(y_d, x_d, set_of_instance=soi_d)
    h2 = est.estimate(y_d * 2, x_d, set_of_instance=soi_d)     # scaling by 2 is exact through every step
    torch.cuda.synchronize()
    assert torch.equal(torch.view_as_real(h2), torch.view_as_real(h1) * 2)
    ha = est.estimate(y_d * (0.37 - 0.81j), x_d, set_of_instance=soi_d)
    ref = oracle.block_lmmse(y, x, r, s2, soi, cfg.b, cfg.stride)
    assert_parity(ha.cpu().numpy(), ref * (0.37 - 0.81j), N, cfg.b, cfg.stride)
    bad = torch.tensor([0, 57, 1], dtype=torch.int32, device="cuda")   # set 57 does not exist (20 sets)
    hb = est.estimate(y_d, x_d, set_of_instance=bad).cpu().numpy()
    assert np.isnan(hb[1]).all() and np.isfinite(hb[[0, 2]]).all()
    assert np.array_equal(hb[[0, 2]].view(np.float32), h1.cpu().numpy()[[0, 2]].view(np.float32))
    lib = ce.ce.lib
    assert lib.ce_estimate(est.handle, y_d.data_ptr(), x_d.data_ptr(), y_d.data_ptr(), T, M, K, None, None) == ce.CE_EINVAL
    assert lib.ce_estimate(est.handle, y_d.data_ptr() + 4, x_d.data_ptr(), h1.data_ptr(), 1, 1, 1, None, None) == ce.CE_EINVAL
    assert lib.ce_estimate(est.handle, y_d.data_ptr(), x_d.data_ptr(), h1.data_ptr(), 0, M, K, None, None) == ce.CE_EINVAL
    with pytest.raises(ValueError):
        est.estimate_host(y, x, out=np.empty((T, M, K, N - 1), np.complex64))
    with pytest.raises(ValueError):
        est.estimate_host(y, x[:, :, :-1])
    with pytest.raises(ValueError):
        est.estimate_host(y, x, set_of_instance=soi[:1])
    with pytest.raises(ValueError):
        est.estimate(y_d, x_d, out=torch.empty((T, M, K, N), dtype=torch.complex128, device="cuda"))
    est.close()


def _random_problem(N, b, M, K, T, seed):
    rng = np.random.default_rng(seed)
    L = 6
    p = np.exp(-np.arange(L) / 2.5)
    p /= p.sum()
    tau = np.sort(rng.uniform(0, 12, L))
    d = np.arange(N)
    r = (p[None] * np.exp(-2j * np.pi * np.outer(d, tau) / (2 * N))).sum(1)[None]
    y = (rng.standard_normal((T, M, K, N)) + 1j * rng.standard_normal((T, M, K, N))).astype(np.complex64)
    x = (np.exp(2j * np.pi * rng.random((T, K, N))) * rng.uniform(0.5, 2.0, (T, K, N))).astype(np.complex64)
    return r, np.array([0.03]), y, x


@pytest.mark.parametrize("kernel", TC_KERNELS)
@pytest.mark.parametrize("N,b,s,M,K,T", [
    (1200, 12, 12, 8, 12, 1),     # the paper's 12-tone groups: 100 windows (> 32 in the kernel parameters)
    (3276, 50, 50, 4, 24, 2),     # 66 windows, NR numerology, two instances
    (1200, 12, 6, 3, 12, 1),      # overlapping 12-tone windows (even starts): 199 windows
    (40, 2, 2, 6, 3, 1),          # b = 2, even starts
    (300, 100, 50, 11, 7, 2),     # cols = 77: ragged column tile, overlapping
])
def test_many_windows_and_small_b(N, b, s, M, K, T, kernel):
    r, s2, y, x = _random_problem(N, b, M, K, T, N + 7 * b + s)
    est = _est(N, b, s, r, s2, kernel)
    h = est.estimate(torch.from_numpy(y).cuda(), torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    assert est.selected_kernel() == kernel
    ref = oracle.block_lmmse(y, x, r, s2, None, b, s)
    assert_parity(h.cpu().numpy(), ref, N, b, s)
    est.close()


def test_host_async_calls_in_flight():
    """ce_estimate_host_async: three calls enqueued back to back on one stream (two staging slots, so the third
    waits on the device for the first's last copy), different inputs and outputs -- each result bitwise equal to
    the device-pointer call."""
    cfg, r, s2, x, y, soi = _geometry(3, 16)
    est = _est(cfg.N, cfg.b, cfg.stride, r, s2, 3)
    ys = [torch.from_numpy(y * np.complex64(f)).pin_memory() for f in (1.0, -0.5 + 0.25j, 3.0)]
    xs = torch.from_numpy(x).pin_memory()
    outs = [torch.empty(y.shape, dtype=torch.complex64).pin_memory() for _ in ys]
    for yi, oi in zip(ys, outs):
        est.estimate_host(yi, xs, out=oi, set_of_instance=soi, sync=False)
    est.host_wait()
    torch.cuda.current_stream().synchronize()
    for yi, oi in zip(ys, outs):
        ref = est.estimate(yi.cuda(), xs.cuda(), set_of_instance=torch.from_numpy(soi).cuda()).cpu()
        assert torch.equal(torch.view_as_real(oi), torch.view_as_real(ref))
    est.close()
