"""Guard-band (canary) checks of every estimate entry point: the stand-in for compute-sanitizer memcheck, which is
closed on this GPU pool.

Each caller-owned tensor sits inside a larger allocation between two guard bands:
- input guards (y, x) are NaN: an out-of-bounds read that reaches the arithmetic turns outputs non-finite and fails
  the parity bar against the oracle (Eq. 12 per block; comb path PAPER.md:345-403);
- output guards (h) hold a sentinel bit pattern and the output interior starts as NaN: an out-of-bounds write changes
  a guard (compared bitwise), a missed write leaves a NaN inside (caught by the parity check).
Shapes are the ones where masks matter: ragged 128-row tiles (cols = 96, 288), edge windows, overlapping windows,
odd window starts, the comb path's ragged row tiles, and the host-buffer entry point.
"""
import dataclasses

import numpy as np
import pytest

import oracle
import workload
from _parity import assert_parity
from workload import CONFIGS

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

G = 4096                                   # guard elements (complex64): 32 KB, keeps the 256-byte alignment
SENT = np.complex64(complex(1234.5, -6789.25))


def _ce():
    import paper_1802_05427_b200 as ce
    return ce


def _guard_in(a: np.ndarray):
    """device copy of `a` between two NaN guard bands; returns (whole allocation, view of a's shape)"""
    big = torch.full((a.size + 2 * G,), complex(float("nan"), float("nan")), dtype=torch.complex64, device="cuda")
    big[G:G + a.size] = torch.from_numpy(np.ascontiguousarray(a).reshape(-1)).cuda()
    return big, big[G:G + a.size].view(*a.shape)


def _guard_out(shape):
    n = int(np.prod(shape))
    big = torch.full((n + 2 * G,), complex(SENT), dtype=torch.complex64, device="cuda")
    big[G:G + n] = complex(float("nan"), float("nan"))
    return big, big[G:G + n].view(*shape)


def _guards_intact(big, n):
    g = big.cpu().numpy()
    want = np.full(G, SENT).view(np.uint64)
    return (np.array_equal(g[:G].view(np.uint64), want) and np.array_equal(g[G + n:].view(np.uint64), want))


def _inputs(cfg, T, m_hi):
    """the first T instances and m_hi antennas of a configuration (same draws as the full configuration's)"""
    r, s2 = workload.channel_stats(cfg, 0)
    x = workload.gen_pilots(cfg, 0, 0, T)
    y = workload.gen_instances(cfg, 0, 0, T, 0, m_hi, x=x)
    return r, s2, x, y, workload.set_of_instance(cfg)[:T].copy()


@pytest.mark.parametrize("kernel", [0, 1, 2, 3])
@pytest.mark.parametrize("cfg_id,T,m_hi", [(3, 1, 8), (3, 1, 24), (4, 3, 8), (2, 2, 5)])
def test_estimate_guard_bands(cfg_id, T, m_hi, kernel):
    ce = _ce()
    cfg = CONFIGS[cfg_id]
    r, s2, x, y, soi = _inputs(cfg, T, m_hi)
    est = ce.ChannelEstimator(cfg.N, cfg.b, cfg.stride, r, s2)
    try:
        ce.ce_set_kernel(est.handle, kernel)
    except ce.CEError as e:
        est.close()
        if e.status == ce.CE_EINVAL:
            pytest.skip(f"kernel {kernel} not applicable to config {cfg_id}: {e}")
        raise
    est.build()
    yb, yv = _guard_in(y)
    xb, xv = _guard_in(x)
    hb, hv = _guard_out(y.shape)
    est.estimate(yv, xv, out=hv, set_of_instance=torch.from_numpy(soi).cuda())
    torch.cuda.synchronize()
    est.close()
    assert _guards_intact(hb, y.size), "ce_estimate wrote outside h"
    ref = oracle.block_lmmse(y, x, r, s2, soi, cfg.b, cfg.stride)
    assert_parity(hv.cpu().numpy(), ref, cfg.N, cfg.b, cfg.stride)


def test_estimate_host_guard_bands():
    ce = _ce()
    cfg = CONFIGS[3]
    r, s2, x, y, soi = _inputs(cfg, 1, 24)
    est = ce.ChannelEstimator(cfg.N, cfg.b, cfg.stride, r, s2).build()
    nan = np.complex64(complex(np.nan, np.nan))
    yb = np.full(y.size + 2 * G, nan)
    yb[G:G + y.size] = y.reshape(-1)
    xb = np.full(x.size + 2 * G, nan)
    xb[G:G + x.size] = x.reshape(-1)
    hb = np.full(y.size + 2 * G, SENT)
    hb[G:G + y.size] = nan
    hv = hb[G:G + y.size].reshape(y.shape)
    est.estimate_host(yb[G:G + y.size].reshape(y.shape), xb[G:G + x.size].reshape(x.shape), out=hv,
                      set_of_instance=soi)
    est.close()
    want = np.full(G, SENT).view(np.uint64)
    assert np.array_equal(hb[:G].view(np.uint64), want) and np.array_equal(hb[G + y.size:].view(np.uint64), want), \
        "ce_estimate_host wrote outside h"
    ref = oracle.block_lmmse(y, x, r, s2, soi, cfg.b, cfg.stride)
    assert_parity(hv, ref, cfg.N, cfg.b, cfg.stride)


@pytest.mark.parametrize("kernel", ["tc", "simt"])
@pytest.mark.parametrize("name,M", [("comb_small12", 5), ("paper_12w", 9), ("comb_small3", 5)])
def test_comb_guard_bands(name, M, kernel):
    ce = _ce()
    cfg = dataclasses.replace(workload.get_comb_config(name), M=M)
    r, s2 = workload.comb_stats(cfg)
    x = workload.comb_pilots(cfg)
    y = workload.comb_instances(cfg, x=x)
    est = ce.CombEstimator(cfg.N, cfg.S, cfg.n_ue, cfg.G, cfg.mode, r, s2).build()
    if kernel == "tc" and not (cfg.mode == "full" and cfg.G <= 13 and cfg.N % 2 == 0):
        est.close()
        pytest.skip("K10 serves the 12W shapes only")
    est.set_kernel(kernel)
    yb, yv = _guard_in(y)
    xb, xv = _guard_in(x)
    shape = (cfg.T, cfg.M, cfg.n_ue, cfg.N)
    hb, hv = _guard_out(shape)
    est.estimate(yv, xv, out=hv)
    torch.cuda.synchronize()
    est.close()
    assert _guards_intact(hb, int(np.prod(shape))), "ce_comb_estimate wrote outside h"
    ref = oracle.comb_estimate(y, x, r, s2, cfg.N, cfg.S, cfg.G, cfg.mode, cfg.n_ue)
    h = hv.cpu().numpy()
    assert np.isfinite(h).all()
    d = (h.astype(np.complex128) - ref).reshape(ref.shape[0], -1)
    err = np.linalg.norm(d, axis=1) / np.linalg.norm(ref.reshape(ref.shape[0], -1), axis=1)
    assert np.all(err <= 1e-4), err


@pytest.mark.parametrize("cfg_id,T,m_hi,D,B", [(2, 2, 5, 20, 32), (3, 1, 24, 100, 32)])
def test_stats_guard_bands(cfg_id, T, m_hi, D, B):
    ce = _ce()
    cfg = CONFIGS[cfg_id]
    _r, _s2, x, y, _soi = _inputs(cfg, T, m_hi)
    yb, yv = _guard_in(y)
    xb, xv = _guard_in(x)
    rg, s2g = ce.ce_stats_estimate(yv, xv, D, B)
    torch.cuda.synchronize()
    ro, s2o = oracle.estimate_stats(y, x, D, B)
    rg, s2g = rg.cpu().numpy(), s2g.cpu().numpy()
    assert np.isfinite(rg).all() and np.isfinite(s2g).all(), "an out-of-bounds (NaN guard) read reached the statistics"
    assert abs(s2g[0] / s2o - 1) < 1e-4 and np.max(np.abs(rg[0] - ro)) < 1e-4 * abs(ro[0])
