"""C-ABI checks that need no GPU: the library loads, exports every function declared in
include/ce.h, and rejects invalid parameters before touching CUDA."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1802_05427_b200 as ce

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "ce.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(ce_\w+)\s*\(", src, flags=re.M)))


def test_header_functions_exported():
    names = _declared()
    assert len(names) >= 12, names
    for n in names:
        assert hasattr(ce.ce.lib, n), n            # dlsym succeeds
    assert sorted(ce.EXPORTED) == names


def test_status_strings_and_version():
    for st in (0, -1, -2, -3, -4, -5, -6, 7):
        assert isinstance(ce.ce_status_string(st), str) and ce.ce_status_string(st)
    assert "sm_100a" in ce.ce_version()
    assert ce.ce_last_error() is not None


def test_window_table_errors():
    with pytest.raises(ce.CEError) as e:
        ce.ce_window_table(10, 11, 1)
    assert e.value.status == ce.CE_EINVAL
    with pytest.raises(ce.CEError):
        ce.ce_window_table(10, 4, 5)
    with pytest.raises(ce.CEError):
        ce.ce_window_table(0, 1, 1)
    buf = (ctypes.c_int32 * 3)()
    assert ce.ce.lib.ce_window_table(100, 12, 1, buf, 1) == ce.CE_EINVAL     # capacity too small
    assert ce.ce.lib.ce_window_table(100, 12, 1, None, 0) == 89


def _raw(N, b, s, n_sets, r=None, s2=None):
    r = np.ones((max(n_sets, 1), max(N, 1)), np.complex128) if r is None else r
    s2 = np.full(max(n_sets, 1), 0.1) if s2 is None else s2
    return ce.ce.ce_init_raw(N, b, s, n_sets, r.ctypes.data, s2.ctypes.data)


def test_init_validation():
    assert _raw(0, 1, 1, 1) == ce.CE_EINVAL
    assert _raw(10, 11, 1, 1) == ce.CE_EINVAL
    assert _raw(10, 0, 1, 1) == ce.CE_EINVAL
    assert _raw(10, 4, 0, 1) == ce.CE_EINVAL
    assert _raw(10, 4, 5, 1) == ce.CE_EINVAL
    assert _raw(10, 4, 4, 0) == ce.CE_EINVAL
    assert _raw(10, 4, 4, 1, s2=np.array([0.0])) == ce.CE_EINVAL
    assert _raw(10, 4, 4, 1, s2=np.array([-1.0])) == ce.CE_EINVAL
    assert _raw(10, 4, 4, 1, s2=np.array([np.nan])) == ce.CE_EINVAL
    r = np.ones((1, 10), np.complex128)
    r[0, 3] = np.inf
    assert _raw(10, 4, 4, 1, r=r) == ce.CE_EINVAL
    r = np.ones((1, 10), np.complex128)
    r[0, 0] = 1 + 0.5j                                     # r[0] must be real
    assert _raw(10, 4, 4, 1, r=r) == ce.CE_EINVAL
    r[0, 0] = -1
    assert _raw(10, 4, 4, 1, r=r) == ce.CE_EINVAL
    assert ce.ce.lib.ce_init(None, None) == ce.CE_EINVAL


def test_null_handle_calls():
    lib = ce.ce.lib
    assert lib.ce_free(None) == ce.CE_OK
    assert lib.ce_build_filters(None, None) == ce.CE_EINVAL
    assert lib.ce_estimate(None, None, None, None, 1, 1, 1, None, None) == ce.CE_EINVAL
    assert lib.ce_estimate_host(None, None, None, None, 1, 1, 1, None, None) == ce.CE_EINVAL
    assert lib.ce_set_kernel(None, 0) == ce.CE_EINVAL
    assert lib.ce_get_filters(None, None) == ce.CE_EINVAL
    assert lib.ce_launch_count(None, None) == ce.CE_EINVAL
    assert lib.ce_selected_kernel(None, None) == ce.CE_EINVAL


def test_no_device_is_loud():
    """Valid parameters on a machine without an sm_100 device: CE_ENODEV, never a CPU fallback."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a CUDA device is present")
    except ImportError:
        pass
    assert _raw(72, 12, 12, 1) == ce.CE_ENODEV


def test_comb_init_validation():
    """ce_comb_init rejects bad geometry before touching CUDA (CE_EINVAL); valid params on a machine
    without a GPU are CE_ENODEV."""
    r = np.zeros(96, np.complex128)
    r[0] = 1.0
    bad = [dict(N=96, S=5, n_ue=1, G=2, mode=0),        # N % S != 0
           dict(N=96, S=4, n_ue=5, G=2, mode=0),        # n_ue > S
           dict(N=96, S=4, n_ue=1, G=25, mode=0),       # G > K
           dict(N=96, S=4, n_ue=1, G=3, mode=1),        # sub mode needs S % G == 0
           dict(N=96, S=4, n_ue=1, G=2, mode=7)]        # unknown mode
    for kw in bad:
        with pytest.raises(ce.CEError) as e:
            ce.ce_comb_init(r_hh=r, sigma2=0.1, **kw)
        assert e.value.status == ce.CE_EINVAL, kw
    with pytest.raises(ce.CEError) as e:
        ce.ce_comb_init(96, 4, 4, 4, 0, r, -1.0)
    assert e.value.status == ce.CE_EINVAL
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        with pytest.raises(ce.CEError) as e:
            ce.ce_comb_init(96, 4, 4, 4, 0, r, 0.1)
        assert e.value.status == ce.CE_ENODEV
