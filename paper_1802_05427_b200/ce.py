"""ctypes binding of libce (include/ce.h) -- argument marshalling only.

Every step of the estimator runs inside libce's CUDA kernels; this module only
converts Python/NumPy/torch arguments to pointers and sizes.  There is no CPU
fallback: importing this module fails loudly if libce.so has not been built.
Function names match the C ABI.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_void_p

import numpy as np

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libce.so")

if not os.path.exists(_LIB_PATH):
    raise ImportError(
        f"libce.so not found at {_LIB_PATH}: build it with "
        "`python -c 'import __graft_entry__ as g; g.build()'` (nvcc, sm_100a)")

lib = ctypes.CDLL(_LIB_PATH)

CE_OK, CE_EINVAL, CE_ENOMEM, CE_ECUDA, CE_ENOTPD, CE_ESTATE, CE_ENODEV = 0, -1, -2, -3, -4, -5, -6
CE_KERNEL_AUTO, CE_KERNEL_SIMT, CE_KERNEL_TF32X3, CE_KERNEL_BF16X3 = 0, 1, 2, 3   # 4 (K5) retired: CE_EINVAL

# every function declared in include/ce.h (tests check the .so exports all of them)
EXPORTED = ("ce_init", "ce_build_filters", "ce_estimate", "ce_estimate_host", "ce_estimate_host_async",
            "ce_estimate_host_wait", "ce_free",
            "ce_set_kernel",
            "ce_selected_kernel",
            "ce_get_filters", "ce_window_table", "ce_launch_count", "ce_status_string", "ce_last_error",
            "ce_version", "ce_comb_init", "ce_comb_build_filters", "ce_comb_estimate", "ce_comb_get_filters",
            "ce_comb_launch_count", "ce_comb_set_kernel", "ce_comb_selected_kernel", "ce_comb_free",
            "ce_stats_workspace_bytes", "ce_stats_estimate")
CE_COMB_FULL, CE_COMB_SUB = 0, 1
CE_COMB_KERNEL_AUTO, CE_COMB_KERNEL_SIMT, CE_COMB_KERNEL_TC = 0, 1, 2


class ce_params(ctypes.Structure):
    _fields_ = [("N", c_int32), ("b", c_int32), ("stride", c_int32), ("n_sets", c_int32),
                ("r_hh", POINTER(c_double)), ("sigma2", POINTER(c_double))]


class ce_comb_params(ctypes.Structure):
    _fields_ = [("N", c_int32), ("S", c_int32), ("n_ue", c_int32), ("G", c_int32), ("mode", c_int32),
                ("r_hh", POINTER(c_double)), ("sigma2", c_double)]


lib.ce_init.argtypes = [POINTER(ce_params), POINTER(c_void_p)]
lib.ce_comb_init.argtypes = [POINTER(ce_comb_params), POINTER(c_void_p)]
lib.ce_comb_build_filters.argtypes = [c_void_p, c_void_p]
lib.ce_comb_estimate.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_void_p]
lib.ce_comb_get_filters.argtypes = [c_void_p, c_void_p]
lib.ce_comb_launch_count.argtypes = [c_void_p, POINTER(c_int64)]
lib.ce_comb_free.argtypes = [c_void_p]
lib.ce_comb_set_kernel.argtypes = [c_void_p, c_int32]
lib.ce_comb_selected_kernel.argtypes = [c_void_p, c_int32, c_int32, POINTER(c_int32)]
lib.ce_stats_workspace_bytes.argtypes = [c_int32, c_int32, c_int32, c_int32, POINTER(c_int64)]
lib.ce_stats_estimate.argtypes = [c_void_p, c_void_p, c_int32, c_int32, c_int32, c_int32, c_void_p, c_int32, c_int32,
                                  c_int32, c_void_p, c_void_p, c_void_p, c_void_p]
lib.ce_build_filters.argtypes = [c_void_p, c_void_p]
lib.ce_estimate.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_int32, c_void_p, c_void_p]
lib.ce_estimate_host.argtypes = lib.ce_estimate.argtypes
lib.ce_estimate_host_async.argtypes = lib.ce_estimate.argtypes
lib.ce_estimate_host_wait.argtypes = [c_void_p, c_void_p]
lib.ce_free.argtypes = [c_void_p]
lib.ce_set_kernel.argtypes = [c_void_p, c_int32]
lib.ce_selected_kernel.argtypes = [c_void_p, POINTER(c_int32)]
lib.ce_get_filters.argtypes = [c_void_p, c_void_p]
lib.ce_window_table.argtypes = [c_int32, c_int32, c_int32, POINTER(c_int32), c_int32]
lib.ce_launch_count.argtypes = [c_void_p, POINTER(c_int64)]
lib.ce_status_string.argtypes = [c_int]
lib.ce_status_string.restype = c_char_p
lib.ce_last_error.argtypes = []
lib.ce_last_error.restype = c_char_p
lib.ce_version.argtypes = []
lib.ce_version.restype = c_char_p
for _n in ("ce_init", "ce_build_filters", "ce_estimate", "ce_estimate_host", "ce_estimate_host_async",
           "ce_estimate_host_wait", "ce_free",
           "ce_set_kernel",
           "ce_selected_kernel",
           "ce_get_filters", "ce_window_table", "ce_launch_count", "ce_comb_init", "ce_comb_build_filters",
           "ce_comb_estimate", "ce_comb_get_filters", "ce_comb_launch_count", "ce_comb_set_kernel",
           "ce_comb_selected_kernel", "ce_comb_free"):
    getattr(lib, _n).restype = c_int


class CEError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {ce_status_string(status)} -- {ce_last_error()}")


def _check(status: int, where: str) -> int:
    if status < 0:
        raise CEError(status, where)
    return status


def ce_status_string(status: int) -> str:
    return lib.ce_status_string(status).decode()


def ce_last_error() -> str:
    return lib.ce_last_error().decode()


def ce_version() -> str:
    return lib.ce_version().decode()


def ce_window_table(N: int, b: int, stride: int):
    """Host-only window table [(a_w, o_w, o_{w+1}), ...] computed by the C++ library."""
    n = _check(lib.ce_window_table(N, b, stride, None, 0), "ce_window_table")
    buf = (c_int32 * (3 * n))()
    _check(lib.ce_window_table(N, b, stride, buf, n), "ce_window_table")
    return [(buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]) for i in range(n)]


window_table = ce_window_table


def ce_init(N: int, b: int, stride: int, r_hh, sigma2) -> int:
    """r_hh: complex [n_sets][N] (Toeplitz first columns); sigma2: float [n_sets]. Returns a handle."""
    r = np.ascontiguousarray(np.asarray(r_hh, np.complex128).reshape(-1, N))
    s2 = np.ascontiguousarray(np.asarray(sigma2, np.float64).reshape(-1))
    n_sets = r.shape[0]
    rv = r.view(np.float64)
    p = ce_params(N, b, stride, n_sets if s2.shape[0] == n_sets else -1,
                  rv.ctypes.data_as(POINTER(c_double)), s2.ctypes.data_as(POINTER(c_double)))
    h = c_void_p()
    _check(lib.ce_init(ctypes.byref(p), ctypes.byref(h)), "ce_init")
    return h.value


def ce_init_raw(N: int, b: int, stride: int, n_sets: int, r_ptr, s2_ptr) -> int:
    """Unchecked-argument variant used by the ABI validation tests; returns the status."""
    p = ce_params(N, b, stride, n_sets, ctypes.cast(r_ptr, POINTER(c_double)), ctypes.cast(s2_ptr, POINTER(c_double)))
    h = c_void_p()
    st = lib.ce_init(ctypes.byref(p), ctypes.byref(h))
    if st == CE_OK:
        lib.ce_free(h)
    return st


def ce_build_filters(h: int, stream: int = 0) -> None:
    _check(lib.ce_build_filters(h, c_void_p(stream)), "ce_build_filters")


def ce_estimate(h: int, d_y: int, d_x: int, d_h: int, T: int, M: int, K: int, d_soi: int = 0,
                stream: int = 0) -> None:
    _check(lib.ce_estimate(h, c_void_p(d_y), c_void_p(d_x), c_void_p(d_h), T, M, K,
                           c_void_p(d_soi or None), c_void_p(stream)), "ce_estimate")


def ce_estimate_host(h: int, y_ptr: int, x_ptr: int, h_ptr: int, T: int, M: int, K: int, soi_ptr: int = 0,
                     stream: int = 0) -> None:
    _check(lib.ce_estimate_host(h, c_void_p(y_ptr), c_void_p(x_ptr), c_void_p(h_ptr), T, M, K,
                                c_void_p(soi_ptr or None), c_void_p(stream)), "ce_estimate_host")


def ce_estimate_host_async(h: int, y_ptr: int, x_ptr: int, h_ptr: int, T: int, M: int, K: int, soi_ptr: int = 0,
                           stream: int = 0) -> None:
    _check(lib.ce_estimate_host_async(h, c_void_p(y_ptr), c_void_p(x_ptr), c_void_p(h_ptr), T, M, K,
                                      c_void_p(soi_ptr or None), c_void_p(stream)), "ce_estimate_host_async")


def ce_estimate_host_wait(h: int, stream: int = 0) -> None:
    _check(lib.ce_estimate_host_wait(h, c_void_p(stream)), "ce_estimate_host_wait")


def ce_free(h: int) -> None:
    _check(lib.ce_free(h), "ce_free")


def ce_set_kernel(h: int, kernel: int) -> None:
    _check(lib.ce_set_kernel(h, kernel), "ce_set_kernel")


def ce_selected_kernel(h: int) -> int:
    v = c_int32()
    _check(lib.ce_selected_kernel(h, ctypes.byref(v)), "ce_selected_kernel")
    return v.value


def ce_get_filters(h: int, n_sets: int, b: int) -> np.ndarray:
    out = np.empty((n_sets, b, b), np.complex64)
    _check(lib.ce_get_filters(h, out.ctypes.data), "ce_get_filters")
    return out


def ce_launch_count(h: int) -> int:
    v = c_int64()
    _check(lib.ce_launch_count(h, ctypes.byref(v)), "ce_launch_count")
    return v.value


class ChannelEstimator:
    """Owns one libce handle (one device).  torch tensors in, torch tensors out.

    est = ChannelEstimator(N, b, stride, r_hh, sigma2); est.build()
    h = est.estimate(y, x)            # y complex64 cuda [T][M][K][N], x [T][K][N]
    """

    def __init__(self, N: int, b: int, stride: int, r_hh, sigma2, kernel: int = CE_KERNEL_AUTO):
        self.N, self.b, self.stride = int(N), int(b), int(stride)
        self.n_sets = int(np.asarray(sigma2).reshape(-1).shape[0])
        self.handle = ce_init(N, b, stride, r_hh, sigma2)
        if kernel != CE_KERNEL_AUTO:
            ce_set_kernel(self.handle, kernel)

    def build(self, stream=None) -> "ChannelEstimator":
        ce_build_filters(self.handle, _stream_ptr(stream))
        return self

    def filters(self) -> np.ndarray:
        return ce_get_filters(self.handle, self.n_sets, self.b)

    def estimate(self, y, x, out=None, set_of_instance=None, stream=None):
        import torch
        if y.dtype != torch.complex64 or x.dtype != torch.complex64:
            raise TypeError("y and x must be complex64")
        if not (y.is_cuda and x.is_cuda):
            raise TypeError("ChannelEstimator.estimate takes CUDA tensors; use estimate_host for host arrays")
        if y.dim() != 4:
            raise ValueError(f"y must be [T][M][K][N], got shape {tuple(y.shape)}")
        T, M, K, N = y.shape
        if N != self.N or tuple(x.shape) != (T, K, N):
            raise ValueError(f"shape mismatch: y {tuple(y.shape)}, x {tuple(x.shape)}, N={self.N}")
        if not (y.is_contiguous() and x.is_contiguous()):
            raise ValueError("y and x must be contiguous")
        if x.device != y.device:
            raise ValueError("y and x must be on the same device")
        if out is None:
            out = torch.empty_like(y)
        elif (out.dtype != torch.complex64 or not out.is_cuda or out.device != y.device or
              tuple(out.shape) != tuple(y.shape) or not out.is_contiguous()):
            raise ValueError("out must be a contiguous complex64 CUDA tensor with y's shape, on y's device")
        soi = 0
        if set_of_instance is not None:
            if set_of_instance.dtype != torch.int32 or not set_of_instance.is_cuda:
                raise TypeError("set_of_instance must be a CUDA int32 tensor")
            if set_of_instance.device != y.device or not set_of_instance.is_contiguous():
                raise ValueError("set_of_instance must be contiguous and on y's device")
            if set_of_instance.numel() < T:
                raise ValueError(f"set_of_instance needs >= T = {T} entries, got {set_of_instance.numel()}")
            soi = set_of_instance.data_ptr()
        ce_estimate(self.handle, y.data_ptr(), x.data_ptr(), out.data_ptr(), T, M, K, soi, _stream_ptr(stream))
        return out

    def estimate_host(self, y, x, out=None, set_of_instance=None, stream=None, sync=True):
        """End-to-end path through ce_estimate_host: host (NumPy or pinned torch) buffers in and out.

        ce_estimate_host copies T*M*K*N elements to and from the raw host pointers, so every shape is checked
        here before the call (a mismatch would over-read y / x or over-write out).  sync=False uses
        ce_estimate_host_async: the call returns once enqueued; the host buffers (pinned) must stay alive and out
        unread until host_wait(stream) has been called and the stream has reached that point."""
        if len(tuple(y.shape)) != 4:
            raise ValueError(f"y must be [T][M][K][N], got shape {tuple(y.shape)}")
        T, M, K, N = (int(v) for v in y.shape)
        if N != self.N or tuple(int(v) for v in x.shape) != (T, K, N):
            raise ValueError(f"shape mismatch: y {tuple(y.shape)}, x {tuple(x.shape)}, N={self.N}")
        if out is None:
            out = np.empty((T, M, K, N), np.complex64)
        elif tuple(int(v) for v in out.shape) != (T, M, K, N):
            raise ValueError(f"out must have y's shape {(T, M, K, N)}, got {tuple(out.shape)}")
        soi_ptr = 0
        if set_of_instance is not None:
            set_of_instance = np.ascontiguousarray(set_of_instance, np.int32).reshape(-1)
            if set_of_instance.shape[0] < T:
                raise ValueError(f"set_of_instance needs >= T = {T} entries, got {set_of_instance.shape[0]}")
            soi_ptr = set_of_instance.ctypes.data
        fn = ce_estimate_host if sync else ce_estimate_host_async
        fn(self.handle, _host_ptr(y), _host_ptr(x), _host_ptr(out), T, M, K, soi_ptr, _stream_ptr(stream))
        if not sync:                                       # keep the host buffers of the calls in flight alive
            self._inflight = (getattr(self, "_inflight", ()) + ((y, x, out, set_of_instance),))[-2:]
        return out

    def host_wait(self, stream=None) -> None:
        """Make `stream` wait for every estimate_host(..., sync=False) call enqueued so far."""
        ce_estimate_host_wait(self.handle, _stream_ptr(stream))

    def selected_kernel(self) -> int:
        return ce_selected_kernel(self.handle)

    def launch_count(self) -> int:
        return ce_launch_count(self.handle)

    def close(self):
        if getattr(self, "handle", None):
            ce_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ce_comb_init(N: int, S: int, n_ue: int, G: int, mode: int, r_hh, sigma2: float) -> int:
    r = np.ascontiguousarray(np.asarray(r_hh, np.complex128).reshape(-1))
    if r.shape[0] != N:
        raise ValueError("r_hh must have N entries")
    rv = r.view(np.float64)
    p = ce_comb_params(N, S, n_ue, G, mode, rv.ctypes.data_as(POINTER(c_double)), float(sigma2))
    h = c_void_p()
    _check(lib.ce_comb_init(ctypes.byref(p), ctypes.byref(h)), "ce_comb_init")
    return h.value


def ce_comb_build_filters(h: int, stream: int = 0) -> None:
    _check(lib.ce_comb_build_filters(h, c_void_p(stream)), "ce_comb_build_filters")


def ce_comb_estimate(h: int, d_y: int, d_x: int, d_h: int, T: int, M: int, stream: int = 0) -> None:
    _check(lib.ce_comb_estimate(h, c_void_p(d_y), c_void_p(d_x), c_void_p(d_h), T, M, c_void_p(stream)),
           "ce_comb_estimate")


def ce_comb_free(h: int) -> None:
    _check(lib.ce_comb_free(h), "ce_comb_free")


class CombEstimator:
    """The paper's comb-pilot 3W / 12W-LMMSE (NEXT-1) on one device (libce ce_comb_* entry points).

    est = CombEstimator(N, S, n_ue, G, mode, r_hh, sigma2).build()
    h = est.estimate(y, x)     # y complex64 cuda [T][M][N], x [T][N] -> h [T][M][n_ue][N]
    """

    def __init__(self, N: int, S: int, n_ue: int, G: int, mode, r_hh, sigma2: float):
        if isinstance(mode, str):
            mode = {"full": CE_COMB_FULL, "sub": CE_COMB_SUB}[mode]
        self.N, self.S, self.n_ue, self.G, self.mode = int(N), int(S), int(n_ue), int(G), int(mode)
        self.handle = ce_comb_init(N, S, n_ue, G, mode, r_hh, sigma2)

    def build(self, stream=None) -> "CombEstimator":
        ce_comb_build_filters(self.handle, _stream_ptr(stream))
        return self

    def filters(self) -> np.ndarray:
        n_w = self.n_ue if self.mode == CE_COMB_FULL else 1
        n_out = self.S if self.mode == CE_COMB_FULL else self.G
        out = np.empty((n_w, self.G, n_out, self.G), np.complex64)
        _check(lib.ce_comb_get_filters(self.handle, out.ctypes.data), "ce_comb_get_filters")
        return out

    def estimate(self, y, x, out=None, stream=None):
        import torch
        if y.dtype != torch.complex64 or x.dtype != torch.complex64 or not (y.is_cuda and x.is_cuda):
            raise TypeError("y and x must be complex64 CUDA tensors")
        T, M, N = y.shape
        if N != self.N or tuple(x.shape) != (T, N) or not (y.is_contiguous() and x.is_contiguous()):
            raise ValueError(f"shape mismatch: y {tuple(y.shape)}, x {tuple(x.shape)}, N={self.N}")
        if out is None:
            out = torch.empty((T, M, self.n_ue, N), dtype=torch.complex64, device=y.device)
        elif (out.dtype != torch.complex64 or out.device != y.device or not out.is_contiguous()
              or tuple(out.shape) != (T, M, self.n_ue, N)):
            raise ValueError(f"out must be a contiguous complex64 tensor of shape {(T, M, self.n_ue, N)} on "
                             f"{y.device}")
        if x.device != y.device:
            raise ValueError("y and x must be on the same device")
        ce_comb_estimate(self.handle, y.data_ptr(), x.data_ptr(), out.data_ptr(), T, M, _stream_ptr(stream))
        return out

    def set_kernel(self, kernel) -> "CombEstimator":
        """CE_COMB_KERNEL_AUTO / _SIMT (K6b) / _TC (K10), or "auto" / "simt" / "tc"."""
        if isinstance(kernel, str):
            kernel = {"auto": CE_COMB_KERNEL_AUTO, "simt": CE_COMB_KERNEL_SIMT, "tc": CE_COMB_KERNEL_TC}[kernel]
        _check(lib.ce_comb_set_kernel(self.handle, int(kernel)), "ce_comb_set_kernel")
        return self

    def selected_kernel(self, T: int = 1, M: int = 1) -> int:
        """The kernel an estimate() of T instances x M antennas will use (CE_COMB_KERNEL_SIMT / _TC)."""
        v = c_int32()
        _check(lib.ce_comb_selected_kernel(self.handle, int(T), int(M), ctypes.byref(v)), "ce_comb_selected_kernel")
        return v.value

    def launch_count(self) -> int:
        v = c_int64()
        _check(lib.ce_comb_launch_count(self.handle, ctypes.byref(v)), "ce_comb_launch_count")
        return v.value

    def close(self):
        if getattr(self, "handle", None):
            ce_comb_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ce_stats_estimate(y, x, D: int, B: int, set_of_instance=None, n_sets: int = 1, stream=None):
    """NEXT-3 statistics from device tensors y [T][M][K][N], x [T][K][N] (complex64, CUDA).

    Returns (r_hat complex128 CUDA tensor [n_sets][D], sigma2_hat float64 CUDA tensor [n_sets])."""
    import torch
    if y.dtype != torch.complex64 or x.dtype != torch.complex64 or not (y.is_cuda and x.is_cuda):
        raise TypeError("y and x must be complex64 CUDA tensors")
    T, M, K, N = y.shape
    if tuple(x.shape) != (T, K, N) or not (y.is_contiguous() and x.is_contiguous()):
        raise ValueError("shape mismatch or non-contiguous input")
    soi = 0
    if set_of_instance is not None:
        if set_of_instance.dtype != torch.int32 or not set_of_instance.is_cuda:
            raise TypeError("set_of_instance must be a CUDA int32 tensor")
        soi = set_of_instance.data_ptr()
    nb = c_int64()
    _check(lib.ce_stats_workspace_bytes(N, n_sets, D, B, ctypes.byref(nb)), "ce_stats_workspace_bytes")
    work = torch.empty(nb.value // 8, dtype=torch.float64, device=y.device)
    r = torch.empty((n_sets, D), dtype=torch.complex128, device=y.device)
    s2 = torch.empty((n_sets,), dtype=torch.float64, device=y.device)
    _check(lib.ce_stats_estimate(c_void_p(y.data_ptr()), c_void_p(x.data_ptr()), T, M, K, N, c_void_p(soi or None),
                                 n_sets, D, B, c_void_p(r.data_ptr()), c_void_p(s2.data_ptr()),
                                 c_void_p(work.data_ptr()), c_void_p(_stream_ptr(stream))), "ce_stats_estimate")
    return r, s2


def _host_ptr(a) -> int:
    """Pointer of a C-contiguous complex64 host array (NumPy, or a CPU / pinned torch tensor)."""
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"] or a.dtype != np.complex64:
            raise ValueError("host arrays must be C-contiguous complex64")
        return a.ctypes.data
    import torch
    if not isinstance(a, torch.Tensor) or a.is_cuda or not a.is_contiguous() or a.dtype != torch.complex64:
        raise ValueError("host tensors must be contiguous complex64 CPU tensors")
    return a.data_ptr()


def _stream_ptr(stream) -> int:
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except ImportError:
            pass
        return 0
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream
