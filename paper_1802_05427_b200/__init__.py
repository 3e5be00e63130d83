"""B200-native block-LMMSE pilot channel estimator (arXiv 1802.05427).

The product path: libce.so (include/ce.h; CUDA kernels for sm_100a) behind a thin
ctypes binding with the same function names.  No CPU fallback, no oracle import.
"""
from .ce import (  # noqa: F401
    CE_COMB_FULL,
    CE_COMB_KERNEL_AUTO,
    CE_COMB_KERNEL_SIMT,
    CE_COMB_KERNEL_TC,
    CE_COMB_SUB,
    CE_EINVAL,
    CE_ENODEV,
    CE_ENOMEM,
    CE_ENOTPD,
    CE_ESTATE,
    CE_KERNEL_AUTO,
    CE_KERNEL_BF16X3,
    CE_KERNEL_SIMT,
    CE_KERNEL_TF32X3,
    CE_OK,
    EXPORTED,
    CEError,
    ChannelEstimator,
    CombEstimator,
    ce_build_filters,
    ce_comb_build_filters,
    ce_comb_estimate,
    ce_comb_free,
    ce_comb_init,
    ce_estimate,
    ce_estimate_host,
    ce_estimate_host_async,
    ce_estimate_host_wait,
    ce_free,
    ce_get_filters,
    ce_init,
    ce_last_error,
    ce_launch_count,
    ce_selected_kernel,
    ce_set_kernel,
    ce_stats_estimate,
    ce_status_string,
    ce_version,
    ce_window_table,
    window_table,
)

__version__ = "0.1.0"
