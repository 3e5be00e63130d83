"""Oracle for arXiv 1802.05427's block-LMMSE pilot channel estimator.

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline / reference legs.  The product package
(paper_1802_05427_b200) never imports it.  See oracle/lmmse.py.
"""
from .lmmse import (  # noqa: F401
    block_apply,
    block_filter,
    block_lmmse,
    block_lmmse_general,
    block_mse,
    block_mse_per_tone,
    error_cov,
    full_lmmse,
    full_lmmse_general,
    full_mse_per_tone,
    lmmse_filter,
    ls_estimate,
    rd_uniform,
    rel_fro_error_per_instance,
    toeplitz_hermitian,
    window_table,
)
from .comb import (  # noqa: F401
    comb_estimate,
    comb_filters,
    comb_full_lmmse,
    comb_geometry,
    comb_ls,
    comb_mse_per_tone,
    comb_out_tones,
    rect_filter,
    zoh_fill,
)
from .stats import (  # noqa: F401,E402
    correlation_estimate,
    estimate_stats,
    ls_rows,
    mismatched_block_mse,
    noise_bins,
    noise_variance_estimate,
)
