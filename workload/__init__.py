"""Seeded synthetic workload generator shared by the oracle and the GPU path.

This package holds NO estimator arithmetic (no LS division, no filter build, no
block apply).  It only draws the inputs the estimator consumes:

* the received pilot symbols ``y`` and the pilots ``x`` (Eq. 5),
* the per-set channel statistics ``r[d]`` (first column of the Toeplitz R_hh,
  PAPER.md:287 "only depends on the difference") and ``sigma2``.

Recipe: SURVEY.md §8(d) "Synthetic inputs" and the readings A3/A4/A6/A12 of
SURVEY.md §8(c), restated in DESIGN.md §3.
"""
from .configs import COMB_CONFIGS, CONFIGS, CombConfig, Config, get_comb_config, get_config  # noqa: F401
from .gen import (  # noqa: F401
    channel_stats,
    gen_instances,
    gen_pilots,
    pdp,
    rms_spread_taps,
    set_of_instance,
)
from .comb import comb_instances, comb_pilots, comb_stats, comb_true_stats  # noqa: F401,E402
