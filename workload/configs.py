"""The five BASELINE.json presets (BASELINE.json "configs").

Notation follows BASELINE.json: M = BS antennas (paper's R),
K = users (paper's S), N = used subcarriers, L = PDP tap count (paper's M).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Tuple


@dataclass(frozen=True)
class Config:
    cfg_id: int
    name: str
    M: int                 # BS antennas
    K: int                 # users (time-orthogonal pilots, one symbol per user)
    N: int                 # used subcarriers, contiguous tones 0..N-1 (reading A10)
    Nfft: int
    slots: int
    pilots_per_slot: int   # estimation instances per slot (reading A3)
    b: int                 # block / window length
    stride: int            # window stride s (== b: non-overlapping)
    n_taps: int            # L, exponential PDP tap count (3 dB/tap, reading A6)
    tap_spacing: Optional[float] = None            # fixed delay spacing in samples (configs 1-2)
    tau_rms_s: Optional[float] = None              # fixed rms delay spread (configs 3, 5)
    tau_rms_range_s: Optional[Tuple[float, float]] = None  # per-slot U[lo, hi] (config 4)
    fs_hz: Optional[float] = None                  # sampling rate Nfft * subcarrier spacing
    snr_db: Optional[float] = None                 # fixed SNR
    snr_choice_db: Optional[Tuple[float, ...]] = None      # per-slot choice (config 2)
    snr_range_db: Optional[Tuple[float, float]] = None     # per-slot U[lo, hi] (config 4)
    per_slot_stats: bool = False                   # reading A4: matched per-slot statistics

    @property
    def T(self) -> int:
        """Estimation instances = slots x pilot symbols per slot."""
        return self.slots * self.pilots_per_slot

    @property
    def n_sets(self) -> int:
        return self.slots if self.per_slot_stats else 1

    @property
    def cols(self) -> int:
        return self.M * self.K

    @property
    def estimates(self) -> int:
        """E = M*K*N*T channel estimates (antenna x user x subcarrier x instance)."""
        return self.M * self.K * self.N * self.T


CONFIGS = {
    1: Config(1, "tiny", M=8, K=2, N=72, Nfft=128, slots=1, pilots_per_slot=1,
              b=12, stride=12, n_taps=4, tap_spacing=1.0, snr_db=10.0),
    2: Config(2, "small", M=32, K=4, N=300, Nfft=512, slots=2, pilots_per_slot=1,
              b=50, stride=25, n_taps=8, tap_spacing=1.0,
              snr_choice_db=(0.0, 10.0, 20.0), per_slot_stats=True),
    3: Config(3, "paper", M=128, K=12, N=1200, Nfft=2048, slots=1, pilots_per_slot=1,
              b=100, stride=100, n_taps=16, tau_rms_s=1e-6, fs_hz=30.72e6, snr_db=15.0),
    4: Config(4, "paper_batched", M=128, K=12, N=1200, Nfft=2048, slots=20, pilots_per_slot=2,
              b=150, stride=100, n_taps=16, tau_rms_range_s=(0.3e-6, 2e-6), fs_hz=30.72e6,
              snr_range_db=(0.0, 25.0), per_slot_stats=True),
    5: Config(5, "scale_out", M=256, K=24, N=3276, Nfft=4096, slots=20, pilots_per_slot=1,
              b=126, stride=126, n_taps=24, tau_rms_s=0.5e-6, fs_hz=122.88e6, snr_db=20.0),
    # NEXT-2: the full-band LMMSE the paper calls infeasible on its CPU,
    # b = N on config 3's statistics -- one 1200 x 1200 filter, tensor-bound.
    6: Config(6, "full_band", M=128, K=12, N=1200, Nfft=2048, slots=1, pilots_per_slot=1,
              b=1200, stride=1200, n_taps=16, tau_rms_s=1e-6, fs_hz=30.72e6, snr_db=15.0),
}


def get_config(cfg) -> Config:
    if isinstance(cfg, Config):
        return cfg
    if isinstance(cfg, str):
        for c in CONFIGS.values():
            if c.name == cfg:
                return c
        return CONFIGS[int(cfg)]
    return CONFIGS[int(cfg)]


# ------------------------------------------------------------------------------------------------
# NEXT-1: the paper's comb-pilot grouped estimators (3W / 12W-LMMSE, Tables I-II).
# Channel per Table III: 6 taps at delays 0..5 samples (Nfft rate) with powers
# [-2, -8, -10, -12, -15, -18] dB.  The estimator uses the paper's FIXED design: r_d of Eq. eqrd with
# the assumed path count L (reading A5: normalised by Nfft) and SNR_fixed
# (Table III: L = 8, 40 dB).
# ------------------------------------------------------------------------------------------------
@dataclass(frozen=True)
class CombConfig:
    name: str
    M: int                 # BS antennas (paper's R)
    S: int                 # comb spacing = pilot-interleaved UE slots (12 in Fig. fig1)
    n_ue: int              # active UEs estimated (the first n_ue comb offsets; 4 in Table III)
    N: int
    Nfft: int
    T: int                 # estimation instances (slots)
    G: int                 # pilots per group window (12 -> 12W, 3 -> 3W)
    mode: str              # "full" (12W: every tone) or "sub" (3W: G tones per group, then ZOH)
    tap_delays: Tuple[float, ...] = (0, 1, 2, 3, 4, 5)
    tap_db: Tuple[float, ...] = (-2, -8, -10, -12, -15, -18)
    snr_db: float = 25.0   # true SNR of the synthetic channel
    L_assumed: float = 8.0
    snr_fixed_db: float = 40.0

    @property
    def K(self) -> int:
        return self.N // self.S

    @property
    def estimates(self) -> int:
        return self.T * self.M * self.n_ue * self.N


COMB_CONFIGS = {
    "comb_tiny12": CombConfig("comb_tiny12", M=4, S=4, n_ue=4, N=96, Nfft=128, T=2, G=4, mode="full",
                              tap_delays=(0, 1, 2), tap_db=(-1, -6, -9), snr_db=10.0, L_assumed=4.0,
                              snr_fixed_db=20.0),
    "comb_tiny3": CombConfig("comb_tiny3", M=3, S=6, n_ue=3, N=96, Nfft=128, T=2, G=3, mode="sub",
                             tap_delays=(0, 1, 2), tap_db=(-1, -6, -9), snr_db=10.0, L_assumed=4.0,
                             snr_fixed_db=20.0),
    "comb_small12": CombConfig("comb_small12", M=9, S=12, n_ue=5, N=288, Nfft=512, T=2, G=12, mode="full"),
    "comb_small3": CombConfig("comb_small3", M=5, S=12, n_ue=7, N=240, Nfft=512, T=2, G=3, mode="sub"),
    "paper_12w": CombConfig("paper_12w", M=16, S=12, n_ue=4, N=1200, Nfft=2048, T=18, G=12, mode="full"),
    "paper_3w": CombConfig("paper_3w", M=16, S=12, n_ue=4, N=1200, Nfft=2048, T=18, G=3, mode="sub"),
    "massive_12w": CombConfig("massive_12w", M=128, S=12, n_ue=12, N=1200, Nfft=2048, T=20, G=12,
                              mode="full"),
}


def get_comb_config(name) -> CombConfig:
    return name if isinstance(name, CombConfig) else COMB_CONFIGS[name]
