"""Antenna sharding across ranks -- host logic only.

Antennas are independent and the filters depend only on the statistics, not on the
antenna (Eq. 17: the weights bear "no relation with the receiving
antennas"), so the estimator shards by antenna with no collective on the hot path.
Each rank owns a contiguous antenna block [m_lo, m_hi) of every instance and runs
ce_estimate on its own [T][m_hi-m_lo][K][N] tensors.

The only collective is the optional verification gather of the estimate shards
(torch.distributed all-gather: NCCL on GPUs, gloo in the CPU tests), outside any
timed region.
"""
from __future__ import annotations

from typing import List, Tuple


def antenna_shard(M_total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block [m_lo, m_hi) of antennas owned by `rank`; blocks partition [0, M_total).

    The first M_total % world ranks own one extra antenna (ragged split allowed)."""
    if world < 1 or not (0 <= rank < world) or M_total < 0:
        raise ValueError("need world >= 1, 0 <= rank < world, M_total >= 0")
    q, r = divmod(M_total, world)
    m_lo = rank * q + min(rank, r)
    return m_lo, m_lo + q + (1 if rank < r else 0)


def shard_table(M_total: int, world: int) -> List[Tuple[int, int]]:
    return [antenna_shard(M_total, world, g) for g in range(world)]


def gather_antenna_shards(h_local, M_total: int, group=None):
    """All-gather every rank's estimate shard h_local [T][m_g][K][N] (complex64, any device)
    and reassemble the full [T][M_total][K][N] tensor on every rank.

    Shards may be ragged: each is zero-padded to the largest block, gathered as float32
    (gloo has no complex dtype), and the padding is dropped on reassembly."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    blocks = shard_table(M_total, world)
    T, m_loc, K, N = h_local.shape
    rank = dist.get_rank(group)
    if m_loc != blocks[rank][1] - blocks[rank][0]:
        raise ValueError(f"rank {rank}: shard has {m_loc} antennas, expected {blocks[rank]}")
    m_max = max(hi - lo for lo, hi in blocks)
    pad = torch.zeros((T, m_max, K, N, 2), dtype=torch.float32, device=h_local.device)
    pad[:, :m_loc] = torch.view_as_real(h_local)
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    full = torch.empty((T, M_total, K, N, 2), dtype=torch.float32, device=h_local.device)
    for g, (lo, hi) in enumerate(blocks):
        full[:, lo:hi] = parts[g][:, :hi - lo]
    return torch.view_as_complex(full)
