"""Multi-rank host logic of the antenna-sharded path on CPU with gloo, world size 2.

The estimate on each rank is the oracle's (a stand-in for the per-rank ce_estimate, which needs a
GPU): what is tested is the partition, the per-rank seeded generation of an antenna block, and the
gather + reassembly that the verification path uses.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_1802_05427_b200.shard import antenna_shard, gather_antenna_shards, shard_table  # noqa: E402


@pytest.mark.parametrize("M,world", [(128, 8), (5, 2), (3, 4), (256, 8), (1, 1), (7, 3)])
def test_shard_table_partitions(M, world):
    blocks = shard_table(M, world)
    covered = [m for lo, hi in blocks for m in range(lo, hi)]
    assert covered == list(range(M))
    sizes = [hi - lo for lo, hi in blocks]
    assert max(sizes) - min(sizes) <= 1


def test_shard_bad_args():
    with pytest.raises(ValueError):
        antenna_shard(8, 0, 0)
    with pytest.raises(ValueError):
        antenna_shard(8, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg_id, M_total, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import dataclasses

        import oracle
        import workload
        cfg = dataclasses.replace(workload.get_config(cfg_id), M=M_total)
        r, s2 = workload.channel_stats(cfg, 0)
        soi = workload.set_of_instance(cfg)
        x = workload.gen_pilots(cfg, 0)
        lo, hi = antenna_shard(M_total, world, rank)
        y_loc = workload.gen_instances(cfg, 0, m_lo=lo, m_hi=hi, x=x)
        h_loc = oracle.block_lmmse(y_loc, x, r, s2, soi, cfg.b, cfg.stride).astype(np.complex64)
        full = gather_antenna_shards(torch.from_numpy(h_loc), M_total)
        if rank == 0:
            y = workload.gen_instances(cfg, 0, x=x)
            assert np.array_equal(y[:, lo:hi], y_loc)            # shard draws == slice of the full draw
            ref = oracle.block_lmmse(y, x, r, s2, soi, cfg.b, cfg.stride).astype(np.complex64)
            err = np.abs(full.numpy() - ref).max()
            q.put(("ok", float(err), tuple(full.shape)))
        dist.barrier()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(("fail", repr(e), None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg_id,M_total", [(2, 32), (1, 5)])
def test_gloo_world2_gather_matches_full(cfg_id, M_total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, cfg_id, M_total, q), nprocs=2, join=True, start_method="spawn")
    status, err, shape = q.get(timeout=60)
    assert status == "ok", err
    assert err < 1e-6
    assert shape[1] == M_total
