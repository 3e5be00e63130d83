"""DRAM traffic per launch over a range of back-to-back ce_estimate calls (for roofline.traffic).

    ncu --replay-mode range --profile-from-start off \
        --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
        python tools/traffic_range.py --config 3 --kernel 3 --steps 50

A single-launch `ncu --set full` capture misses the write-back of that launch's output (it stays dirty in L2 until
later traffic evicts it); summed over a range of launches on rotating buffers larger than L2, read + write / steps
is the steady-state DRAM traffic of one launch.  The range is bracketed by cudaProfilerStart / Stop."""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workload  # noqa: E402
import paper_1802_05427_b200 as ce  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--kernel", type=int, default=0)
    ap.add_argument("--steps", type=int, default=50)
    a = ap.parse_args()
    cfg = workload.get_config(a.config)
    r, s2 = workload.channel_stats(cfg, 0)
    est = ce.ChannelEstimator(cfg.N, cfg.b, cfg.stride, r, s2, kernel=a.kernel).build()
    x = torch.from_numpy(workload.gen_pilots(cfg, 0)).cuda()
    soi = torch.from_numpy(workload.set_of_instance(cfg)).cuda()
    shape = (cfg.T, cfg.M, cfg.K, cfg.N)
    nbuf = max(2, int(np.ceil(1.25 * 126 * 2**20 / (16 * np.prod(shape)))) + 1)
    ys = [torch.randn(shape, dtype=torch.complex64, device="cuda") for _ in range(nbuf)]
    hs = [torch.empty_like(ys[0]) for _ in range(nbuf)]
    for i in range(2 * nbuf):
        est.estimate(ys[i % nbuf], x, out=hs[i % nbuf], set_of_instance=soi)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    for i in range(a.steps):
        est.estimate(ys[i % nbuf], x, out=hs[i % nbuf], set_of_instance=soi)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print(f"kernel {est.selected_kernel()} steps {a.steps} nbuf {nbuf} algorithmic bytes per launch "
          f"{16 * cfg.estimates + 8 * cfg.T * cfg.K * cfg.N}")
    est.close()


if __name__ == "__main__":
    main()
