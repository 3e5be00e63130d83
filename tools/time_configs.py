"""Device time of ce_estimate on configs 3/4/5 (CUDA-graph replay over rotating > L2 buffers, device-drawn y),
one line per config; env vars select kernel experiments.  python tools/time_configs.py [kernel] [configs]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workload  # noqa: E402
import paper_1802_05427_b200 as ce  # noqa: E402


def time_cfg(cid, kernel, reps=3):
    cfg = workload.get_config(cid)
    r, s2 = workload.channel_stats(cfg, 0)
    x_d = torch.from_numpy(workload.gen_pilots(cfg, 0)).cuda()
    soi_d = torch.from_numpy(workload.set_of_instance(cfg)).cuda()
    shape = (cfg.T, cfg.M, cfg.K, cfg.N)
    nbuf = max(2, int(np.ceil(1.25 * 126 * 2**20 / (16 * np.prod(shape)))) + 1)
    ys = [torch.randn(shape, dtype=torch.complex64, device="cuda") for _ in range(nbuf)]
    hs = [torch.empty_like(ys[0]) for _ in range(nbuf)]
    est = ce.ChannelEstimator(cfg.N, cfg.b, cfg.stride, r, s2, kernel=kernel).build()
    steps = 400 if cid == 3 else (40 if cid == 4 else 10)
    for i in range(nbuf + 3):
        est.estimate(ys[i % nbuf], x_d, out=hs[i % nbuf], set_of_instance=soi_d)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            for i in range(steps):
                est.estimate(ys[i % nbuf], x_d, out=hs[i % nbuf], set_of_instance=soi_d, stream=st)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / steps)
    frac = (16 * cfg.estimates + 8 * cfg.T * cfg.K * cfg.N) / (best * 1e-6) / 6556.2e9
    sel = est.selected_kernel()
    est.close()
    del g, ys, hs
    torch.cuda.empty_cache()
    return best, frac, sel


if __name__ == "__main__":
    kernel = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    cfgs = [int(c) for c in sys.argv[2].split(",")] if len(sys.argv) > 2 else [3, 4, 5]
    tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("CE_"))
    for cid in cfgs:
        us, frac, sel = time_cfg(cid, kernel)
        print(f"config{cid} kernel {sel} [{tag}]: {us:8.2f} us/step  HBM frac {frac:.3f}", flush=True)
