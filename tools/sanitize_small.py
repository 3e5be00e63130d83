"""Tiny end-to-end run of every kernel for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

usage: compute-sanitizer --tool memcheck python tools/sanitize_small.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1802_05427_b200 as ce  # noqa: E402
import workload  # noqa: E402


def main():
    torch.cuda.set_device(0)
    for cfg_id in (1, 2):
        cfg = workload.get_config(cfg_id)
        r, s2 = workload.channel_stats(cfg, 0)
        x = workload.gen_pilots(cfg, 0)
        y = workload.gen_instances(cfg, 0, x=x)
        soi = torch.from_numpy(workload.set_of_instance(cfg)).cuda()
        for k in (1, 2, 3, 4):
            est = ce.ChannelEstimator(cfg.N, cfg.b, cfg.stride, r, s2)
            try:
                ce.ce_set_kernel(est.handle, k)
            except ce.CEError:
                est.close()
                continue
            est.build()
            h = est.estimate(torch.from_numpy(y).cuda(), torch.from_numpy(x).cuda(), set_of_instance=soi)
            torch.cuda.synchronize()
            print(f"config {cfg_id} kernel {k} -> {est.selected_kernel()} ok {float(h.abs().mean()):.4f}", flush=True)
            est.close()
    for name in ("comb_tiny12", "comb_tiny3", "comb_small12", "comb_small3"):
        cfg = workload.get_comb_config(name)
        r, s2 = workload.comb_stats(cfg)
        x = workload.comb_pilots(cfg)
        y = workload.comb_instances(cfg, x=x)
        est = ce.CombEstimator(cfg.N, cfg.S, cfg.n_ue, cfg.G, cfg.mode, r, s2).build()
        h = est.estimate(torch.from_numpy(y).cuda(), torch.from_numpy(x).cuda())
        torch.cuda.synchronize()
        print(f"comb {name} ok {float(h.abs().mean()):.4f}", flush=True)
        est.close()


if __name__ == "__main__":
    main()
