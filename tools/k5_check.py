"""K5 (CTA pair, filter in TMEM) bring-up: parity vs the oracle on small shapes, then K4 vs K5 device times.
Run under `timeout` on the GPU box: python tools/k5_check.py [--time]"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import workload  # noqa: E402
import paper_1802_05427_b200 as ce  # noqa: E402
from _parity import row_rel_err_max  # noqa: E402


def run(N, b, s, r, s2, y, x, soi, kernel):
    est = ce.ChannelEstimator(N, b, s, r, s2, kernel=kernel).build()
    soi_t = None if soi is None else torch.from_numpy(np.ascontiguousarray(soi, np.int32)).cuda()
    h = est.estimate(torch.from_numpy(y).cuda(), torch.from_numpy(x).cuda(), set_of_instance=soi_t)
    torch.cuda.synchronize()
    sel = est.selected_kernel()
    est.close()
    return h.cpu().numpy(), sel


def rand_problem(N, b, M, K, T, seed):
    rng = np.random.default_rng(seed)
    p = np.exp(-np.arange(6) / 2.5)
    p /= p.sum()
    tau = np.sort(rng.uniform(0, 12, 6))
    r = (p[None] * np.exp(-2j * np.pi * np.outer(np.arange(N), tau) / (2 * N))).sum(1)[None]
    y = (rng.standard_normal((T, M, K, N)) + 1j * rng.standard_normal((T, M, K, N))).astype(np.complex64)
    x = (np.exp(2j * np.pi * rng.random((T, K, N))) * rng.uniform(0.5, 2.0, (T, K, N))).astype(np.complex64)
    return r, np.array([0.03]), y, x


def check(name, N, b, s, r, s2, y, x, soi, kernel=4):
    t0 = time.time()
    h, sel = run(N, b, s, r, s2, y, x, soi, kernel)
    ref = oracle.block_lmmse(y, x, r, s2, soi, b, s)
    err = oracle.rel_fro_error_per_instance(h, ref).max()
    row = row_rel_err_max(h, ref, N, b, s)
    ok = err <= 1e-4 and row <= 1e-3 and np.isfinite(h).all()
    print(f"{'OK  ' if ok else 'FAIL'} {name}: kernel {sel} inst {err:.2e} row {row:.2e} ({time.time() - t0:.1f}s)",
          flush=True)
    if not ok:
        d = np.abs(h - ref)
        idx = np.unravel_index(np.nanargmax(d), d.shape)
        print("   worst at", idx, h[idx], ref[idx], "nan count", np.isnan(h).sum(), flush=True)
    return ok


CASES = [("cfg", 3, 16), ("cfg", 1, None), ("cfg", 4, 8), ("cfg", 5, 4),
         ("rand", (1200, 12, 12, 8, 12, 1)), ("rand", (40, 2, 2, 6, 3, 1)), ("rand", (300, 100, 50, 11, 7, 2)),
         ("rand", (96, 96, 96, 2, 3, 1)), ("rand", (1200, 150, 100, 4, 12, 1)), ("rand", (400, 200, 200, 3, 5, 1))]


def run_case(i):
    c = CASES[i]
    if c[0] == "cfg":
        cid, mh = c[1], c[2]
        cfg = workload.get_config(cid)
        r, s2 = workload.channel_stats(cfg, 0)
        x = workload.gen_pilots(cfg, 0)
        T = min(cfg.T, 4)
        y = workload.gen_instances(cfg, 0, x=x, m_hi=mh, t_hi=T)
        soi = workload.set_of_instance(cfg)[:T]
        return check(f"config{cid}", cfg.N, cfg.b, cfg.stride, r, s2, y, x[:T], soi)
    N, b, s, M, K, T = c[1]
    r, s2, y, x = rand_problem(N, b, M, K, T, N + b)
    return check(f"N{N} b{b} s{s} M{M} K{K} T{T}", N, b, s, r, s2, y, x, None)


def main():
    torch.cuda.set_device(0)
    if "--case" in sys.argv:
        ok = run_case(int(sys.argv[sys.argv.index("--case") + 1]))
        sys.exit(0 if ok else 1)
    import subprocess
    ok = True
    for i in range(len(CASES)):      # one process per case: a fault in one does not hide the others
        res = subprocess.run([sys.executable, __file__, "--case", str(i)], capture_output=True, text=True, timeout=120)
        print(res.stdout.strip() or f"case {i}: rc {res.returncode} {res.stderr.strip().splitlines()[-1:]}", flush=True)
        ok &= res.returncode == 0
    print("K5 parity", "OK" if ok else "FAILED", flush=True)
    if "--time" in sys.argv and ok:
        for cid in (3, 4, 5):
            cfg = workload.get_config(cid)
            r, s2 = workload.channel_stats(cfg, 0)
            x_d = torch.from_numpy(workload.gen_pilots(cfg, 0)).cuda()
            soi_d = torch.from_numpy(workload.set_of_instance(cfg)).cuda()
            shape = (cfg.T, cfg.M, cfg.K, cfg.N)
            nbuf = max(2, int(np.ceil(1.25 * 126 * 2**20 / (16 * np.prod(shape)))) + 1)
            ys = [torch.randn(shape, dtype=torch.complex64, device="cuda") for _ in range(nbuf)]
            hs = [torch.empty_like(ys[0]) for _ in range(nbuf)]
            for kern in (3, 4):
                est = ce.ChannelEstimator(cfg.N, cfg.b, cfg.stride, r, s2, kernel=kern).build()
                steps = 200 if cid == 3 else 20
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
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) * 1e3 / steps
                frac = 16 * cfg.estimates / (us * 1e-6) / 6556.2e9
                print(f"config{cid} kernel {est.selected_kernel()}: {us:.2f} us/step, HBM frac {frac:.3f}", flush=True)
                est.close()
                del g
            del ys, hs
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
