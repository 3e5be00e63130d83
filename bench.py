#!/usr/bin/env python
"""Benchmark of the block-LMMSE pilot channel estimator (arXiv 1802.05427 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

One step = one pass of the hot path (LS + block-LMMSE contraction, a3-a5 of SURVEY.md §8(a))
over one estimation batch of the configured workload (default: config 3, the paper-scale
128 x 12 x 1200 slot, b = 100).  The filters W_b (a1-a2) are per-statistics, precomputed
before the slot loop exactly as the paper does offline; their
build time is reported separately as `filter_build_ms`.

Multi-GPU (`--gpus N`: spawned through torch.distributed.run unless a launcher already set WORLD_SIZE; one rank
per GPU): each rank estimates its own antenna block with no data-path collective -> weak scaling by default (the
task's rule for independent units), `--strong` splits the configuration's own antennas; at N > 1 the line also
carries the strong-scaled record of the same configuration and the config 4 / 5 sweep split across the ranks.
Time = max over ranks of CUDA-event time on the launching stream.

Prints ONE JSON line (rank 0).  See DESIGN.md §7 for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workload  # noqa: E402  (seeded input generator: no estimator arithmetic)

L2_BYTES = 126 * 1024 * 1024


def _peaks():
    """MEASURED_PEAKS.json (driver-written: HBM copy, cuBLAS bf16) plus the committed FFMA microbenchmark
    (profiles/ffma_peak_r02.json, tools/ffma_peak.cu run on this pool's B200s) as fp32_tflops."""
    d = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
    except Exception:
        pass
    try:
        with open(os.path.join(ROOT, "profiles", "ffma_peak_r02.json")) as f:
            d["fp32_tflops"] = float(json.load(f)["fp32_tflops_burst"])
    except Exception:
        pass
    return d


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
    }

    def __init__(self, device_index: int, period_s: float = 0.005):
        self.samples, self.reasons = [], set()
        self.period = period_s
        self._stop = threading.Event()
        self.ok = False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False

    def _run(self):
        nv = self.nvml
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _spawn(args) -> int:
    """`bench.py --gpus N` without a launcher: re-exec through torch.distributed.run, one rank per GPU."""
    import socket
    import subprocess
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


class Dist:
    """torch.distributed plumbing for the bench: device per rank, barrier, max over ranks, gather of shards.

    NCCL over NVLink on a multi-GPU node (one GPU per rank); `--backend gloo` lets several ranks share one GPU
    (the 2-rank test on a single leased B200) -- the data path has no collective either way."""

    def __init__(self, backend: str):
        import torch
        import torch.distributed as dist
        self.world, self.rank, self.local = _dist_env()
        if not torch.cuda.is_available():
            raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
        self.dev = torch.device("cuda", self.local % torch.cuda.device_count())
        torch.cuda.set_device(self.dev)
        self.backend = backend
        self.dist = dist
        if self.world > 1:
            if backend == "nccl":
                dist.init_process_group("nccl", device_id=self.dev)
            else:
                dist.init_process_group("gloo")

    def _coll(self, t):
        return t if self.backend == "nccl" else t.cpu()

    def barrier(self):
        if self.world > 1:
            if self.backend == "nccl":
                self.dist.barrier(device_ids=[self.dev.index])
            else:
                self.dist.barrier()

    def max(self, v: float) -> float:
        import torch
        if self.world == 1:
            return float(v)
        t = self._coll(torch.tensor([float(v)], dtype=torch.float64, device=self.dev))
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def all_values(self, v: float):
        import torch
        if self.world == 1:
            return [float(v)]
        t = self._coll(torch.tensor([float(v)], dtype=torch.float64, device=self.dev))
        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t)
        return [float(p.item()) for p in parts]

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def _cfg_json(cfg, extra):
    d = {"workload": f"config{cfg.cfg_id}_{cfg.name}_{cfg.M}x{cfg.K}x{cfg.N}_T{cfg.T}_b{cfg.b}_s{cfg.stride}",
         "M": cfg.M, "K": cfg.K, "N": cfg.N, "T": cfg.T, "b": cfg.b, "stride": cfg.stride,
         "n_sets": cfg.n_sets}
    d.update(extra)
    return d


def _cores():
    for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        if os.environ.get(var):
            return int(os.environ[var])
    return len(os.sched_getaffinity(0))


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def _blas_vendor() -> str:
    try:
        cfg = np.show_config(mode="dicts")
        b = cfg["Build Dependencies"]["blas"]
        return f"{b.get('name')} {b.get('version', '')}".strip()
    except Exception:
        return "unknown"


def _oracle_sample_timing(cfg, x, y, r, s2, soi, budget_s: float, threads=None, min_runs: int = 3):
    """Per-run times of the oracle's LS + block apply (no generation, no filter build) on (y, x): a list of
    seconds, >= min_runs runs and about budget_s in total; `threads` caps the BLAS pool (threadpoolctl)."""
    import contextlib

    import oracle
    filters = {}
    for st in set(int(v) for v in soi):
        filters[st] = [oracle.block_filter(r[st], s2[st], cfg.b)] * len(oracle.window_table(cfg.N, cfg.b, cfg.stride))
    ctx = contextlib.nullcontext()
    if threads is not None:
        from threadpoolctl import threadpool_limits
        ctx = threadpool_limits(limits=threads)
    times, out = [], None
    with ctx:
        t_start = time.perf_counter()
        while True:
            t0 = time.perf_counter()
            H_ls = oracle.ls_estimate(y, x)
            out = np.stack([oracle.block_apply(H_ls[t], filters[int(soi[t])], cfg.b, cfg.stride)
                            for t in range(y.shape[0])])
            times.append(time.perf_counter() - t0)
            if len(times) >= min_runs and time.perf_counter() - t_start >= budget_s:
                break
    return times, out


def run_reference(args, cfg):
    """--impl reference: the CPU oracle (the slow program the ratio divides by), rank 0 only."""
    world, rank, _ = _dist_env()
    if rank != 0:
        return
    x = workload.gen_pilots(cfg, 0)
    r, s2 = workload.channel_stats(cfg, 0)
    soi = workload.set_of_instance(cfg)
    # bounded sample: antennas [0, m) of instance 0, sized for <= ~0.03 s of oracle work per step
    m = max(1, min(cfg.M, args.ref_antennas))
    y = workload.gen_instances(cfg, 0, t_lo=0, t_hi=1, m_lo=0, m_hi=m, x=x[:1])
    import oracle
    filters = [oracle.block_filter(r[soi[0]], s2[soi[0]], cfg.b)] * len(oracle.window_table(cfg.N, cfg.b, cfg.stride))

    def step():
        H_ls = oracle.ls_estimate(y, x[:1])
        oracle.block_apply(H_ls[0], filters, cfg.b, cfg.stride)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    est = m * cfg.K * cfg.N
    value = est * args.steps / el
    sample = (f"oracle LS+block apply (complex128 NumPy, {_blas_vendor()}) on antennas [0,{m}) of config "
              f"{cfg.cfg_id} instance 0 per step")
    line = {
        "impl": "reference", "metric": "channel estimates/s (antenna*user*subcarrier)", "value": value,
        "unit": "estimates/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128 (oracle)", "data": "synthetic (seeded workload generator)",
        "config": _cfg_json(cfg, {"sample_antennas": m}),
        "cpu_baseline": {"value": value, "unit": "estimates/s", "cores": _cores(), "kind": "oracle",
                         "sample": sample, "cpu_model": _cpu_model(), "blas": _blas_vendor()},
        "e2e": {"value": value, "unit": "estimates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


KERNEL_NAMES = {0: "auto", 1: "k2_simt", 2: "k3_tf32x3", 3: "k4_bf16x3"}
KERNEL_DTYPE = {1: "c64 I/O, fp32 SIMT products, fp32 accumulate",
                2: "c64 I/O, tf32x3 (error-compensated) products, fp32 accumulate",
                3: "c64 I/O, bf16x3 (error-compensated) products, fp32 accumulate"}


def _rotating_buffers(make_y, step_bytes: int, dev):
    """nbuf (y, h) pairs whose total exceeds the 126 MB L2 (inputs larger than L2 between timed steps)."""
    import torch
    nbuf = max(2, int(np.ceil(1.25 * L2_BYTES / step_bytes)) + 1)
    y0 = make_y()
    ys = [y0] + [y0.clone() for _ in range(nbuf - 1)]
    hs = [torch.empty_like(y0) for _ in range(nbuf)]
    return ys, hs, nbuf


def _queue_ahead(stream, cycles: int = 200_000):
    """Keep the device busy (a ~0.1 ms spin kernel, outside the timed region) while the timed region's start event and
    first launches are enqueued: the start event then fires when the device reaches the first timed kernel, not while
    the host is still submitting it (a 20-step graph replay otherwise carried ~9 us of idle submission latency)."""
    import torch
    with torch.cuda.stream(stream):
        torch.cuda._sleep(cycles)


def time_estimator(est, ys, hs, x_d, soi_d, steps: int, warmup: int, launch: str, dist, clock_s: float = 0.0):
    """W warm-up steps, then EXACTLY `steps` timed steps (one ce_estimate each, rotating over the buffers),
    bracketed by a barrier + synchronize on both sides; CUDA events on the launching stream; max over ranks.

    launch = "graph": the `steps` calls are captured once into a CUDA graph (programmatic-dependent-launch edges
    kept) and the timed region is one replay of it -- the same kernels, no host launch cost between them;
    launch = "direct": the calls are issued from Python through the C-ABI inside the timed region.
    Every buffer is primed (its tensor maps encoded) before the warm-up; the first call's host cost is returned."""
    import torch

    import paper_1802_05427_b200 as ce
    nbuf = len(ys)
    T, M, K, _ = ys[0].shape
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    soi_ptr = soi_d.data_ptr() if soi_d is not None else 0

    def step(i, sp=sptr):
        ce.ce_estimate(est.handle, ys[i % nbuf].data_ptr(), x_d.data_ptr(), hs[i % nbuf].data_ptr(), T, M, K,
                       soi_ptr, sp)

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    step(0)
    first_call_us = (time.perf_counter() - t0) * 1e6         # includes encoding buffer 0's tensor maps
    t0 = time.perf_counter()
    step(0)
    second_call_us = (time.perf_counter() - t0) * 1e6
    for i in range(1, nbuf):                                  # prime every rotating buffer
        step(i)
    for i in range(warmup):
        step(i)
    torch.cuda.synchronize()
    graph, n_graph = None, 0
    if launch == "graph":
        l0 = est.launch_count()
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(stream)
        with torch.cuda.stream(cap):
            with torch.cuda.graph(graph, stream=cap):
                for i in range(steps):
                    step(i, cap.cuda_stream)
        n_graph = est.launch_count() - l0
        torch.cuda.synchronize()
        graph.replay()                                        # untimed: first replay uploads the graph
        torch.cuda.synchronize()
    clk = ClockSampler(dist.dev.index)
    with clk:
        if clock_s > 0:                                       # load window for the clock record (untimed)
            tw = time.perf_counter()
            while time.perf_counter() - tw < clock_s:
                if graph is not None:
                    graph.replay()
                else:
                    for i in range(steps):
                        step(i)
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        l0 = est.launch_count()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        _queue_ahead(stream)
        ev0.record(stream)
        if graph is not None:
            graph.replay()
        else:
            for i in range(steps):
                step(i)
        ev1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
    launches = n_graph if graph is not None else est.launch_count() - l0
    ms = ev0.elapsed_time(ev1)
    del graph
    return {"ms": ms, "ms_max": dist.max(ms), "ms_ranks": dist.all_values(ms), "launches": int(launches),
            "first_call_us": first_call_us, "steady_call_host_us": second_call_us, "clocks": clk.summary()}


def _roofline(sel, cfg, E_local, kernel_s, peaks, props, sm_max):
    """Roofline of the dominant kernel: algorithmic bytes (16 B per estimate + pilots) and flops (8b per estimate)."""
    import paper_1802_05427_b200 as ce
    fp32_meas = peaks.get("fp32_tflops")
    fp32_peak = (fp32_meas * 1e12 if fp32_meas else props.multi_processor_count * 128 * 2 * sm_max * 1e6)
    hbm_bw = peaks.get("hbm_gbs", 6548.8) * 1e9
    T_loc = cfg.T
    flops = 8.0 * cfg.b * E_local
    alg_bytes = 16 * E_local + 8 * T_loc * cfg.K * cfg.N
    kname = KERNEL_NAMES.get(sel, "?")
    if sel in (ce.CE_KERNEL_TF32X3, ce.CE_KERNEL_BF16X3):
        bf16 = peaks.get("bf16_tflops", 1605.7) * 1e12
        if sel == ce.CE_KERNEL_TF32X3:
            tc_peak = bf16 * 0.5 / 3.0
            src = "MEASURED_PEAKS bf16_tflops x 1/2 (tf32:bf16 nominal) / 3 (3xTF32 MMAs per product)"
        else:
            tc_peak = bf16 / 3.0
            src = "MEASURED_PEAKS bf16_tflops / 3 (BF16x3 MMAs per product)"
        t_tc, t_hbm = flops / tc_peak, alg_bytes / hbm_bw
        if t_tc >= t_hbm:
            roof = {"bound": "tensor", "achieved": flops / kernel_s / 1e12, "peak": tc_peak / 1e12,
                    "unit": "TFLOP/s", "frac": (flops / kernel_s) / tc_peak, "peak_source": src}
        else:
            roof = {"bound": "hbm", "achieved": alg_bytes / kernel_s / 1e9, "peak": hbm_bw / 1e9, "unit": "GB/s",
                    "frac": (alg_bytes / kernel_s) / hbm_bw, "peak_source": "MEASURED_PEAKS hbm_gbs (burst copy)"}
        roof["roofline_time_us"] = max(t_tc, t_hbm) * 1e6
    else:
        roof = {"bound": "alu", "achieved": flops / kernel_s / 1e12, "peak": fp32_peak / 1e12, "unit": "TFLOP/s",
                "frac": (flops / kernel_s) / fp32_peak,
                "peak_source": ("MEASURED_PEAKS fp32_tflops (FFMA microbenchmark)" if fp32_meas else
                                f"{props.multi_processor_count} SMs x 128 FP32 lanes x 2 x {sm_max:.0f} MHz (nominal)"),
                "roofline_time_us": max(flops / fp32_peak, alg_bytes / hbm_bw) * 1e6}
    roof.update({"kernel": kname, "kernel_us": kernel_s * 1e6, "algorithmic_flops_per_launch": flops,
                 "algorithmic_bytes_per_launch": alg_bytes, "hbm_frac": (alg_bytes / kernel_s) / hbm_bw,
                 "fp32_simt_frac": (flops / kernel_s) / fp32_peak})
    return roof


def _traffic(kname: str, cfg_id: int):
    """dram read+write bytes per launch from the committed ncu range capture (profiles/traffic_r02.json): the
    counters summed over a range of back-to-back launches on rotating > L2 buffers, divided by the launch count
    (a single-launch capture misses the write-back of that launch's output, which stays dirty in L2)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic_r02.json")) as f:
            d = json.load(f)
        e = d[f"config{cfg_id}"][kname]
        return {"bytes_per_launch": e["dram_bytes_per_launch"], "source": "profiles/traffic_r02.json: " + e["how"]}
    except Exception:
        return None


def _device_inputs(cfg, m_lo, m_hi, dev, seed=11):
    """Timing-only inputs for the sweep lines: y drawn on the device (torch.randn, unit power), the seeded pilots
    and the configuration's statistics -- the kernels' work does not depend on the values (parity of configs 4-5
    at full size is tests/test_gpu_parity.py::test_full_size_sampled)."""
    import torch
    g = torch.Generator(device=dev)
    g.manual_seed(seed)

    def make_y():
        re = torch.randn((cfg.T, m_hi - m_lo, cfg.K, cfg.N), generator=g, device=dev, dtype=torch.float32)
        im = torch.randn((cfg.T, m_hi - m_lo, cfg.K, cfg.N), generator=g, device=dev, dtype=torch.float32)
        return torch.complex(re, im) * np.float32(np.sqrt(0.5))
    return make_y


def _k4_variant(sel, cfg, m_local, props):
    """The K4 launch shape the library's policy picks for this call (mirrors bf16x3_pair_wanted in
    csrc/k4p_block_lmmse_pair.cu, CE_K4_PAIR overrides it): CTA pairs (tcgen05 cta_group::2) when every CTA walks
    more than two 128-row tiles, single CTAs otherwise.  Windows too wide for one accumulator (config 6) are split
    by the library; the unsplit count used here only matters at that boundary."""
    if sel != 3:
        return None
    import paper_1802_05427_b200 as ce
    n_ct = -(-m_local * cfg.K // 128)
    n_win = len(ce.ce_window_table(cfg.N, cfg.b, cfg.stride))
    env = os.environ.get("CE_K4_PAIR")
    pair = n_ct >= 2 and (env == "1" if env in ("0", "1") else cfg.T * n_win * n_ct > 2 * props.multi_processor_count)
    return "k4_bf16x3_pair (clusters of two CTAs, cta_group::2)" if pair else "k4_bf16x3 (single CTAs)"


def sweep_line(cfg_id, args, dist, peaks, props, sm_max):
    """Device-time line of another configuration (strong-scaled: its own M antennas split across the ranks)."""
    import torch

    import paper_1802_05427_b200 as ce
    from paper_1802_05427_b200.shard import antenna_shard
    cfg = workload.get_config(cfg_id)
    m_lo, m_hi = antenna_shard(cfg.M, dist.world, dist.rank)
    r, s2 = workload.channel_stats(cfg, 0)
    soi_d = torch.from_numpy(workload.set_of_instance(cfg)).to(dist.dev)
    x_d = torch.from_numpy(workload.gen_pilots(cfg, 0)).to(dist.dev)
    est = ce.ChannelEstimator(cfg.N, cfg.b, cfg.stride, r, s2, kernel=args.kernel).build()
    E_loc = cfg.T * (m_hi - m_lo) * cfg.K * cfg.N
    ys, hs, nbuf = _rotating_buffers(_device_inputs(cfg, m_lo, m_hi, dist.dev), 16 * E_loc, dist.dev)
    res = time_estimator(est, ys, hs, x_d, soi_d, args.sweep_steps, 3, args.launch, dist, clock_s=0.2)
    sel = est.selected_kernel()
    kernel_s = res["ms"] / args.sweep_steps * 1e-3
    roof = _roofline(sel, cfg, E_loc, kernel_s, peaks, props, sm_max)
    est.close()
    del ys, hs
    torch.cuda.empty_cache()
    return {"workload": _cfg_json(cfg, {})["workload"], "n_gpus": dist.world, "scaling": "strong",
            "steps": args.sweep_steps, "warmup": 3, "ms_per_step": res["ms_max"] / args.sweep_steps,
            "per_rank_ms_per_step": [v / args.sweep_steps for v in res["ms_ranks"]],
            "value": cfg.estimates * args.sweep_steps / (res["ms_max"] * 1e-3), "unit": "estimates/s",
            "kernel": KERNEL_NAMES.get(sel), "kernel_variant": _k4_variant(sel, cfg, m_hi - m_lo, props),
            "dtype": KERNEL_DTYPE.get(sel),
            "roofline": {k: roof[k] for k in ("bound", "achieved", "peak", "unit", "frac", "roofline_time_us")},
            "gpu_launches": res["launches"], "clocks": res["clocks"],
            "l2": f"rotating {nbuf} y/h buffer pairs (> L2)", "data": "y drawn on device (timing only), seeded pilots"}


def run_ours(args, cfg):
    import torch

    import paper_1802_05427_b200 as ce
    from paper_1802_05427_b200.shard import antenna_shard

    dist = Dist(args.backend)
    world, rank = dist.world, dist.rank
    dev = dist.dev

    r, s2 = workload.channel_stats(cfg, 0)
    soi = workload.set_of_instance(cfg)
    x = workload.gen_pilots(cfg, 0)
    # weak scaling (default, one rank = one GPU's own slot stream): the global batch has world*M antennas and
    # rank r owns [r*M, (r+1)*M) drawn with the per-(t, m) seeds of the full draw; --strong splits the
    # configuration's own M antennas across the ranks.  Either way no data-path collective.
    M_glob = cfg.M if args.strong else world * cfg.M
    m_lo, m_hi = antenna_shard(M_glob, world, rank)
    y = workload.gen_instances(cfg, 0, m_lo=m_lo, m_hi=m_hi, x=x)
    est = ce.ChannelEstimator(cfg.N, cfg.b, cfg.stride, r, s2, kernel=args.kernel)
    torch.cuda.synchronize()
    tb0 = time.perf_counter()
    est.build()
    build_ms = (time.perf_counter() - tb0) * 1e3

    y_t = torch.from_numpy(y)
    ys, hs, nbuf = _rotating_buffers(lambda: y_t.to(dev), 2 * y.nbytes, dev)
    x_d = torch.from_numpy(x).to(dev)
    soi_d = torch.from_numpy(soi).to(dev)
    T, M, K, N = y.shape
    res = time_estimator(est, ys, hs, x_d, soi_d, args.steps, args.warmup, args.launch, dist,
                         clock_s=args.clock_window_s)
    ms_max = res["ms_max"]
    m_par = max(1, min(cfg.M, args.ref_antennas * 4))
    h_sample = hs[0][:1, :min(m_par, m_hi - m_lo)].cpu().numpy()   # parity sample, before the buffers are reused
    E_glob = cfg.estimates * M_glob // cfg.M          # estimates of the whole job per step
    E = cfg.estimates * (m_hi - m_lo) // cfg.M        # this rank's estimates per launch (roofline)
    value = E_glob * args.steps / (ms_max * 1e-3)
    kernel_s = res["ms"] / args.steps * 1e-3          # one contraction launch per step on this stream
    direct = None
    if args.launch == "graph":                        # the same K steps issued one by one from Python (record)
        rd = time_estimator(est, ys, hs, x_d, soi_d, args.steps, 3, "direct", dist)
        direct = {"ms_per_step": rd["ms_max"] / args.steps, "gpu_launches": rd["launches"]}

    # practical ceiling for this traffic (outside the timed region): a plain device copy y -> h of the same
    # bytes over the same rotating buffers, back to back (torch's copy kernel, not ours)
    stream = torch.cuda.current_stream()
    copy_steps = min(max(args.steps, 50), 500)
    for i in range(10):
        hs[i % nbuf].copy_(ys[i % nbuf])
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    _queue_ahead(stream)
    c0.record(stream)
    for i in range(copy_steps):
        hs[i % nbuf].copy_(ys[i % nbuf])
    c1.record(stream)
    torch.cuda.synchronize()
    copy_us = c0.elapsed_time(c1) * 1e3 / copy_steps

    # end-to-end through the public host-buffer API: pinned host y, x in, pinned host h out, every step
    y_pin = y_t.pin_memory()
    x_pin = torch.from_numpy(x).pin_memory()
    h_pin = torch.empty(y.shape, dtype=torch.complex64).pin_memory()
    # each step copies its inputs in and its estimates out (ce_estimate_host_async: two staging slots, so one step's
    # device->host copies overlap the next step's host->device copies); two pinned output buffers alternate
    e2e_steps = max(3, min(args.steps, args.e2e_steps))
    h_pins = [h_pin, torch.empty(y.shape, dtype=torch.complex64).pin_memory()]
    for i in range(2):
        est.estimate_host(y_pin, x_pin, out=h_pins[i], set_of_instance=soi)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(e2e_steps):
        est.estimate_host(y_pin, x_pin, out=h_pins[i % 2], set_of_instance=soi, sync=False)
    est.host_wait(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = dist.max(e0.elapsed_time(e1))
    e2e_value = E_glob * e2e_steps / (e2e_ms * 1e-3)
    e2e_sync = None
    if args.e2e_sync_steps > 0:                       # the synchronous call, for the record
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for i in range(args.e2e_sync_steps):
            est.estimate_host(y_pin, x_pin, out=h_pins[i % 2], set_of_instance=soi)
        s1.record(stream)
        torch.cuda.synchronize()
        e2e_sync = E_glob * args.e2e_sync_steps / (dist.max(s0.elapsed_time(s1)) * 1e-3)

    props = torch.cuda.get_device_properties(dev)
    peaks = _peaks()
    sel = est.selected_kernel()
    sm_max = peaks.get("sm_max_mhz") or res["clocks"].get("sm_max_mhz") or 1965.0
    roof = _roofline(sel, cfg, E, kernel_s, peaks, props, sm_max)
    roof["copy_ceiling"] = {"us": copy_us, "frac": (2 * y.nbytes / (copy_us * 1e-6)) / (peaks.get("hbm_gbs", 6548.8) * 1e9),
                            "what": "torch copy y -> h (same 2 x y bytes, same rotating buffers), back to back: "
                                    "the practical ceiling for this read + write traffic"}
    tr = _traffic(KERNEL_NAMES.get(sel, "?"), cfg.cfg_id) if world == 1 else None
    roof["traffic"] = tr["bytes_per_launch"] if tr else None
    roof["traffic_source"] = tr["source"] if tr else "not measured for this kernel / config"

    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the oracle as it stands, on a bounded sample of the same workload (antennas [0, m) of instance 0),
        # all host cores then one core; its output doubles as the parity sample of the timed buffers
        m = h_sample.shape[1]
        times, ref = _oracle_sample_timing(cfg, x[:1], y[:1, :m], r, s2, soi[:1], budget_s=args.cpu_budget_s)
        times1, _ = _oracle_sample_timing(cfg, x[:1], y[:1, :m], r, s2, soi[:1], budget_s=args.cpu_budget_s / 2,
                                          threads=1)
        est_per_run = m * cfg.K * cfg.N
        med, med1 = float(np.median(times)), float(np.median(times1))
        cpu = {"value": est_per_run / med, "unit": "estimates/s", "cores": _cores(), "kind": "oracle",
               "sample": f"oracle LS+block apply (complex128) on antennas [0,{m}) of config {cfg.cfg_id} instance 0; "
                         f"median of {len(times)} runs ({sum(times):.1f} s)",
               "runs": len(times), "cpu_model": _cpu_model(), "blas": _blas_vendor(),
               "one_thread": {"value": est_per_run / med1, "unit": "estimates/s", "runs": len(times1),
                              "note": "BLAS limited to 1 thread (threadpoolctl): per-core figure beside the paper's "
                                      "Table V per-core cycle counts (PAPER.md:545-548)"}}
        import oracle
        h0 = h_sample.astype(np.complex128)                          # every y buffer holds the same draw
        d = (h0 - ref).reshape(-1, N)
        row_err = 0.0
        for (_a, o, o1) in oracle.window_table(N, cfg.b, cfg.stride):
            nr = np.linalg.norm(ref.reshape(-1, N)[:, o:o1], axis=1)
            row_err = max(row_err, float((np.linalg.norm(d[:, o:o1], axis=1) / np.maximum(nr, 1e-300)).max()))
        parity = {"max_rel_err_per_instance": float(oracle.rel_fro_error_per_instance(h0, ref).max()),
                  "max_row_rel_err": row_err, "bar": "1e-4 per instance (north_star), 1e-3 per row",
                  "sample": f"the timed buffers' estimates of antennas [0,{m}) of instance 0 vs the oracle"}

    # multi-GPU verification (outside the timed region): all-gather of the antenna shards, and rank 0
    # recomputes the whole global batch on its own GPU -- the sharded result must match it bit for bit
    # (SURVEY.md §8(e) shard invariance)
    verify = None
    if world > 1 and not args.no_verify:
        try:
            from paper_1802_05427_b200.shard import gather_antenna_shards
            h_loc = est.estimate(ys[0], x_d, set_of_instance=soi_d)      # the h buffers were reused by the copy ceiling
            torch.cuda.synchronize()
            full = gather_antenna_shards(h_loc if dist.backend == "nccl" else h_loc.cpu(), M_glob)
            if rank == 0:
                y_all = workload.gen_instances(cfg, 0, m_lo=0, m_hi=M_glob, x=x)
                h_ref = est.estimate(torch.from_numpy(y_all).to(dev), x_d, set_of_instance=soi_d)
                torch.cuda.synchronize()
                verify = {"gather_bytes": int(full.numel() * 8), "backend": dist.backend,
                          "bitwise_equal_to_single_gpu": bool(torch.equal(torch.view_as_real(full.to(dev)),
                                                                          torch.view_as_real(h_ref)))}
            del full
        except Exception as exc:       # never let the check take the measurement down
            verify = {"error": repr(exc)[:200]}
        dist.barrier()

    # strong scaling of the configuration's own M antennas (when the primary line is weak and N > 1)
    strong = None
    if world > 1 and not args.strong:
        s_lo, s_hi = antenna_shard(cfg.M, world, rank)
        ys_s = workload.gen_instances(cfg, 0, m_lo=s_lo, m_hi=s_hi, x=x)
        ys_t = torch.from_numpy(ys_s)
        yss, hss, _ = _rotating_buffers(lambda: ys_t.to(dev), max(2 * ys_s.nbytes, 1), dev)
        rs = time_estimator(est, yss, hss, x_d, soi_d, args.steps, args.warmup, args.launch, dist)
        strong = {"scaling": "strong", "antennas_per_rank": [list(antenna_shard(cfg.M, world, g)) for g in range(world)],
                  "ms_per_step": rs["ms_max"] / args.steps, "value": cfg.estimates * args.steps / (rs["ms_max"] * 1e-3),
                  "unit": "estimates/s", "per_rank_ms_per_step": [v / args.steps for v in rs["ms_ranks"]]}
        del yss, hss

    sweep = None
    if args.sweep:
        sweep = [sweep_line(int(c), args, dist, peaks, props, sm_max) for c in args.sweep.split(",") if c]

    if rank == 0:
        line = {
            "metric": "channel estimates/s (antenna*user*subcarrier)", "value": value, "unit": "estimates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong" if args.strong else "weak", "vs_baseline": None,
            "dtype": KERNEL_DTYPE.get(sel, "c64"),
            "data": "synthetic (seeded workload generator, SURVEY.md §8(d) recipe)",
            "config": _cfg_json(cfg, {"l2": f"inputs larger than L2: rotating {nbuf} y/h buffer pairs "
                                            f"({nbuf * 2 * y.nbytes / 2**20:.0f} MiB > 126 MiB)",
                                      "kernel": KERNEL_NAMES[args.kernel] + f"->{KERNEL_NAMES.get(sel)}",
                                      "kernel_variant": _k4_variant(sel, cfg, M, props),
                                      "launch": args.launch, "global_antennas": M_glob,
                                      "parallelism": f"antenna shard x{world} ({dist.backend}), no data-path collective"}),
            "roofline": roof,
            "cpu_baseline": cpu,
            "parity": parity,
            "e2e": {"value": e2e_value, "unit": "estimates/s",
                    "h2d_bytes_per_step": int(y.nbytes + x.nbytes + soi.nbytes),
                    "d2h_bytes_per_step": int(y.nbytes), "steps": e2e_steps, "api": "ce_estimate_host_async",
                    "synchronous_call_value": e2e_sync},
            "gpu_launches": res["launches"],
            "per_rank_ms_per_step": [v / args.steps for v in res["ms_ranks"]],
            "direct_launch": direct,
            "first_call": {"first_call_host_us": res["first_call_us"], "steady_call_host_us": res["steady_call_host_us"],
                           "what": "host cost of the first ce_estimate on a new buffer (tensor-map encodes) vs a "
                                   "repeated call; every rotating buffer is primed before the warm-up"},
            "strong": strong,
            "multi_gpu_verify": verify,
            "sweep": sweep,
            "clocks": res["clocks"],
            "filter_build_ms": build_ms,
            "device": props.name,
        }
        print(json.dumps(line), flush=True)
    est.close()
    dist.close()


def run_comb(args):
    """--comb NAME: the paper's comb-pilot 3W / 12W-LMMSE path (NEXT-1; K10 on tcgen05 for the 12W, K6b FP32 SIMT
    otherwise or with --comb-kernel simt) on one of workload.COMB_CONFIGS."""
    import torch

    import paper_1802_05427_b200 as ce
    from paper_1802_05427_b200.shard import antenna_shard

    dd = Dist(args.backend)
    world, rank, local, dev = dd.world, dd.rank, dd.local, dd.dev
    cfg = workload.get_comb_config(args.comb)
    r, s2 = workload.comb_stats(cfg)
    x = workload.comb_pilots(cfg)
    m_lo, m_hi = antenna_shard(world * cfg.M, world, rank)
    y = workload.comb_instances(cfg, x=x, m_lo=m_lo, m_hi=m_hi)
    est = ce.CombEstimator(cfg.N, cfg.S, cfg.n_ue, cfg.G, cfg.mode, r, s2).build()
    est.set_kernel(args.comb_kernel)
    T, M, N = y.shape
    tc = est.selected_kernel(T, M) == ce.CE_COMB_KERNEL_TC
    out_bytes = T * M * cfg.n_ue * N * 8
    nbuf = max(2, int(np.ceil(1.25 * L2_BYTES / (y.nbytes + out_bytes))) + 1)
    y_dev = [torch.from_numpy(y).to(dev) for _ in range(nbuf)]
    h_dev = [torch.empty((T, M, cfg.n_ue, N), dtype=torch.complex64, device=dev) for _ in range(nbuf)]
    x_dev = torch.from_numpy(x).to(dev)
    stream = torch.cuda.current_stream()
    for i in range(args.warmup):
        est.estimate(y_dev[i % nbuf], x_dev, out=h_dev[i % nbuf])
    torch.cuda.synchronize()
    dd.barrier()
    torch.cuda.synchronize()
    l0 = est.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        _queue_ahead(stream)
        ev0.record(stream)
        for i in range(args.steps):
            est.estimate(y_dev[i % nbuf], x_dev, out=h_dev[i % nbuf])
        ev1.record(stream)
        torch.cuda.synchronize()
        dd.barrier()
    launches = est.launch_count() - l0
    ms = ev0.elapsed_time(ev1)
    ms_max = dd.max(ms)
    E = cfg.estimates
    value = world * E * args.steps / (ms_max * 1e-3)
    kernel_s = ms / args.steps * 1e-3
    # end to end: pinned host y -> device, estimate, device -> pinned host h, every step
    y_pin = torch.from_numpy(y).pin_memory()
    h_pin = torch.empty((T, M, cfg.n_ue, N), dtype=torch.complex64).pin_memory()
    e2e_steps = max(3, min(args.steps, args.e2e_steps))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        yd = y_pin.to(dev, non_blocking=True)
        hd = est.estimate(yd, x_dev)
        h_pin.copy_(hd, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_value = world * E * e2e_steps / (dd.max(e0.elapsed_time(e1)) * 1e-3)
    peaks = _peaks()
    hbm_bw = peaks.get("hbm_gbs", 6548.8) * 1e9
    alg_bytes = out_bytes + y.nbytes + x.nbytes
    # K10: the step is two kernels (k10_ls, k10_comb_tc); the fraction is taken over the whole step
    roof = {"bound": "hbm", "achieved": alg_bytes / kernel_s / 1e9, "peak": hbm_bw / 1e9, "unit": "GB/s",
            "frac": alg_bytes / kernel_s / hbm_bw, "peak_source": "MEASURED_PEAKS hbm_gbs", "traffic": None,
            "kernel": "k10_ls + k10_comb_tc (whole step)" if tc else "k6_estimate_g" if cfg.S == 12 else "k6_estimate",
            "kernel_us": kernel_s * 1e6, "algorithmic_bytes_per_launch": alg_bytes,
            "algorithmic_flops_per_launch": 8.0 * cfg.G * E,
            "alu_bound_us_simt": 8.0 * cfg.G * E / (peaks.get("fp32_tflops", 69.13) * 1e12) * 1e6}
    if rank == 0:
        line = {
            "metric": "channel estimates/s (antenna*user*subcarrier)", "value": value, "unit": "estimates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": ("c64 I/O, bf16x3 (error-compensated) tensor products, fp32 accumulate" if tc
                      else "c64 I/O, fp32 FFMA2 products, fp32 accumulate"),
            "data": "synthetic (workload.comb: Table III channel, fixed-design r_d / SNR_fixed)",
            "config": {"workload": f"comb_{cfg.name}_{cfg.M}x{cfg.n_ue}of{cfg.S}x{cfg.N}_T{cfg.T}_G{cfg.G}_{cfg.mode}",
                       "M": cfg.M, "S": cfg.S, "n_ue": cfg.n_ue, "N": cfg.N, "T": cfg.T, "G": cfg.G,
                       "mode": cfg.mode, "kernel": "k10_comb_tc (tcgen05)" if tc else "k6 (fp32 simt)",
                       "l2": f"rotating {nbuf} y/h buffer pairs (> L2)",
                       "parallelism": f"antenna shard x{world}"},
            "roofline": roof, "cpu_baseline": None,
            "e2e": {"value": e2e_value, "unit": "estimates/s", "h2d_bytes_per_step": int(y.nbytes),
                    "d2h_bytes_per_step": int(out_bytes), "steps": e2e_steps},
            "gpu_launches": int(launches), "clocks": clk.summary(), "device": torch.cuda.get_device_name(dev),
        }
        if world == 1 and not args.no_cpu_baseline:
            # the oracle on a bounded sample (antenna 0 of every instance), timed on the host cores; the timed buffers'
            # estimates of that antenna are its parity sample (every y buffer holds the same draw)
            import oracle
            times = []
            t_start = time.perf_counter()
            while len(times) < 3 or time.perf_counter() - t_start < args.cpu_budget_s / 2:
                t0 = time.perf_counter()
                ref = oracle.comb_estimate(y[:, :1], x, r, s2, cfg.N, cfg.S, cfg.G, cfg.mode, cfg.n_ue)
                times.append(time.perf_counter() - t0)
            med = float(np.median(times))
            line["cpu_baseline"] = {"value": T * cfg.n_ue * N / med, "unit": "estimates/s", "cores": _cores(),
                                    "kind": "oracle", "runs": len(times), "cpu_model": _cpu_model(),
                                    "blas": _blas_vendor(),
                                    "sample": f"oracle comb_estimate (complex128) on antenna 0 of all {T} instances; "
                                              f"median of {len(times)} runs"}
            hs = h_dev[0][:, :1].cpu().numpy().astype(np.complex128)
            d = (hs - ref).reshape(T, -1)
            inst = np.linalg.norm(d, axis=1) / np.linalg.norm(ref.reshape(T, -1), axis=1)
            rows = np.linalg.norm(hs - ref, axis=-1) / np.maximum(np.linalg.norm(ref, axis=-1), 1e-300)
            line["parity"] = {"max_rel_err_per_instance": float(inst.max()), "max_row_rel_err": float(rows.max()),
                              "bar": "1e-4 per instance, 1e-3 per row",
                              "sample": "the timed buffers' estimates of antenna 0 (all instances, all UEs) vs the oracle"}
        print(json.dumps(line), flush=True)
    est.close()
    dd.close()


def run_stats(args):
    """--stats: the NEXT-3 statistics estimator (K7) on the configured workload (1 GPU line)."""
    import torch

    import paper_1802_05427_b200 as ce

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    cfg = workload.get_config(args.config)
    x = workload.gen_pilots(cfg, 0)
    y = workload.gen_instances(cfg, 0, x=x)
    soi = torch.from_numpy(workload.set_of_instance(cfg)).cuda()
    D, B = cfg.b, 32          # 32 noise-window bins: sigma2_hat from C x 32 samples (rel. s.e. < 1% on config 3)
    nbuf = max(2, int(np.ceil(1.25 * L2_BYTES / y.nbytes)) + 1)
    y_dev = [torch.from_numpy(y).cuda() for _ in range(nbuf)]
    x_dev = torch.from_numpy(x).cuda()
    for i in range(args.warmup):
        ce.ce_stats_estimate(y_dev[i % nbuf], x_dev, D, B, soi, cfg.n_sets)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        _queue_ahead(stream)
        ev0.record(stream)
        for i in range(args.steps):
            ce.ce_stats_estimate(y_dev[i % nbuf], x_dev, D, B, soi, cfg.n_sets)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    samples = cfg.T * cfg.M * cfg.K * cfg.N
    cols = cfg.T * cfg.M * cfg.K
    peaks = _peaks()
    fp32_peak = peaks.get("fp32_tflops", 69.13) * 1e12
    hbm_bw = peaks.get("hbm_gbs", 6548.8) * 1e9
    bf16 = peaks.get("bf16_tflops", 1605.7) * 1e12
    # the library's policy (k7_stats.cu, k9_spectrum.cu): lags through the power spectrum (K9: FP32 FFT of length
    # L = 2^l >= max(64, N + D - 1) per LS row, l <= 13) and the noise window on the tensor cores (K4 power mode:
    # one BF16x3 pass over y against the inverse-DFT bank) when K4 can stream y (N even, K <= 32)
    L = 64
    while L < cfg.N + D - 1:
        L *= 2
    k9 = L <= 8192 and cfg.n_sets <= 65535
    k4n = k9 and cfg.N % 2 == 0 and cfg.K <= 32 and B <= 4096
    y_bytes = float(y.nbytes)
    x_bytes = float(x.nbytes)
    fft_flops = 5.0 * L * np.log2(L) * cols                # the standard radix-2 count, per zero-padded row
    lag_flops = 8.0 * cols * sum(cfg.N - d for d in range(D))
    noise_flops = 8.0 * cols * cfg.N * B
    if k9 and k4n:
        # K9 bound by the FP32 pipes or by its read of y; K4's noise pass bound by its read of y (HBM)
        t_k9 = max(fft_flops / fp32_peak, (y_bytes + x_bytes) / hbm_bw)
        t_k4 = (y_bytes + x_bytes) / hbm_bw
        t_ideal = t_k9 + t_k4
        bound, kern = "alu+hbm", "k9_spectrum (lags) + k4_bf16x3 power mode (noise window)"
        note = ("sum of the two kernels' bounds: K9 = max(FFT flops 5 L log2 L per row at the FP32 FFMA peak, y + x "
                "bytes at HBM), K4 noise pass = y + x bytes at HBM")
        flops = fft_flops + 3 * 8.0 * cols * cfg.N * B
    else:
        t_ideal = lag_flops / (bf16 / 3) + noise_flops / fp32_peak
        bound, kern = "tensor+alu", "k8_gram / k7_accumulate (lags) + k7_noise (noise window)"
        note = "lag flops at the BF16 peak / 3 plus noise-window flops at the FP32 SIMT peak"
        flops = lag_flops + noise_flops
    t_direct = lag_flops / (bf16 / 3) + noise_flops / fp32_peak
    line = {"metric": "LS samples/s through the statistics estimator (NEXT-3)", "value": samples / (ms * 1e-3),
            "unit": "samples/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": ("c64 I/O; lags fp32 FFT, noise window bf16x3 tensor products; fp64 accumulation per set"
                      if k9 and k4n else "c64 I/O; lags bf16x3 tensor products (K8) or fp32 FFMA; fp64 accumulation per set"),
            "data": "synthetic (seeded workload generator)",
            "config": _cfg_json(cfg, {"D": D, "B": B, "L_fft": L if k9 else None,
                                      "l2": f"rotating {nbuf} y buffers (> L2)"}),
            "roofline": {"bound": bound, "achieved": None, "peak": None, "unit": "us", "frac": t_ideal / (ms * 1e-3),
                         "traffic": None, "roofline_time_us": t_ideal * 1e6, "kernel": kern,
                         "flops_per_launch": flops, "note": note,
                         "direct_method_roofline_us": t_direct * 1e6,
                         "frac_vs_direct_method": t_direct / (ms * 1e-3),
                         "direct_method_note": ("round-1/2a definition: the direct lag sums 8 C sum_d (N - d) at the "
                                                "BF16 peak / 3 plus the noise-window DFT 8 C N B at the FP32 peak")},
            "gpu_launches": (5 if k9 and k4n else 3) * args.steps, "clocks": clk.summary(),
            "device": torch.cuda.get_device_properties(0).name}
    if not args.no_cpu_baseline:
        # the oracle as it stands on a bounded sample (instance 0, antennas [0, m)), timed on the host cores; the same
        # sample through ce_stats_estimate (outside the timed region) is its parity check
        import oracle
        m = max(1, min(cfg.M, 8))
        ys, xs = y[:1, :m], x[:1]
        times = []
        t_start = time.perf_counter()
        while len(times) < 3 or time.perf_counter() - t_start < args.cpu_budget_s / 2:
            t0 = time.perf_counter()
            r_o, s2_o = oracle.estimate_stats(ys, xs, D, B)
            times.append(time.perf_counter() - t0)
        rg, s2g = ce.ce_stats_estimate(torch.from_numpy(np.ascontiguousarray(ys)).cuda(),
                                       torch.from_numpy(np.ascontiguousarray(xs)).cuda(), D, B)
        torch.cuda.synchronize()
        rg, s2g = rg.cpu().numpy()[0], float(s2g.cpu().numpy()[0])
        med = float(np.median(times))
        line["cpu_baseline"] = {"value": m * cfg.K * cfg.N / med, "unit": "samples/s", "cores": _cores(),
                                "kind": "oracle", "runs": len(times), "cpu_model": _cpu_model(), "blas": _blas_vendor(),
                                "sample": f"oracle estimate_stats (complex128) on antennas [0,{m}) of config "
                                          f"{cfg.cfg_id} instance 0; median of {len(times)} runs"}
        line["parity"] = {"max_rel_err_r": float(np.max(np.abs(rg - r_o)) / abs(r_o[0])),
                          "rel_err_sigma2": abs(s2g / s2_o - 1.0), "bar": "1e-4 (tests/test_gpu_stats.py)",
                          "sample": "ce_stats_estimate on the same sample vs the oracle"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1,
                    help="ranks (one per GPU); without a launcher's WORLD_SIZE, bench.py spawns them itself")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--kernel", type=int, default=0, help="0 auto, 1 simt, 2 tf32x3, 3 bf16x3")
    ap.add_argument("--launch", choices=["graph", "direct"], default="graph",
                    help="timed steps replayed from one CUDA graph (default) or issued one by one from Python")
    ap.add_argument("--backend", choices=["nccl", "gloo"], default="nccl",
                    help="process-group backend for N > 1 (gloo lets several ranks share one GPU: tests only)")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--e2e-sync-steps", type=int, default=5, help="steps of the synchronous ce_estimate_host (record)")
    ap.add_argument("--ref-antennas", type=int, default=4)
    ap.add_argument("--cpu-budget-s", type=float, default=8.0)
    ap.add_argument("--clock-window-s", type=float, default=0.3,
                    help="untimed load window right before the timed region, sampled for the clocks record")
    ap.add_argument("--sweep", default="4,5",
                    help="comma-separated configurations timed after the main line (device time, strong-scaled "
                         "across the ranks); '' to skip")
    ap.add_argument("--sweep-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-verify", action="store_true", help="skip the N>1 gather + single-GPU bitwise check")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: split the configuration's M antennas across the ranks (default: weak, "
                         "M antennas per rank; a strong-scaled record of the same configuration rides along at N > 1)")
    ap.add_argument("--stats", action="store_true", help="time the NEXT-3 statistics estimator instead")
    ap.add_argument("--comb", default=None, help="run the comb-pilot 3W/12W path on workload.COMB_CONFIGS[NAME]")
    ap.add_argument("--comb-kernel", choices=["auto", "simt", "tc"], default="auto",
                    help="comb estimator kernel: auto (K10 tcgen05 for 12W shapes), simt (K6b), tc (K10)")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn(args))
    if args.comb:
        if args.impl == "reference":
            raise SystemExit("--impl reference times the block path's oracle; use it without --comb")
        run_comb(args)
        return
    if args.stats:
        run_stats(args)
        return
    cfg = workload.get_config(args.config)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
