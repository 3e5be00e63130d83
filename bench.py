#!/usr/bin/env python
"""Benchmark of the block-LMMSE pilot channel estimator (arXiv 1802.05427 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

One step = one pass of the hot path (LS + block-LMMSE contraction, a3-a5 of SURVEY.md §8(a))
over one estimation batch of the configured workload (default: config 3, the paper-scale
128 x 12 x 1200 slot, b = 100).  The filters W_b (a1-a2) are per-statistics, precomputed
before the slot loop exactly as the paper does offline; their
build time is reported separately as `filter_build_ms`.

Multi-GPU (torchrun, one rank per GPU): each rank estimates its own batch (antenna-sharded
global batch, no data-path collective) -> weak scaling; time = max over ranks.

Prints ONE JSON line (rank 0).  See DESIGN.md §6 for every field.
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
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def _ncu_traffic(kernel_key: str):
    """dram read+write bytes per launch from the committed ncu --set full summary, or None."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d["kernels"][kernel_key]["dram_bytes_per_launch"]
    except Exception:
        return None


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


def _cfg_json(cfg, extra):
    d = {"workload": f"config{cfg.cfg_id}_{cfg.name}_{cfg.M}x{cfg.K}x{cfg.N}_T{cfg.T}_b{cfg.b}_s{cfg.stride}",
         "M": cfg.M, "K": cfg.K, "N": cfg.N, "T": cfg.T, "b": cfg.b, "stride": cfg.stride,
         "n_sets": cfg.n_sets}
    d.update(extra)
    return d


def _oracle_rate(cfg, x, y, r, s2, soi, budget_s: float, min_runs: int = 3):
    """Time the oracle's LS + block apply (no generation, no filter build) on (y, x)."""
    import oracle
    filters = {}
    for st in set(int(v) for v in soi):
        filters[st] = [oracle.block_filter(r[st], s2[st], cfg.b)] * len(oracle.window_table(cfg.N, cfg.b, cfg.stride))
    runs, t0 = 0, time.perf_counter()
    while True:
        H_ls = oracle.ls_estimate(y, x)
        for t in range(y.shape[0]):
            oracle.block_apply(H_ls[t], filters[int(soi[t])], cfg.b, cfg.stride)
        runs += 1
        el = time.perf_counter() - t0
        if runs >= min_runs and el >= budget_s:
            break
    return runs, el


def _cores():
    for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        if os.environ.get(var):
            return int(os.environ[var])
    return len(os.sched_getaffinity(0))


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
    sample = f"oracle LS+block apply (complex128 NumPy/OpenBLAS) on antennas [0,{m}) of config {cfg.cfg_id} instance 0 per step"
    line = {
        "impl": "reference", "metric": "channel estimates/s (antenna*user*subcarrier)", "value": value,
        "unit": "estimates/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded workload generator)",
        "config": _cfg_json(cfg, {"sample_antennas": m}),
        "cpu_baseline": {"value": value, "unit": "estimates/s", "cores": _cores(), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": "estimates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_1802_05427_b200 as ce
    from paper_1802_05427_b200.shard import antenna_shard

    world, rank, local = _dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    r, s2 = workload.channel_stats(cfg, 0)
    soi = workload.set_of_instance(cfg)
    x = workload.gen_pilots(cfg, 0)
    # weak scaling (default): the global batch has world*M antennas; rank r owns the contiguous block
    # [r*M, (r+1)*M) (shard.antenna_shard), drawn with the per-(t, m) seeds of the full draw.
    # --strong: the configuration's own M antennas are split across the ranks (config 5's
    # 256 antennas on 8 GPUs)
    M_glob = cfg.M if args.strong else world * cfg.M
    m_lo, m_hi = antenna_shard(M_glob, world, rank)
    y = workload.gen_instances(cfg, 0, m_lo=m_lo, m_hi=m_hi, x=x)
    est = ce.ChannelEstimator(cfg.N, cfg.b, cfg.stride, r, s2, kernel=args.kernel)
    stream = torch.cuda.current_stream()
    tb0 = time.perf_counter()
    est.build()
    build_ms = (time.perf_counter() - tb0) * 1e3

    # inputs larger than L2: rotate over nbuf (y, h) buffer pairs, total > 126 MB
    step_bytes = 2 * y.nbytes
    nbuf = max(2, int(np.ceil(1.25 * L2_BYTES / step_bytes)) + 1)
    y_dev = [torch.from_numpy(y).to(dev) for _ in range(nbuf)]
    h_dev = [torch.empty_like(y_dev[0]) for _ in range(nbuf)]
    x_dev = torch.from_numpy(x).to(dev)
    soi_dev = torch.from_numpy(soi).to(dev)
    T, M, K, N = y.shape
    sptr = stream.cuda_stream

    def step(i):
        ce.ce_estimate(est.handle, y_dev[i % nbuf].data_ptr(), x_dev.data_ptr(), h_dev[i % nbuf].data_ptr(),
                       T, M, K, soi_dev.data_ptr(), sptr)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = est.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for i in range(args.steps):
            step(i)
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = est.launch_count() - l0
    ms = ev0.elapsed_time(ev1)
    graph = None
    if args.graph_steps > 0:
        # the same step loop replayed from a CUDA graph (launch overhead off the host; PDL edges kept)
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(stream)
        with torch.cuda.stream(cap):
            with torch.cuda.graph(g, stream=cap):
                for i in range(args.graph_steps):
                    ce.ce_estimate(est.handle, y_dev[i % nbuf].data_ptr(), x_dev.data_ptr(), h_dev[i % nbuf].data_ptr(),
                                   T, M, K, soi_dev.data_ptr(), cap.cuda_stream)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        g0.record(stream)
        for _ in range(reps):
            g.replay()
        g1.record(stream)
        torch.cuda.synchronize()
        graph = {"ms_per_step": g0.elapsed_time(g1) / (reps * args.graph_steps), "steps_per_graph": args.graph_steps,
                 "replays": reps}
        del g
    # practical ceiling for this traffic (outside the timed region): a plain device copy y -> h of the same
    # bytes over the same rotating buffers, back to back (torch's copy kernel, not ours)
    copy_steps = min(args.steps, 500)
    with torch.cuda.stream(stream):
        for i in range(10):
            h_dev[i % nbuf].copy_(y_dev[i % nbuf])
        torch.cuda.synchronize()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        for i in range(copy_steps):
            h_dev[i % nbuf].copy_(y_dev[i % nbuf])
        c1.record(stream)
        torch.cuda.synchronize()
    copy_us = c0.elapsed_time(c1) * 1e3 / copy_steps
    t_local = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    ms_max = float(t_local.item())
    E_glob = cfg.estimates * M_glob // cfg.M          # estimates of the whole job per step
    E = cfg.estimates * (m_hi - m_lo) // cfg.M        # this rank's estimates per launch (roofline)
    value = E_glob * args.steps / (ms_max * 1e-3)
    kernel_s = ms / args.steps * 1e-3      # one contraction launch per step on this stream

    # end-to-end through the public host-buffer API: pinned host in, pinned host out
    y_pin = torch.from_numpy(y).pin_memory()
    x_pin = torch.from_numpy(x).pin_memory()
    h_pin = torch.empty(y.shape, dtype=torch.complex64).pin_memory()
    e2e_steps = max(3, min(args.steps, args.e2e_steps))
    for _ in range(2):
        est.estimate_host(y_pin, x_pin, out=h_pin, set_of_instance=soi)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        est.estimate_host(y_pin, x_pin, out=h_pin, set_of_instance=soi)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = E_glob * e2e_steps / (float(e2e_ms.item()) * 1e-3)

    # roofline of the dominant kernel (the contraction, one launch per step)
    props = torch.cuda.get_device_properties(dev)
    peaks = _peaks()
    sel = est.selected_kernel()
    sm_max = peaks.get("sm_max_mhz") or clk.summary().get("sm_max_mhz") or 1965.0
    fp32_peak = props.multi_processor_count * 128 * 2 * sm_max * 1e6     # FFMA lanes x 2 flops x clock
    hbm_bw = peaks.get("hbm_gbs", 6548.8) * 1e9
    flops = 8.0 * cfg.b * E                                  # 4 real MACs per complex MAC, b per estimate
    alg_bytes = 16 * E + 8 * cfg.T * cfg.K * cfg.N            # y read + h written + pilots
    if sel in (ce.CE_KERNEL_TF32X3, ce.CE_KERNEL_BF16X3, ce.CE_KERNEL_BF16X3_PAIR):
        bf16 = peaks.get("bf16_tflops", 1605.7) * 1e12
        if sel == ce.CE_KERNEL_TF32X3:
            # TF32 = 1/2 bf16 (nominal ratio); 3 MMAs per product (hi/lo split)
            tc_peak, kname = bf16 * 0.5 / 3.0, "k3_tf32x3"
            src = "MEASURED_PEAKS bf16_tflops x 1/2 (tf32:bf16 nominal) / 3 (3xTF32 MMAs per product)"
        else:
            tc_peak, kname = bf16 / 3.0, ("k4_bf16x3" if sel == ce.CE_KERNEL_BF16X3 else "k5_pair")
            src = "MEASURED_PEAKS bf16_tflops / 3 (BF16x3 MMAs per product)"
        t_tc, t_hbm = flops / tc_peak, alg_bytes / hbm_bw
        if t_tc >= t_hbm:
            roof = {"bound": "tensor", "achieved": flops / kernel_s / 1e12, "peak": tc_peak / 1e12,
                    "unit": "TFLOP/s", "frac": (flops / kernel_s) / tc_peak, "peak_source": src}
        else:
            roof = {"bound": "hbm", "achieved": alg_bytes / kernel_s / 1e9, "peak": hbm_bw / 1e9, "unit": "GB/s",
                    "frac": (alg_bytes / kernel_s) / hbm_bw, "peak_source": "MEASURED_PEAKS hbm_gbs"}
        roof["roofline_time_us"] = max(t_tc, t_hbm) * 1e6
    else:
        kname = "k2_simt"
        roof = {"bound": "alu", "achieved": flops / kernel_s / 1e12, "peak": fp32_peak / 1e12, "unit": "TFLOP/s",
                "frac": (flops / kernel_s) / fp32_peak,
                "peak_source": f"{props.multi_processor_count} SMs x 128 FP32 lanes x 2 x {sm_max:.0f} MHz",
                "roofline_time_us": max(flops / fp32_peak, alg_bytes / hbm_bw) * 1e6}
    roof["copy_ceiling"] = {"us": copy_us, "frac": (2 * y.nbytes / (copy_us * 1e-6)) / hbm_bw,
                            "what": "torch copy y -> h (same 2 x y bytes, same rotating buffers), back to back: "
                                    "the practical ceiling for this read + write traffic"}
    roof.update({"traffic": _ncu_traffic(kname), "kernel": kname, "kernel_us": kernel_s * 1e6,
                 "algorithmic_flops_per_launch": flops, "algorithmic_bytes_per_launch": alg_bytes,
                 "hbm_frac": (alg_bytes / kernel_s) / hbm_bw, "fp32_simt_frac": (flops / kernel_s) / fp32_peak})

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle  # noqa: F401  (cpu_baseline leg only)
        m = max(1, min(cfg.M, args.ref_antennas * 4))
        ys = y[:1, :m]
        runs, el = _oracle_rate(cfg, x[:1], ys, r, s2, soi[:1], budget_s=args.cpu_budget_s)
        cpu = {"value": runs * m * cfg.K * cfg.N / el, "unit": "estimates/s", "cores": _cores(), "kind": "oracle",
               "sample": f"{runs} runs of oracle LS+block apply (complex128) on antennas [0,{m}) of config "
                         f"{cfg.cfg_id} instance 0, {el:.1f} s"}

    # multi-GPU verification (outside the timed region): NCCL all-gather of the antenna shards, and rank 0
    # recomputes the whole global batch on its own GPU -- the sharded result must match it bit for bit
    # (SURVEY.md §8(e) shard invariance)
    verify = None
    if world > 1 and not args.no_verify:
        try:
            from paper_1802_05427_b200.shard import gather_antenna_shards
            full = gather_antenna_shards(h_dev[(args.steps - 1) % nbuf], M_glob)
            if rank == 0:
                y_all = workload.gen_instances(cfg, 0, m_lo=0, m_hi=M_glob, x=x)
                h_ref = est.estimate(torch.from_numpy(y_all).to(dev), x_dev, set_of_instance=soi_dev)
                torch.cuda.synchronize()
                verify = {"nccl_all_gather_bytes": int(full.numel() * 8),
                          "bitwise_equal_to_single_gpu": bool(torch.equal(torch.view_as_real(full),
                                                                          torch.view_as_real(h_ref)))}
            del full
        except Exception as exc:       # never let the check take the measurement down
            verify = {"error": repr(exc)[:200]}
        dist.barrier()

    if rank == 0:
        line = {
            "metric": "channel estimates/s (antenna*user*subcarrier)", "value": value, "unit": "estimates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong" if args.strong else "weak", "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (seeded workload generator, SURVEY.md §8(d) recipe)",
            "config": _cfg_json(cfg, {"l2": f"rotating {nbuf} y/h buffer pairs ({nbuf * step_bytes / 2**20:.0f} MiB > L2)",
                                      "kernel": {0: "auto", 1: "simt", 2: "tf32x3", 3: "bf16x3", 4: "bf16x3_pair"}[args.kernel] + f"->{kname}",
                                      "global_antennas": M_glob,
                                      "parallelism": f"antenna/batch shard x{world}"}),
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "estimates/s",
                    "h2d_bytes_per_step": int(y.nbytes + x.nbytes + soi.nbytes),
                    "d2h_bytes_per_step": int(y.nbytes), "steps": e2e_steps},
            "gpu_launches": int(launches),
            "cuda_graph": graph,
            "multi_gpu_verify": verify,
            "clocks": clk.summary(),
            "filter_build_ms": build_ms,
            "device": props.name,
        }
        print(json.dumps(line), flush=True)
    est.close()
    if world > 1:
        dist.destroy_process_group()


def run_comb(args):
    """--comb NAME: the paper's comb-pilot 3W / 12W-LMMSE path (NEXT-1, K6) on one of workload.COMB_CONFIGS."""
    import torch
    import torch.distributed as dist

    import paper_1802_05427_b200 as ce
    from paper_1802_05427_b200.shard import antenna_shard

    world, rank, local = _dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = workload.get_comb_config(args.comb)
    r, s2 = workload.comb_stats(cfg)
    x = workload.comb_pilots(cfg)
    m_lo, m_hi = antenna_shard(world * cfg.M, world, rank)
    y = workload.comb_instances(cfg, x=x, m_lo=m_lo, m_hi=m_hi)
    est = ce.CombEstimator(cfg.N, cfg.S, cfg.n_ue, cfg.G, cfg.mode, r, s2).build()
    T, M, N = y.shape
    out_bytes = T * M * cfg.n_ue * N * 8
    nbuf = max(2, int(np.ceil(1.25 * L2_BYTES / (y.nbytes + out_bytes))) + 1)
    y_dev = [torch.from_numpy(y).to(dev) for _ in range(nbuf)]
    h_dev = [torch.empty((T, M, cfg.n_ue, N), dtype=torch.complex64, device=dev) for _ in range(nbuf)]
    x_dev = torch.from_numpy(x).to(dev)
    stream = torch.cuda.current_stream()
    for i in range(args.warmup):
        est.estimate(y_dev[i % nbuf], x_dev, out=h_dev[i % nbuf])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    l0 = est.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for i in range(args.steps):
            est.estimate(y_dev[i % nbuf], x_dev, out=h_dev[i % nbuf])
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = est.launch_count() - l0
    ms = ev0.elapsed_time(ev1)
    t_local = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    ms_max = float(t_local.item())
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
    e2e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = world * E * e2e_steps / (float(e2e_ms.item()) * 1e-3)
    peaks = _peaks()
    hbm_bw = peaks.get("hbm_gbs", 6548.8) * 1e9
    alg_bytes = out_bytes + y.nbytes + x.nbytes
    roof = {"bound": "hbm", "achieved": alg_bytes / kernel_s / 1e9, "peak": hbm_bw / 1e9, "unit": "GB/s",
            "frac": alg_bytes / kernel_s / hbm_bw, "peak_source": "MEASURED_PEAKS hbm_gbs", "traffic": None,
            "kernel": "k6_estimate", "kernel_us": kernel_s * 1e6, "algorithmic_bytes_per_launch": alg_bytes,
            "algorithmic_flops_per_launch": 8.0 * cfg.G * E}
    if rank == 0:
        line = {
            "metric": "channel estimates/s (antenna*user*subcarrier)", "value": value, "unit": "estimates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (workload.comb: Table III channel, fixed-design r_d / SNR_fixed)",
            "config": {"workload": f"comb_{cfg.name}_{cfg.M}x{cfg.n_ue}of{cfg.S}x{cfg.N}_T{cfg.T}_G{cfg.G}_{cfg.mode}",
                       "M": cfg.M, "S": cfg.S, "n_ue": cfg.n_ue, "N": cfg.N, "T": cfg.T, "G": cfg.G,
                       "mode": cfg.mode, "l2": f"rotating {nbuf} y/h buffer pairs (> L2)",
                       "parallelism": f"antenna shard x{world}"},
            "roofline": roof, "cpu_baseline": None,
            "e2e": {"value": e2e_value, "unit": "estimates/s", "h2d_bytes_per_step": int(y.nbytes),
                    "d2h_bytes_per_step": int(out_bytes), "steps": e2e_steps},
            "gpu_launches": int(launches), "clocks": clk.summary(), "device": torch.cuda.get_device_name(dev),
        }
        print(json.dumps(line), flush=True)
    est.close()
    if world > 1:
        dist.destroy_process_group()


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
        ev0.record(stream)
        for i in range(args.steps):
            ce.ce_stats_estimate(y_dev[i % nbuf], x_dev, D, B, soi, cfg.n_sets)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    samples = cfg.T * cfg.M * cfg.K * cfg.N
    cols = cfg.T * cfg.M * cfg.K
    lag_flops = 8.0 * cols * sum(cfg.N - d for d in range(D))
    noise_flops = 8.0 * cols * cfg.N * B
    flops = lag_flops + noise_flops
    props = torch.cuda.get_device_properties(0)
    fp32_peak = props.multi_processor_count * 128 * 2 * 1965e6
    # the library's policy (k7_stats.cu): lags on the tensor cores (K8, BF16x3) from 16384 columns, noise window then
    # streamed by K7c; below, K7a does both on the FP32 pipes
    k8 = cols >= 16384 and cfg.K <= 24 and D <= 512 and cfg.N % 2 == 0
    bf16 = _peaks().get("bf16_tflops", 1605.7) * 1e12
    t_ideal = (lag_flops / (bf16 / 3) + noise_flops / fp32_peak) if k8 else flops / fp32_peak
    line = {"metric": "LS samples/s through the statistics estimator (NEXT-3)", "value": samples / (ms * 1e-3),
            "unit": "samples/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded workload generator)",
            "config": _cfg_json(cfg, {"D": D, "B": B, "l2": f"rotating {nbuf} y buffers (> L2)"}),
            "roofline": {"bound": "tensor+alu" if k8 else "alu", "achieved": flops / (ms * 1e-3) / 1e12,
                         "peak": flops / t_ideal / 1e12, "unit": "TFLOP/s", "frac": t_ideal / (ms * 1e-3),
                         "traffic": None, "roofline_time_us": t_ideal * 1e6,
                         "kernel": "k8_gram (lags) + k7_noise (noise window)" if k8 else "k7_accumulate",
                         "algorithmic_flops_per_launch": flops,
                         "note": ("effective peak of the mix: lag flops at the BF16 peak / 3 (BF16x3) plus noise-window "
                                  "flops at the FP32 SIMT peak" if k8 else "lag + noise-window flops vs the FP32 SIMT peak")},
            "gpu_launches": (3 if k8 else 2) * args.steps, "clocks": clk.summary(), "device": props.name}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--kernel", type=int, default=0, help="0 auto, 1 simt, 2 tf32x3, 3 bf16x3, 4 bf16x3_pair")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--graph-steps", type=int, default=100, help="steps per CUDA-graph replay (0: skip)")
    ap.add_argument("--ref-antennas", type=int, default=4)
    ap.add_argument("--cpu-budget-s", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-verify", action="store_true", help="skip the N>1 NCCL gather + single-GPU bitwise check")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: split the configuration's M antennas across the ranks (default: weak, M per rank)")
    ap.add_argument("--stats", action="store_true", help="time the NEXT-3 statistics estimator instead")
    ap.add_argument("--comb", default=None, help="run the comb-pilot 3W/12W path on workload.COMB_CONFIGS[NAME]")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
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
