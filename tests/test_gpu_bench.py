"""bench.py end to end on the GPU: every mode prints one parseable JSON line with the contract's keys
(short runs; the numbers themselves are the bench's business)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=900, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("extra", [
    ["--config", "3"],
    ["--config", "3", "--launch", "direct"],
    ["--config", "1"],
    ["--config", "2", "--strong"],
    ["--comb", "paper_12w"],
    ["--comb", "paper_3w"],
    ["--stats"],
])
def test_bench_modes(extra):
    d = _run("--steps", "5", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "3", "--sweep", "", *extra)
    keys = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
            "roofline", "gpu_launches", "clocks"]
    if "--stats" not in extra:            # the statistics line has no host-buffer path
        keys.append("e2e")
    for key in keys:
        assert key in d, key
    assert d["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["frac"] > 0


def test_bench_default_fields():
    """The fields the round-2 review asked for: kernel dtype label, parity sample, CPU-baseline details, sweep."""
    d = _run("--steps", "20", "--warmup", "5", "--cpu-budget-s", "1", "--sweep", "4", "--sweep-steps", "3")
    assert "bf16x3" in d["dtype"] or "tf32x3" in d["dtype"]
    assert d["parity"]["max_rel_err_per_instance"] <= 1e-4 and d["parity"]["max_row_rel_err"] <= 1e-3
    cpu = d["cpu_baseline"]
    assert cpu["runs"] >= 3 and cpu["cpu_model"] and cpu["blas"] and cpu["one_thread"]["value"] > 0
    assert d["sweep"][0]["workload"].startswith("config4_") and d["sweep"][0]["roofline"]["frac"] > 0
    assert d["gpu_launches"] == 20 and d["first_call"]["first_call_host_us"] > 0


@pytest.mark.parametrize("strong", [False, True])
def test_bench_two_ranks_on_one_gpu(strong):
    """The real multi-rank path on the single leased GPU: bench.py spawns 2 ranks (gloo: both on cuda:0), each
    runs ce_estimate on its antenna shard, the max over ranks is reduced, the shards are gathered and rank 0
    compares them bit for bit with its own single-GPU estimate of the whole batch (antennas are
    independent).  The ranks' kernels never wait on one another."""
    extra = ["--strong"] if strong else []
    d = _run("--gpus", "2", "--backend", "gloo", "--config", "1", "--steps", "5", "--warmup", "3",
             "--no-cpu-baseline", "--e2e-steps", "3", "--sweep", "", *extra)
    assert d["n_gpus"] == 2 and len(d["per_rank_ms_per_step"]) == 2
    assert d["scaling"] == ("strong" if strong else "weak")
    assert d["config"]["global_antennas"] == (8 if strong else 16)
    assert d["multi_gpu_verify"]["bitwise_equal_to_single_gpu"] is True, d["multi_gpu_verify"]
    if not strong:
        assert d["strong"]["value"] > 0 and len(d["strong"]["per_rank_ms_per_step"]) == 2


def test_bench_reference_arm():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
