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
    ["--config", "1"],
    ["--config", "2", "--strong"],
    ["--comb", "paper_12w"],
    ["--comb", "paper_3w"],
    ["--stats"],
])
def test_bench_modes(extra):
    d = _run("--steps", "5", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "3", "--graph-steps", "0", *extra)
    keys = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
            "roofline", "gpu_launches", "clocks"]
    if "--stats" not in extra:            # the statistics line has no host-buffer path
        keys.append("e2e")
    for key in keys:
        assert key in d, key
    assert d["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["frac"] > 0


def test_bench_reference_arm():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
