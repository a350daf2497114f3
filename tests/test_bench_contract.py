"""The bench.py JSON-line contract (the driver parses these keys).

CPU: the reference arm (the oracle on the host cores) for C1, and `--gpus N`
failing loudly without N GPUs.  GPU: the default line's keys, on C1 (seconds)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def _run(args, timeout=600):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT, env=env)
    return r


def test_reference_arm_line():
    r = _run(["--impl", "reference", "--config", "C1", "--steps", "3", "--warmup", "3"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and BASE_KEYS <= set(d)
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("C1")


def test_gpus_more_than_available_fails_loudly():
    import torch
    n = torch.cuda.device_count() + 1
    r = _run(["--gpus", str(n), "--steps", "1", "--warmup", "3"], timeout=300)
    assert r.returncode == 1 and "needs" in r.stderr


@pytest.mark.gpu
def test_default_line_keys_on_c1():
    r = _run(["--config", "C1", "--steps", "5", "--warmup", "3", "--cpu-seconds", "0.5", "--no-other-configs"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert BASE_KEYS <= set(d) and {"roofline", "gpu_launches", "clocks"} <= set(d)
    rf = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(rf) and rf["frac"] == pytest.approx(
        rf["achieved"] / rf["peak"], abs=2e-4)
    assert {"value", "unit", "cores", "kind", "sample"} <= set(d["cpu_baseline"])
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(d["e2e"])
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["n_gpus"] == 1 and d["higher_is_better"] is True


@pytest.mark.gpu
def test_sustained_leg_and_c1_cold_on_c2():
    """The burst-vs-sustained leg (DESIGN 8.1) on C2, and C1's cold-L2 figure from
    `other_configs` is covered by the default run; here: the `sustained` object."""
    r = _run(["--config", "C2", "--steps", "5", "--warmup", "3", "--no-cpu-baseline", "--no-other-configs",
              "--no-ceilings", "--no-e2e"])
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    s = d["sustained"]
    assert {"steps", "seconds", "first_ms_per_step", "first_frac", "last_ms_per_step", "value", "unit", "frac",
            "clocks"} <= set(s)
    assert s["steps"] >= 20 and s["seconds"] > 0.3 and s["unit"] == "GB/s"
    assert 0.2 < s["frac"] <= s["first_frac"] * 1.05  # the sustained rate never beats the burst by more than noise
    assert s["value"] == pytest.approx(2 ** 28 * 6 / s["last_ms_per_step"] / 1e6, rel=1e-3)
