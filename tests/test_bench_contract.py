"""bench.py's JSON contract, checked on the CPU through the reference arm (the GPU arm
prints the same keys plus roofline/e2e/clocks; it runs in the GPU suite and the bench)."""

import json
import subprocess
import sys

from conftest import REPO


def test_reference_arm_prints_one_contract_line():
    r = subprocess.run([sys.executable, str(REPO / "bench.py"), "--impl", "reference", "--workload", "c1",
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600,
                       cwd=str(REPO))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "gpu_launches"):
        assert key in d, key
    assert d["impl"] == "reference" and d["unit"] == "Gpoints/s" and d["higher_is_better"] is True
    assert d["config"]["workload"] == "c1" and d["value"] > 0
    cb = d["cpu_baseline"]
    # config 1 is rank 2 and small: the reference's own Machine (baseline/_ref) is timed,
    # on the full config for exactly the requested steps
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["config"]["same_config"] is True and cb["steps"] == d["steps"]
    assert abs(d["ms_per_step"] * d["steps"] / 1e3 - cb["seconds"]) < 0.01


def test_reference_arm_port_on_a_3d_config_states_its_sample():
    """The port path (rank 3, which the reference Machine rejects): with a tight budget it
    times a slab sample and says so (same_config false, measured ms_per_step)."""
    import os
    env = dict(os.environ, LOPE_BENCH_REF_BUDGET_S="3")
    r = subprocess.run([sys.executable, str(REPO / "bench.py"), "--impl", "reference", "--workload", "c3",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600,
                       cwd=str(REPO), env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.strip()][-1])
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["same_config"] is False and "slab of the full" in cb["sample"]
    assert d["config"]["same_config"] is False and d["value"] > 0
    assert d["e2e"] == {"value": d["value"], "unit": "Gpoints/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["gpu_launches"] == 0


def test_config1_defaults_to_its_own_step_count():
    """Without --steps, config 1 is timed over its own 100 steps (BASELINE config 1)."""
    r = subprocess.run([sys.executable, str(REPO / "bench.py"), "--impl", "reference", "--workload", "c1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=str(REPO))
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.strip()][-1])
    assert d["steps"] == 100 and d["cpu_baseline"]["steps"] == 100
