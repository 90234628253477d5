"""bench.py's reference arm (the CPU oracle, the one place besides tests that
runs it) prints one JSON line with the contract's keys; runs on CPU."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "2", "--warmup", "1", "--cpu-sample", "2000"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in j, key
    assert j["impl"] == "reference" and j["unit"] == "epochs/s" and j["value"] > 0
    import os
    assert j["cpu_baseline"]["kind"] == "oracle" and j["cpu_baseline"]["cores"] == len(os.sched_getaffinity(0))
    assert j["cpu_baseline"]["cpu_model"] and "OMP_NUM_THREADS" in j["cpu_baseline"]
    # the line reports what it timed: K steps of ms_per_step fit in the run's wall time
    assert j["steps"] * j["ms_per_step"] <= j["wall_s"] * 1e3
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["e2e"]["value"] == j["value"]
    assert j["config"]["workload"].startswith("c1")
