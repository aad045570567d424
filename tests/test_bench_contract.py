"""bench.py's reference arm on CPU: one JSON line with the contract keys the
driver reads (impl, metric, value, unit, e2e, cpu_baseline), at the tiny
config so it finishes in seconds; and the planner-time baseline (the
reference's own CPU path) returns a median per scenario."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_prints_one_contract_line():
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "tiny",
                          "--steps", "2", "--warmup", "3", "--cpu-sample-tokens", "64"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "cpu_baseline", "e2e", "config", "dtype"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1


def test_planner_baseline_times_the_reference_plan():
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2508_19373_b200.config import get_config

    out = bench.planner_baseline(get_config("mixtral-8x7b"), 8, reps=2)
    for k in ("prefill_8x2048_roofline_ms", "prefill_8x2048_measured_tables_ms", "decode_b64_roofline_ms",
              "decode_b64_measured_tables_ms"):
        assert out[k] > 0
