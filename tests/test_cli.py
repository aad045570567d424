"""CLI in the reference's conventions (moeplan cli.py): JSON payload with a
manifest, exit codes 0 / 2 (config) / 3 (infeasible) / 4 (internal)."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def run(*args):
    r = subprocess.run([sys.executable, "-m", "paper_2508_19373_b200", *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    return r.returncode, r.stdout, r.stderr


def test_plan_matches_library_and_carries_manifest():
    from paper_2508_19373_b200.config import get_config
    from paper_2508_19373_b200.plan import plan_for

    rc, out, _ = run("plan", "--preset", "mixtral-8x7b", "--devices", "8", "--batch", "8", "--input", "2048")
    assert rc == 0
    d = json.loads(out)
    ref = plan_for(get_config("mixtral-8x7b"), 8, 8, 2048, 0).plan
    assert d["plan"]["attention"] == ref.attention.label()
    assert d["plan"]["expert_prefill"] == ref.expert_prefill.label()
    assert d["baseline_tp"]["attention"] == "attn(tp=8,dp=1)"
    m = d["manifest"]
    assert m["command"] == "plan" and m["flags"]["devices"] == 8 and m["config_paths"]["hw"].endswith("b200.cfg")


def test_plan_reads_reference_format_hardware_file(tmp_path):
    hw = tmp_path / "slow.cfg"
    hw.write_text("[hardware]\nn_devices = 4\npeak_flops = 1e15\ndevice_mem_bytes = 180e9\n"
                  "intra_node_bw = 1e9\nhost_to_device_bw = 1e9\n")
    rc, out, _ = run("plan", "--preset", "mixtral-8x7b", "--hw", str(hw), "--batch", "8", "--input", "2048")
    assert rc == 0 and json.loads(out)["n_devices"] == 4


def test_exit_codes():
    rc, _, err = run("plan", "--preset", "no-such-model")
    assert rc == 2 and json.loads(err)["error"] == "config"
    rc, _, _ = run("plan", "--preset", "mixtral-8x7b", "--hw", "/nonexistent.cfg")
    assert rc == 2


@pytest.mark.gpu
def test_run_tiny_prefill_and_decode():
    rc, out, err = run("run", "--preset", "tiny", "--batch", "4", "--input", "128", "--output-len", "64",
                       "--steps", "2")
    assert rc == 0, err
    d = json.loads(out)
    assert d["prefill"]["tokens"] == 512 and d["prefill"]["tokens_per_s"] > 0
    assert d["decode"]["kv_len"] == 128 + 32


@pytest.mark.gpu
def test_measure_writes_reference_calibration_csv(tmp_path):
    from paper_2508_19373_b200.config import import_moeplan

    import_moeplan()
    from moeplan.costmodel import read_samples_csv

    csv = tmp_path / "cal.csv"
    rc, out, err = run("measure", "--preset", "tiny", "--devices", "2", "--batch", "4", "--input", "128",
                       "--stage", "prefill", "--reps", "1", "--out-csv", str(csv))
    assert rc == 0, err
    samples = read_samples_csv(str(csv))
    assert len(samples) == json.loads(out)["n_samples"] > 0
