"""Measure the stage-switch inputs on B200: dequant-time table (reference CSV
format, transition.py:100-124) and pinned H2D bandwidth.

  python scripts/measure_transition.py [--out-dir gpurun_out]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2508_19373_b200.config import import_moeplan  # noqa: E402
from paper_2508_19373_b200.transition import dequant_table, measure_dequant_seconds, measure_h2d_bandwidth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out-dir", default="gpurun_out")
args = ap.parse_args()
mp = import_moeplan()
from moeplan.transition import table_to_csv  # noqa: E402

meas = measure_dequant_seconds(range(10, 32))
table = dequant_table(meas)
out = Path(args.out_dir)
out.mkdir(parents=True, exist_ok=True)
table_to_csv(table, str(out / "r01_dequant_table.csv"))
h2d = measure_h2d_bandwidth()
top = max(meas)
rep = {"dequant_seconds_measured": {str(k): v for k, v in meas.items()},
       "dequant_params_per_s_at_2^31": top / meas[top],
       "dequant_bytes_per_s_at_2^31": top * (0.5 + 2 + 16 / 128) / meas[top],
       "h2d_pinned_bytes_per_s": h2d,
       "reference_default_rate_params_per_s": 20e9}
(out / "r01_transition_measurements.json").write_text(json.dumps(rep, indent=1))
print(json.dumps({k: v for k, v in rep.items() if k != "dequant_seconds_measured"}, indent=1))
