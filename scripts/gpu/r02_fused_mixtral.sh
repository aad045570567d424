# Mixtral-8x7B decode B=1: fused norm+QKV vs two launches, alternating, then per-kernel launch lists of each
mkdir -p gpurun_out
for rep in 1 2 3; do for f in 0 1; do HAP_FUSED_NORM=$f python scripts/decode_ab.py mixtral-8x7b 1 2 2>&1 | tail -1 | sed "s/^/fused=$f /"; done; done > gpurun_out/fused_mixtral_ab.txt
cat gpurun_out/fused_mixtral_ab.txt
for f in 0 1; do
  HAP_FUSED_NORM=$f timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fused_launch_$f.csv python scripts/decode_ab.py mixtral-8x7b 1 > /dev/null 2>&1
done
python - <<'P'
import csv, io
for f in (0, 1):
    rows = list(csv.DictReader(io.StringIO("".join(l for l in open(f"gpurun_out/fused_launch_{f}.csv") if not l.startswith("==")))))
    names = [(r["Kernel Name"][:60], float(r["Metric Value"])) for r in rows if r.get("Metric Name") == "gpu__time_duration.sum"]
    tail = names[-14:]
    print(f"fused={f}: last {len(tail)} launches", [(n.split("(")[0][-38:], round(v / 1e3, 1)) for n, v in tail])
P
