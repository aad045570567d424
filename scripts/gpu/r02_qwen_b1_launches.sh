mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qwen_b1_launch.csv python scripts/decode_ab.py qwen2-57b-a14b 1 > /dev/null 2>&1
python - <<'P'
import csv, io
rows = list(csv.DictReader(io.StringIO("".join(l for l in open("gpurun_out/qwen_b1_launch.csv") if not l.startswith("==")))))
names = [(r["Kernel Name"], float(r["Metric Value"])) for r in rows if r.get("Metric Name") == "gpu__time_duration.sum"]
tail = names[-18:]
tot = 0
for n, v in tail:
    tot += v
    print(f"{v/1e3:8.1f} us  {n.split('(')[0][-60:]}")
print("sum", tot / 1e3)
P
