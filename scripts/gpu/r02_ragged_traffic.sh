# expert GEMMs in isolation: DRAM bytes with balanced (4096 rows per expert) vs ragged (multinomial) segments
for r in 0 1; do
  SWEEP_RAGGED=$r timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:grouped_gemm -c 6 --csv python scripts/gemm_l2_sweep.py 1 2>/dev/null > gpurun_out/ragged_$r.csv
  python - "$r" <<'P'
import csv, io, sys
txt = open(f"gpurun_out/ragged_{sys.argv[1]}.csv").read()
rows = list(csv.DictReader(io.StringIO(txt[txt.find('"ID"'):])))
by = {}
for r in rows:
    by.setdefault(int(r["ID"]), {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
for i, m in sorted(by.items()):
    print(f"ragged={sys.argv[1]} launch {i}: read {m['dram__bytes_read.sum']/1e9:.2f} GB write {m['dram__bytes_write.sum']/1e9:.2f} GB {m['gpu__time_duration.sum']/1e6:.3f} ms")
P
done
