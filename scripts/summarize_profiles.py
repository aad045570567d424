"""Summarise ncu output for profiles/: python scripts/summarize_profiles.py <round_tag>.

Inputs (in gpurun_out/): launches_block.csv (ncu --metrics gpu__time_duration.sum
--csv of scripts/profile_block.py 2 2), full_block.ncu-rep (ncu --set full of
scripts/profile_block.py 1 0).  Outputs: profiles/<tag>_summary.json (per-kernel
times of the last prefill and decode block forward; launches are serialised and
cold-L2, so compare shares, not absolutes) and profiles/<tag>_ncu_full.json
(selected --set full counters per kernel of one prefill forward)."""
import csv
import io
import json
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
FULL_KEYS = [
    "Kernel Name", "launch__grid_size", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
    "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
]


def short(name: str) -> str:
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"\(.*$", "", name)
    return name.replace("hap::", "")


def launches(path: Path):
    text = path.read_text()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    out = []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        us = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
        out.append((short(r["Kernel Name"]), round(us, 1)))
    return out


def forwards(ls):
    """Split the launch list at combine kernels (the last kernel of a block forward)."""
    segs, cur = [], []
    for k in ls:
        cur.append(k)
        if "combine" in k[0]:
            segs.append(cur)
            cur = []
    return segs


def main(tag: str) -> None:
    prof = ROOT / "profiles"
    src = OUT / "launches_block.csv"
    if src.exists():
        segs = forwards(launches(src))
        pre = [s for s in segs if any("attn_pair" in k or "attn_tc" in k for k, _ in s)]
        dec = [s for s in segs if any("decode_mma" in k for k, _ in s)]
        summ = {"source": "ncu --metrics gpu__time_duration.sum --clock-control none, scripts/profile_block.py 2 2 "
                          "(launches are serialised, cold L2: compare shares)"}
        for name, ss in (("prefill_forward", pre), ("decode_forward", dec)):
            if ss:
                s = ss[-1]
                summ[name] = {"total_us": round(sum(t for _, t in s), 1), "kernels": s}
        (prof / f"{tag}_summary.json").write_text(json.dumps(summ, indent=1))
    rep = OUT / "full_block.ncu-rep"
    raw_csv = OUT / "full_block_raw.csv"  # written on the GPU box when the .ncu-rep is too big to bring back
    raw = None
    if rep.exists():
        raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    elif raw_csv.exists():
        raw = raw_csv.read_text()
    if raw:
        rows = list(csv.reader(io.StringIO(raw[raw.find('"ID"'):])))
        hdr, units, data = rows[0], rows[1], rows[2:]
        out = []
        gemm_phase = iter(["qkv", "o_proj", "gate_up", "down"])  # grouped_gemm launches of one prefill forward
        for r in data:
            d = dict(zip(hdr, r))
            u = dict(zip(hdr, units))
            e = {k: (d.get(k, "") + (" " + u[k] if u.get(k) else "")).strip() for k in FULL_KEYS if k in d}
            if "grouped_gemm_kernel" in d.get("Kernel Name", ""):
                e["phase"] = next(gemm_phase, "?")
            out.append(e)
        (prof / f"{tag}_ncu_full.json").write_text(json.dumps(
            {"source": "ncu --set full --clock-control none --import-source on, scripts/profile_block.py 1 0 "
                       "(Mixtral-8x7B prefill 8x2048, one block forward)", "launches": out}, indent=1))
        # DRAM traffic of the expert GEMMs against their algorithmic bytes (bench.py reads this file)
        T, h, I, E, k = 8 * 2048, 4096, 14336, 8, 2
        algo = {"gate_up": T * k * h * 2 + E * 2 * I * h * 2 + T * k * I * 2,
                "down": T * k * I * 2 + E * h * I * 2 + T * k * h * 2}
        tr = {"source": f"profiles/{tag}_ncu_full.json (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum)",
              "kernel": "hap::gemm::grouped_gemm_kernel (Mixtral-8x7B, 32768 routed rows)"}
        for e in out:
            ph = e.get("phase")
            if ph in algo:
                def num(key):
                    v, _, unit = e[key].partition(" ")
                    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
                    return float(v.replace(",", "")) * scale
                dram = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
                tr[ph] = {"dram_bytes_per_launch": dram, "algorithmic_bytes": algo[ph],
                          "traffic_over_algorithmic": dram / algo[ph]}
        if "gate_up" in tr:
            tr["dram_bytes_per_launch"] = tr["gate_up"]["dram_bytes_per_launch"]
            tr["algorithmic_bytes"] = tr["gate_up"]["algorithmic_bytes"]
            (prof / f"{tag}_gemm_traffic.json").write_text(json.dumps(tr, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
