"""Key metrics of the round-2 ncu captures (tools/ncu_r02.sh) into profiles/:
  r02_ncu_full_summaries.txt      one line per profiled launch (time, DRAM bytes, throughput, issue)
  k2_ncu_summary.json             K2's DRAM bytes per launch (bench.py scales it for roofline_k2)
  k1b_tp8_ncu_summary.json        K1b (tensor-map TMA) over an HBM pool at TP8
  r02_ncu_bench_launches_summary.json   the bench command's launch list, split per stage pass
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic"]
MULT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Tbyte": 1e12}
TMUL = {"ms": 1e3, "msecond": 1e3, "us": 1.0, "usecond": 1.0, "ns": 1e-3, "nsecond": 1e-3}

# algorithmic bytes of each capture (read + write of the payload the launch moves)
ALG = {
    "r02_prof_k2": ("K2 paged scatter, HBM staging -> pages: one layer x 128 Llama-3.1-8B chunks",
                    2 * 128 * 2 * 256 * 8 * 128 * 2),
    "r02_prof_k1b_tp8": ("K1b tensor-map TMA over an HBM pool, Llama-3-70B TP8 rank 7, 128 chunks, flash-attn pages",
                         2 * 128 * 80 * 2 * 256 * 1 * 128 * 2),
    "r02_prof_k1b_tp8_hnd": ("K1b tensor-map TMA over an HBM pool, Llama-3-70B TP8 rank 7, 128 chunks, HND pages",
                             2 * 128 * 80 * 2 * 256 * 1 * 128 * 2),
    "r02_prof_k1b_full": ("K1b tensor-map TMA over an HBM pool, Llama-3.1-8B, 128 chunks, full heads",
                          2 * 128 * 32 * 2 * 256 * 8 * 128 * 2),
}


def rows(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        return []
    return [(r[0], r[1], v) for v in r[2:]]


def value(h, units, v, key):
    i = h.index(key)
    x = float(v[i].replace(",", ""))
    if key.startswith("dram__bytes"):
        return x * MULT.get(units[i], 1)
    if key == "gpu__time_duration.sum":
        return x * TMUL.get(units[i], 1.0)
    return x


def main():
    lines, summaries = [], {}
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    for name in ["r02_prof_k2", "r02_prof_k1b_tp8", "r02_prof_k1b_tp8_hnd", "r02_prof_k1b_full", "r02_prof_hash"]:
        rep = OUT / f"{name}.ncu-rep"
        if not rep.exists():
            continue
        for h, units, v in rows(rep):
            kn = v[h.index("Kernel Name")].split("(")[0].replace("(anonymous namespace)::", "")
            parts = [f"{k.split('.')[0]}={v[h.index(k)]} {units[h.index(k)]}".strip() for k in KEYS if k in h]
            lines.append(f"{name} | {kn} | " + " | ".join(parts))
            if name in ALG and name not in summaries:
                t = value(h, units, v, "gpu__time_duration.sum")
                rd, wr = value(h, units, v, "dram__bytes_read.sum"), value(h, units, v, "dram__bytes_write.sum")
                what, alg = ALG[name]
                summaries[name] = {"kernel": kn + " -- " + what, "source": f"ncu --set full --clock-control none ({name})",
                                   "gpu_time_us": t, "dram_bytes_read": int(rd), "dram_bytes_write": int(wr),
                                   "dram_bytes_per_launch": int(rd + wr), "algorithmic_bytes_per_launch": alg,
                                   "achieved_GBps_cold": alg / (t * 1e-6) / 1e9,
                                   "frac_of_hbm_peak_cold": alg / (t * 1e-6) / 1e9 / peak,
                                   "note": "ncu times are cold-cache and serialised; DRAM reads vs the algorithmic "
                                           "read bytes show re-reads; writes still in L2 at kernel end are uncounted"}
    (ROOT / "profiles" / "r02_ncu_full_summaries.txt").write_text("\n".join(lines) + "\n")
    if "r02_prof_k2" in summaries:
        (ROOT / "profiles" / "k2_ncu_summary.json").write_text(json.dumps(summaries["r02_prof_k2"], indent=1) + "\n")
    for k in ("r02_prof_k1b_tp8", "r02_prof_k1b_tp8_hnd", "r02_prof_k1b_full"):
        if k in summaries:
            (ROOT / "profiles" / f"{k.replace('r02_prof_', '')}_ncu_summary.json").write_text(
                json.dumps(summaries[k], indent=1) + "\n")
    launches = OUT / "r02_ncu_bench_launches.csv"
    if launches.exists():
        out = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_launch_summary.py"), str(launches)],
                             capture_output=True, text=True).stdout
        (ROOT / "profiles" / "r02_ncu_bench_launches_summary.json").write_text(out)
    print("\n".join(lines))


if __name__ == "__main__":
    sys.exit(main())
