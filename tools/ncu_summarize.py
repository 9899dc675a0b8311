"""Key metrics of the ncu --set full reports in gpurun_out/ (tools/ncu_full.sh), one line per
kernel launch, into profiles/r01_ncu_full_summaries.txt; K2's DRAM bytes into k2_ncu_summary.json."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size"]


def rows(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        return []
    h, units = r[0], r[1]
    return [(h, units, v) for v in r[2:]]


def main():
    lines = []
    k2 = None
    for name in ["prof_hash", "prof_score", "prof_k2", "prof_bulk", "prof_k1hbm", "prof_index"]:
        rep = ROOT / "gpurun_out" / f"{name}.ncu-rep"
        if not rep.exists():
            continue
        for h, units, v in rows(rep):
            kn = v[h.index("Kernel Name")].split("(")[0].replace("(anonymous namespace)::", "")
            parts = [f"{k.split('.')[0]}={v[h.index(k)]} {units[h.index(k)]}".strip() for k in KEYS if k in h]
            lines.append(f"{name} | {kn} | " + " | ".join(parts))
            if name == "prof_k2" and k2 is None:
                mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
                rd = float(v[h.index("dram__bytes_read.sum")]) * mult[units[h.index("dram__bytes_read.sum")]]
                wr = float(v[h.index("dram__bytes_write.sum")]) * mult[units[h.index("dram__bytes_write.sum")]]
                tu = units[h.index("gpu__time_duration.sum")]
                t = float(v[h.index("gpu__time_duration.sum")]) * {"ms": 1e3, "us": 1.0, "ns": 1e-3}.get(tu, 1.0)
                alg = 2 * 128 * (2 * 256 * 8 * 128 * 2)  # read + write of one layer of 128 Llama-8B chunks
                k2 = {"kernel": kn + " (K2 paged scatter, HBM staging -> pages), one layer x 128 chunks of Llama-3.1-8B KV (per-layer fences)",
                      "source": "ncu --set full --clock-control none -k regex:k_ingest_ldg -s 2 -c 1 python tools/prof_targets.py ingest-ce (final r01 code)",
                      "gpu_time_us": t, "dram_bytes_read": int(rd), "dram_bytes_write": int(wr),
                      "dram_bytes_per_launch": int(rd + wr), "algorithmic_bytes_per_launch": alg,
                      "note": "reads equal the staged payload (no re-reads); writes still in L2 at kernel end are not counted"}
    (ROOT / "profiles" / "r01_ncu_full_summaries.txt").write_text("\n".join(lines) + "\n")
    if k2:
        (ROOT / "profiles" / "k2_ncu_summary.json").write_text(json.dumps(k2, indent=1) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    sys.exit(main())
