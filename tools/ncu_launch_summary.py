"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list of `bench.py`.

Each stage pass starts with the scorer (k_score), so the list splits into passes: value-arm
warm-up, value-arm timed pass (+ the live K1 roofline launches), e2e-arm warm-up, e2e-arm timed
pass (+ the live K2 roofline launches).  Per segment: launches and summed ncu time per kernel.
ncu times are cold-cache and serialised: compare shares of a pass, not absolute times.
    python tools/ncu_launch_summary.py launches.csv > summary.json
"""
import csv
import json
import sys
from collections import OrderedDict


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, mi, ui, vi = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    gi = h.index("Grid Size")
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}
    segs, cur = [], None
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")
        if name == "k_score" or cur is None:
            cur = OrderedDict()
            segs.append(cur)
        us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        k = f"{name} grid={r[gi]}"
        a = cur.setdefault(k, {"launches": 0, "total_ms": 0.0, "max_us": 0.0})
        a["launches"] += 1
        a["total_ms"] += us / 1e3
        a["max_us"] = max(a["max_us"], us)
    out = []
    for s in segs:
        tot = sum(v["total_ms"] for v in s.values())
        out.append({"total_ms": round(tot, 3),
                    "kernels": {k: {**v, "total_ms": round(v["total_ms"], 3), "max_us": round(v["max_us"], 1),
                                    "share": round(v["total_ms"] / tot, 4) if tot else 0} for k, v in s.items()}})
    print(json.dumps({"source": path, "segments": out}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
