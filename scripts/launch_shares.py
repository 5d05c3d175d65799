"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel.

    python scripts/launch_shares.py gpurun_out/launches.csv --source "<ncu command>" > profiles/rNN_launch_shares.json

Per kernel family: launches, total and mean device time, share of the listed
time.  ncu serialises launches and runs them cold-cache, so compare SHARES
with the bench's CUDA-event breakdown, not absolute times.
"""
import csv
import io
import json
import re
import sys

FAMILIES = [
    ("gemm_pair", r"gemm_pair_kernel"), ("gemm_tn", r"gemm_tn_kernel"),
    ("gemm_skinny", r"gemm_skinny_kernel"), ("chunk_attn_fa", r"chunk_attn_fa_kernel"),
    ("fa_combine", r"fa_combine_kernel"), ("chunk_attn_mma", r"chunk_attn_kernel"),
    ("attn_combine", r"attn_combine_kernel"), ("decode_attn", r"decode_attn"),
    ("norm", r"norm_kernel"), ("kv_write", r"kv_write"), ("embed", r"embed"),
    ("argmax", r"argmax"), ("gather_rows", r"gather_rows"),
]


def family(name: str) -> str:
    for fam, pat in FAMILIES:
        if re.search(pat, name):
            return fam
    return name.split("(")[0][-60:]


def main():
    path = sys.argv[1]
    source = sys.argv[sys.argv.index("--source") + 1] if "--source" in sys.argv else ""
    text = open(path).read()
    lines = text[text.index('"ID"'):] if '"ID"' in text else text
    rows = list(csv.DictReader(io.StringIO(lines)))
    agg: dict = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1e3 if unit == "ns" else v * 1e3 if unit == "ms" else v
        f = family(r["Kernel Name"])
        a = agg.setdefault(f, {"launches": 0, "us": 0.0})
        a["launches"] += 1
        a["us"] += us
    total = sum(a["us"] for a in agg.values())
    out = {"source": source, "launches": sum(a["launches"] for a in agg.values()),
           "total_us": round(total, 1), "by_kernel": {}}
    for f, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
        out["by_kernel"][f] = {"launches": a["launches"], "us": round(a["us"], 1),
                               "mean_us": round(a["us"] / a["launches"], 2),
                               "share": round(a["us"] / total, 4) if total else 0.0}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
