"""Busiest execution pipe per kernel from an ncu --set full raw page.

    python tools/pipe_util.py profiles/r01/r01_full_raw.csv profiles/pipe_util.json

Writes {kernel: {"pipe": name, "pct": % of that pipe's peak, "issue_pct": %}}
(sm__inst_executed_pipe_*.avg.pct_of_peak_sustained_active); bench.py quotes
the dominant kernel's entry next to its HBM roofline.
"""
import csv, json, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
PIPES = ["alu", "fma", "fmaheavy", "fp64", "lsu", "xu", "uniform", "tensor"]
out = {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").strip()
    if "<" in name and not name.startswith("<"):
        name = name[: name.index("<")]  # template arguments
    best = None
    for p in PIPES:
        col = f"sm__inst_executed_pipe_{p}.avg.pct_of_peak_sustained_active"
        if col in hdr:
            try:
                v = float(r[hdr.index(col)])
            except ValueError:
                continue
            if best is None or v > best[1]:
                best = (p, v)
    issue = hdr.index("smsp__issue_active.avg.pct_of_peak_sustained_active")
    if best and name not in out:
        out[name] = {"pipe": best[0], "pct": round(best[1], 1), "issue_pct": round(float(r[issue]), 1)}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
