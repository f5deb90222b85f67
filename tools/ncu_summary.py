"""Summarise an ncu --set full report (per kernel) as markdown + DRAM traffic per pixel and stage (json).

    python tools/ncu_summary.py REPORT.ncu-rep|RAW.csv NPIX OUT.json
"""
import csv, io, json, subprocess, sys
from collections import defaultdict

rep, npx = sys.argv[1], float(sys.argv[2])
raw = (open(rep).read() if rep.endswith(".csv")
       else subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
idx = {w: hdr.index(w) for w in want if w in hdr}
SCALE = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
         "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
STAGE = {"k_lum_log": "tonemap", "k_tm_nodes": "tonemap", "k_tm_scalars": "tonemap", "k_base_layer": "base",
         "k_sdr_ycc": "base", "k_sdr_fix": "base", "k_prefilter_cols": "prefilter",
         "k_prefilter_fused": "prefilter", "k_prefilter_v": "prefilter", "k_prefilter_h": "prefilter",
         "k_sort_hist": "fit", "k_sort_scan": "fit", "k_sort_scatter": "fit", "k_seg_setup": "fit", "k_seg_nodes": "fit",
         "k_seg_dot": "fit", "k_seg_reduce_coef": "fit", "k_estimate": "estimate", "k_crc_chunks": "crc",
         "k_crc_combine": "crc", "k_entropy_dct": "entropy_dct", "k_entropy_plane": "entropy_plane",
         "k_entropy_fixup": "entropy_plane", "k_assemble": "assemble"}


def val(r, k):
    try:
        return float(r[idx[k]].replace(",", "")) * SCALE.get(units[idx[k]], 1.0)
    except Exception:
        return float("nan")


out = ["| kernel | ms | DRAM read GB | DRAM write GB | DRAM % peak | SM % | issue active % | warps active % | regs | warp instr |",
       "|---|---|---|---|---|---|---|---|---|---|"]
traffic = defaultdict(float)
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    name = name.split("<")[0].replace("void ", "")
    name = name.split("(")[0].split("::")[-1].strip()
    rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
    out.append(f"| {name} | {val(r, 'gpu__time_duration.sum'):.3f} | {rd:.3f} | {wr:.3f} | "
               f"{val(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
               f"{val(r, 'sm__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
               f"{val(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
               f"{val(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
               f"{float(r[idx['launch__registers_per_thread']]):.0f} | {float(r[idx['smsp__inst_executed.sum']].replace(',', '')):.3g} |")
    if name in STAGE:
        traffic[STAGE[name]] += (rd + wr) * 1e9 / npx
print("\n".join(out))
json.dump(dict(traffic), open(sys.argv[3], "w"), indent=1)
