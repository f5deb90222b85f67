"""Summarise an ncu --set full report (per kernel) as markdown + traffic per pixel json."""
import csv, io, json, subprocess, sys
rep, npx = sys.argv[1], float(sys.argv[2])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size"]
idx = {w: hdr.index(w) for w in want if w in hdr}
out = ["| kernel | ms | DRAM read GB | DRAM write GB | DRAM % peak | SM % | warps active % | regs | warp instr |",
       "|---|---|---|---|---|---|---|---|---|"]
traffic = {}
def val(r, k, scale=1.0):
    try: return float(r[idx[k]].replace(",", "")) * scale
    except Exception: return float("nan")
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0]
    gb = lambda k: val(r, k) * (1.0 if units[idx[k]] == "Gbyte" else 1e-3 if units[idx[k]] == "Mbyte" else 1e-9 if units[idx[k]] == "byte" else 1.0)
    rd, wr = gb("dram__bytes_read.sum"), gb("dram__bytes_write.sum")
    out.append(f"| {name} | {val(r,'gpu__time_duration.sum'):.3f} | {rd:.3f} | {wr:.3f} | "
               f"{val(r,'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
               f"{val(r,'sm__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
               f"{val(r,'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | {val(r,'launch__registers_per_thread'):.0f} | "
               f"{val(r,'smsp__inst_executed.sum'):.3g} |")
    key = {"k_entropy_plane": "entropy_plane", "k_entropy_dct": "entropy_dct", "k_base_layer": "base",
           "k_prefilter_fused": "prefilter"}.get(name.split("::")[-1])
    if key:
        traffic[key] = (rd + wr) * 1e9 / npx
print("\n".join(out))
json.dump(traffic, open(sys.argv[3], "w"), indent=1)
