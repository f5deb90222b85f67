#!/usr/bin/env python3
"""Per-stage compute ceilings of the encode step.

    python tools/ceilings.py <ncu metrics csv> <peaks_fp64_alu.json> profiles/ceilings.json [images_in_capture]

Input 1: `ncu --metrics <tools/gpu/session_a.sh list> --csv` over
`tools/steptimes.py 16 1 2` (16 config-1 images, two steps; the second step's
launches are used).  Input 2: the pipe rates measured on the B200 by
tools/peaks_fp64_alu.cu.  For every kernel launch the lower bound on its
duration is the largest of
  * fp64 pipe: warp instructions on the fp64 pipe / measured DADD|DMUL|DFMA rate,
  * ALU pipe:  warp instructions on the alu pipe / measured LOP3 rate,
  * issue:     warp instructions executed / measured issue rate (1 per SMSP per clock),
  * DRAM:      dram bytes read + written / measured HBM copy bandwidth;
the stage's ceiling is the sum over its launches, scaled to the 64-image bench
step.  bench.py reports measured stage time against it (`compute_ceilings`).
"""

from __future__ import annotations

import csv
import json
import sys
from collections import defaultdict
from pathlib import Path

STAGE_OF = {  # kernel -> stage (api.cu run_batch order)
    "k_stage": "staging", "k_tm_nodes": "tonemap", "k_tm_scalars": "tonemap",
    "k_sdr_ycc": "base", "k_sdr_fix": "base", "k_base_layer": "base",
    "k_prefilter_cols": "prefilter", "k_prefilter_fused": "prefilter", "k_prefilter_h": "prefilter",
    "k_prefilter_v": "prefilter",
    "k_sort_hist": "fit", "k_sort_scan": "fit", "k_sort_scatter": "fit", "k_seg_setup": "fit", "k_seg_nodes": "fit",
    "k_seg_dot": "fit", "k_seg_reduce_coef": "fit", "k_fit_int": "fit", "k_fit_int_coef": "fit",
    "k_estimate": "estimate", "k_crc_chunks": "crc", "k_crc_combine": "crc",
    "k_entropy_dct": "entropy_dct", "k_entropy_plane": "entropy_plane", "k_entropy_fixup": None,
    "k_chain_maps": None, "k_assemble": "assemble",
}


def kname(full: str) -> str:
    n = full.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").split("(")[0].replace("void ", "").strip()
    if "<" in n:
        n = n[: n.index("<")]
    return n.split("::")[-1]


def main():
    lines = open(sys.argv[1]).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))  # after ncu's ==PROF== lines
    rows = list(csv.DictReader(lines[start:]))
    peaks = json.loads(Path(sys.argv[2]).read_text())
    images = int(sys.argv[4]) if len(sys.argv) > 4 else 16
    hbm = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] * 1e9
    r = peaks["rates"]
    fp64 = max(r["dadd"]["warp_inst_per_s"], r["dmul"]["warp_inst_per_s"], r["dfma"]["warp_inst_per_s"])
    alu = r["lop3"]["warp_inst_per_s"]
    # issue: one warp instruction per SMSP per clock (4 per SM) at the max SM
    # clock -- the FFMA+LOP3 microbenchmark reaches 2.66 of those 4 and some of
    # the encoder's kernels issue faster than it, so it is no ceiling
    issue = 4 * peaks["sms"] * 1.965e9
    launches: dict = defaultdict(dict)
    names = {}
    for row in rows:
        lid = int(row["ID"])
        v = row["Metric Value"].replace(",", "")
        try:
            launches[lid][row["Metric Name"]] = float(v)
        except ValueError:
            continue
        names[lid] = kname(row["Kernel Name"])
    ids = sorted(launches)
    # the second step: launches after the second k_stage
    starts = [i for i in ids if names[i] == "k_stage"]
    if len(starts) >= 2:
        ids = [i for i in ids if i >= starts[1]]
    stages: dict = defaultdict(lambda: {"measured_ms": 0.0, "fp64_ms": 0.0, "alu_ms": 0.0, "issue_ms": 0.0,
                                        "dram_ms": 0.0, "min_ms": 0.0, "launches": []})
    scale = 64.0 / images
    for i in ids:
        m = launches[i]
        st = STAGE_OF.get(names[i], "other")
        if st is None:
            st = "entropy_plane" if "plane" in names[i] else "entropy_dct"
        t = {
            "fp64": m.get("sm__inst_executed_pipe_fp64.sum", 0.0) / fp64,
            "alu": m.get("sm__inst_executed_pipe_alu.sum", 0.0) / alu,
            "issue": m.get("smsp__inst_executed.sum", 0.0) / issue,
            "dram": (m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)) / hbm,
        }
        bound = max(t, key=t.get)
        dur = m.get("gpu__time_duration.sum", 0.0) * 1e-9
        e = stages[st]
        e["measured_ms"] += dur * 1e3 * scale
        for k in t:
            e[f"{k}_ms"] += t[k] * 1e3 * scale
        e["min_ms"] += t[bound] * 1e3 * scale
        e["launches"].append({"kernel": names[i], "bound": bound, "ncu_ms": round(dur * 1e3, 4),
                              "ceiling_ms": round(t[bound] * 1e3, 4),
                              "frac": round(t[bound] / dur, 3) if dur else None,
                              **{f"{k}_ms": round(v * 1e3, 4) for k, v in t.items()}})
    out = {"source": f"{sys.argv[1]} (ncu, {images} config-1 images, cold-cache serialised launches) x {sys.argv[2]}",
           "scaled_to_images": 64,
           "peaks": {"fp64_warp_inst_per_s": fp64, "alu_warp_inst_per_s": alu, "issue_warp_inst_per_s": issue,
                     "hbm_bytes_per_s": hbm},
           "stages": {}}
    for st, e in stages.items():
        b = max(("fp64", "alu", "issue", "dram"), key=lambda k: e[f"{k}_ms"])
        out["stages"][st] = {"bound": b, **{k: (round(v, 4) if isinstance(v, float) else v) for k, v in e.items()},
                             "frac": round(e["min_ms"] / e["measured_ms"], 3) if e["measured_ms"] else None}
    Path(sys.argv[3]).write_text(json.dumps(out, indent=1) + "\n")
    for st, e in out["stages"].items():
        print(f"{st:14s} ncu {e['measured_ms']:8.3f} ms  ceiling {e['min_ms']:8.3f} ms ({e['bound']}, frac {e['frac']})")


if __name__ == "__main__":
    main()
