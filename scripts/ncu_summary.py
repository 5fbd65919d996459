"""Summarise an `ncu --set full` report (read here with `ncu -i --page raw --csv`)
into profiles/<name>_ncu_full_summary.json and, with --traffic, the per-phase
DRAM bytes per launch bench.py reads as roofline.traffic (profiles/traffic.json,
keyed by config and cell count; one launch per kernel in the report).

    python scripts/ncu_summary.py gpurun_out/x.ncu-rep profiles/r02_x_ncu_full_summary.json --traffic 3 8388608
"""
import argparse
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

PHASE = {"k_central": "central", "k_troubled": "cwenoz+muscl", "k_cwenoz": "cwenoz+muscl", "k_muscl": "cwenoz+muscl",
         "k_face_flux": "flux+RK", "k_gather_rk": "flux+RK", "k_spread": "spread+compaction"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--traffic", nargs=2, metavar=("CONFIG", "CELLS"))
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]

    units = rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "ms": 1e6,
             "msecond": 1e6, "second": 1e9}

    def num(r, k):  # bytes in B, times in ns
        try:
            i = hdr.index(k)
            return float(r[i].replace(",", "")) * scale.get(units[i], 1.0)
        except (ValueError, IndexError):
            return None

    stall_cols = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and
                  h.endswith("_per_issue_active.ratio")]
    out, traffic = [], {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        short = name.split("(")[0].replace("void ", "")
        stalls = {c[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]: num(r, c)
                  for c in stall_cols}
        tot = sum(v for v in stalls.values() if v) or 1.0
        top = dict(sorted(((k, round(100 * v / tot, 1)) for k, v in stalls.items() if v), key=lambda x: -x[1])[:4])
        rd, wr = num(r, "dram__bytes_read.sum"), num(r, "dram__bytes_write.sum")
        dur_ns = num(r, "gpu__time_duration.sum")
        e = {"kernel": short, "duration_us": round(dur_ns / 1e3, 3) if dur_ns else None, "dram_read_B": rd,
             "dram_write_B": wr,
             "dram_GBps": round((rd + wr) / dur_ns, 1) if dur_ns else None,
             "achieved_occupancy_pct": num(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
             "regs": num(r, "launch__registers_per_thread"),
             "fp64_pipe_pct": num(r, "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
             "l2_hit_pct": num(r, "lts__t_sector_hit_rate.pct"),
             "dyn_smem_B": num(r, "launch__shared_mem_per_block_dynamic"),
             "warp_inst": num(r, "smsp__inst_executed.sum"),
             "top_stalls_pct": top}
        out.append(e)
        for k, ph in PHASE.items():
            if short.startswith(k):
                traffic[ph] = traffic.get(ph, 0.0) + (rd or 0) + (wr or 0)
                break
    Path(a.out).write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))
    if a.traffic:
        tf = Path(__file__).resolve().parents[1] / "profiles" / "traffic.json"
        try:
            allt = json.loads(tf.read_text())
            if not all(k.startswith("config") for k in allt):
                allt = {}
        except Exception:
            allt = {}
        allt[f"config{a.traffic[0]}"] = {"cells": int(a.traffic[1]), "source": a.report, **traffic}
        tf.write_text(json.dumps(allt, indent=1) + "\n")
        print("traffic:", allt, file=sys.stderr)


if __name__ == "__main__":
    main()
