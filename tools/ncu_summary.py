#!/usr/bin/env python
"""Summarise ncu reports (--page raw) into a short text table + traffic JSON.

usage: python tools/ncu_summary.py OUT_DIR key=report.ncu-rep [key=report.ncu-rep ...]
Writes OUT_DIR/ncu_<key>.txt and merges {key: {bytes: dram bytes per launch, kernel,
capture: that summary file, date: capture date}} into profiles/ncu_traffic.json
(read by bench.py for roofline.traffic and roofline.traffic_source).
"""
import csv
import io
import json
import os
import subprocess
import sys
import time

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe % active"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma pipe % active"),
    ("sm__warps_active.avg.per_cycle_active", "warps active / SM"),
    ("smsp__issue_active.avg.per_cycle_active", "issue active / SMSP"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem st bank conflicts"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
]


def to_bytes(v, unit):
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(v) * f


def main():
    out_dir = sys.argv[1]
    os.makedirs(out_dir, exist_ok=True)
    tpath = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                         "profiles", "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for arg in sys.argv[2:]:
        key, rep = arg.split("=", 1)
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units, vals = rows[0], rows[1], rows[2]
        kname = vals[hdr.index("Kernel Name")]
        lines = [f"ncu --set full capture: {os.path.basename(rep)}", f"kernel: {kname}"]
        got = {}
        for m, label in METRICS:
            if m in hdr:
                i = hdr.index(m)
                got[m] = (vals[i], units[i])
                lines.append(f"  {label:28s} {vals[i]:>16s} {units[i]}")
        stalls = [(h, vals[i]) for i, h in enumerate(hdr)
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
        stalls = sorted(((float(v or 0), h.replace("smsp__pcsamp_warps_issue_stalled_", ""))
                         for h, v in stalls), reverse=True)[:8]
        lines.append("  top stall reasons (pc samples): " +
                     ", ".join(f"{n}={int(c)}" for c, n in stalls))
        if "dram__bytes_read.sum" in got:
            b = to_bytes(*got["dram__bytes_read.sum"]) + to_bytes(*got["dram__bytes_write.sum"])
            when = time.strftime("%Y-%m-%d", time.gmtime(os.path.getmtime(rep)))
            traffic[key] = {"bytes": b, "kernel": kname.split("(")[0],
                            "capture": os.path.join(out_dir, f"ncu_{key}.txt"), "date": when}
            lines.append(f"  dram bytes read+write per launch: {b:.4e}")
        open(os.path.join(out_dir, f"ncu_{key}.txt"), "w").write("\n".join(lines) + "\n")
        print("\n".join(lines))
    json.dump(traffic, open(tpath, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
