"""Summarise an `ncu --set full` report into the JSON kept under profiles/.

  python scripts/ncu_summary.py REPORT.ncu-rep "capture command" "reading" > profiles/X.json

One entry per profiled launch: time, DRAM bytes, SM/issue utilisation,
occupancy, pipe utilisation and the warp-stall breakdown (cycles per issued
instruction, the ncu "Warp State" numbers).
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct",
]
PIPES = ["fp64", "fma", "alu", "xu", "lsu", "adu", "cbu"]


def main(rep, capture, reading):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    out = {"capture": capture, "reading": reading, "launches": []}
    for r in rows[2:]:
        m = dict(zip(head, r))
        u = dict(zip(head, units))
        e = {"kernel": m.get("Kernel Name", ""), "metrics": {}}
        for k in KEYS:
            if k in m:
                e["metrics"][k] = [m[k], u.get(k, "")]
        e["pipes_pct_of_peak"] = {
            p: m.get(f"sm__inst_executed_pipe_{p}.avg.pct_of_peak_sustained_active")
            for p in PIPES}
        stalls = {}
        for k, v in m.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith(
                    "_per_issue_active.ratio"):
                name = k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]
                try:
                    if float(v) >= 0.05:
                        stalls[name] = round(float(v), 2)
                except ValueError:
                    pass
        e["stall_cycles_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        out["launches"].append(e)
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
