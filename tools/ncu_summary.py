"""Summarise one kernel of an ``ncu --set full`` report (read here, no GPU):

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [--algorithmic BYTES] [--json out.json]

Prints duration, DRAM bytes, traffic / algorithmic ratio, occupancy, issue
utilisation and the warp-stall breakdown (per issue-active cycle)."""
import argparse
import csv
import io
import json
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--launch", type=int, default=0)
    ap.add_argument("--algorithmic", type=float, default=None, help="algorithmic bytes per launch")
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    h, units, rows = raw(a.rep)
    v = dict(zip(h, rows[a.launch]))
    u = dict(zip(h, units))

    def g(k, scale=1.0):
        x = num(v.get(k, ""))
        return None if x is None else x * scale

    unit_scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    rd = g("dram__bytes_read.sum", unit_scale.get(u.get("dram__bytes_read.sum"), 1.0))
    wr = g("dram__bytes_write.sum", unit_scale.get(u.get("dram__bytes_write.sum"), 1.0))
    dur_unit = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}
    dur = g("gpu__time_duration.sum", dur_unit.get(u.get("gpu__time_duration.sum"), 1.0))
    s = {"kernel": v.get("Kernel Name"), "duration_ms_ncu": dur, "dram_read_bytes": rd, "dram_write_bytes": wr,
         "bytes_per_launch": (rd or 0) + (wr or 0),
         "dram_GBps_ncu": ((rd or 0) + (wr or 0)) / (dur * 1e-3) / 1e9 if dur else None,
         "registers": g("launch__registers_per_thread"), "grid": g("launch__grid_size"),
         "block": g("launch__block_size"),
         "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
         "sm_issue_active_pct": g("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
         "l2_hit_pct": g("lts__t_sector_hit_rate.pct")}
    if a.algorithmic:
        s["algorithmic_bytes"] = a.algorithmic
        s["traffic_over_algorithmic"] = s["bytes_per_launch"] / a.algorithmic
    pre, post = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
    stalls = {k[len(pre):-len(post)]: num(x) for k, x in v.items() if k.startswith(pre) and k.endswith(post)}
    s["stalls_per_issue"] = {k: round(x, 3) for k, x in sorted(stalls.items(), key=lambda t: -(t[1] or 0))
                             if x and x > 0.01}
    text = json.dumps(s, indent=1)
    print(text)
    if a.json:
        with open(a.json, "w") as f:
            f.write(text + "\n")


if __name__ == "__main__":
    sys.exit(main())
