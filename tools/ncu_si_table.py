"""Per-launch table of an ncu --set full raw CSV export (ncu -i rep --page raw --csv):
duration, DRAM read/write, DMMA sub-pipe utilisation, achieved occupancy, registers.
Usage: python tools/ncu_si_table.py gpurun_out/x_raw.csv > profiles/x.txt"""
import csv
import sys

COLS = {
    "ms": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "dmma_pct": "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "warps_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}
SCALE = {"ms": {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "msecond": 1.0, "usecond": 1e-3, "nsecond": 1e-6},
         "dram_rd": {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0},
         "dram_wr": {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}}


def main(path):
    rows = [r for r in csv.reader(open(path)) if r]
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    head, units, data = rows[start], rows[start + 1], rows[start + 2:]
    idx = {k: head.index(v) for k, v in COLS.items() if v in head}
    kn = head.index("Kernel Name")
    print("kernel | ms | DRAM R GB | DRAM W GB | GB/s | DMMA % | warps % | regs | grid x block")
    for r in data:
        out = {}
        for k, i in idx.items():
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                v = float("nan")
            out[k] = v * SCALE.get(k, {}).get(units[i], 1.0)
        gbs = (out.get("dram_rd", 0) + out.get("dram_wr", 0)) / (out["ms"] * 1e-3) if out.get("ms") else 0
        name = r[kn].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")
        print(f"{name} | {out.get('ms', 0):.3f} | {out.get('dram_rd', 0):.2f} | {out.get('dram_wr', 0):.2f} | "
              f"{gbs:.0f} | {out.get('dmma_pct', 0):.1f} | {out.get('warps_pct', 0):.1f} | {out.get('regs', 0):.0f} | "
              f"{out.get('grid', 0):.0f} x {out.get('block', 0):.0f}")


if __name__ == "__main__":
    main(sys.argv[1])
