"""One-line roofline summary per ncu report: duration, DRAM bytes and GB/s, FP64/DMMA pipe use, occupancy.
Usage: python tools/ncu_summary.py rep1.ncu-rep [rep2 ...]   (needs ncu on PATH)"""
import csv
import io
import subprocess
import sys

KEYS = {
    "dur_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_rd_GB": ("dram__bytes_read.sum", 1e-9),
    "dram_wr_GB": ("dram__bytes_write.sum", 1e-9),
    "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "dmma_pct": ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "fp64_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "grid": ("launch__grid_size", 1),
    "regs": ("launch__registers_per_thread", 1),
}
UNIT = {"ms": 1e6, "us": 1e3, "ns": 1.0, "s": 1e9, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0,
        "Tbyte": 1e12}

for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        print(rep, "no data")
        continue
    hdr, units, vals = rows[0], rows[1], rows[2]
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    res = {}
    for k, (metric, scale) in KEYS.items():
        if metric in hdr:
            i = hdr.index(metric)
            try:
                v = float(vals[i].replace(",", ""))
            except ValueError:
                continue
            v *= UNIT.get(units[i], 1.0) if k.endswith(("_ms", "_GB")) else 1.0
            res[k] = v * scale
    if "dur_ms" in res and "dram_rd_GB" in res:
        res["dram_GBps"] = (res["dram_rd_GB"] + res.get("dram_wr_GB", 0.0)) / (res["dur_ms"] * 1e-3)
    print(rep.split("/")[-1], name.split("(")[0][:60], {k: round(v, 3) for k, v in res.items()})
