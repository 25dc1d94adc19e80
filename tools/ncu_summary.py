#!/usr/bin/env python3
"""Key metrics of every kernel in an ncu --set full report (reads `ncu -i --page raw --csv`)."""
import csv
import io
import re
import subprocess
import sys

KEYS = [
    ("time_us", "gpu__time_duration.sum"),
    ("dram_rd_MB", "dram__bytes_read.sum"),
    ("dram_wr_MB", "dram__bytes_write.sum"),
    ("dram_%pk", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("sm_%pk", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("l1_%pk", "l1tex__throughput.avg.pct_of_peak_sustained_active"),
    ("l2_%pk", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("l1_hit%", "l1tex__t_sector_hit_rate.pct"),
    ("l2_hit%", "lts__t_sector_hit_rate.pct"),
    ("warps_act%", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("regs", "launch__registers_per_thread"),
    ("tensor%", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    ("grid", "launch__grid_size"),
    ("l2_rd_sect_M", "lts__t_sectors_srcunit_tex_op_read.sum"),
    ("l1_rd_sect_M", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"),
    ("lsu_wavefr%", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
    ("issue%", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
]


def unit_scale(unit, key):
    if key.endswith("_sect_M"):
        return {"sector": 1e-6, "Ksector": 1e-3, "Msector": 1.0, "Gsector": 1e3}.get(unit, 1e-6)
    if key.startswith("dram_") and key.endswith("MB"):
        return {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
    if key == "time_us":
        return {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
    return 1.0


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    stall_cols = [i for i, c in enumerate(h) if re.match(r"smsp__average_warp_latency_issue_stalled_\w+$", c)
                  or re.match(r"smsp__pcsamp_warps_issue_stalled_\w+$", c)]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].replace("(anonymous namespace)::", "")
        name = re.sub(r"\(.*", "", name)
        parts = []
        for lab, key in KEYS:
            if key in h:
                i = h.index(key)
                try:
                    v = float(r[i].replace(",", "")) * unit_scale(units[i], lab)
                    parts.append(f"{lab}={v:.4g}")
                except ValueError:
                    parts.append(f"{lab}={r[i]}")
        stalls = []
        for i in stall_cols:
            try:
                stalls.append((float(r[i].replace(",", "")), h[i].split("stalled_")[-1]))
            except ValueError:
                pass
        stalls.sort(reverse=True)
        print(name)
        print("   " + " ".join(parts))
        if stalls:
            print("   stalls: " + ", ".join(f"{n}={v:.3g}" for v, n in stalls[:5]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
