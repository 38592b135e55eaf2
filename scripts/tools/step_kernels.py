"""Per-kernel table of a one-step ncu --set full capture (scripts/tools/profile_step.py
under `ncu -k regex:k_ --launch-skip 8 --launch-count 8`): duration, DRAM and L2
bytes / bandwidth, issue and pipe utilisation, instruction counts.
usage: step_kernels.py step.ncu-rep > profiles/rNN/step_kernels_ncu.json"""
import csv
import io
import json
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
col = {h: i for i, h in enumerate(hdr)}


def num(r, k, default=0.0):
    try:
        return float(r[col[k]].replace(",", ""))
    except (KeyError, ValueError):
        return default


out = []
for r in rows[2:]:
    us = num(r, "gpu__time_duration.sum")
    unit = rows[1][col["gpu__time_duration.sum"]]
    us = us * {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(unit, 1.0)
    dram = num(r, "dram__bytes_read.sum") + num(r, "dram__bytes_write.sum")
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        pass
    du = rows[1][col["dram__bytes_read.sum"]]
    dram *= {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(du, 1.0)
    l2 = num(r, "lts__t_sectors.sum") * 32.0
    cyc = num(r, "smsp__cycles_elapsed.avg")
    fp64 = sum(num(r, f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed")
               for op in ("dadd", "dmul", "dfma")) * cyc
    out.append({
        "kernel": r[col["Kernel Name"]].split("(")[0],
        "us": round(us, 1),
        "dram_MB": round(dram / 1e6, 1), "dram_GBs": round(dram / us / 1e3, 1),
        "l2_MB": round(l2 / 1e6, 1), "l2_GBs": round(l2 / us / 1e3, 1),
        "l2_pct": num(r, "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        "sm_pct": num(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        "issue": num(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "fp64_pipe": num(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "xu_pipe": num(r, "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
        "warp_inst": num(r, "smsp__inst_executed.sum"),
        "fp64_thread_inst": round(fp64),
        "regs": int(num(r, "launch__registers_per_thread")),
    })
json.dump(out, sys.stdout, indent=1)
print()
