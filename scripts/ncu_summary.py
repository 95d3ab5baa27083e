"""Summarise `ncu --page raw --csv` exports (one row per profiled launch):
duration, DRAM bytes, throughputs, occupancy, issue activity.  Prints a
markdown table; with --traffic PATH also writes {kernel: dram bytes per
launch} (the bench's roofline.traffic).
usage: python scripts/ncu_summary.py [--traffic profiles/traffic.json] a_raw.csv ..."""
import csv
import json
import sys

COLS = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "DRAM rd"), ("dram__bytes_write.sum", "DRAM wr"),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem thr %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM thr %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
        ("smsp__average_warp_latency_per_inst_issued.ratio", "cyc/issue"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid")]
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3}

args = sys.argv[1:]
traffic_out = None
if args and args[0] == "--traffic":
    traffic_out, args = args[1], args[2:]
traffic = {}
print("| kernel | " + " | ".join(c[1] for c in COLS) + " |")
print("|---" * (len(COLS) + 1) + "|")
for path in args:
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        vals = []
        for key, _ in COLS:
            i = h.index(key)
            v = float(r[i].replace(",", "")) * UNIT.get(units[i], 1.0)
            vals.append(v)
        short = name.split("(")[0].replace("void ", "")
        traffic[short.split("<")[0]] = vals[1] + vals[2]
        fmt = [f"{vals[0]:.2f}", f"{vals[1] / 1e6:.2f} MB", f"{vals[2] / 1e6:.2f} MB"] + [f"{v:.1f}" for v in vals[3:8]] + \
              [f"{int(vals[8])}", f"{int(vals[9])}"]
        print(f"| {short} | " + " | ".join(fmt) + " |")
if traffic_out:
    json.dump({"source": "ncu --set full --clock-control none (cache control flush-all) via scripts/gpu_profile.sh: "
                         "dram__bytes_read.sum + dram__bytes_write.sum of one launch", **traffic},
              open(traffic_out, "w"), indent=1)
