"""Summarise an ncu --set full report (.ncu-rep) and a launch list (.csv)
into profiles/ text files; update profiles/ncu_traffic.json with the DRAM
bytes per launch of the profiled kernel (bench.py's roofline.traffic).

  python scripts/ncu_summary.py REPORT.ncu-rep OUT.txt [--key KEY]
  python scripts/ncu_summary.py --launches LAUNCHES.csv OUT.txt
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes_read.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_op_imma.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum", "smsp__inst_executed.sum",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active"]


def summarize_report(rep, out, key=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = []
    traffic = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        lines.append(f"kernel: {name}")
        for i, h in enumerate(hdr):
            if h in KEYS or "stalled" in h and "pcsamp" in h and not h.endswith("not_issued"):
                lines.append(f"  {h} [{units[i]}] = {r[i]}")
        try:
            rd = float(r[hdr.index("dram__bytes_read.sum")].replace(",", ""))
            wr = float(r[hdr.index("dram__bytes_write.sum")].replace(",", ""))
            ur = units[hdr.index("dram__bytes_read.sum")]
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(ur, 1)
            traffic[name] = (rd + wr) * mult
        except ValueError:
            pass
    with open(out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    if key and traffic:
        p = os.path.join(os.path.dirname(out), "ncu_traffic.json")
        d = json.load(open(p)) if os.path.exists(p) else {}
        d[key] = list(traffic.values())[0]
        json.dump(d, open(p, "w"), indent=1)
    print("\n".join(lines[:60]))


def summarize_launches(path, out):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[i]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    d = defaultdict(list)
    for r in rows[i + 1:]:
        if len(r) > vi:
            d[r[ki]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    lines = ["kernel | launches | mean ns | share of GPU time"]
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k[:90]} | {len(v)} | {sum(v)/len(v):.0f} | {sum(v)/tot:.3f}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        summarize_launches(sys.argv[2], sys.argv[3])
    else:
        key = sys.argv[sys.argv.index("--key") + 1] if "--key" in sys.argv else None
        summarize_report(sys.argv[1], sys.argv[2], key)
