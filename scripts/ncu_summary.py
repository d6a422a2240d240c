"""Summarise ncu captures (`ncu -i REP --page raw --csv`) and a launch list
(`--metrics gpu__time_duration.sum --csv`) into markdown rows.

    python scripts/ncu_summary.py rep1.ncu-rep [rep2 ...] [--launches launches.csv]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__instruction_throughput.avg.pct_of_peak_sustained_active": "issue_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "launch__registers_per_thread": "regs",
    "sm__warps_active.avg.per_cycle_active": "warps_per_sm",
    "launch__shared_mem_per_block_dynamic": "smem_dyn",
    "smsp__inst_executed.sum": "warp_inst",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        rec = {"kernel": d.get("Kernel Name", "")[:80]}
        for m, k in METRICS.items():
            if m in d:
                rec[k] = d[m] + (" " + units[hdr.index(m)] if units[hdr.index(m)] else "")
        res.append(rec)
    return res


def launches(path):
    tot = defaultdict(lambda: [0, 0.0])
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")[:60]
        tot[name][0] += 1
        tot[name][1] += float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)
    all_us = sum(v[1] for v in tot.values())
    print("| kernel | launches | total us | share |\n|---|---|---|---|")
    for name, (n, us) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"| {name} | {n} | {us:.1f} | {100 * us / all_us:.1f} % |")


if __name__ == "__main__":
    args = sys.argv[1:]
    if "--launches" in args:
        i = args.index("--launches")
        launches(args[i + 1])
        args = args[:i] + args[i + 2:]
    for rep in args:
        for rec in raw(rep):
            print(rep, rec)
