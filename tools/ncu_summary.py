"""Summarise ncu output for profiles/ (run here, on the CPU box, after gpurun brings files back).

  python tools/ncu_summary.py launches <launches.csv>          per-kernel launch list shares
  python tools/ncu_summary.py report <prof.ncu-rep> [<prof2>]   key metrics of a --set full capture
"""
import collections
import csv
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
    "sass__inst_executed_local_loads", "sass__inst_executed_local_stores",
    "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def _us(unit, v):
    return v / 1000.0 if unit == "nsecond" or unit == "ns" else (v * 1000.0 if unit in ("msecond", "ms") else v)


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    d = collections.defaultdict(list)
    for r in rows[1:]:
        d[r[ki].split("(")[0].replace("(anonymous namespace)::", "")].append(
            _us(r[ui], float(r[vi].replace(",", ""))))
    tot = sum(sum(v) for v in d.values())
    print(f"{'kernel':44s} {'launches':>8s} {'mean us':>10s} {'total ms':>10s} {'share':>6s}")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k[:44]:44s} {len(v):8d} {sum(v) / len(v):10.1f} {sum(v) / 1000:10.2f} {sum(v) / tot:6.3f}")
    print(f"{'TOTAL':44s} {sum(len(v) for v in d.values()):8d} {'':>10s} {tot / 1000:10.2f}")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0]
        print(f"== {name}")
        for k in KEYS:
            if k in h:
                print(f"  {k:64s} {r[h.index(k)]} {units[h.index(k)]}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        for p in sys.argv[2:]:
            report(p)
