"""Summarise an ncu report: per kernel, top stall reasons and the source lines with most stall samples.
usage: python tools/ncu_stalls.py report.ncu-rep [kernel-regex ...]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
un = dict(zip(hdr, units))
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print("==", d["Kernel Name"][:60], "time", d["gpu__time_duration.sum"], un.get("gpu__time_duration.sum"),
          "dram r/w", d.get("dram__bytes_read.sum"), un.get("dram__bytes_read.sum"),
          d.get("dram__bytes_write.sum"), un.get("dram__bytes_write.sum"))
    st = []
    for k, v in d.items():
        if "warps_issue_stalled" in k and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    print("   stalls:", ", ".join("%s %.2f" % (k, v) for v, k in sorted(st, reverse=True)[:6]))
    for k in ["smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
              "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
              "launch__occupancy_limit_registers"]:
        print("   ", k, d.get(k))
for kre in sys.argv[2:]:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass", "-k", "regex:" + kre],
                         capture_output=True, text=True).stdout
    cur = None
    out = []
    for r in csv.reader(io.StringIO(src)):
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) > 6 and r[0] and r[0] not in ("Function Name", "Line No"):
            try:
                out.append((int(r[4]), cur, r[0], r[1][:100]))
            except ValueError:
                pass
    tot = sum(o[0] for o in out) or 1
    print("-- stall samples by line:", kre)
    for o in sorted(out, reverse=True)[:14]:
        print("  %5.1f%% %s:%s %s" % (100 * o[0] / tot, o[1], o[2], o[3]))
