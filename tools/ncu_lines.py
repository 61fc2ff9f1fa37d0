"""Per-source-line hot spots of one kernel in an ncu report (instructions, stall samples, shared
wavefronts).  usage: python tools/ncu_lines.py report.ncu-rep kernel-regex [n]"""
import csv, io, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = None
fname = None
out = []
for r in rows:
    if r and r[0] in ("File Name", "File Path"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        d = dict(zip(hdr, r))
        def num(k):
            try:
                return float(d.get(k, 0) or 0)
            except ValueError:
                return 0.0
        out.append((num("Warp Stall Sampling (All Samples)"), num("Instructions Executed"),
                    num("L1 Wavefronts Shared"), num("L1 Wavefronts Shared Ideal"), fname, d["Line No"], d["Source"].strip()[:90]))
ts = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
print("total warp-instructions %.3e, stall samples %d" % (ti, ts))
print("  stall%   inst%   shWF(ideal)  line")
for o in sorted(out, key=lambda o: -o[0])[:n]:
    print("  %5.1f  %5.1f  %9.2e(%8.2e) %s:%s  %s" % (100 * o[0] / ts, 100 * o[1] / ti, o[2], o[3], o[4], o[5], o[6]))
