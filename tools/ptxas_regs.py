"""name -> registers / spill bytes from a ptxas -v log.  usage: python tools/ptxas_regs.py LOG [regex]"""
import re, subprocess, sys
cur = None
out = {}
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        out.setdefault(cur, {})["spill"] = int(m.group(1)) + int(m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        out.setdefault(cur, {})["regs"] = int(m.group(1))
names = list(out)
dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
for n, d in zip(names, dem):
    if pat and not pat.search(d):
        continue
    print("%4s regs %5s spill  %s" % (out[n].get("regs"), out[n].get("spill"), d))
