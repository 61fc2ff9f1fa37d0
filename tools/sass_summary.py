"""SASS evidence for profiles/: per hot kernel, counts of the instructions that prove the
design (DMMA tensor-core FP64, UTMALDG / UBLKCP TMA copies, SYNCS mbarriers, LDGSTS cp.async,
DFMA) and a short excerpt of the inner loop.  usage: python tools/sass_summary.py > out.txt"""
import re
import subprocess
import sys

OBJS = {"p3m": "paper_2004_02609_b200/_build/p3m.o", "operator": "paper_2004_02609_b200/_build/operator.o"}
WANT = [("p3m", r"k_p3mILi3ELi10ELb0E"), ("operator", r"k_p4sILi1024ELi32ELb0E"),
        ("operator", r"k_p5ILi1024ELb0E"), ("operator", r"k_p2ILi1024ELb0E"),
        ("operator", r"k_p1ILi1024ELb0E"), ("operator", r"k_p3ILi256ELi3EE")]
KEYS = ["DMMA", "DFMA", "DMUL", "DADD", "UTMALDG", "UBLKCP", "SYNCS", "LDGSTS", "LDS", "STS", "LDG", "STG",
        "SHFL", "BAR"]
for obj, pat in WANT:
    txt = subprocess.run(["cuobjdump", "-sass", OBJS[obj]], capture_output=True, text=True).stdout
    parts = re.split(r"\n\s*Function : ", txt)
    for p in parts[1:]:
        name = p.split("\n", 1)[0].strip()
        if not re.search(pat, name):
            continue
        ins = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", p)
        ops = [o for _, o in ins]
        print("==", name, "instructions:", len(ops))
        print("   " + ", ".join("%s %d" % (k, sum(1 for o in ops if o.split(".")[0] == k)) for k in KEYS))
        lines = [l.strip() for l in p.split("\n") if re.search(r"/\*[0-9a-f]{4,}\*/", l)]
        hit = next((i for i, l in enumerate(lines) if re.search(r"\b(DMMA|UTMALDG|UBLKCP)\b", l)), None)
        if hit is not None:
            print("   excerpt:")
            for l in lines[max(0, hit - 6):hit + 10]:
                print("     " + re.sub(r"\s*/\* 0x[0-9a-f]+ \*/", "", l))
