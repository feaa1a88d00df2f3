"""Summarise ptxas -v output: registers / spills per kernel (demangled)."""
import re
import subprocess
import sys

log = open(sys.argv[1] if len(sys.argv) > 1 else "paper_2605_11215_b200/csrc/ptxas.log").read()
pat = sys.argv[2] if len(sys.argv) > 2 else ""
cur = None
rows = []
for line in log.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = {"name": m.group(1)}
        rows.append(cur)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        cur["spill"] = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        cur["regs"] = int(m.group(1))
names = subprocess.run(["c++filt"], input="\n".join(r["name"] for r in rows), capture_output=True,
                       text=True).stdout.splitlines()
for r, n in zip(rows, names):
    if pat in n:
        print("%3s regs spill %-10s %s" % (r.get("regs"), r.get("spill"), n[:150]))
