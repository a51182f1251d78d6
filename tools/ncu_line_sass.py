"""Opcode histogram (executed warp-instructions) of the SASS mapped to given
source lines: python tools/ncu_line_sass.py report.ncu-rep file.cuh L1[-L2] ..."""
import csv
import io
import subprocess
import sys

rep, fname = sys.argv[1], sys.argv[2]
want = []
for a in sys.argv[3:]:
    lo, _, hi = a.partition("-")
    want.append((int(lo), int(hi or lo)))
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = hdr = ln = None
cnt = {}
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0].isdigit():
        ln = int(r[0])
        continue
    if cur != fname or ln is None or not any(lo <= ln <= hi for lo, hi in want):
        continue
    ins = r[3].split()
    if not ins:
        continue
    op = ins[1] if ins[0].startswith("@") else ins[0]
    try:
        n = int(r[7])
    except ValueError:
        continue
    cnt[op] = cnt.get(op, 0) + n
tot = sum(cnt.values())
print("total", tot)
for k, v in sorted(cnt.items(), key=lambda kv: -kv[1])[:25]:
    print(f"{k:28s} {v:12d} {100 * v / max(tot, 1):5.1f}%")
