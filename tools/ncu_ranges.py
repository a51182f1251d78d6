"""Sum an ncu report's source-page instructions / stall samples over line ranges
of one file: python tools/ncu_ranges.py report.ncu-rep file.cuh a-b:name c-d:name ...
(lines outside every range are summed as 'other'; other files as 'elsewhere')."""
import csv
import io
import subprocess
import sys

rep, fname = sys.argv[1], sys.argv[2]
ranges = []
for a in sys.argv[3:]:
    r, name = a.split(":", 1)
    lo, hi = r.split("-")
    ranges.append((int(lo), int(hi), name))
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
acc, cur, hdr = {}, None, None
tot_i = tot_s = 0
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
    d = dict(zip(hdr[2:], r[2:]))
    try:
        ln, ins, s = int(r[0]), int(d["Instructions Executed"]), int(d["Warp Stall Sampling (All Samples)"])
    except (KeyError, ValueError):
        continue
    key = "elsewhere:" + str(cur)
    if cur == fname:
        key = "other"
        for lo, hi, name in ranges:
            if lo <= ln <= hi:
                key = name
                break
    a = acc.setdefault(key, [0, 0])
    a[0] += ins
    a[1] += s
    tot_i += ins
    tot_s += s
for k, (i, s) in sorted(acc.items(), key=lambda kv: -kv[1][0]):
    print(f"{100 * i / tot_i:5.1f}%i {100 * s / max(tot_s, 1):5.1f}%s  {k}")
