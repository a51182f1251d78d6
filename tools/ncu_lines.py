"""Summarise an ncu report's source page by CUDA source line:
python tools/ncu_lines.py report.ncu-rep [top] [--by-instr]  -> lines sorted by stall samples
(or by executed warp instructions)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 40
by_instr = "--by-instr" in sys.argv
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cur_file, hdr, out = None, None, []
tot_s = tot_i = 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        s = int(d["Warp Stall Sampling (All Samples)"])
        ins = int(d["Instructions Executed"])
    except (KeyError, ValueError):
        continue
    stalls = {k: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit()}
    topst = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
    out.append((s, ins, f"{cur_file}:{r[0]}", r[1][:70], topst))
    tot_s += s
    tot_i += ins
out.sort(key=lambda t: -(t[1] if by_instr else t[0]))
print(f"total samples {tot_s}  total warp-instructions {tot_i}")
for s, ins, loc, src, st in out[:top]:
    sts = " ".join(f"{k[6:]}={v}" for k, v in st if v)
    print(f"{100*s/max(tot_s,1):5.1f}% {100*ins/max(tot_i,1):5.1f}%i {loc:22s} {src:70s} {sts}")
