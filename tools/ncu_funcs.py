"""Aggregate an ncu source page by enclosing function (of the given .cuh files):
python tools/ncu_funcs.py report.ncu-rep"""
import csv, io, re, subprocess, sys, os
rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
funcs = {}
def func_map(fname):
    if fname in funcs: return funcs[fname]
    path = os.path.join(root, "paper_2405_07122_b200", "csrc", fname)
    m = {}
    if os.path.exists(path):
        cur = "?"
        for i, line in enumerate(open(path), 1):
            mm = re.match(r"^(?:template <[^>]*>\s*)?(?:__device__|__global__|static|inline|__host__)[^(]*?\b(\w+)\s*\(", line)
            if mm: cur = mm.group(1)
            m[i] = cur
    funcs[fname] = m
    return m
agg, tot_s, tot_i, cur_file, hdr = {}, 0, 0, None, None
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or r[0] in ("", "Function Name"): continue
    d = dict(zip(hdr[2:], r[2:]))
    try: s = int(d["Warp Stall Sampling (All Samples)"]); ins = int(d["Instructions Executed"])
    except (KeyError, ValueError): continue
    fn = func_map(cur_file).get(int(r[0]), cur_file) if r[0].isdigit() else cur_file
    key = f"{cur_file}:{fn}"
    a = agg.setdefault(key, [0, 0]); a[0] += s; a[1] += ins
    tot_s += s; tot_i += ins
print(f"total samples {tot_s}  warp-instr {tot_i}")
for k, (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"{100*s/tot_s:5.1f}%stall {100*i/tot_i:5.1f}%instr  {k}")
