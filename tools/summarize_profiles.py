"""Summaries of a profile_round.sh / profile_r02.sh pass for profiles/<round>/:
python tools/summarize_profiles.py gpurun_out/prof profiles/r01 [c2]
python tools/summarize_profiles.py gpurun_out/prof2 profiles/r02 c5f
 - launches_bench_c2.txt : per-kernel time share of one bench step (ncu launch list, cold, serialised)
 - <kernel>_<cfg>.txt    : key metrics of the ncu --set full capture + top source lines
 - traffic.json (repo profiles/): dram bytes per launch of the bench's dominant kernel (bench.py reads it)"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

src, dst = sys.argv[1], sys.argv[2]
CFG = sys.argv[3] if len(sys.argv) > 3 else "c2"
os.makedirs(dst, exist_ok=True)
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# ---- launch list: one bench step = the kernels between two consecutive k_minmax launches
rows = list(csv.reader(open(os.path.join(src, f"launches_bench_{CFG}.csv"))))
hdr, out = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(d["Metric Unit"], 1.0)
        if "pcf::" not in d["Kernel Name"]:
            continue   # the L2 flush between steps is not part of the sort
        out.append((d["Kernel Name"].split("(")[0], v * scale))
starts = [i for i, (k, _) in enumerate(out) if "k_minmax" in k]
seg = out[starts[-2]:starts[-1]] if len(starts) >= 2 else out
agg = defaultdict(lambda: [0, 0.0])
for k, us in seg:
    agg[k][0] += 1
    agg[k][1] += us
tot = sum(v[1] for v in agg.values())
with open(os.path.join(dst, f"launches_bench_{CFG}.txt"), "w") as f:
    f.write(f"# one {CFG} sort from `ncu --metrics gpu__time_duration.sum --clock-control none`\n")
    f.write("# of `python bench.py --steps 2 --warmup 3 --no-cpu-baseline`: cold-cache, serialised launches -> compare shares\n")
    f.write(f"# {len(seg)} launches, {tot:.1f} us total\n")
    for k, (cnt, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        f.write(f"{us:10.1f} us {100 * us / tot:5.1f}%  x{cnt:<3d} {k}\n")

# ---- full captures
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic"]
traffic = {}
for fn in sorted(os.listdir(src)):
    if not fn.endswith(".ncu-rep"):
        continue
    rep = os.path.join(src, fn)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) < 3:
        continue
    h, units, v = rr[0], rr[1], rr[2]
    met = {n: (v[i], units[i]) for i, n in enumerate(h)}
    stalls = sorted(((n.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v[i] or 0)) for i, n in enumerate(h)
                     if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")),
                    key=lambda t: -t[1])
    tots = sum(s for _, s in stalls) or 1
    lines = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, "25"],
                           capture_output=True, text=True).stdout
    name = fn[:-8]
    with open(os.path.join(dst, name + ".txt"), "w") as f:
        f.write(f"# ncu --set full --import-source on --clock-control none, first launch: {name}\n")
        for n in WANT:
            if n in met:
                f.write(f"{n:55s} {met[n][0]:>18s} {met[n][1]}\n")
        f.write("\n# warp stall samples\n")
        for s, c in stalls[:12]:
            f.write(f"{s:28s} {100 * c / tots:5.1f}%\n")
        f.write("\n# top source lines by stall samples (tools/ncu_lines.py)\n")
        f.write(lines)
    if name.startswith("k7_kernel_") and "dram__bytes_read.sum" in met:
        def b(n):
            val, u = met[n]
            return float(val.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        traffic[name[len("k7_kernel_"):]] = {"smem_subtree": b("dram__bytes_read.sum") + b("dram__bytes_write.sum"),
                                             "_from": f"{dst}/{name}.txt (one K7 launch = the sort's K7 work)"}
if traffic:   # merged into profiles/traffic.json (bench.py's roofline.traffic) by tools/merge_traffic.py
    with open(os.path.join(dst, "traffic_fragment.json"), "w") as f:
        json.dump(traffic, f, indent=1)
print("wrote", dst)
