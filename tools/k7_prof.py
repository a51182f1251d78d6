"""Print K7's per-phase cycle breakdown (PCF_FLAG_PROFILE) for a workload.
python tools/k7_prof.py --config c2"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_07122_b200 as pcf
import synth
NAMES = ["claim", "load", "group placement (CTA)", "CTA node: minmax+samples", "CTA-run nodes", "node groups", "sort tasks", "#group nodes",
         "group node keys", "#CTA nodes", "CTA node keys", "tasks", "keys", "store", "CTA node: fit+classify", "CTA node: columns+place"]
SLOTS = [0, 1, 2, 3, 14, 15, 4, 5, 6, 13]
ap = argparse.ArgumentParser(); ap.add_argument("--config", default="c2"); ap.add_argument("--n", type=int, default=None)
a = ap.parse_args()
x = torch.from_numpy(synth.config(a.config, n=a.n)).cuda()
out = torch.empty_like(x)
pcf.sort(x, out)
_, info = pcf.sort(x, out, profile=True)
cy = info.stats["k7_cycles"]
tot = sum(cy[i] for i in SLOTS)
print(f"{a.config}: tasks {cy[11]} keys {cy[12]}  total CTA-cycles {tot:.3e}  cycles/key {tot / max(cy[12], 1):.1f}")
for i in SLOTS:
    print(f"  {NAMES[i]:28s} {cy[i]:.3e}  {100 * cy[i] / max(tot, 1):5.1f}%  {cy[i] / max(cy[12], 1):6.2f} cyc/key")
for i in (7, 8, 9, 10):
    print(f"  {NAMES[i]:28s} {cy[i]:.0f}")
print(f"  mean group node {cy[8] / max(cy[7], 1):.1f} keys, mean CTA node {cy[10] / max(cy[9], 1):.1f} keys")
# warp utilisation of the node phases (slots 16-19: per-warp cycles, summed over warps and CTAs)
nodes_cta = cy[4] + cy[5]   # thread 0's cycles from the end of the group placement to the end of the task
busy = cy[16] + cy[17] + cy[18]
print(f"  warp-cycles in node steps: double teams {cy[16]:.3e}, teams {cy[17]:.3e}, warps {cy[18]:.3e}; "
      f"small-list waits {cy[19]:.3e}")
print(f"  node-phase warp utilisation {busy / max(16 * nodes_cta, 1):.3f} (busy warp-cycles / (16 warps x node-phase cycles))")
tp = [cy[i] for i in (3, 14, 15, 20, 21, 22, 23)]
if sum(tp) and not cy[9] - cy[11]:   # PCF_K7_NPROF build: phases of the 4-warp team nodes
    names = ["minmax", "samples", "fit", "classify+count", "columns", "placement", "leaves+record"]
    print("  team-node phases (team-cycles, PCF_K7_NPROF): " + ", ".join(f"{n} {100 * v / sum(tp):.1f}%" for n, v in zip(names, tp))
          + f"; total {sum(tp):.3e}")
