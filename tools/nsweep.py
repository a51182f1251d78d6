"""GPU analogue of the paper's Fig. 2 (ops/n vs n): device time per
key of the whole sort vs n, for the paper's four synthetic distributions
(Uniform(0,1), Normal(0,1), Exponential(1), LogNormal(0,1); SPEC.md:395-396 recipes via synth/).
python tools/nsweep.py [--max-log10 9] > profiles/r01/nsweep.txt   (one GPU)"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_07122_b200 as pcf  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--max-log10", type=int, default=9)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
dists = ["uniform", "normal", "exponential", "lognormal"]
print("# ns per key of one sort (median of reps, L2 flushed), 1 x B200")
print("n          " + " ".join(f"{d:>12s}" for d in dists))
l2 = torch.cuda.get_device_properties(0).L2_cache_size
flush = torch.empty(2 * l2, dtype=torch.uint8, device="cuda")
for e in range(3, a.max_log10 + 1):
    n = 10 ** e
    row = []
    for d in dists:
        x = torch.from_numpy(synth.generate(d, n, 7)).cuda()
        out = torch.empty_like(x)
        ws = torch.empty(pcf.workspace_bytes(n), dtype=torch.uint8, device="cuda")
        pcf.sort(x, out, workspace=ws)
        ts = []
        for _ in range(a.reps):
            flush.fill_(1)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            pcf.sort(x, out, workspace=ws)
            s1.record()
            s1.synchronize()
            ts.append(s0.elapsed_time(s1))
        ts.sort()
        row.append(ts[len(ts) // 2] * 1e6 / n)
        del x, out, ws
        torch.cuda.empty_cache()
    print(f"{n:<10d} " + " ".join(f"{v:12.3f}" for v in row), flush=True)
