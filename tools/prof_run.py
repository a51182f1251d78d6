"""Minimal driver for ncu captures: sorts one workload `--reps` times (no timing,
no oracle).  Usage: python tools/prof_run.py --config c2 [--n N] [--reps 2]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2405_07122_b200 as pcf  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
x = torch.from_numpy(synth.config(a.config, n=a.n)).cuda()
out = torch.empty_like(x)
ws = torch.empty(pcf.workspace_bytes(x.numel()), dtype=torch.uint8, device="cuda")
for _ in range(a.reps):
    pcf.sort(x, out, workspace=ws)
torch.cuda.synchronize()
print("ok", x.numel())
