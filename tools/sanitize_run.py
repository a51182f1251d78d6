"""Workload for compute-sanitizer: a few sorts through the C ABI
that exercise every kernel family -- the single-task K7 path, the split rounds
(bulk-copy count kernel, scatter, taskgen), K7's team / warp node lists and
mbarrier bulk copies, the batched global nodes, the radix Standard-Sort -- each checked against the
oracle.  Sizes are kept small (sanitizers slow kernels down 10-1000x).

  python tools/sanitize_run.py [scale]     # scale 1.0 = default sizes
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2405_07122_b200 as pcf  # noqa: E402
import synth  # noqa: E402


def check(x, name, **kw):
    ref = oracle.learned_sort(x, log=True, **kw)
    out, info = pcf.sort(torch.from_numpy(x).cuda(), log=True, **kw)
    ok = np.array_equal(out.cpu().numpy().view(np.uint64), ref.out.view(np.uint64))
    a, b = oracle.sort_nodes(ref.nodes), np.sort(info.nodes, order=["level", "offset"])
    ok = ok and len(a) == len(b) and all(np.array_equal(a[f], b[f]) for f in a.dtype.names)
    print(f"{name}: n={len(x)} {'OK' if ok else 'MISMATCH'}", flush=True)
    return ok


def main():
    scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
    s = lambda n: max(1000, int(n * scale))  # noqa: E731
    ok = True
    ok &= check(synth.generate("uniform", 5000, 1), "k7_single_task")
    ok &= check(synth.config("c1", n=s(200_000)), "c1_uniform")
    ok &= check(synth.config("c2", n=s(1_000_000)), "c2_lognormal")
    x = synth.generate("uniform", s(600_000), 3)          # oversized recursing buckets -> batched global nodes
    rng = np.random.default_rng(5)
    for v in (0.25, 0.5):
        x[rng.choice(x.size, 12_000, replace=False)] = v
    ok &= check(x, "batched_global_nodes")
    ok &= check(synth.config("c4", n=s(300_000)), "c4_fallback_k8")
    ok &= check(synth.config("c5u", n=s(300_000)), "c5u_u64")
    print("ALL OK" if ok else "FAILED")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
