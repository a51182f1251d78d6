"""The paper's bucketing-failure experiment on the GPU (§4.3, Fig. 4).

alpha = floor(n^a), beta = floor(n^b), gamma = floor(n^c), delta = floor(n^d) for
a, b, c, d in {0.05, ..., 0.95}; the two exponents not on a panel's axes are
0.75.  Each cell runs `trials` bucketing steps M_PCF of n = 10^6 uniform keys
(a fresh seeded array and sampler seed per trial) through pcf_bucket_counts_f64
and counts "failures", max_j |c_j| > delta.  Lemma 3 bounds
that probability by (2n/delta) exp{-(alpha K / 2 gamma)(1 - 1/K)^2} when K >= 1,
K = gamma delta / 2n - 2 sigma_2 gamma / (sigma_1 beta); for the uniform density
sigma_2 / sigma_1 = 1.  The paper's white line is where that bound equals 0.5.

  python tools/failure_grid.py [--n 1000000] [--trials 100] [--out FILE]

Prints, per panel, the failure frequency of every cell (in %) and marks the cells
where the bound is <= 0.5 ('<'), then counts the marked cells whose observed
frequency exceeds 0.5 (Lemma 3 says the true probability there is below 0.5).
Inputs are synthetic (synth.generate('uniform', n, seed)); no dataset is used.
"""
import argparse
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

Q = 20                        # exponents are p / 20, p = 1..19  (0.05 .. 0.95)
GRID = list(range(1, 20))
FIXED = 15                    # 0.75
PANELS = [("a", "b"), ("a", "c"), ("a", "d"), ("b", "c"), ("b", "d"), ("c", "d")]   # Fig. 4 order


def exp_floor(n: int, p: int, q: int = Q) -> int:
    """floor(n^(p/q)) exactly: the largest c with c^q <= n^p (integer arithmetic)."""
    t = n ** p
    c = int(round(n ** (p / q)))
    while c > 0 and c ** q > t:
        c -= 1
    while (c + 1) ** q <= t:
        c += 1
    return c


def lemma3_bound(n: int, alpha: int, beta: int, gamma: int, delta: int, s21: float = 1.0):
    """Right side of Lemma 3, or None when K < 1 (no claim)."""
    K = gamma * delta / (2.0 * n) - 2.0 * s21 * gamma / beta
    if K < 1.0:
        return None
    return (2.0 * n / delta) * math.exp(-(alpha * K / (2.0 * gamma)) * (1.0 - 1.0 / K) ** 2)


def cell_params(n: int, panel, px: int, py: int):
    e = {"a": FIXED, "b": FIXED, "c": FIXED, "d": FIXED}
    e[panel[0]], e[panel[1]] = px, py
    return tuple(exp_floor(n, e[k]) for k in "abcd")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--trials", type=int, default=100)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    import torch

    import paper_2405_07122_b200 as pcf
    import synth

    n, T = args.n, args.trials
    dev = "cuda:0"
    xs = [torch.from_numpy(synth.generate("uniform", n, 5000 + t)).to(dev) for t in range(T)]
    bmax = max(exp_floor(n, p) for p in GRID) + 1
    b = torch.empty(bmax, dtype=torch.uint32, device=dev)
    H = torch.empty(bmax, dtype=torch.uint32, device=dev)
    lines = [f"# PCF bucketing-failure frequency (PAPER.md:516-531, Fig. 4): n={n} uniform, {T} trials per cell,",
             "# failure = exists j |c_j| > delta; '<' marks cells where the Lemma-3 bound <= 0.5 (sigma2/sigma1 = 1).",
             "# rows: y exponent (0.95 top), columns: x exponent 0.05..0.95; entries: failure frequency in %."]
    calls, t0, viol, marked = 0, time.perf_counter(), 0, 0
    for panel in PANELS:
        lines.append(f"\n## x = {panel[0]}, y = {panel[1]}  (others 0.75)")
        lines.append("   y\\x " + " ".join(f"{p * 5:>4d}" for p in GRID))
        for py in reversed(GRID):
            row = []
            for px in GRID:
                alpha, beta, gamma, delta = cell_params(n, panel, px, py)
                fails = 0
                for t in range(T):
                    _, _, mx = pcf.bucket_counts(xs[t], alpha, beta, gamma, seed=t, b=b, H=H)
                    fails += mx > delta
                    calls += 1
                bound = lemma3_bound(n, alpha, beta, gamma, delta)
                mark = "<" if bound is not None and bound <= 0.5 else " "
                if mark == "<":
                    marked += 1
                    viol += fails > T // 2
                row.append(f"{100 * fails // T:>3d}{mark}")
            lines.append(f"  {py * 5:>4d} " + " ".join(row))
    dt = time.perf_counter() - t0
    lines.append(f"\n# {calls} bucketing steps in {dt:.1f} s ({1e6 * dt / calls:.1f} us per step incl. host sync)")
    lines.append(f"# cells with Lemma-3 bound <= 0.5: {marked}; of those with observed frequency > 0.5: {viol}")
    txt = "\n".join(lines)
    print(txt)
    if args.out:
        with open(args.out, "w") as f:
            f.write(txt + "\n")


if __name__ == "__main__":
    main()
