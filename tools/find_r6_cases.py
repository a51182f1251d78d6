"""Find bin-edge keys for the R6 pins (tests/golden/r6_bin_edges.json).

Reading R6 evaluates i(x) = floor(t) + 1 with
    d = RN(x - x_min),  r = RN(x_max - x_min),  q = RN(d / r),  t = RN(q * beta)
(RN = IEEE binary64 round-to-nearest-even).  This script derives those values
WITHOUT the FPU's sub/div/mul: every step is done in exact rational arithmetic
(fractions.Fraction) and rounded once with CPython's correctly rounded int/int
true division (RN).  It keeps keys where the R6 value differs from the exact
rational i(x) = floor((x - x_min) / (x_max - x_min) * beta) + 1 and/or from the
other plausible op order fl(d * fl(beta / r)) -- so a pin on these keys fails if
an implementation uses the rational value, a different op order, an FMA, or a
reciprocal.  It calls nothing from oracle/ or the CUDA path.

  python tools/find_r6_cases.py > tests/golden/r6_bin_edges.json
"""
import json
import math
import random
from fractions import Fraction as F


def rn(q: F) -> float:
    return q.numerator / q.denominator   # correctly rounded (CPython long true division)


def r6(x, lo, hi, beta):
    d = rn(F(x) - F(lo))
    r = rn(F(hi) - F(lo))
    q = rn(F(d) / F(r))
    t = rn(F(q) * beta)
    return math.floor(t) + 1, dict(d=d.hex(), r=r.hex(), q=q.hex(), t=t.hex())


def exact(x, lo, hi, beta):
    return math.floor((F(x) - F(lo)) / (F(hi) - F(lo)) * beta) + 1


def other_order(x, lo, hi, beta):
    d = rn(F(x) - F(lo))
    r = rn(F(hi) - F(lo))
    s = rn(F(beta) / F(r))
    return math.floor(rn(F(d) * F(s))) + 1


def iroot34(m):
    c = int(round(m ** 0.75))
    while c ** 4 > m ** 3:
        c -= 1
    while (c + 1) ** 4 <= m ** 3:
        c += 1
    return c


def search(m, lo, hi, want, rng):
    beta = iroot34(m)
    out = []
    tried = 0
    while len(out) < want and tried < 200000:
        tried += 1
        k = rng.randrange(1, beta)
        e = F(lo) + (F(hi) - F(lo)) * k / beta          # exact bin edge k
        x = rn(e)
        x = x + rng.randrange(-3, 4) * math.ulp(x)
        if not (lo < x < hi):
            continue
        i6, steps = r6(x, lo, hi, beta)
        ie, io = exact(x, lo, hi, beta), other_order(x, lo, hi, beta)
        if i6 != ie or i6 != io:
            if any(c["x"] == x.hex() for c in out):
                continue
            out.append(dict(x=x.hex(), i_r6=i6, i_exact=ie, i_other_order=io, steps=steps))
    return dict(m=m, beta=beta, lo=lo.hex(), hi=hi.hex(), cases=out)


def main():
    rng = random.Random(20240512)
    groups = [
        search(1000, 0.1, 0.7, 12, rng),                 # K7 path (m <= 8192), beta = 177
        search(1000, -3.0, 1e3 / 3, 12, rng),
        search(20000, 0.3, 1.1, 12, rng),                # global path (m > 8192), beta = 1681
        search(20000, -1e-3, 7e5 / 9, 12, rng),
    ]
    doc = {
        "_source": "tools/find_r6_cases.py (exact rationals + one correct rounding per step; "
                   "no oracle/ or CUDA code).  Reading R6: DESIGN.md §2, PAPER.md:293-295 (i(x)).",
        "groups": groups,
    }
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
