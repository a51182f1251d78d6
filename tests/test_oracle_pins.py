"""Pins for the CPU oracle (oracle/pcf_oracle.c) against things other than itself.

Every test here runs without a GPU.  The oracle is pinned by
  * worked examples hand-derived from the paper's definitions (tests/golden/),
  * closed forms (perfect fourth powers for floor(n^{3/4}), exact rationals),
  * brute force over every tiny array (vs. an independent totalOrder sort),
  * the paper's invariants (order property, b monotone with b_{beta+1}=alpha, ...),
  * the published SplitMix64 output vector (the sampler's hash).
"""
import itertools
import json
import os
import struct
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def total_order_key(x: float):
    """IEEE-754 totalOrder as a Python sort key, written from the standard's text
    (sign first; among negatives larger magnitude first; -0 < +0)."""
    bits = struct.unpack("<Q", struct.pack("<d", x))[0]
    neg = bits >> 63
    mag = bits & 0x7FFFFFFFFFFFFFFF
    return (0, -mag) if neg else (1, mag)


def tsorted_bits(xs):
    return [struct.unpack("<Q", struct.pack("<d", v))[0] for v in sorted(xs, key=total_order_key)]


# ---------------------------------------------------------------- level parameters (R5)
def test_level_params_golden():
    for n, p in _gold("spec_examples.json")["level_params"]["cases"]:
        assert oracle.iroot34(n) == p


def test_iroot34_perfect_fourth_powers():
    # closed form: (k^4)^{3/4} = k^3 exactly
    for k in list(range(1, 200)) + [1000, 1024, 1448]:   # k^4 <= 2^42 (documented range)
        assert oracle.iroot34(k ** 4) == k ** 3
        if k > 1:
            assert oracle.iroot34(k ** 4 - 1) == k ** 3 - 1


def test_iroot34_definition_bruteforce():
    rng = np.random.default_rng(5)
    ms = list(range(1, 3000)) + [int(v) for v in rng.integers(1, 2 ** 40, 2000)]
    for m in ms:
        c = oracle.iroot34(m)
        assert c ** 4 <= m ** 3 < (c + 1) ** 4


# ---------------------------------------------------------------- i(x)
def test_interval_index_golden():
    for x, lo, hi, beta, want in _gold("spec_examples.json")["interval_index"]["cases"]:
        assert oracle.interval_index(x, lo, hi, beta) == want


def test_interval_index_endpoints_monotone_and_rational():
    rng = np.random.default_rng(1)
    off_by_one = 0
    for _ in range(300):
        lo, hi = sorted(rng.normal(0, 100, 2))
        beta = int(rng.integers(1, 10 ** 6))
        assert oracle.interval_index(lo, lo, hi, beta) == 1
        assert oracle.interval_index(hi, lo, hi, beta) == beta + 1
        xs = np.sort(rng.uniform(lo, hi, 50))
        idx = [oracle.interval_index(x, lo, hi, beta) for x in xs]
        assert all(1 <= i <= beta + 1 for i in idx)
        assert idx == sorted(idx)                       # non-decreasing in x
        for x, i in zip(xs, idx):                       # exact-rational definition, +-1 only at edges
            t = (Fraction(float(x)) - Fraction(float(lo))) / (Fraction(float(hi)) - Fraction(float(lo))) * beta
            exact = int(t) + 1
            assert abs(exact - i) <= 1
            off_by_one += exact != i
    assert off_by_one <= 3


def test_interval_index_u64_exact_difference():
    # R15: the u64 difference is exact before rounding; x = xmin + (xmax-xmin)/2 lands mid-range
    lo, hi = 2 ** 63 + 12345, 2 ** 64 - 1
    mid = lo + (hi - lo) // 2
    assert oracle.interval_index_u64(lo, lo, hi, 1000) == 1
    assert oracle.interval_index_u64(hi, lo, hi, 1000) == 1001
    assert oracle.interval_index_u64(mid, lo, hi, 1000) == 501
    assert oracle.interval_index_u64(5, 0, 10, 5) == 3


# ---------------------------------------------------------------- PCF training / inference
def test_train_pcf_golden():
    for c in _gold("spec_examples.json")["train_pcf"]["cases"]:
        b = oracle.train_pcf(np.array(c["sample"], float), float(c["xmin"]), float(c["xmax"]), c["beta"])
        assert b.tolist() == c["b"]


def test_train_pcf_bruteforce_set_counting():
    # b_i = |{ j : i(a_j) <= i }|, counted by brute force over the set
    rng = np.random.default_rng(2)
    for _ in range(300):
        alpha = int(rng.integers(1, 100))
        beta = int(rng.integers(1, 21))
        a = rng.normal(0, 1, alpha)
        lo, hi = float(a.min()) - abs(rng.normal()), float(a.max()) + abs(rng.normal())
        if rng.random() < 0.5:
            lo, hi = float(a.min()), float(a.max())
            if lo == hi:
                continue
        b = oracle.train_pcf(a, lo, hi, beta)
        ia = [oracle.interval_index(v, lo, hi, beta) for v in a]
        want = [sum(1 for v in ia if v <= i) for i in range(1, beta + 2)]
        assert b.tolist() == want
        assert b[-1] == alpha and all(np.diff(b.astype(np.int64)) >= 0)


def test_infer_cdf_golden_and_properties():
    g = _gold("spec_examples.json")["infer_cdf"]
    md = g["model"]
    b = np.array(md["b"], np.uint32)
    for x, want in g["cases"]:
        assert oracle.infer_cdf(b, md["alpha"], float(x), float(md["xmin"]), float(md["xmax"]), md["beta"]) == want
    rng = np.random.default_rng(3)
    a = rng.random(200)
    b = oracle.train_pcf(a, 0.0, 1.0, 37)
    xs = np.sort(rng.random(1000))
    F = [oracle.infer_cdf(b, 200, x, 0.0, 1.0, 37) for x in xs]
    assert all(0.0 <= f <= 1.0 for f in F) and F == sorted(F)


def test_bucket_index_exact_integer_form():
    # R7: j = floor(b*gamma/alpha)+1 equals floor(F~ * gamma)+1 with exact rationals
    rng = np.random.default_rng(4)
    for _ in range(5000):
        alpha = int(rng.integers(1, 10 ** 7))
        gamma = int(rng.integers(1, 10 ** 7))
        b = int(rng.integers(0, alpha + 1))
        assert oracle.bucket_of(b, alpha, gamma) == int(Fraction(b, alpha) * gamma) + 1
    assert oracle.bucket_of(7, 7, 7) == 8 and oracle.bucket_of(0, 5, 9) == 1


# ---------------------------------------------------------------- bucketing (Alg. 1 body)
def test_bucketing_golden():
    g = _gold("spec_examples.json")["bucketing"]
    x = np.array(g["x"], float)
    b, H, bid, out = oracle.bucketing(x, np.array(g["sample"], float), g["beta"], g["gamma"])
    got, pos = [], 0
    for h in H:
        got.append(out[pos:pos + h].tolist())
        pos += h
    assert [c for c in got if c] == g["buckets"]


def test_bucketing_order_property_and_conservation():
    rng = np.random.default_rng(6)
    for dist in ["uniform", "normal", "exponential", "lognormal"]:
        x = synth.generate(dist, 1000, int(rng.integers(1 << 30)))
        p = oracle.iroot34(1000)
        sample = x[rng.integers(0, 1000, p)]
        b, H, bid, out = oracle.bucketing(x, sample, p, p)
        assert H.sum() == 1000 and sorted(out.tolist()) == sorted(x.tolist())
        pos, prev = 0, None
        for j, h in enumerate(H):
            if h == 0:
                continue
            c = out[pos:pos + h]
            assert np.all(bid[np.isin(x, c)] == j + 1)
            if prev is not None:
                assert prev < c.min()
            prev = c.max()
            pos += h
        # stability (Append in index order)
        order = np.argsort(bid, kind="stable")
        assert np.array_equal(out, x[order])


# ---------------------------------------------------------------- sampler (R3/R4)
def test_mix64_published_splitmix64_vector():
    want = [int(h, 16) for h in _gold("splitmix64.json")["outputs_seed0"]]
    got = [oracle.mix64(k * 0x9E3779B97F4A7C15) for k in range(1, 5)]
    assert got == want


def test_sample_positions_uniform_and_deterministic():
    m, alpha = 1000, 200000
    p = oracle.sample_positions(7, 1, 0, m, alpha)
    assert p.max() < m
    assert np.array_equal(p, oracle.sample_positions(7, 1, 0, m, alpha))
    counts = np.bincount(p.astype(np.int64), minlength=m)
    chi2 = ((counts - alpha / m) ** 2 / (alpha / m)).sum()
    assert chi2 < m + 6 * np.sqrt(2 * m)                  # ~6 sigma
    q = oracle.sample_positions(7, 2, 0, m, 1000)
    r = oracle.sample_positions(7, 1, 64, m, 1000)
    assert not np.array_equal(p[:1000], q) and not np.array_equal(p[:1000], r)


def test_digest_position_sensitive():
    v = np.arange(1, 100, dtype=np.uint32)
    assert oracle.digest(v) != oracle.digest(v[::-1])
    assert oracle.digest(np.zeros(0, np.uint32)) == 0
    w = v.copy(); w[50] += 1
    assert oracle.digest(v) != oracle.digest(w)


# ---------------------------------------------------------------- the full sort
def test_learned_sort_golden():
    for c in _gold("spec_examples.json")["learned_sort"]["cases"]:
        r = oracle.learned_sort(np.array(c["x"], float), tau=c["tau"])
        assert r.out.tolist() == c["out"]


ALPHABETS = [
    [-np.inf, -1.5, -0.0, 0.0, 5e-324, 1e300],
    [-1e308, -2.0, 0.0, 1.0, 1e308, np.inf],
    [1.0, 2.0, 2.0000000000000004, 3.0, 1e-300, -0.0],
]


def test_bruteforce_every_tiny_array():
    """Every array of length <= 5 (<= 6 for tau=2) over small alphabets incl. +-0,
    subnormals, +-inf and overflowing ranges: output bits == totalOrder sort."""
    for alph in ALPHABETS:
        for tau in (2, 3, 64):
            maxlen = 6 if tau == 2 else 5
            for L in range(0, maxlen + 1):
                for xs in itertools.product(alph, repeat=L):
                    x = np.array(xs, dtype=np.float64)
                    r = oracle.learned_sort(x, tau=tau, seed=L)
                    assert r.out.view(np.uint64).tolist() == tsorted_bits(xs), (xs, tau)


def test_random_arrays_vs_independent_sort():
    """SPEC.md:633 acceptance: >= 1000 random arrays incl. all-equal and 50% duplicates."""
    rng = np.random.default_rng(11)
    dists = ["uniform", "normal", "exponential", "lognormal"]
    for t in range(1000):
        n = int(rng.integers(0, 3000))
        kind = t % 6
        if kind < 4:
            x = synth.generate(dists[kind], n, t)
        elif kind == 4:
            x = np.full(n, rng.normal())
        else:
            x = synth.generate("normal", n, t)
            if n:
                x[rng.random(n) < 0.5] = x[0]
        tau = int(rng.choice([2, 16, 64]))
        r = oracle.learned_sort(x, tau=tau, seed=t)
        assert np.array_equal(r.out.view(np.uint64), np.sort(x).view(np.uint64)) or \
            r.out.view(np.uint64).tolist() == tsorted_bits(x.tolist())


def test_u64_keys():
    rng = np.random.default_rng(12)
    for t in range(50):
        n = int(rng.integers(0, 5000))
        x = synth.generate("u64", n, t)
        if t % 3 == 0:
            x = (x >> np.uint64(rng.integers(0, 60))).astype(np.uint64)
        r = oracle.learned_sort(x, tau=int(rng.choice([2, 64])), seed=t)
        assert np.array_equal(r.out, np.sort(x))


def test_nan_rejected_before_work():
    x = np.array([3.0, np.nan, 1.0])
    with pytest.raises(oracle.OracleError) as e:
        oracle.learned_sort(x)
    assert e.value.rc == oracle.ERR_NAN


def test_node_invariants_and_log_level1():
    """Per-node invariant checks run inside the oracle (check=True): sum H = m,
    b monotone with b_{beta+1} = alpha, T[beta+1] = gamma+1, H[gamma+1] >= 1,
    the order property; the level-1 log equals a direct recomputation."""
    x = synth.generate("lognormal", 200_000, 3)
    r = oracle.learned_sort(x, log=True)
    n = len(x)
    p = oracle.iroot34(n)
    assert len(r.l1_b) == p + 1 and len(r.l1_h) == p + 1
    assert r.l1_h.sum() == n and r.l1_b[-1] == p
    root = oracle.sort_nodes(r.nodes)[0]
    assert root["level"] == 1 and root["m"] == n and root["alpha"] == p
    assert root["digest_b"] == oracle.digest(r.l1_b) and root["digest_h"] == oracle.digest(r.l1_h)
    # recompute level 1 independently from the published pieces: sample -> b -> H
    pos = oracle.sample_positions(0, 1, 0, n, p)
    b = oracle.train_pcf(x[pos.astype(np.int64)], float(x.min()), float(x.max()), p)
    assert np.array_equal(b, r.l1_b)
    b2, H2, _, _ = oracle.bucketing(x, x[pos.astype(np.int64)], p, p)
    assert np.array_equal(H2, r.l1_h)
    # children bookkeeping: counts of fallback/small/recurse buckets
    nz = r.l1_h[r.l1_h > 0]
    assert root["n_fallback"] == (nz >= p).sum()
    assert root["n_small"] == ((nz < p) & (nz < 64)).sum()
    assert root["n_recurse"] == ((nz < p) & (nz >= 64)).sum()


def test_sample_all_mode_is_rng_free():
    """R14 test mode: a = the whole segment, alpha = m, beta = gamma = floor(m^{3/4})."""
    x = synth.generate("normal", 5000, 9)
    r1 = oracle.learned_sort(x, flags=oracle.FLAG_SAMPLE_ALL, seed=1, log=True)
    r2 = oracle.learned_sort(x, flags=oracle.FLAG_SAMPLE_ALL, seed=99, log=True)
    assert np.array_equal(r1.l1_b, r2.l1_b) and np.array_equal(r1.l1_h, r2.l1_h)
    p = oracle.iroot34(5000)
    lo, hi = float(x.min()), float(x.max())
    ix = np.array([oracle.interval_index(v, lo, hi, p) for v in x])
    cnt = np.bincount(ix, minlength=p + 2)[1:]
    assert np.array_equal(r1.l1_b, np.cumsum(cnt))
    j = [int(Fraction(int(r1.l1_b[i - 1]) * p, 5000)) + 1 for i in ix]
    assert np.array_equal(r1.l1_h, np.bincount(j, minlength=p + 2)[1:])
    assert np.array_equal(r1.out, np.sort(x))


def test_depth_bound_and_observed_depth():
    for n, tau, want in _gold("spec_examples.json")["depth_bound"]["cases"]:
        assert oracle.depth_bound(n, tau) == want
    for seed in range(5):
        x = synth.generate("uniform", 10 ** 5, seed)
        r = oracle.learned_sort(x, seed=seed)
        assert r.max_depth <= oracle.depth_bound(10 ** 5)


def test_lemma3_no_failures_uniform():
    """Lemma 3 at alpha=beta=gamma=delta=floor(n^{3/4}), n=1e5
    uniform: the bound is < 1e-30, so no level-1 bucket reaches delta."""
    for seed in range(10):
        x = synth.generate("uniform", 10 ** 5, 100 + seed)
        r = oracle.learned_sort(x, seed=seed, log=True)
        root = oracle.sort_nodes(r.nodes)[0]
        assert root["n_fallback"] == 0


def test_determinism():
    x = synth.generate("exponential", 100_000, 2)
    a = oracle.learned_sort(x, seed=5, log=True)
    b = oracle.learned_sort(x, seed=5, log=True)
    assert np.array_equal(a.nodes, b.nodes) and np.array_equal(a.out, b.out)


# ---------------------------------------------------------------- R6 at bin edges
def _rn(q):
    return q.numerator / q.denominator   # one correct rounding (CPython int/int true division)


def r6_by_rationals(x, lo, hi, beta):
    """Reading R6 derived in exact rationals, one RN per step (no FPU sub/div/mul)."""
    d = _rn(Fraction(x) - Fraction(lo))
    r = _rn(Fraction(hi) - Fraction(lo))
    q = _rn(Fraction(d) / Fraction(r))
    t = _rn(Fraction(q) * beta)
    return int(t // 1) + 1


def r6_cases():
    g = _gold("r6_bin_edges.json")
    for grp in g["groups"]:
        lo, hi, beta = float.fromhex(grp["lo"]), float.fromhex(grp["hi"]), grp["beta"]
        for c in grp["cases"]:
            yield lo, hi, beta, float.fromhex(c["x"]), c


def test_r6_golden_derivation():
    """Each stored case is re-derived here: the R6 value, and that it differs from the
    exact rational floor and/or from the fl(d * fl(beta / r)) op order (so the pin
    discriminates between the readings)."""
    n = 0
    for lo, hi, beta, x, c in r6_cases():
        assert r6_by_rationals(x, lo, hi, beta) == c["i_r6"]
        ex = int((Fraction(x) - Fraction(lo)) / (Fraction(hi) - Fraction(lo)) * beta // 1) + 1
        assert ex == c["i_exact"]
        assert c["i_r6"] != c["i_exact"] or c["i_r6"] != c["i_other_order"]
        n += 1
    assert n >= 40


def test_r6_oracle_at_bin_edges():
    """The oracle's i(x) follows reading R6 (not the exact rational, not another op
    order) on keys within a few ulps of bin edges."""
    for lo, hi, beta, x, c in r6_cases():
        assert oracle.interval_index(x, lo, hi, beta) == c["i_r6"], (x.hex(), c)
