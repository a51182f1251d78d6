"""key-value / argsort mode.

CPU (-m "not gpu"): the oracle's stable permutation (oracle.stable_argsort, the plain
definition: reading R18) pinned against Python's stable `sorted` (a library routine)
over every small array of an alphabet with duplicates, -0.0/+0.0 and infinities, and
against numpy's stable argsort on random arrays; invariants.
GPU (-m gpu): pcf_argsort_* / pcf_sort_pairs_* against the oracle, element by element.
"""
import itertools
import struct

import numpy as np
import pytest

import oracle
import synth


def tokey(v):
    """totalOrder key of a float64 (an int whose order is IEEE totalOrder)."""
    b = struct.unpack("<q", struct.pack("<d", v))[0]
    return b ^ ((b >> 63) & 0x7FFFFFFFFFFFFFFF)


ALPHA = [-np.inf, -1.5, -0.0, 0.0, 2.0, 2.0, np.inf]


def test_argsort_brute_force_small():
    for n in range(0, 6):
        for t in itertools.product(range(len(ALPHA)), repeat=n):
            x = np.array([ALPHA[i] for i in t], dtype=np.float64)
            want = sorted(range(n), key=lambda i: tokey(float(x[i])))   # Python's sort is stable
            assert list(oracle.stable_argsort(x)) == want, x


def test_argsort_random_vs_numpy_stable():
    rng = np.random.default_rng(3)
    for trial in range(200):
        n = int(rng.integers(1, 3000))
        x = np.round(rng.normal(0, 3, n), int(rng.integers(0, 3)))      # many ties
        x[rng.random(n) < 0.05] = -0.0
        k = x.view(np.int64)
        k = k ^ ((k >> 63) & 0x7FFFFFFFFFFFFFFF)
        assert np.array_equal(oracle.stable_argsort(x), np.argsort(k, kind="stable"))
        u = rng.integers(0, 50, n).astype(np.uint64)
        assert np.array_equal(oracle.stable_argsort(u), np.argsort(u, kind="stable"))


def test_argsort_invariants():
    x = synth.config("c3", n=100_000)                 # 10 % of the keys equal
    p = oracle.stable_argsort(x).astype(np.int64)
    assert np.array_equal(np.sort(p), np.arange(len(x)))
    y = x[p]
    assert np.array_equal(y.view(np.uint64), oracle.learned_sort(x).out.view(np.uint64))
    eq = y[1:] == y[:-1]
    assert np.all(p[1:][eq] > p[:-1][eq])             # equal keys in input order


# ---------------------------------------------------------------- GPU
torch = pytest.importorskip("torch")
DEV = "cuda:0"


@pytest.fixture(scope="module")
def pcf():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2405_07122_b200 as m
    m.build()
    m.lib()
    return m


def check_argsort(pcf, x, **kw):
    want = oracle.stable_argsort(x)
    keys = oracle.learned_sort(x, check=False).out
    xt = torch.from_numpy(x.copy()).to(DEV)
    out, perm = pcf.argsort(xt, **kw)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), keys.view(np.uint64)), "keys differ"
    got = perm.view(torch.int32).cpu().numpy().view(np.uint32).astype(np.uint64)
    if not np.array_equal(got, want):
        bad = np.nonzero(got != want)[0][:5]
        raise AssertionError(f"permutation differs at {bad}: gpu {got[bad]} oracle {want[bad]}")


@pytest.mark.gpu
@pytest.mark.parametrize("name,n", [("c1", None), ("c2", 3_000_000), ("c3", 3_000_000), ("c4", 3_000_000),
                                    ("c5f", 2_000_000), ("c5u", 2_000_000)])
def test_argsort_configs(pcf, name, n):
    check_argsort(pcf, synth.config(name, n=n))


@pytest.mark.gpu
@pytest.mark.parametrize("n", [0, 1, 17, 63, 64, 65, 1000, 8192, 8193, 50_000])
def test_argsort_sizes(pcf, n):
    check_argsort(pcf, synth.generate("lognormal", n, 4))


@pytest.mark.gpu
def test_argsort_patterns(pcf):
    rng = np.random.default_rng(11)
    for n in (3000, 40_000, 400_000):
        base = rng.normal(0, 1, n)
        for x in [np.full(n, 2.5), np.where(rng.random(n) < 0.5, -0.0, 0.0), np.round(base * 4) / 4,
                  rng.integers(0, 3, n).astype(np.float64), np.sort(base)[::-1].copy(),
                  np.where(rng.random(n) < 0.2, 7.0, base)]:
            check_argsort(pcf, np.ascontiguousarray(x))
    check_argsort(pcf, rng.integers(0, 40, 300_000).astype(np.uint64))


@pytest.mark.gpu
def test_argsort_full_size_c3(pcf):
    """c3 at its BASELINE.json size (1e8, a 10^7-key duplicate bucket: the radix Standard-Sort + stability)."""
    check_argsort(pcf, synth.config("c3"))


@pytest.mark.gpu
def test_argsort_batched_global_nodes(pcf):
    check_argsort(pcf, synth.config("c2", n=20_000_000))


@pytest.mark.gpu
@pytest.mark.parametrize("vdt", ["u32", "u64"])
@pytest.mark.parametrize("kdt", ["f64", "u64"])
def test_sort_pairs(pcf, kdt, vdt):
    n = 2_000_000
    x = synth.config("c3", n=n) if kdt == "f64" else (synth.generate("u64", n, 2) >> np.uint64(44))
    rng = np.random.default_rng(1)
    vnp = rng.integers(0, 2 ** 32 if vdt == "u32" else 2 ** 62, n).astype(np.uint32 if vdt == "u32" else np.uint64)
    tdt = torch.int32 if vdt == "u32" else torch.int64
    vt = torch.from_numpy(vnp.view(np.int32 if vdt == "u32" else np.int64)).to(DEV)
    ko, vo = pcf.sort_pairs(torch.from_numpy(x).to(DEV), vt)
    assert vo.dtype == tdt
    perm = oracle.stable_argsort(x).astype(np.int64)
    assert np.array_equal(ko.cpu().numpy().view(np.uint64), x[perm].view(np.uint64))
    assert np.array_equal(vo.cpu().numpy().view(vnp.dtype), vnp[perm])


@pytest.mark.gpu
def test_argsort_small_tau_rejected(pcf):
    x = torch.from_numpy(synth.generate("uniform", 1000, 1)).to(DEV)
    with pytest.raises(pcf.PCFError) as e:
        pcf.argsort(x, tau=8)
    assert e.value.status == 1
