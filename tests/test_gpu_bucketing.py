"""GPU parity of pcf_bucket_counts_f64 (the §4.3 failure experiment's bucketing
step) against the oracle's M_PCF step (oracle.bucketing):
b[1..beta+1] and H[1..gamma+1] bit-exact, max_j |c_j| exact, with decoupled
alpha, beta, gamma = floor(n^{p/20}) as in Fig. 4."""
import os
import sys

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
from failure_grid import exp_floor  # noqa: E402

DEV = "cuda:0"


@pytest.fixture(scope="module")
def pcf():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2405_07122_b200 as m
    m.build()
    m.lib()
    return m


def u32(t):
    return t.view(torch.int32).cpu().numpy().view(np.uint32)


def check(pcf, x, alpha, beta, gamma, seed):
    pos = oracle.sample_positions(seed, 1, 0, len(x), alpha)
    b_ref, H_ref, _, _ = oracle.bucketing(x, x[pos.astype(np.int64)], beta, gamma)
    b, H, mx = pcf.bucket_counts(torch.from_numpy(x).to(DEV), alpha, beta, gamma, seed=seed)
    np.testing.assert_array_equal(u32(b), b_ref)
    np.testing.assert_array_equal(u32(H), H_ref)
    assert mx == int(H_ref.max())
    assert int(H_ref.sum()) == len(x)


@pytest.mark.parametrize("n", [10_000, 100_003])
@pytest.mark.parametrize("abc", [(15, 15, 15), (1, 1, 1), (19, 19, 19), (15, 6, 18), (8, 19, 4), (19, 2, 19),
                                 (12, 17, 9), (3, 19, 19)])
def test_bucket_counts_uniform(pcf, n, abc):
    x = synth.generate("uniform", n, 77 + n)
    a, b, c = (exp_floor(n, p) for p in abc)
    for seed in (0, 7):
        check(pcf, x, a, b, c, seed)


@pytest.mark.parametrize("dist", ["lognormal", "exponential", "gauss_mix8", "exp700u4"])
def test_bucket_counts_skewed(pcf, dist):
    n = 50_000
    x = synth.generate(dist, n, 5)
    for abc in [(15, 15, 15), (10, 18, 12)]:
        check(pcf, x, *(exp_floor(n, p) for p in abc), seed=3)


def test_bucket_counts_paper_size_and_oversampling(pcf):
    n = 1_000_000                                           # the §4.3 size, in the harness's launch configuration
    x = synth.generate("uniform", n, 5000)
    check(pcf, x, exp_floor(n, 15), exp_floor(n, 15), exp_floor(n, 15), seed=0)
    check(pcf, x, exp_floor(n, 19), exp_floor(n, 19), exp_floor(n, 19), seed=1)
    check(pcf, synth.generate("uniform", 1000, 1), 3000, 64, 5000, seed=2)     # alpha > n (with replacement), gamma > n


def test_bucket_counts_small_and_ties(pcf):
    check(pcf, np.array([2.0, 1.0]), 1, 1, 1, seed=0)
    x = np.repeat(np.array([0.0, 1.0, 2.0, 3.0]), 257)     # many ties; samples hit few distinct keys
    check(pcf, x, 31, 7, 5, seed=4)
    check(pcf, np.array([-0.0, 0.0, 1.0, -1.0, 5e-324, -5e-324]), 4, 3, 6, seed=9)


def test_bucket_counts_errors(pcf):
    with pytest.raises(pcf.PCFError) as e:
        pcf.bucket_counts(torch.full((1000,), 3.5, dtype=torch.float64, device=DEV), 10, 10, 10)
    assert e.value.status == 8                                 # PCF_ERR_DEGENERATE
    x = torch.rand(1000, dtype=torch.float64, device=DEV)
    x[500] = float("nan")
    with pytest.raises(pcf.PCFError) as e:
        pcf.bucket_counts(x, 10, 10, 10)
    assert e.value.status == 2                                 # PCF_ERR_NAN
