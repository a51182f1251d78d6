"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

The bar (integer/index work): bit-exact sorted output AND bit-exact per-node
records -- (level, offset, m, alpha, x_min/x_max bits, digest of b, digest of H,
#fallback/#small/#recurse buckets) -- plus the full level-1 b and H arrays.
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pcf():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2405_07122_b200 as m
    m.build()
    m.lib()
    return m


DEV = "cuda:0"


def compare(pcf, x, tau=64, seed=0, sample_all=False, check_nodes=True, inplace=False, exact_ranks=False):
    flags = oracle.FLAG_SAMPLE_ALL if sample_all else 0
    ref = oracle.learned_sort(x, tau=tau, seed=seed, flags=flags, log=check_nodes, check=True)
    xt = torch.from_numpy(x.copy()).to(DEV)
    if inplace:
        out, info = pcf.sort(xt, xt, tau=tau, seed=seed, sample_all=sample_all, log=check_nodes, stats=True)
        assert out.data_ptr() == xt.data_ptr()
    else:
        out, info = pcf.sort(xt, tau=tau, seed=seed, sample_all=sample_all, log=check_nodes, stats=True,
                             exact_ranks=exact_ranks)
        assert np.array_equal(xt.cpu().numpy().view(np.uint64), x.view(np.uint64)), "input was modified"
    got = out.cpu().numpy()
    assert np.array_equal(got.view(np.uint64), ref.out.view(np.uint64)), "sorted output differs"
    if check_nodes:
        a = oracle.sort_nodes(ref.nodes)
        b = np.sort(info.nodes, order=["level", "offset"])
        assert len(a) == len(b), f"node count {len(b)} != oracle {len(a)}"
        for f in a.dtype.names:
            if not np.array_equal(a[f], b[f]):
                bad = np.nonzero(a[f] != b[f])[0][:5]
                raise AssertionError(f"node field {f} differs at {bad}: gpu {b[bad]} oracle {a[bad]}")
        if ref.l1_b is not None and len(ref.l1_b):
            assert np.array_equal(info.level1_b[: len(ref.l1_b)], ref.l1_b), "level-1 b differs"
            assert np.array_equal(info.level1_h[: len(ref.l1_h)], ref.l1_h), "level-1 H differs"
    return ref, info


@pytest.mark.parametrize("n", [0, 1, 2, 3, 63, 64, 65, 100, 1000, 1024, 1025, 4097, 8191, 8192, 8193,
                               10_000, 50_000, 100_000, 1_000_000, 3_000_000])
def test_n_sweep_uniform(pcf, n):
    compare(pcf, synth.generate("uniform", n, 17))


@pytest.mark.parametrize("name,n", [("c1", None), ("c2", 2_000_000), ("c3", 2_000_000), ("c4", 2_000_000),
                                    ("c5f", 2_000_000), ("c5u", 2_000_000)])
def test_configs_reduced(pcf, name, n):
    compare(pcf, synth.config(name, n=n))


@pytest.mark.parametrize("dist", ["normal", "exponential", "lognormal", "gauss_mix8", "exp700u4", "u64"])
@pytest.mark.parametrize("n", [5_000, 20_000, 300_000])
def test_distributions(pcf, dist, n):
    compare(pcf, synth.generate(dist, n, 3))


@pytest.mark.parametrize("tau", [2, 3, 16, 300, 5000])
def test_tau(pcf, tau):
    compare(pcf, synth.generate("lognormal", 200_000, 5), tau=tau)
    compare(pcf, synth.generate("uniform", 3000, 5), tau=tau)


@pytest.mark.parametrize("seed", [1, 2, 12345678901234567])
def test_seeds(pcf, seed):
    compare(pcf, synth.generate("exponential", 100_000, 8), seed=seed)


@pytest.mark.parametrize("n", [500, 6000, 100_000])
def test_sample_all_mode(pcf, n):
    compare(pcf, synth.generate("normal", n, 4), sample_all=True)


def _patterns(n, rng):
    base = rng.normal(0, 1, n)
    out = {
        "sorted": np.sort(base),
        "reverse": np.sort(base)[::-1].copy(),
        "all_equal": np.full(n, 3.25),
        "two_values": np.where(rng.random(n) < 0.5, -1.0, 2.0),
        "mixed_zero": np.where(rng.random(n) < 0.5, -0.0, 0.0),
        "zeros_and_values": np.where(rng.random(n) < 0.3, rng.choice([-0.0, 0.0], n), base),
        "overflow_range": np.where(rng.random(n) < 0.5, -1e308, 1e308) * rng.random(n),
        "with_inf": np.where(rng.random(n) < 0.01, np.inf, base),
        "with_neg_inf": np.where(rng.random(n) < 0.01, -np.inf, base),
        "subnormal": rng.random(n) * 5e-320,
        "dup_heavy": np.round(base * 3) / 3,
        "few_distinct": rng.integers(0, 5, n).astype(np.float64),
        "ties_at_edges": np.concatenate([np.zeros(n // 3), np.ones(n - n // 3)]),
    }
    return out


@pytest.mark.parametrize("n", [50, 3000, 9000, 120_000])
def test_patterns(pcf, n):
    rng = np.random.default_rng(n)
    for name, x in _patterns(n, rng).items():
        try:
            compare(pcf, np.ascontiguousarray(x, dtype=np.float64))
        except AssertionError as e:
            raise AssertionError(f"pattern {name}: {e}")


def test_u64_patterns(pcf):
    rng = np.random.default_rng(9)
    for x in [np.arange(100_000, dtype=np.uint64)[::-1].copy(),
              np.full(20_000, 7, dtype=np.uint64),
              (synth.generate("u64", 200_000, 1) >> np.uint64(40)).astype(np.uint64),
              np.array([0, 2 ** 64 - 1] * 5000, dtype=np.uint64),
              rng.integers(0, 3, 50_000).astype(np.uint64)]:
        compare(pcf, x)


def test_inplace(pcf):
    compare(pcf, synth.generate("lognormal", 500_000, 11), inplace=True)
    compare(pcf, synth.generate("uniform", 3000, 11), inplace=True)


@pytest.mark.parametrize("n", [10, 5000, 100_000])
def test_nan_is_error(pcf, n):
    x = synth.generate("uniform", n, 1)
    x[n // 2] = np.nan
    with pytest.raises(pcf.PCFError) as e:
        pcf.sort(torch.from_numpy(x).to(DEV))
    assert e.value.status == 2


def test_determinism(pcf):
    x = torch.from_numpy(synth.generate("lognormal", 1_000_000, 2)).to(DEV)
    outs = [pcf.sort(x, log=True) for _ in range(5)]
    for o, info in outs[1:]:
        assert torch.equal(o, outs[0][0])
        assert np.array_equal(np.sort(info.nodes, order=["level", "offset"]),
                              np.sort(outs[0][1].nodes, order=["level", "offset"]))


def test_host_entry(pcf):
    x = synth.generate("exponential", 200_000, 6)
    got = pcf.sort_host(x)
    assert np.array_equal(got.view(np.uint64), oracle.learned_sort(x).out.view(np.uint64))
    u = synth.generate("u64", 100_000, 6)
    assert np.array_equal(pcf.sort_host(u), np.sort(u))


def test_full_size_c2_exact(pcf):
    """configs[1] at its BASELINE.json size (1e7): full output and all node records."""
    compare(pcf, synth.config("c2"))


def test_full_size_c1_exact(pcf):
    compare(pcf, synth.config("c1"))


@pytest.mark.parametrize("name,n", [("c2", 2_000_000), ("c5f", 1_000_000), ("c3", 500_000)])
def test_split_scatter_exact_rank_path(pcf, name, n):
    """The split scatter's fallback (exact re-rank of every same-chunk, same-digit
    group by source index), forced on every tile: identical output and records."""
    compare(pcf, synth.config(name, n=n), exact_ranks=True)


def test_batched_global_nodes(pcf):
    """LogNormal at 2e7 keys: hundreds of level-1 buckets are too large for a K7 CTA and
    become global nodes fitted in one batch (k_minmax_batch / k_fit_sample_batch /
    k_fit_batch); output, every node record and level-1 b/H must still match."""
    _, info = compare(pcf, synth.config("c2", n=20_000_000))
    assert info.stats["global_nodes"] > 100


def test_batched_degenerate_and_sample_all_nodes(pcf):
    """Oversized recursing buckets that are degenerate (one repeated value: R9, the
    whole node goes to Standard-Sort) or fitted in SAMPLE_ALL mode, through the
    batched global-node path."""
    rng = np.random.default_rng(5)
    x = synth.generate("uniform", 3_000_000, 3)
    for v in (0.25, 0.5, 0.75):                  # 20 000 copies each: buckets > S_CAP, < delta
        idx = rng.choice(x.size, 20_000, replace=False)
        x[idx] = v
    _, info = compare(pcf, x)
    assert info.stats["global_nodes"] > 1
    compare(pcf, synth.config("c2", n=3_000_000), sample_all=True)


# ---------------------------------------------------------------- asynchronous calls
@pytest.mark.parametrize("name,n", [("c2", None), ("c4", 2_000_000), ("c2", 100_000_000)])
def test_async_no_host_sync(pcf, name, n):
    """Without PCF_FLAG_SYNC the call never waits for the GPU: the recursion over
    oversized buckets and the fallback sort are decided on the
    device.  c2 (one device batch), c4 (a ~10^8-key Standard-Sort bucket: radix splits)
    and LogNormal 1e8 (thousands of oversized recursing buckets, several device
    batches); output and the status word must match the synchronous call / oracle."""
    x = synth.config(name, n=n)
    xt = torch.from_numpy(x).to(DEV)
    status = torch.full((1,), -1, dtype=torch.int32, device=DEV)
    out, info = pcf.sort(xt, sync=False, stats=True, status=status)
    assert info.stats["host_syncs"] == 0
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    if n is None or n <= 2_000_000:
        ref = oracle.learned_sort(x, check=False).out
        assert np.array_equal(out.cpu().numpy().view(np.uint64), ref.view(np.uint64))
    else:
        s = xt.view(torch.int64)
        key = s ^ ((s >> 63) & 0x7FFFFFFFFFFFFFFF)
        o = out.view(torch.int64)
        assert torch.equal(o ^ ((o >> 63) & 0x7FFFFFFFFFFFFFFF), torch.sort(key).values)
    _, sinfo = pcf.sort(xt, stats=True)
    assert sinfo.stats["host_syncs"] == 1
    if name == "c2" and n is not None:
        assert sinfo.stats["device_batches"] >= 1 and sinfo.stats["global_nodes"] > 100


@pytest.mark.parametrize("n", [5000, 100_000, 3_000_000])
def test_async_nan_status(pcf, n):
    """NaN input without SYNC: PCF_OK returned after enqueueing, PCF_ERR_NAN (2) in the status word."""
    x = synth.generate("uniform", n, 1)
    x[n // 3] = np.nan
    status = torch.full((1,), -1, dtype=torch.int32, device=DEV)
    out, info = pcf.sort(torch.from_numpy(x).to(DEV), sync=False, stats=True, status=status)
    assert info.stats["host_syncs"] == 0
    torch.cuda.synchronize()
    assert int(status.item()) == 2


def test_host_entry_nan(pcf):
    x = synth.generate("exponential", 300_000, 6)
    x[7] = np.nan
    with pytest.raises(pcf.PCFError) as e:
        pcf.sort_host(x)
    assert e.value.status == 2


def test_repeated_calls_reuse_graphs(pcf):
    """The device-driven tail is a cached CUDA graph keyed on the workspace: repeated
    sorts with one workspace, then a different workspace, then the first again."""
    xs = [synth.generate("lognormal", 3_000_000, s) for s in (1, 2)]
    ws = [torch.empty(pcf.workspace_bytes(3_000_000), dtype=torch.uint8, device=DEV) for _ in range(2)]
    for k in (0, 1, 0, 0, 1):
        x = xs[k % 2]
        out = pcf.sort(torch.from_numpy(x).to(DEV), workspace=ws[k])
        assert np.array_equal(out.cpu().numpy().view(np.uint64), oracle.learned_sort(x, check=False).out.view(np.uint64))


# ---------------------------------------------------------------- reading R6 at bin edges
def test_r6_bin_edges_gpu(pcf):
    """Keys within a few ulps of PCF bin edges (tests/golden/r6_bin_edges.json, derived in
    exact rationals by tools/find_r6_cases.py): with the whole segment as the sample
    (R14 test mode) the level-1 b[] counts every key's i(x), so b must equal the counts of
    the R6 values -- and differs from the counts of the exact-rational values.  m = 1000
    runs in K7 (one CTA), m = 20000 on the global path (min/max, fit, split kernels)."""
    import json
    import os
    from fractions import Fraction
    from test_oracle_pins import r6_by_rationals
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "r6_bin_edges.json")))
    rng = np.random.default_rng(7)
    for grp in g["groups"]:
        m, beta = grp["m"], grp["beta"]
        lo, hi = float.fromhex(grp["lo"]), float.fromhex(grp["hi"])
        cases = [float.fromhex(c["x"]) for c in grp["cases"]]
        ks = rng.integers(0, beta, m - 2 - len(cases))
        filler = [(Fraction(lo) + (Fraction(hi) - Fraction(lo)) * (2 * int(k) + 1) / (2 * beta)) for k in ks]
        filler = [f.numerator / f.denominator for f in filler]   # bin centres: far from every edge
        x = np.array([lo, hi] + cases + filler, dtype=np.float64)
        rng.shuffle(x)
        i6 = np.array([r6_by_rationals(float(v), lo, hi, beta) for v in x])
        iex = np.array([int((Fraction(float(v)) - Fraction(lo)) / (Fraction(hi) - Fraction(lo)) * beta // 1) + 1
                        for v in x])
        b_r6 = np.cumsum(np.bincount(i6, minlength=beta + 2)[1:]).astype(np.uint32)
        b_ex = np.cumsum(np.bincount(iex, minlength=beta + 2)[1:]).astype(np.uint32)
        assert not np.array_equal(b_r6, b_ex)
        _, info = compare(pcf, x, sample_all=True)
        assert np.array_equal(info.level1_b[: beta + 1], b_r6), f"m={m}: GPU i(x) differs from reading R6"


def _cluster_input(n0, k1, k2, seed, embedded):
    """Uniform keys plus a cluster of k1 + k2 keys whose k2 keys sit in one tiny interval:
    the node holding the cluster (the root when not embedded, else one level-2 node)
    has a recursing bucket of ~k2 keys, larger than one warp's
    register capacity in the 1024-thread K7 build."""
    r = np.random.default_rng(seed)
    if embedded:
        beta = oracle.iroot34(n0 + k1 + k2)
        parts = [r.random(n0), 0.25 + r.random(k1) * (0.5 / beta), 0.25 + 1e-5 + r.random(k2) * 1e-15]
    else:
        parts = [r.random(n0), 0.5 + r.random(k2) * 1e-9]
    x = np.concatenate(parts)
    r.shuffle(x)
    return x


@pytest.mark.parametrize("n0,k1,k2,embedded", [(1720, 0, 280, False), (3580, 0, 420, False), (2650, 0, 350, False),
                                                (200_000, 2500, 300, True), (200_000, 1900, 250, True),
                                                (200_000, 3500, 350, True)])
def test_team_children_over_warp_capacity(pcf, n0, k1, k2, embedded):
    """Nodes run by multi-warp groups whose recursing children exceed one warp's keys."""
    x = _cluster_input(n0, k1, k2, 3, embedded)
    ref, _ = compare(pcf, x)
    nd = ref.nodes
    assert ((nd["level"] >= 2) & (nd["m"] > 256)).any()
