"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

* c3, c4 (10^8 keys): the whole output and every node record against the oracle.
* c5f, c5u (10^9 keys): the whole output, every node record of every level and the
  level-1 b[1..beta+1] / H[1..gamma+1] dumps against the oracle run on the full
  array; the output also against an independent library sort on the device.
* F4: Normal / Exponential / LogNormal / Uniform at 10^8 keys (the large end of
  the n-sweep), output and node records against the oracle.
"""
import numpy as np
import pytest

import oracle
import synth
from test_gpu_parity import compare

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


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_full_size_exact(pcf, name):
    compare(pcf, synth.config(name))


def _total_order_i64(t):
    """int64 keys whose signed order is totalOrder (f64) / unsigned order (u64)."""
    s = t.view(torch.int64)
    if t.dtype == torch.float64:
        return s ^ ((s >> 63) & 0x7FFFFFFFFFFFFFFF)
    return s ^ torch.tensor(-(1 << 63), dtype=torch.int64, device=t.device)


@pytest.mark.parametrize("name", ["c5f", "c5u"])
def test_full_size_1e9(pcf, name):
    """c5f / c5u at 10^9 keys in bench.py's launch configuration: the whole output, every
    node record (all levels: ~1.5 M bucketing nodes) and the level-1 b/H arrays against
    the oracle run on the full array (Alg. 1)."""
    x = synth.config(name)
    n = len(x)
    dev = "cuda:0"
    xt = torch.from_numpy(x).to(dev)
    out, info = pcf.sort(xt, log=True, node_capacity=8_000_000)
    torch.cuda.synchronize()
    # (1) output == an independent library sort of the same keys (unique under totalOrder)
    ref = torch.sort(_total_order_i64(xt)).values
    assert torch.equal(_total_order_i64(out), ref), "sorted output differs from the library sort"
    del ref
    got = out.cpu().numpy()
    got_b, got_h, got_nodes = info.level1_b, info.level1_h, info.nodes
    del out, xt, info
    torch.cuda.empty_cache()
    # (2) the oracle on the full array: output, every node record, level-1 b and H
    res = oracle.learned_sort(x, log=True, check=False, node_cap=8_000_000)
    assert np.array_equal(got.view(np.uint64), res.out.view(np.uint64)), "output differs from the oracle"
    del got
    a = oracle.sort_nodes(res.nodes)
    b = np.sort(got_nodes, order=["level", "offset"])
    assert len(a) == len(b), f"node count {len(b)} != oracle {len(a)}"
    for f in a.dtype.names:
        if not np.array_equal(a[f], b[f]):
            bad = np.nonzero(a[f] != b[f])[0][:5]
            raise AssertionError(f"node field {f} differs at {bad}: gpu {b[bad]} oracle {a[bad]}")
    P = oracle.iroot34(n)
    assert np.array_equal(got_b[: P + 1], res.l1_b), "level-1 b differs"
    assert np.array_equal(got_h[: P + 1], res.l1_h), "level-1 H differs"
    assert len(a) > 100_000 and a["level"].max() >= 2


@pytest.mark.parametrize("dist", ["normal", "exponential", "lognormal", "uniform"])
def test_nsweep_scale_parity(pcf, dist):
    """SURVEY.md 8(f) F4 (the Fig. 2 n-sweep) at its large end: the
    sweep's distributions at 10^8 keys, output and every node record vs the oracle."""
    compare(pcf, synth.generate(dist, 100_000_000, 7))
