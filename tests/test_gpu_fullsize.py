"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

* c3, c4 (10^8 keys): the whole output and every node record against the oracle.
* c5f, c5u (10^9 keys): the oracle's level-1 bucketing of the full array (its seeded
  sample, b[1..beta+1] and H[1..gamma+1]) against the GPU's
  level-1 dumps and node record; the whole output against an independent library
  sort of the same keys on the device (the sorted permutation is unique under
  totalOrder, so equality there is the plain definition of the result).
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
    x = synth.config(name)
    n = len(x)
    dev = "cuda:0"
    xt = torch.from_numpy(x).to(dev)
    out, info = pcf.sort(xt, log=True, node_capacity=8_000_000)
    torch.cuda.synchronize()
    # (1) output == library sort of the same keys (unique under totalOrder)
    ref = torch.sort(_total_order_i64(xt)).values
    assert torch.equal(_total_order_i64(out), ref), "sorted output differs from the library sort"
    del ref
    got_b = info.level1_b
    got_h = info.level1_h
    rec = info.nodes[(info.nodes["level"] == 1)]
    del out, xt
    torch.cuda.empty_cache()
    # (2) level-1 bucketing node vs the oracle, on the full array
    P = oracle.iroot34(n)
    pos = oracle.sample_positions(0, 1, 0, n, P).astype(np.int64)
    sample = x[pos]
    b, H, _, _ = oracle.bucketing(x, sample, P, P)
    assert np.array_equal(got_b[: P + 1], b), "level-1 b differs"
    assert np.array_equal(got_h[: P + 1], H), "level-1 H differs"
    assert len(rec) == 1
    r = rec[0]
    bits = x.view(np.uint64)
    if x.dtype == np.float64:
        okey = bits ^ np.where(bits >> np.uint64(63), np.uint64(0xFFFFFFFFFFFFFFFF), np.uint64(1 << 63))
    else:
        okey = bits
    assert int(r["xmin_bits"]) == int(bits[np.argmin(okey)]) and int(r["xmax_bits"]) == int(bits[np.argmax(okey)])
    assert int(r["m"]) == n and int(r["alpha"]) == P
    assert int(r["digest_b"]) == oracle.digest(b) and int(r["digest_h"]) == oracle.digest(H)
