"""the sharded sort.

GPU (-m gpu): R = 1..4 ranks as threads of one process on one GPU (LoopbackComm,
each rank on its own stream, host-side exchanges: no rank's kernel waits on
another's), shards of uneven sizes; the concatenation of the ranks' slices must be
the oracle's output and the union of their node records the oracle's records.
CPU (-m "not gpu"): the TorchComm adapter's collectives (the ones the driver uses
with NCCL) under gloo, world size 2.
"""
import os
import threading

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")


def run_sharded(pcf_sharded, x, R, cuts=None, log=True, **kw):
    n = len(x)
    if cuts is None:
        cuts = [n * r // R for r in range(R + 1)]
    hub = pcf_sharded.LoopbackHub(R)
    res = [None] * R
    err = [None] * R

    def rank_main(r):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                xt = torch.from_numpy(x[cuts[r]: cuts[r + 1]].copy()).cuda()
                out, info = pcf_sharded.sort_sharded(xt, pcf_sharded.LoopbackComm(hub, r), log=log, stream=s, **kw)
                s.synchronize()
                res[r] = (out.cpu().numpy(), info)
        except BaseException as e:   # noqa: BLE001 -- reported below
            err[r] = e
            hub.barrier.abort()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in err:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    return res


@pytest.fixture(scope="module")
def sharded():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2405_07122_b200 as m
    m.build()
    from paper_2405_07122_b200 import sharded as sh
    return sh


def check(sharded, x, R, cuts=None, **kw):
    ref = oracle.learned_sort(x, log=True, check=False, **{k: v for k, v in kw.items() if k in ("tau", "seed")})
    res = run_sharded(sharded, x, R, cuts, **kw)
    off = 0
    for r, (out, info) in enumerate(res):
        assert info.offset == off, f"rank {r} offset {info.offset} != {off}"
        off += len(out)
    got = np.concatenate([o for o, _ in res])
    assert np.array_equal(got.view(np.uint64), ref.out.view(np.uint64)), "sharded output differs from the oracle"
    nodes = np.concatenate([i.nodes for _, i in res])
    a = oracle.sort_nodes(ref.nodes)
    b = np.sort(nodes, order=["level", "offset"])
    assert len(a) == len(b), f"node count {len(b)} != oracle {len(a)}"
    for f in a.dtype.names:
        if not np.array_equal(a[f], b[f]):
            bad = np.nonzero(a[f] != b[f])[0][:5]
            raise AssertionError(f"node field {f} differs at {bad}: shards {b[bad]} oracle {a[bad]}")
    if len(ref.l1_b):
        i0 = res[0][1]
        assert np.array_equal(i0.level1_b[: len(ref.l1_b)], ref.l1_b)
        assert np.array_equal(i0.level1_h[: len(ref.l1_h)], ref.l1_h)


@pytest.mark.gpu
@pytest.mark.parametrize("R", [1, 2, 3, 4])
@pytest.mark.parametrize("name,n", [("c1", 1_000_000), ("c2", 2_000_000), ("c5u", 1_000_000)])
def test_sharded_configs(sharded, R, name, n):
    check(sharded, synth.config(name, n=n), R)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c3", "c4"])
def test_sharded_fallback_paths(sharded, name):
    check(sharded, synth.config(name, n=3_000_000), 3)


@pytest.mark.gpu
def test_sharded_uneven_and_empty_shards(sharded):
    x = synth.generate("lognormal", 1_500_000, 9)
    check(sharded, x, 4, cuts=[0, 10, 700_000, 700_000, len(x)])


@pytest.mark.gpu
def test_sharded_degenerate_and_skewed(sharded):
    check(sharded, np.full(200_000, 2.5), 2)
    rng = np.random.default_rng(1)
    x = synth.generate("uniform", 2_000_000, 4)
    x[rng.random(len(x)) < 0.3] = 0.125          # one bucket with 30 % of the keys
    check(sharded, x, 4)


@pytest.mark.gpu
def test_sharded_nan(sharded):
    import paper_2405_07122_b200 as pcf
    x = synth.generate("uniform", 300_000, 2)
    x[123_456] = np.nan
    with pytest.raises(pcf.PCFError) as e:
        run_sharded(sharded, x, 2)
    assert e.value.status == 2


# ---------------------------------------------------------------- CPU: the NCCL adapter's semantics under gloo
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _comm_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2405_07122_b200.sharded import TorchComm
    c = TorchComm()
    t = torch.tensor([10 - rank, -5 + rank, rank], dtype=torch.int64)
    c.allreduce(t[0:1], "min"); c.allreduce(t[1:2], "max"); c.allreduce(t[2:3], "max")
    u = torch.from_numpy(np.array([2 ** 31 - 1 + rank, 7], dtype=np.uint32).view(np.int32))   # u32 counts as int32
    c.allreduce(u, "sum")
    g = torch.empty(2 * world, dtype=torch.int32)
    c.allgather_into(g, torch.tensor([rank, 100 + rank], dtype=torch.int32))
    sizes = c.sizes(3 + rank, "cpu")
    send = [1, 2] if rank == 0 else [3, 0]                           # rank r sends send[q] keys to q
    inp = torch.arange(sum(send), dtype=torch.int64) + 1000 * rank
    recv = [1, 3] if rank == 0 else [2, 0]
    out = torch.empty(sum(recv), dtype=torch.int64)
    c.alltoall(out, inp, recv, send)
    q.put((rank, t.tolist(), u.tolist(), g.tolist(), sizes, out.tolist()))
    dist.destroy_process_group()


def test_torchcomm_gloo_world2():
    import multiprocessing as mp
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    ps = [ctx.Process(target=_comm_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    got = dict()
    for _ in ps:
        r, *v = q.get()
        got[r] = v
    for r in (0, 1):
        t, u, g, sizes, out = got[r]
        assert t == [9, -4, 1]
        assert np.array(u, dtype=np.int32).view(np.uint32).tolist() == [(2 * (2 ** 31 - 1) + 1) % 2 ** 32, 14]
        assert g == [0, 100, 1, 101] and sizes == [3, 4]
    assert got[0][4] == [0, 1000, 1001, 1002] and got[1][4] == [1, 2]


@pytest.mark.gpu
def test_sharded_nccl_world1(sharded):
    """The production communicator (TorchComm over NCCL) in a world of one GPU: the
    collectives the driver issues run through NCCL on device tensors."""
    import socket
    import torch.distributed as dist
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        x = synth.config("c2", n=1_000_000)
        out, info = sharded.sort_sharded(torch.from_numpy(x).cuda(), sharded.TorchComm(), log=True)
        ref = oracle.learned_sort(x, log=True, check=False)
        assert info.offset == 0
        assert np.array_equal(out.cpu().numpy().view(np.uint64), ref.out.view(np.uint64))
        a, b = oracle.sort_nodes(ref.nodes), np.sort(info.nodes, order=["level", "offset"])
        assert len(a) == len(b) and all(np.array_equal(a[f], b[f]) for f in a.dtype.names)
    finally:
        dist.destroy_process_group()
