"""CPU oracle for PCF Learned Sort -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path (``paper_2405_07122_b200``) never imports it and shares no code
with it.  The arithmetic lives in ``pcf_oracle.c`` (plain single-threaded C,
compiled with ``-O2 -ffp-contract=off``); this module is ctypes marshalling.

Pins (``tests/test_oracle_pins.py``): SPEC.md worked examples, closed forms
for floor(n^{3/4}), brute force over every tiny array, std-library sort of the
same bits, the paper's invariants.  ``sample_positions`` is "parity unpinned"
by the paper (its sampler is unspecified); it is pinned only by
the published SplitMix64 output vector (for ``mix64``) and statistical checks.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pcf_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

KEY_F64 = 0
KEY_U64 = 1
FLAG_SAMPLE_ALL = 2

OK, ERR_INVALID_ARG, ERR_NAN, ERR_OOM, ERR_INVARIANT = 0, 1, 2, 4, 8


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, -O2 -ffp-contract=off, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class Node(ctypes.Structure):
    _fields_ = [("level", ctypes.c_uint32), ("alpha", ctypes.c_uint32),
                ("offset", ctypes.c_uint64), ("m", ctypes.c_uint64),
                ("xmin_bits", ctypes.c_uint64), ("xmax_bits", ctypes.c_uint64),
                ("digest_b", ctypes.c_uint64), ("digest_h", ctypes.c_uint64),
                ("n_fallback", ctypes.c_uint32), ("n_small", ctypes.c_uint32),
                ("n_recurse", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


assert ctypes.sizeof(Node) == 72

NODE_DTYPE = np.dtype([("level", "<u4"), ("alpha", "<u4"), ("offset", "<u8"), ("m", "<u8"),
                       ("xmin_bits", "<u8"), ("xmax_bits", "<u8"), ("digest_b", "<u8"),
                       ("digest_h", "<u8"), ("n_fallback", "<u4"), ("n_small", "<u4"),
                       ("n_recurse", "<u4"), ("reserved", "<u4")])


class Ctx(ctypes.Structure):
    _fields_ = [("tau", ctypes.c_uint32), ("flags", ctypes.c_uint32), ("seed", ctypes.c_uint64),
                ("check", ctypes.c_int), ("violation", ctypes.c_int),
                ("nodes", ctypes.c_void_p), ("nodes_cap", ctypes.c_uint64),
                ("nodes_count", ctypes.c_uint64),
                ("l1_b", ctypes.c_void_p), ("l1_h", ctypes.c_void_p),
                ("l1_cap", ctypes.c_uint64), ("l1_b_len", ctypes.c_uint64),
                ("l1_h_len", ctypes.c_uint64),
                ("max_depth", ctypes.c_uint32),
                ("base_case_calls", ctypes.c_uint64), ("fallback_buckets", ctypes.c_uint64),
                ("fallback_keys", ctypes.c_uint64), ("degenerate_calls", ctypes.c_uint64),
                ("bucketing_calls", ctypes.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        u64, u32, i32, dbl, vp = (ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int,
                                  ctypes.c_double, ctypes.c_void_p)
        L.orc_iroot34.argtypes = [u64]; L.orc_iroot34.restype = u64
        L.orc_interval_index_f64.argtypes = [dbl, dbl, dbl, u64]; L.orc_interval_index_f64.restype = u64
        L.orc_interval_index_u64.argtypes = [u64, u64, u64, u64]; L.orc_interval_index_u64.restype = u64
        L.orc_mix64.argtypes = [u64]; L.orc_mix64.restype = u64
        L.orc_sample_position.argtypes = [u64, u32, u64, u64, u64]; L.orc_sample_position.restype = u64
        L.orc_sample_positions.argtypes = [u64, u32, u64, u64, u64, vp]; L.orc_sample_positions.restype = None
        L.orc_digest.argtypes = [vp, u64]; L.orc_digest.restype = u64
        L.orc_train_pcf.argtypes = [i32, vp, u64, u64, u64, u64, vp]; L.orc_train_pcf.restype = i32
        L.orc_bucket_of.argtypes = [u64, u64, u64]; L.orc_bucket_of.restype = u64
        L.orc_infer_cdf.argtypes = [i32, vp, u64, u64, u64, u64, u64]; L.orc_infer_cdf.restype = dbl
        L.orc_bucketing.argtypes = [i32, vp, u64, vp, u64, u64, u64, u64, u64, vp, vp, vp, vp]
        L.orc_bucketing.restype = i32
        L.orc_standard_sort.argtypes = [vp, u64, i32]; L.orc_standard_sort.restype = None
        L.orc_learned_sort.argtypes = [i32, vp, u64, ctypes.POINTER(Ctx)]; L.orc_learned_sort.restype = i32
        L.orc_depth_bound.argtypes = [u64, u32]; L.orc_depth_bound.restype = u32
        L.orc_stable_argsort.argtypes = [i32, vp, u64, vp]; L.orc_stable_argsort.restype = i32
        _lib = L
    return _lib


def _bits(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x)
    if x.dtype == np.float64:
        return x.view(np.uint64).copy()
    if x.dtype == np.uint64:
        return x.copy()
    raise TypeError(f"keys must be float64 or uint64, got {x.dtype}")


def _kt(x: np.ndarray) -> int:
    return KEY_F64 if x.dtype == np.float64 else KEY_U64


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _key_bits(v, kt):
    if kt == KEY_F64:
        return int(np.array([v], dtype=np.float64).view(np.uint64)[0])
    return int(v)


# ---- small functions (for pins) -------------------------------------------------------------

def iroot34(m: int) -> int:
    return int(lib().orc_iroot34(m))


def interval_index(x: float, xmin: float, xmax: float, beta: int) -> int:
    """i(x) for float64 keys (reading R6)."""
    return int(lib().orc_interval_index_f64(float(x), float(xmin), float(xmax), beta))


def interval_index_u64(x: int, xmin: int, xmax: int, beta: int) -> int:
    return int(lib().orc_interval_index_u64(x, xmin, xmax, beta))


def mix64(z: int) -> int:
    return int(lib().orc_mix64(z & 0xFFFFFFFFFFFFFFFF))


def sample_positions(seed: int, level: int, offset: int, m: int, alpha: int) -> np.ndarray:
    out = np.empty(alpha, dtype=np.uint64)
    lib().orc_sample_positions(seed, level, offset, m, alpha, _ptr(out))
    return out


def digest(v: np.ndarray) -> int:
    v = np.ascontiguousarray(v, dtype=np.uint32)
    return int(lib().orc_digest(_ptr(v), len(v)))


def train_pcf(sample: np.ndarray, xmin, xmax, beta: int) -> np.ndarray:
    """b[1..beta+1], returned 0-based."""
    kt = _kt(sample)
    a = _bits(sample)
    b = np.zeros(beta + 1, dtype=np.uint32)
    rc = lib().orc_train_pcf(kt, _ptr(a), len(a), _key_bits(xmin, kt), _key_bits(xmax, kt), beta, _ptr(b))
    if rc:
        raise RuntimeError(f"train_pcf invariant failed rc={rc}")
    return b


def infer_cdf(b: np.ndarray, alpha: int, x, xmin, xmax, beta: int, kt: int = KEY_F64) -> float:
    b = np.ascontiguousarray(b, dtype=np.uint32)
    return float(lib().orc_infer_cdf(kt, _ptr(b), alpha, _key_bits(x, kt), _key_bits(xmin, kt),
                                     _key_bits(xmax, kt), beta))


def bucket_of(b_i: int, alpha: int, gamma: int) -> int:
    return int(lib().orc_bucket_of(b_i, alpha, gamma))


def bucketing(x: np.ndarray, sample: np.ndarray, beta: int, gamma: int):
    """One M_PCF step with an explicit sample.  Returns (b, H, bucket_ids, out)."""
    kt = _kt(x)
    seg = _bits(x)
    a = _bits(sample)
    m = len(seg)
    if kt == KEY_F64:
        mn, mx = float(np.min(x)), float(np.max(x))
    else:
        mn, mx = int(np.min(x)), int(np.max(x))
    b = np.zeros(beta + 1, dtype=np.uint32)
    H = np.zeros(gamma + 1, dtype=np.uint32)
    bid = np.zeros(m, dtype=np.uint32)
    out = np.zeros(m, dtype=np.uint64)
    rc = lib().orc_bucketing(kt, _ptr(seg), m, _ptr(a), len(a), beta, gamma, _key_bits(mn, kt),
                             _key_bits(mx, kt), _ptr(b), _ptr(H), _ptr(bid), _ptr(out))
    if rc:
        raise RuntimeError(f"bucketing rc={rc}")
    return b, H, bid, out.view(x.dtype)


def standard_sort(x: np.ndarray) -> np.ndarray:
    kt = _kt(x)
    a = _bits(x)
    lib().orc_standard_sort(_ptr(a), len(a), kt)
    return a.view(x.dtype)


def stable_argsort(x: np.ndarray) -> np.ndarray:
    """the stable sorting permutation of x (ascending, totalOrder
    for float64; equal keys in increasing index order), as uint64 indices."""
    kt = _kt(x)
    a = _bits(x)
    perm = np.empty(len(a), dtype=np.uint64)
    rc = lib().orc_stable_argsort(kt, _ptr(a), len(a), _ptr(perm))
    if rc:
        raise OracleError(rc)
    return perm


def depth_bound(n: int, tau: int = 64) -> int:
    return int(lib().orc_depth_bound(n, tau))


class SortResult:
    def __init__(self, out, nodes, l1_b, l1_h, ctx):
        self.out = out
        self.nodes = nodes
        self.l1_b = l1_b
        self.l1_h = l1_h
        self.max_depth = ctx.max_depth
        self.base_case_calls = ctx.base_case_calls
        self.fallback_buckets = ctx.fallback_buckets
        self.fallback_keys = ctx.fallback_keys
        self.degenerate_calls = ctx.degenerate_calls
        self.bucketing_calls = ctx.bucketing_calls


class OracleError(RuntimeError):
    def __init__(self, rc):
        super().__init__(f"oracle learned_sort failed rc={rc}")
        self.rc = rc


def learned_sort(x: np.ndarray, tau: int = 64, seed: int = 0, flags: int = 0, log: bool = False,
                 check: bool = True, node_cap: int | None = None) -> SortResult:
    """PCF Learned Sort (Alg. 1) of a float64/uint64 array; returns a SortResult."""
    kt = _kt(x)
    a = _bits(x)
    n = len(a)
    ctx = Ctx()
    ctx.tau, ctx.flags, ctx.seed, ctx.check = tau, flags, seed, 1 if check else 0
    nodes = l1b = l1h = None
    if log:
        # every node has >= tau keys and nodes of one level are disjoint; <= ~12 levels
        cap = node_cap if node_cap is not None else min(n, 12 * (n // max(tau, 1))) + 16
        nodes = np.zeros(cap, dtype=NODE_DTYPE)
        ctx.nodes, ctx.nodes_cap = nodes.ctypes.data, cap
        l1cap = iroot34(n) + 2 if n else 2
        l1b = np.zeros(l1cap, dtype=np.uint32)
        l1h = np.zeros(l1cap, dtype=np.uint32)
        ctx.l1_b, ctx.l1_h, ctx.l1_cap = l1b.ctypes.data, l1h.ctypes.data, l1cap
    rc = lib().orc_learned_sort(kt, _ptr(a), n, ctypes.byref(ctx))
    if rc:
        raise OracleError(rc)
    if log:
        if ctx.nodes_count > ctx.nodes_cap:
            raise RuntimeError("oracle node log overflow")
        nodes = nodes[: ctx.nodes_count]
        l1b = l1b[: ctx.l1_b_len]
        l1h = l1h[: ctx.l1_h_len]
    return SortResult(a.view(x.dtype), nodes, l1b, l1h, ctx)


def sort_nodes(nodes: np.ndarray) -> np.ndarray:
    """Node records in canonical (level, offset) order."""
    return np.sort(nodes, order=["level", "offset"])
