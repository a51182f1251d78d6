"""paper_2405_07122_b200 -- B200-native PCF Learned Sort (arXiv 2405.07122).

Thin ctypes binding over ``libpcfsort.so`` (C ABI in ``include/pcf_sort.h``).
Argument marshalling only: every step of the sort runs in the library's CUDA
kernels.  PyTorch is used for device memory and streams.  There is no CPU
fallback: if the extension is missing or no GPU is present, calls raise.
"""
from __future__ import annotations

import ctypes
import os

from ._build import LIB_PATH, build  # noqa: F401

__all__ = ["build", "lib", "sort", "argsort", "sort_pairs", "bucket_counts", "sort_host", "workspace_bytes", "host_workspace_bytes", "PCFError", "KEY_F64", "KEY_U64",
           "FLAG_SYNC", "FLAG_SAMPLE_ALL", "FLAG_TIMING", "PHASES"]

KEY_F64, KEY_U64 = 0, 1
KEY_ARGSORT, KEY_PAIRS = 0x10, 0x20   # or'ed into key_type for workspace_bytes
FLAG_SYNC, FLAG_SAMPLE_ALL, FLAG_TIMING, FLAG_PROFILE, FLAG_EXACT_RANKS = 1, 2, 4, 8, 16
PHASES = ["minmax", "fit", "classify_hist", "scatter", "smem_subtree", "log_records", "other", "total",
          "deep_batches"]
NPHASES = len(PHASES)
STATUS = {0: "PCF_OK", 1: "PCF_ERR_INVALID_ARG", 2: "PCF_ERR_NAN", 3: "PCF_ERR_WORKSPACE_TOO_SMALL",
          4: "PCF_ERR_OOM", 5: "PCF_ERR_CUDA", 6: "PCF_ERR_LOG_OVERFLOW", 7: "PCF_ERR_INTERNAL",
          8: "PCF_ERR_DEGENERATE"}


class NodeRecord(ctypes.Structure):
    _fields_ = [("level", ctypes.c_uint32), ("alpha", ctypes.c_uint32),
                ("offset", ctypes.c_uint64), ("m", ctypes.c_uint64),
                ("xmin_bits", ctypes.c_uint64), ("xmax_bits", ctypes.c_uint64),
                ("digest_b", ctypes.c_uint64), ("digest_h", ctypes.c_uint64),
                ("n_fallback", ctypes.c_uint32), ("n_small", ctypes.c_uint32),
                ("n_recurse", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


class PassLog(ctypes.Structure):
    _fields_ = [("records", ctypes.c_void_p), ("capacity", ctypes.c_uint64),
                ("count", ctypes.c_void_p), ("level1_b", ctypes.c_void_p),
                ("level1_h", ctypes.c_void_p), ("level1_capacity", ctypes.c_uint64)]


class Stats(ctypes.Structure):
    _fields_ = [("kernel_launches", ctypes.c_uint32), ("rounds", ctypes.c_uint32),
                ("host_syncs", ctypes.c_uint32), ("device_batches", ctypes.c_uint32),
                ("groups_smem", ctypes.c_uint64), ("split_keys_moved", ctypes.c_uint64),
                ("global_nodes", ctypes.c_uint64), ("fallback_keys_global", ctypes.c_uint64),
                ("phase_ms", ctypes.c_float * NPHASES), ("phase_bytes", ctypes.c_uint64 * NPHASES),
                ("k7_cycles", ctypes.c_uint64 * 24)]

    def as_dict(self):
        return {"kernel_launches": self.kernel_launches, "rounds": self.rounds,
                "host_syncs": self.host_syncs, "device_batches": self.device_batches,
                "groups_smem": self.groups_smem,
                "split_keys_moved": self.split_keys_moved, "global_nodes": self.global_nodes,
                "fallback_keys_global": self.fallback_keys_global,
                "phase_ms": {PHASES[i]: float(self.phase_ms[i]) for i in range(NPHASES)},
                "phase_bytes": {PHASES[i]: int(self.phase_bytes[i]) for i in range(NPHASES)},
                "k7_cycles": [int(v) for v in self.k7_cycles]}


class Params(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("tau", ctypes.c_uint32),
                ("seed", ctypes.c_uint64), ("flags", ctypes.c_uint32), ("reserved0", ctypes.c_uint32),
                ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t),
                ("log", ctypes.POINTER(PassLog)), ("stats", ctypes.POINTER(Stats)),
                ("status_out", ctypes.c_void_p)]


class PCFError(RuntimeError):
    def __init__(self, status: int, detail: str = ""):
        super().__init__(f"{STATUS.get(status, status)}: {detail}")
        self.status = status


_lib = None
SYMBOLS = ["pcf_params_init", "pcf_workspace_bytes", "pcf_sort_f64", "pcf_sort_u64", "pcf_sort_f64_host",
           "pcf_sort_u64_host", "pcf_status_string", "pcf_last_error", "pcf_abi_version",
           "pcf_bucket_counts_f64", "pcf_level1_entries", "pcf_argsort_f64", "pcf_argsort_u64",
           "pcf_sort_pairs_f64_u32", "pcf_sort_pairs_f64_u64", "pcf_sort_pairs_u64_u32", "pcf_sort_pairs_u64_u64",
           "pcf_shard_state_bytes", "pcf_shard_workspace_bytes", "pcf_shard_views", "pcf_shard_minmax",
           "pcf_shard_counts", "pcf_shard_histogram", "pcf_shard_partition", "pcf_shard_sort_range"]


def lib():
    """Load libpcfsort.so (built in-tree by ``build()``); raise if it is missing."""
    global _lib
    if _lib is None:
        path = os.environ.get("PCF_LIB", LIB_PATH)   # PCF_LIB: an alternative build (tuning experiments)
        if not os.path.exists(path):
            raise RuntimeError(f"{path} not built: run __graft_entry__.build() "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(path)
        vp, sz, i32, u32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint32
        PP = ctypes.POINTER(Params)
        L.pcf_params_init.argtypes = [PP]; L.pcf_params_init.restype = None
        L.pcf_workspace_bytes.argtypes = [sz, i32, PP]; L.pcf_workspace_bytes.restype = sz
        for name in ["pcf_sort_f64", "pcf_sort_u64", "pcf_sort_f64_host", "pcf_sort_u64_host"]:
            f = getattr(L, name)
            f.argtypes = [vp, vp, sz, PP, vp]
            f.restype = i32
        L.pcf_status_string.argtypes = [i32]; L.pcf_status_string.restype = ctypes.c_char_p
        L.pcf_last_error.argtypes = []; L.pcf_last_error.restype = ctypes.c_char_p
        L.pcf_abi_version.argtypes = []; L.pcf_abi_version.restype = i32
        u64 = ctypes.c_uint64
        L.pcf_bucket_counts_f64.argtypes = [vp, sz, u64, u64, u64, u64, vp, vp, ctypes.POINTER(u64), vp]
        L.pcf_bucket_counts_f64.restype = i32
        L.pcf_level1_entries.argtypes = [sz, PP]; L.pcf_level1_entries.restype = sz
        for name in ["pcf_argsort_f64", "pcf_argsort_u64"]:
            f = getattr(L, name)
            f.argtypes = [vp, vp, vp, sz, PP, vp]
            f.restype = i32
        for name in ["pcf_sort_pairs_f64_u32", "pcf_sort_pairs_f64_u64", "pcf_sort_pairs_u64_u32", "pcf_sort_pairs_u64_u64",
           "pcf_shard_state_bytes", "pcf_shard_workspace_bytes", "pcf_shard_views", "pcf_shard_minmax",
           "pcf_shard_counts", "pcf_shard_histogram", "pcf_shard_partition", "pcf_shard_sort_range"]:
            f = getattr(L, name)
            f.argtypes = [vp, vp, vp, vp, sz, PP, vp]
            f.restype = i32
        _ = u32
        _lib = L
    return _lib


def _check_device_buffer(t, dtype, n, device, name):
    """The library writes n elements of `dtype` through t's pointer: refuse anything else."""
    import torch

    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if t.numel() != n:
        raise ValueError(f"{name} must have {n} elements, got {t.numel()}")
    if t.device != device:
        raise ValueError(f"{name} is on {t.device}, keys are on {device}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def _check_workspace(ws, device):
    import torch

    if not isinstance(ws, torch.Tensor) or not ws.is_cuda or ws.device != device or not ws.is_contiguous():
        raise ValueError(f"workspace must be a contiguous CUDA tensor on {device}")


def make_params(tau: int = 64, seed: int = 0, flags: int = FLAG_SYNC, workspace=None, workspace_bytes=0):
    p = Params()
    lib().pcf_params_init(ctypes.byref(p))
    p.tau, p.seed, p.flags = tau, seed, flags
    if workspace is not None:
        p.workspace, p.workspace_bytes = workspace, workspace_bytes
    return p


def workspace_bytes(n: int, key_type: int = KEY_F64) -> int:
    return int(lib().pcf_workspace_bytes(n, key_type, None))


def _check(rc: int):
    if rc != 0:
        raise PCFError(rc, lib().pcf_last_error().decode())


class SortInfo:
    """Pass log (node records, level-1 b/H) and statistics of one sort."""

    def __init__(self):
        self.nodes = None
        self.level1_b = None
        self.level1_h = None
        self.stats = None


def sort(x, out=None, *, tau: int = 64, seed: int = 0, sample_all: bool = False, log: bool = False,
         timing: bool = False, stats: bool = False, sync: bool = True, workspace=None, node_capacity=None,
         profile: bool = False, exact_ranks: bool = False, stream=None, status=None):
    """Sort a 1-D CUDA tensor of float64 or uint64 keys ascending (totalOrder for f64).

    Returns ``out`` (a new tensor unless given; ``out is x`` sorts in place), or
    ``(out, SortInfo)`` when ``log``/``timing``/``stats`` is requested.
    ``sync=False`` returns right after enqueueing (no host synchronisation); the
    call's status (0 = PCF_OK, 2 = PCF_ERR_NAN, ...) is then written, in stream
    order, to ``status`` (a 1-element CUDA int32 tensor) if given.
    """
    import torch

    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise TypeError("x must be a CUDA tensor (no CPU fallback)")
    if x.dtype == torch.float64:
        fn, kt = lib().pcf_sort_f64, KEY_F64
    elif x.dtype == torch.uint64:
        fn, kt = lib().pcf_sort_u64, KEY_U64
    else:
        raise TypeError(f"keys must be float64 or uint64, got {x.dtype}")
    if x.dim() != 1 or not x.is_contiguous():
        raise ValueError("x must be a contiguous 1-D tensor")
    n = x.numel()
    if out is None:
        out = torch.empty_like(x)
    _check_device_buffer(out, x.dtype, n, x.device, "out")
    if workspace is not None:
        _check_workspace(workspace, x.device)
    flags = (FLAG_SYNC if sync else 0) | (FLAG_SAMPLE_ALL if sample_all else 0) | (FLAG_TIMING if timing else 0) \
        | (FLAG_PROFILE if profile else 0) | (FLAG_EXACT_RANKS if exact_ranks else 0)
    p = make_params(tau, seed, flags)
    if workspace is not None:
        p.workspace, p.workspace_bytes = workspace.data_ptr(), workspace.numel() * workspace.element_size()
    if status is not None:
        _check_device_buffer(status, torch.int32, 1, x.device, "status")
        p.status_out = status.data_ptr()
    info = SortInfo() if (log or timing or stats or profile) else None
    keep = []
    if log:
        cap = node_capacity if node_capacity is not None else min(n, 12 * (n // max(tau, 1))) + 64
        recs = torch.zeros(cap * 9, dtype=torch.int64, device=x.device)   # 72-byte records
        cnt = torch.zeros(1, dtype=torch.int64, device=x.device)
        l1 = int(lib().pcf_level1_entries(n, ctypes.byref(p))) if n else 2   # the library sizes it
        b = torch.zeros(l1, dtype=torch.int32, device=x.device)
        h = torch.zeros(l1, dtype=torch.int32, device=x.device)
        pl = PassLog(recs.data_ptr(), cap, cnt.data_ptr(), b.data_ptr(), h.data_ptr(), l1)
        p.log = ctypes.pointer(pl)
        keep += [recs, cnt, b, h, pl]
    st = Stats()
    if info is not None:
        p.stats = ctypes.pointer(st)
    s = stream if stream is not None else torch.cuda.current_stream(x.device)
    with torch.cuda.device(x.device):
        rc = fn(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()), n, ctypes.byref(p),
                ctypes.c_void_p(s.cuda_stream))
    _check(rc)
    if info is None:
        return out
    info.stats = st.as_dict()
    if log:
        import numpy as np
        k = int(cnt.item())
        arr = recs.view(torch.uint8).cpu().numpy().view(np.uint8)[: k * 72]
        info.nodes = np.frombuffer(arr.tobytes(), dtype=NODE_DTYPE()).copy()
        info.level1_b = b.cpu().numpy().view(np.uint32)
        info.level1_h = h.cpu().numpy().view(np.uint32)
    return out, info


def argsort(x, out=None, perm=None, *, tau: int = 64, seed: int = 0, sync: bool = True, workspace=None,
            stream=None, status=None):
    """Key-value mode: sort 1-D CUDA float64/uint64 keys and return
    ``(out, perm)`` -- the sorted keys and the stable sorting permutation (uint32 CUDA
    tensor, perm[k] = input index of out[k]; equal keys keep their input order)."""
    import torch

    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise TypeError("x must be a CUDA tensor (no CPU fallback)")
    if x.dtype == torch.float64:
        fn = lib().pcf_argsort_f64
    elif x.dtype == torch.uint64:
        fn = lib().pcf_argsort_u64
    else:
        raise TypeError(f"keys must be float64 or uint64, got {x.dtype}")
    if x.dim() != 1 or not x.is_contiguous():
        raise ValueError("x must be a contiguous 1-D tensor")
    n = x.numel()
    if out is None:
        out = torch.empty_like(x)
    if perm is None:
        perm = torch.empty(n, dtype=torch.uint32, device=x.device)
    _check_device_buffer(out, x.dtype, n, x.device, "out")
    _check_device_buffer(perm, torch.uint32, n, x.device, "perm")
    p = make_params(tau, seed, FLAG_SYNC if sync else 0)
    if workspace is not None:
        _check_workspace(workspace, x.device)
        p.workspace, p.workspace_bytes = workspace.data_ptr(), workspace.numel() * workspace.element_size()
    if status is not None:
        _check_device_buffer(status, torch.int32, 1, x.device, "status")
        p.status_out = status.data_ptr()
    s = stream if stream is not None else torch.cuda.current_stream(x.device)
    with torch.cuda.device(x.device):
        rc = fn(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(perm.data_ptr()), n,
                ctypes.byref(p), ctypes.c_void_p(s.cuda_stream))
    _check(rc)
    return out, perm


def sort_pairs(keys, vals, keys_out=None, vals_out=None, *, tau: int = 64, seed: int = 0, sync: bool = True,
               workspace=None, stream=None):
    """Key-value mode: sort keys (CUDA float64/uint64) and move vals (CUDA uint32/uint64,
    same length) with them; equal keys keep their input order.  Returns (keys_out, vals_out)."""
    import torch

    if not isinstance(keys, torch.Tensor) or not keys.is_cuda or not isinstance(vals, torch.Tensor) or not vals.is_cuda:
        raise TypeError("keys and vals must be CUDA tensors (no CPU fallback)")
    kk = {torch.float64: "f64", torch.uint64: "u64"}.get(keys.dtype)
    vk = {torch.uint32: "u32", torch.uint64: "u64", torch.int32: "u32", torch.int64: "u64"}.get(vals.dtype)
    if kk is None or vk is None:
        raise TypeError(f"unsupported key/value dtypes {keys.dtype}/{vals.dtype}")
    if keys.dim() != 1 or vals.dim() != 1 or not keys.is_contiguous() or not vals.is_contiguous():
        raise ValueError("keys and vals must be contiguous 1-D tensors")
    n = keys.numel()
    if vals.numel() != n or vals.device != keys.device:
        raise ValueError("vals must have one value per key, on the keys' device")
    if keys_out is None:
        keys_out = torch.empty_like(keys)
    if vals_out is None:
        vals_out = torch.empty_like(vals)
    _check_device_buffer(keys_out, keys.dtype, n, keys.device, "keys_out")
    _check_device_buffer(vals_out, vals.dtype, n, keys.device, "vals_out")
    fn = getattr(lib(), f"pcf_sort_pairs_{kk}_{vk}")
    p = make_params(tau, seed, FLAG_SYNC if sync else 0)
    if workspace is not None:
        _check_workspace(workspace, keys.device)
        p.workspace, p.workspace_bytes = workspace.data_ptr(), workspace.numel() * workspace.element_size()
    s = stream if stream is not None else torch.cuda.current_stream(keys.device)
    with torch.cuda.device(keys.device):
        rc = fn(ctypes.c_void_p(keys.data_ptr()), ctypes.c_void_p(vals.data_ptr()), ctypes.c_void_p(keys_out.data_ptr()),
                ctypes.c_void_p(vals_out.data_ptr()), n, ctypes.byref(p), ctypes.c_void_p(s.cuda_stream))
    _check(rc)
    return keys_out, vals_out


def bucket_counts(x, alpha: int, beta: int, gamma: int, *, seed: int = 0, b=None, H=None, stream=None):
    """One M_PCF bucketing step with decoupled alpha, beta, gamma (the §4.3
    failure experiment) through ``pcf_bucket_counts_f64``.

    x: 1-D CUDA float64 tensor.  Returns ``(b, H, max_bucket)``: b[1..beta+1]
    and H = |c_1|..|c_{gamma+1}| as CUDA uint32 tensors (0-based), and
    max_j |c_j| (the experiment's failure is ``max_bucket > delta``).
    """
    import torch

    if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype != torch.float64:
        raise TypeError("x must be a CUDA float64 tensor (no CPU fallback)")
    x = x.contiguous()
    if b is None:
        b = torch.empty(beta + 1, dtype=torch.uint32, device=x.device)
    if H is None:
        H = torch.empty(gamma + 1, dtype=torch.uint32, device=x.device)
    _check_device_buffer(b, torch.uint32, beta + 1, x.device, "b")
    _check_device_buffer(H, torch.uint32, gamma + 1, x.device, "H")
    mx = ctypes.c_uint64(0)
    st = stream if stream is not None else torch.cuda.current_stream(x.device).cuda_stream
    _check(lib().pcf_bucket_counts_f64(x.data_ptr(), x.numel(), alpha, beta, gamma, seed & 0xFFFFFFFFFFFFFFFF,
                                       b.data_ptr(), H.data_ptr(), ctypes.byref(mx), st))
    return b, H, int(mx.value)


def NODE_DTYPE():
    import numpy as np
    return np.dtype([("level", "<u4"), ("alpha", "<u4"), ("offset", "<u8"), ("m", "<u8"),
                     ("xmin_bits", "<u8"), ("xmax_bits", "<u8"), ("digest_b", "<u8"),
                     ("digest_h", "<u8"), ("n_fallback", "<u4"), ("n_small", "<u4"),
                     ("n_recurse", "<u4"), ("reserved", "<u4")])


def host_workspace_bytes(n: int) -> int:
    """Device workspace that lets ``sort_host`` run without allocating: the n keys
    (rounded to 256 B) followed by ``workspace_bytes(n)``."""
    return ((8 * n + 255) // 256) * 256 + workspace_bytes(n)


def sort_host(x, out=None, *, tau: int = 64, seed: int = 0, workspace=None, stream=None):
    """End-to-end sort of HOST keys (numpy array or CPU tensor; pinned recommended)
    through ``pcf_sort_*_host``: H2D copy, device sort, D2H copy, synchronise.
    ``workspace`` (a CUDA tensor of >= host_workspace_bytes(n) bytes) avoids allocations."""
    import numpy as np
    import torch

    if isinstance(x, torch.Tensor):
        if x.is_cuda:
            raise TypeError("sort_host expects host memory")
        if x.dtype not in (torch.float64, torch.uint64):
            raise TypeError(f"keys must be float64 or uint64, got {x.dtype}")
        if x.dim() != 1 or not x.is_contiguous():
            raise ValueError("x must be a contiguous 1-D tensor")
        ptr, n, dt = x.data_ptr(), x.numel(), x.dtype
        is_f64 = dt == torch.float64
        if out is None:
            out = torch.empty_like(x)
        if not isinstance(out, torch.Tensor) or out.is_cuda or out.dtype != dt or out.numel() != n \
                or not out.is_contiguous():
            raise ValueError(f"out must be a contiguous host tensor of {n} {dt} keys")
        optr = out.data_ptr()
    else:
        x = np.asarray(x)
        if x.dtype not in (np.float64, np.uint64):
            raise TypeError(f"keys must be float64 or uint64, got {x.dtype}")
        if x.ndim != 1:
            raise ValueError("x must be 1-D")
        x = np.ascontiguousarray(x)
        ptr, n = x.ctypes.data, x.size
        is_f64 = x.dtype == np.float64
        if out is None:
            out = np.empty_like(x)
        if not isinstance(out, np.ndarray) or out.dtype != x.dtype or out.size != n or not out.flags.c_contiguous \
                or not out.flags.writeable:
            raise ValueError(f"out must be a writeable contiguous numpy array of {n} {x.dtype} keys")
        optr = out.ctypes.data
    fn = lib().pcf_sort_f64_host if is_f64 else lib().pcf_sort_u64_host
    p = make_params(tau, seed, FLAG_SYNC)
    if workspace is not None:
        if not isinstance(workspace, torch.Tensor) or not workspace.is_cuda or not workspace.is_contiguous():
            raise ValueError("workspace must be a contiguous CUDA tensor")
        p.workspace, p.workspace_bytes = workspace.data_ptr(), workspace.numel() * workspace.element_size()
    s = stream if stream is not None else torch.cuda.current_stream()
    rc = fn(ctypes.c_void_p(ptr), ctypes.c_void_p(optr), n, ctypes.byref(p), ctypes.c_void_p(s.cuda_stream))
    _check(rc)
    return out
