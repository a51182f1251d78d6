"""CPU-side checks of the C ABI library: it loads, exports every symbol the
header declares, and its host-only entry points behave (no GPU needed)."""
import ctypes
import os
import re

import pytest

import paper_2405_07122_b200 as pcf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pcf_sort.h")


@pytest.fixture(scope="module")
def L():
    pcf.build()
    return pcf.lib()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pcf_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    names = declared_functions()
    assert set(names) == set(pcf.SYMBOLS), names
    for name in names:
        assert hasattr(L, name), f"missing export {name}"


def test_params_defaults(L):
    p = pcf.Params()
    L.pcf_params_init(ctypes.byref(p))
    assert p.struct_size == ctypes.sizeof(pcf.Params)
    assert p.tau == 64 and p.seed == 0 and p.flags == pcf.FLAG_SYNC
    assert p.workspace is None and not p.log and not p.stats
    assert ctypes.sizeof(pcf.NodeRecord) == 72


def test_status_strings_and_version(L):
    for code, name in pcf.STATUS.items():
        assert L.pcf_status_string(code).decode() == name
    assert L.pcf_abi_version() == 2


def test_workspace_bytes(L):
    assert pcf.workspace_bytes(0) == 0
    small = pcf.workspace_bytes(100)
    assert 0 < small < 4096
    prev = 0
    for n in [10_000, 10 ** 5, 10 ** 6, 10 ** 7, 10 ** 8, 10 ** 9]:
        w = pcf.workspace_bytes(n)
        assert w >= 8 * n and w > prev
        prev = w
    assert pcf.workspace_bytes(10 ** 9) < 18 * 10 ** 9   # one extra key buffer + digits + tables/queues


def test_argument_errors_before_any_launch(L):
    p = pcf.make_params()
    # n == 0 is a no-op
    assert L.pcf_sort_f64(None, None, 0, ctypes.byref(p), None) == 0
    # NULL with n > 0
    assert L.pcf_sort_f64(None, None, 10, ctypes.byref(p), None) == 1
    # tau < 2
    p.tau = 1
    assert L.pcf_sort_u64(ctypes.c_void_p(4096), ctypes.c_void_p(8192), 10, ctypes.byref(p), None) == 1
    p.tau = 64
    # overlapping but distinct ranges
    assert L.pcf_sort_f64(ctypes.c_void_p(4096), ctypes.c_void_p(4096 + 8), 10, ctypes.byref(p), None) == 1
    # misaligned
    assert L.pcf_sort_f64(ctypes.c_void_p(4097), ctypes.c_void_p(1 << 20), 10, ctypes.byref(p), None) == 1
    # n >= 2^32
    assert L.pcf_sort_f64(ctypes.c_void_p(4096), ctypes.c_void_p(1 << 40), 1 << 32, ctypes.byref(p), None) == 1
    # struct_size too small
    p.struct_size = 8
    assert L.pcf_sort_f64(ctypes.c_void_p(4096), ctypes.c_void_p(1 << 20), 10, ctypes.byref(p), None) == 1
    assert b"struct_size" in L.pcf_last_error()


def test_bucket_counts_argument_errors_before_any_launch(L):
    f, dp = L.pcf_bucket_counts_f64, ctypes.c_void_p
    assert f(None, 10, 4, 4, 4, 0, dp(8192), dp(16384), None, None) == 1      # NULL keys
    assert f(dp(4096), 10, 4, 4, 4, 0, None, dp(16384), None, None) == 1     # NULL b
    assert f(dp(4096), 1, 4, 4, 4, 0, dp(8192), dp(16384), None, None) == 1  # n < 2
    assert f(dp(4096), 1 << 32, 4, 4, 4, 0, dp(8192), dp(16384), None, None) == 1
    for a, b, g in [(0, 4, 4), (4, 0, 4), (4, 4, 0), (1 << 32, 4, 4), (4, (1 << 32) - 1, 4)]:
        assert f(dp(4096), 10, a, b, g, 0, dp(8192), dp(16384), None, None) == 1
    assert b"alpha" in L.pcf_last_error()
    assert f(dp(4097), 10, 4, 4, 4, 0, dp(8192), dp(16384), None, None) == 1   # misaligned keys
    assert f(dp(4096), 10, 4, 4, 4, 0, dp(8194), dp(16384), None, None) == 1   # misaligned b
    assert b"misaligned" in L.pcf_last_error()


def test_product_path_does_not_touch_oracle():
    """The product package and its CUDA sources never reference oracle/ (③)."""
    pkg = os.path.join(ROOT, "paper_2405_07122_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".c")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "pcf_oracle" not in txt \
                    and "liboracle" not in txt, f
    ora = open(os.path.join(ROOT, "oracle", "pcf_oracle.c")).read()
    assert "#include \"" not in ora   # the oracle includes no project header
