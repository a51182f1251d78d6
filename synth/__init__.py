"""Seeded synthetic inputs -- shared by tests, bench.py and smoke().

This module holds none of the method's arithmetic; it only generates key
arrays on the host (C, OpenMP).  Configs follow BASELINE.json ``configs``:

  c1   n=1e6  float64 Uniform[0,1), seed 0                       (§4.1 uniform)
  c2   n=1e7  float64 LogNormal(0,1), seed 1                     (§4.1 lognormal)
  c3   n=1e8  float64 8-Gaussian mixture + 10% one value, seed 2 (stand-in for skewed real data, §4.2)
  c4   n=1e8  float64 exp(700 U^4), seed 3                       (sigma2/sigma1 -> inf regime)
  c5f  n=1e9  float64 Exponential(1), seed 4                     (§4.1 exponential)
  c5u  n=1e9  uint64 Uniform[0,2^64), seed 5                     (integer keys)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "synth.c")
_LIB = os.path.join(_HERE, "libsynth.so")

DISTS = {"uniform": 0, "normal": 1, "exponential": 2, "lognormal": 3, "gauss_mix8": 4,
         "exp700u4": 5, "u64": 6}

CONFIGS = {
    "c1": dict(dist="uniform", n=1_000_000, seed=0),
    "c2": dict(dist="lognormal", n=10_000_000, seed=1),
    "c3": dict(dist="gauss_mix8", n=100_000_000, seed=2),
    "c4": dict(dist="exp700u4", n=100_000_000, seed=3),
    "c5f": dict(dist="exponential", n=1_000_000_000, seed=4),
    "c5u": dict(dist="u64", n=1_000_000_000, seed=5),
}

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-std=c11", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp,
                               _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _L():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.synth_generate.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p]
        _lib.synth_generate.restype = None
    return _lib


def generate(dist: str, n: int, seed: int, out: np.ndarray | None = None) -> np.ndarray:
    """n keys of distribution ``dist`` from ``seed`` (float64, or uint64 for 'u64')."""
    dt = np.uint64 if dist == "u64" else np.float64
    if out is None:
        out = np.empty(n, dtype=dt)
    assert out.dtype == dt and out.flags.c_contiguous and len(out) == n
    _L().synth_generate(DISTS[dist], seed, n, out.ctypes.data_as(ctypes.c_void_p))
    return out


def config(name: str, n: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
    """BASELINE.json config ``name`` (optionally at a reduced size n, same recipe and seed)."""
    c = CONFIGS[name]
    return generate(c["dist"], c["n"] if n is None else n, c["seed"], out=out)
