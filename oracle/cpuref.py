"""TEST INFRASTRUCTURE ONLY -- ctypes binding of oracle/_build/libcpuref.so (cpu_ref.c): the reference's
element kernels as GMP calls under OpenMP.  Checker for sizes the Python oracle is too slow for, and the
timed CPU baseline of bench.py.  Never imported by the product package."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_PATH = os.path.join(_HERE, "_build", "libcpuref.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-C", _HERE], check=True, capture_output=True)
    return _PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_PATH):
            build()
        _lib = ctypes.CDLL(_PATH)
    return _lib


def threads() -> int:
    """Host threads the CPU baseline uses: every core this process may run on.  Deliberately NOT OpenMP's default:
    torchrun exports OMP_NUM_THREADS=1 to its ranks, which would silently turn the "all host cores" baseline into a
    one-core one; the num_threads clause of cpu_ref.c's parallel regions overrides that variable."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


def _w(vals, width):
    buf = b"".join(int(v).to_bytes(4 * width, "little") for v in vals)
    return np.frombuffer(buf, dtype=np.uint32).reshape(-1, width).copy()


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def widths(n: int):
    kb = n.bit_length()
    return (kb + 31) // 32, ((2 * kb + 7) // 8 + 3) // 4


def encrypt_words(n: int, m: np.ndarray, r: np.ndarray, nthreads: int | None = None) -> np.ndarray:
    wn, wc = widths(n)
    out = np.zeros((m.shape[0], wc), np.uint32)
    lib().cpuref_encrypt(_p(_w([n], wn)), wn, _p(m), wn, _p(r), _p(out), wc, ctypes.c_long(m.shape[0]), 0,
                         nthreads or threads())
    return out


def obfuscate_words(n: int, c: np.ndarray, r: np.ndarray, nthreads: int | None = None) -> np.ndarray:
    wn, wc = widths(n)
    out = np.zeros((c.shape[0], wc), np.uint32)
    lib().cpuref_encrypt(_p(_w([n], wn)), wn, _p(c), wc, _p(r), _p(out), wc, ctypes.c_long(c.shape[0]), 1,
                         nthreads or threads())
    return out


def decrypt_words(key, c: np.ndarray, nthreads: int | None = None) -> np.ndarray:
    """key: oracle Key with p, q, hp, hq, q_inv."""
    wn, wc = widths(key.n)
    hw = (max(key.p, key.q).bit_length() + 31) // 32
    parts = [_w([v], hw) for v in (key.p, key.q, key.hp, key.hq, key.q_inv)]
    out = np.zeros((c.shape[0], wn), np.uint32)
    lib().cpuref_decrypt(*[_p(a) for a in parts], hw, _p(c), wc, _p(out), wn, ctypes.c_long(c.shape[0]),
                         nthreads or threads())
    return out


def mulmod_words(n: int, a: np.ndarray, b: np.ndarray, nthreads: int | None = None) -> np.ndarray:
    wn, wc = widths(n)
    out = np.zeros_like(a)
    lib().cpuref_mulmod(_p(_w([n], wn)), wn, _p(a), _p(b), _p(out), wc, ctypes.c_long(a.shape[0]),
                        nthreads or threads())
    return out


def powscalar_words(n: int, c: np.ndarray, k: np.ndarray, nthreads: int | None = None) -> np.ndarray:
    wn, wc = widths(n)
    out = np.zeros_like(c)
    rc = lib().cpuref_powscalar(_p(_w([n], wn)), wn, _p(c), wc, _p(k), ctypes.c_long(k.shape[0]), _p(out),
                                ctypes.c_long(c.shape[0]), nthreads or threads())
    if rc:
        raise ZeroDivisionError("invert() no inverse exists")
    return out


def matvec_words(n: int, c: np.ndarray, k: np.ndarray, inner: int, d: int, nthreads: int | None = None) -> np.ndarray:
    wn, wc = widths(n)
    out = np.zeros((d, wc), np.uint32)
    rc = lib().cpuref_matvec(_p(_w([n], wn)), wn, _p(c), wc, _p(k), ctypes.c_long(inner), ctypes.c_long(d),
                             _p(out), nthreads or threads())
    if rc:
        raise ZeroDivisionError("invert() no inverse exists")
    return out
