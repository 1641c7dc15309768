"""TEST INFRASTRUCTURE ONLY -- exact big-integer primitives for the oracle.

powmod / invert / is_prime with the semantics of the four gmpy2 entry points the reference uses
(/root/reference/pkg/src/hebatch/paillier.py:93-98,137,190,207-208,217,227,236 and
operators.py:41,46,53-54,61-62,72,79,90).  gmpy2 (unpinned ">=2.1", pkg/pyproject.toml:11) is absent
from this image; the GMP runtime /lib/x86_64-linux-gnu/libgmp.so.10 (GMP 6.3.0) is present and is
driven through ctypes when it can be loaded, otherwise Python's own integers are used.  Both are
exact, so the results are identical; only the speed differs (about 8x at 2048 bits).

Nothing under oracle/ may be imported by the product package.
"""
from __future__ import annotations

import ctypes
import ctypes.util


class _Mpz(ctypes.Structure):
    _fields_ = [("alloc", ctypes.c_int), ("size", ctypes.c_int), ("d", ctypes.c_void_p)]


def _load():
    for name in ("libgmp.so.10", ctypes.util.find_library("gmp")):
        if not name:
            continue
        try:
            return ctypes.CDLL(name)
        except OSError:
            continue
    return None


_g = _load()
HAVE_GMP = _g is not None

if HAVE_GMP:
    _p = ctypes.POINTER(_Mpz)
    _g.__gmpz_init.argtypes = [_p]
    _g.__gmpz_clear.argtypes = [_p]
    _g.__gmpz_import.argtypes = [_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_size_t, ctypes.c_int,
                                 ctypes.c_size_t, ctypes.c_char_p]
    _g.__gmpz_export.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_size_t), ctypes.c_int,
                                 ctypes.c_size_t, ctypes.c_int, ctypes.c_size_t, _p]
    _g.__gmpz_export.restype = ctypes.c_void_p
    _g.__gmpz_powm.argtypes = [_p, _p, _p, _p]
    _g.__gmpz_invert.argtypes = [_p, _p, _p]
    _g.__gmpz_invert.restype = ctypes.c_int
    _g.__gmpz_probab_prime_p.argtypes = [_p, ctypes.c_int]
    _g.__gmpz_probab_prime_p.restype = ctypes.c_int
    _g.__gmpz_sizeinbase.argtypes = [_p, ctypes.c_int]
    _g.__gmpz_sizeinbase.restype = ctypes.c_size_t
    # module-level aliases: a double-underscore attribute inside a class body would be name-mangled
    _z_init = getattr(_g, "__gmpz_init")
    _z_clear = getattr(_g, "__gmpz_clear")
    _z_import = getattr(_g, "__gmpz_import")
    _z_export = getattr(_g, "__gmpz_export")
    _z_powm = getattr(_g, "__gmpz_powm")
    _z_invert = getattr(_g, "__gmpz_invert")
    _z_prime = getattr(_g, "__gmpz_probab_prime_p")
    _z_size = getattr(_g, "__gmpz_sizeinbase")


class _Z:
    """A GMP integer with automatic lifetime."""

    def __init__(self, value: int = 0):
        self.z = _Mpz()
        _z_init(ctypes.byref(self.z))
        if value:
            raw = int(value).to_bytes((int(value).bit_length() + 7) // 8, "little")
            _z_import(ctypes.byref(self.z), len(raw), -1, 1, 0, 0, raw)

    def __del__(self):
        _z_clear(ctypes.byref(self.z))

    def ref(self):
        return ctypes.byref(self.z)

    def to_int(self) -> int:
        nbytes = (_z_size(self.ref(), 2) + 7) // 8
        buf = ctypes.create_string_buffer(nbytes)
        cnt = ctypes.c_size_t()
        _z_export(buf, ctypes.byref(cnt), -1, 1, 0, 0, self.ref())
        return int.from_bytes(buf.raw[:cnt.value], "little")


def powmod(base: int, exp: int, mod: int) -> int:
    base, exp, mod = int(base), int(exp), int(mod)
    if not HAVE_GMP or exp < 0 or base < 0 or mod <= 0:
        return pow(base, exp, mod)
    out, b, e, m = _Z(), _Z(base), _Z(exp), _Z(mod)   # named: temporaries would be freed too early
    _z_powm(out.ref(), b.ref(), e.ref(), m.ref())
    return out.to_int()


def invert(a: int, mod: int) -> int:
    """a^-1 mod `mod`; ZeroDivisionError when it does not exist (as gmpy2.invert)."""
    a, mod = int(a), int(mod)
    if not HAVE_GMP or a < 0 or mod <= 0:
        try:
            return pow(a, -1, mod)
        except ValueError as exc:
            raise ZeroDivisionError("invert() no inverse exists") from exc
    out, x, m = _Z(), _Z(a), _Z(mod)
    if _z_invert(out.ref(), x.ref(), m.ref()) == 0:
        raise ZeroDivisionError("invert() no inverse exists")
    return out.to_int()


def _miller_rabin(n: int, rounds: int) -> bool:
    import random
    if n < 2:
        return False
    for sp in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if n % sp == 0:
            return n == sp
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    rng = random.Random(n)
    for _ in range(rounds):
        a = rng.randrange(2, n - 1)
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def is_prime(n: int, rounds: int = 25) -> bool:
    n = int(n)
    if not HAVE_GMP or n <= 0:
        return _miller_rabin(n, rounds)
    z = _Z(n)
    return _z_prime(z.ref(), rounds) != 0
