"""TEST INFRASTRUCTURE ONLY -- stand-in for the gmpy2 module so the UNMODIFIED reference package
(/root/reference/pkg/src/hebatch) can be imported in the build container, where the gmpy2 wheel is
absent.  Only the four entry points the reference uses exist: powmod, invert, mpz, is_prime.

Used by tools/make_golden.py (fixture generation) and by oracle validation runs with
PYTHONPATH=oracle/gmpy2_shim:/root/reference/pkg/src.  Never on the GPU box's product path.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gmp as _gmp  # noqa: E402  (oracle/gmp.py)

mpz = int


def powmod(base, exp, mod):
    return _gmp.powmod(base, exp, mod)


def invert(a, mod):
    return _gmp.invert(a, mod)


def is_prime(n, rounds=25):
    return _gmp.is_prime(n, rounds)
