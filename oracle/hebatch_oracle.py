"""TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference's homomorphic-operator path.

What it restates (file:line under /root/reference/pkg/src/hebatch):
    paillier.py   :39-66 PublicKey, :69-107 PrivateKey, :130-170 keygen, :173-178 draw_unit,
                  :181-237 scalar encrypt / lift / decrypt / hadd / hmul / obfuscate
    encoding.py   :44-137 fixed-point codec
    operators.py  :39-104 the ten element kernels; :109-317 the batch operators' arithmetic
    bufferpool.py :231-330 HAFB wire format
All big-integer arithmetic goes through oracle/gmp.py (libgmp via ctypes when present, Python integers
otherwise -- both exact).  The reference delegates the same arithmetic to gmpy2 (pyproject.toml:11,
unpinned ">=2.1"), which is not in /root/reference; because every result is an exact integer, any
correct engine reproduces it bit for bit.

Parity is PINNED: tests/test_oracle_golden.py checks this module against (a) the known-answer values
the reference's own tests hold (n=35: encrypt(3, r=2) = 683, decrypt(683) = 3, codec tables, the HAFB
golden bytes) and (b) tests/golden/*.json, produced by importing the unmodified reference in the build
container (tools/make_golden.py; needs /root/reference, which does not exist on the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import this
module.  The product package must never do so.
"""
from __future__ import annotations

import math
import os
import random
import struct
import sys
from fractions import Fraction

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import gmp  # noqa: E402

BASE = 16            # encoding.py:22
LOG2_BASE = 4        # encoding.py:23
MIN_EXPONENT = -32   # encoding.py:24


class Overflow(ArithmeticError):
    """encoding.FixedPointOverflow (encoding.py:27)."""


# ---------------------------------------------------------------- keys (paillier.py:39-170)
class Key:
    """Public part (n) and, when p and q are given, the CRT constants of paillier.py:94-98."""

    def __init__(self, n: int, p: int | None = None, q: int | None = None):
        self.n = int(n)
        self.n2 = self.n * self.n
        self.key_bits = self.n.bit_length()
        self.max_int = self.n // 3                      # paillier.py:56
        self.neg_band = self.n - self.max_int           # operators.py:250
        self.p = self.q = None
        if p is not None:
            p, q = int(p), int(q)
            assert p * q == self.n and p != q
            self.p, self.q = p, q
            self.p2, self.q2 = p * p, q * q
            g = self.n + 1
            self.hp = gmp.invert((gmp.powmod(g, p - 1, self.p2) - 1) // p, p)   # paillier.py:96
            self.hq = gmp.invert((gmp.powmod(g, q - 1, self.q2) - 1) // q, q)   # paillier.py:97
            self.q_inv = gmp.invert(q, p)                                      # paillier.py:98
            self.lam = math.lcm(p - 1, q - 1)
            self.mu = gmp.invert((gmp.powmod(g, self.lam, self.n2) - 1) // self.n, self.n)


def probable_prime(bits: int, rng: random.Random) -> int:
    """paillier.py:130-137: top two bits and the low bit forced, 40 primality rounds."""
    high = 3 << (bits - 2)
    while True:
        cand = rng.getrandbits(bits) | high | 1
        if gmp.is_prime(cand, 40):
            return cand


def keygen(bits: int, rng: random.Random) -> Key:
    """paillier.py:147-170 (size checks omitted: the oracle is fed valid sizes)."""
    half = bits // 2
    while True:
        p = probable_prime(half, rng)
        q = probable_prime(half, rng)
        if p != q and (p * q).bit_length() == bits:
            return Key(p * q, p, q)


def draw_unit(n: int, rng: random.Random) -> int:
    """paillier.py:173-178."""
    while True:
        r = rng.randrange(1, n)
        if math.gcd(r, n) == 1:
            return r


# ---------------------------------------------------------------- element kernels (operators.py:39-104)
def k_encrypt(key: Key, items):
    n, n2 = key.n, key.n2
    return [(1 + m * n) * gmp.powmod(r, n, n2) % n2 for m, r in items]       # operators.py:41


def k_obfuscate(key: Key, items):
    n, n2 = key.n, key.n2
    return [c * gmp.powmod(r, n, n2) % n2 for c, r in items]                 # operators.py:46


def k_decrypt(key: Key, items):
    p, q = key.p, key.q
    out = []
    for c in items:                                                          # operators.py:52-55
        mp = (gmp.powmod(c, p - 1, key.p2) - 1) // p * key.hp % p
        mq = (gmp.powmod(c, q - 1, key.q2) - 1) // q * key.hq % q
        out.append(mq + q * ((mp - mq) * key.q_inv % p))
    return out


def decrypt_textbook(key: Key, c: int) -> int:
    """L-function form, the cross-check the reference runs in tests/test_paillier.py:108-113."""
    return (gmp.powmod(c, key.lam, key.n2) - 1) // key.n * key.mu % key.n


def pow_scalar(key: Key, c: int, k: int) -> int:
    """operators.py:59-62: residues above n - max_int are negative; use the inverse and n - k."""
    if k > key.neg_band:
        return gmp.powmod(gmp.invert(c, key.n2), key.n - k, key.n2)
    return gmp.powmod(c, k, key.n2)


def k_mul(key: Key, items):
    return [pow_scalar(key, c, k) for c, k in items]                          # operators.py:67


def k_add(key: Key, items):
    return [a * b % key.n2 for a, b in items]                                 # operators.py:72


def k_product(key: Key, groups):
    out = []
    for values in groups:                                                     # operators.py:78-82
        acc = 1
        for v in values:
            acc = acc * v % key.n2
        out.append(acc)
    return out


def k_dot(key: Key, rows, cols, items):
    out = []
    for i, j in items:                                                        # operators.py:89-93
        acc = 1
        for c, k in zip(rows[i], cols[j]):
            acc = acc * pow_scalar(key, c, k) % key.n2
        out.append(acc)
    return out


def lift(key: Key, m: int) -> int:
    return (1 + m * key.n) % key.n2                                           # operators.py:211


# ---------------------------------------------------------------- codec (encoding.py:44-137)
def exact_exponent(value) -> int:
    num, den = value.as_integer_ratio()
    if num == 0:
        return 0
    lsb = (num & -num).bit_length() - 1
    return (lsb - (den.bit_length() - 1)) // LOG2_BASE                        # encoding.py:49-51


def encode(key: Key, value, target_exponent=None) -> tuple[int, int]:
    """(mantissa residue, exponent); encoding.py:54-78."""
    if isinstance(value, float) and not math.isfinite(value):
        raise ValueError("cannot encode non-finite values")
    if target_exponent is None:
        exponent = exact_exponent(value)
        num, den = value.as_integer_ratio()
        shift = -LOG2_BASE * exponent - (den.bit_length() - 1)
        scaled = num << shift if shift >= 0 else num >> -shift
    else:
        exponent = int(target_exponent)
        scaled = round(Fraction(value) * Fraction(BASE) ** -exponent)        # half-to-even
    if abs(scaled) >= key.max_int:
        raise Overflow("mantissa beyond max_int")
    return scaled % key.n, exponent


def signed_mantissa(key: Key, m: int) -> int:
    if m >= key.n:
        raise ValueError("mantissa exceeds the modulus")
    if m < key.max_int:
        return m
    if m > key.n - key.max_int:
        return m - key.n
    raise Overflow("overflow band")                                           # encoding.py:86-92


def decode(key: Key, m: int, exponent: int) -> float:
    s = signed_mantissa(key, m)
    if exponent >= 0:
        return float(s * BASE ** exponent)
    return s / BASE ** -exponent                                              # correctly rounded


def rescale(key: Key, m: int, exponent: int, new_exponent: int) -> int:
    if new_exponent > exponent:
        raise ValueError("can only rescale toward a smaller exponent")
    if new_exponent == exponent:
        return m
    s = signed_mantissa(key, m) * BASE ** (exponent - new_exponent)
    if abs(s) >= key.max_int:
        raise Overflow("rescaled mantissa exceeds max_int")
    return s % key.n


def renormalize(key: Key, m: int, exponent: int, min_exponent: int = MIN_EXPONENT) -> tuple[int, int]:
    if exponent >= min_exponent:
        return m, exponent
    value = decode(key, m, exponent)
    return encode(key, value, max(exact_exponent(value), min_exponent))       # encoding.py:135-137


def encode_batch(key: Key, values, target_exponent=None) -> tuple[list[int], int]:
    """batches.py:112-125: shared exponent = min of the exact exponents unless given."""
    flat = [float(v) for v in values]
    if target_exponent is None:
        target_exponent = min((exact_exponent(v) for v in flat), default=0)
    return [encode(key, v, target_exponent)[0] for v in flat], target_exponent


# ---------------------------------------------------------------- HAFB wire format (bufferpool.py:231-330)
HAFB_MAGIC = b"HAFB"
HAFB_HEADER = struct.Struct("<4sIQIIIB3x")      # bufferpool.py:33


def hafb_word_bytes(key_bits: int) -> int:
    return (2 * key_bits + 7) // 8


def hafb_serialize(key_bits: int, shape, exponents, payload, shared: bool, version: int = 1) -> bytes:
    """bufferpool.py:282-294: header (magic, version, count, key_bits, rows, cols, exponent mode),
    i32 exponents, then count little-endian words of ceil(2*key_bits/8) bytes."""
    rows = shape[0]
    cols = shape[1] if len(shape) == 2 else 0
    head = HAFB_HEADER.pack(HAFB_MAGIC, version, len(payload), key_bits, rows, cols, 0 if shared else 1)
    exps = struct.pack(f"<{len(exponents)}i", *exponents)
    wb = hafb_word_bytes(key_bits)
    return head + exps + b"".join(int(v).to_bytes(wb, "little") for v in payload)


def hafb_deserialize(data: bytes):
    """Inverse: (key_bits, shape, exponents, payload, shared); bufferpool.py:311-330."""
    magic, version, count, key_bits, rows, cols, mode = HAFB_HEADER.unpack(data[:HAFB_HEADER.size])
    assert magic == HAFB_MAGIC and version == 1 and mode in (0, 1)
    shape = (rows,) if cols == 0 else (rows, cols)
    nexp = 1 if mode == 0 else count
    off = HAFB_HEADER.size
    exps = struct.unpack_from(f"<{nexp}i", data, off)
    off += 4 * nexp
    wb = hafb_word_bytes(key_bits)
    assert len(data) == off + count * wb
    payload = [int.from_bytes(data[off + i * wb: off + (i + 1) * wb], "little") for i in range(count)]
    return key_bits, shape, tuple(exps), payload, mode == 0
