"""The homomorphic operators, API-compatible with the reference's operators module
(/root/reference/pkg/src/hebatch/operators.py:109-317), running on the B200.

Signatures, broadcast rules, exponent bookkeeping, `obfuscated` propagation and error behaviour follow
the reference operator by operator (cited below).  What differs is the execution: operands are
aggregated word arrays that stay on the GPU between chained operators, each operator is one call into
libhebatch_b200.so, and there is no CPU path -- `backend` must be a CudaBackend (the default).

The `_k_*` functions are the element kernels' names only: they are what CudaBackend.run dispatches
on (and what the reference's own operators pass to a backend); calling one directly is an error.
"""
from __future__ import annotations

import random

import numpy as np

from . import encoding
from .backends import CudaBackend, ExecutionBackend, default_backend
from .batches import (
    CiphertextBatch,
    ExponentMismatch,
    PlaintextBatch,
    ShapeMismatch,
    ct_width,
    plain_rescale,
    pt_width,
    require_same_key,
    shared_exponent_of,
)
from .device import WordArray
from .paillier import PrivateKey, PublicKey, draw_unit

OPERATOR_NAMES = ("encode", "decode", "henc", "hdec", "hmul", "hadd", "hmatmul", "hsum")


def _no_cpu_path(name):
    def marker(common, items):
        raise RuntimeError(f"{name} has no CPU implementation in this package; run it through CudaBackend")
    marker.__name__ = name
    marker.__qualname__ = name
    return marker


_k_encrypt = _no_cpu_path("_k_encrypt")
_k_obfuscate = _no_cpu_path("_k_obfuscate")
_k_decrypt = _no_cpu_path("_k_decrypt")
_k_mul = _no_cpu_path("_k_mul")
_k_add = _no_cpu_path("_k_add")
_k_product = _no_cpu_path("_k_product")
_k_dot = _no_cpu_path("_k_dot")
_k_encode = _no_cpu_path("_k_encode")
_k_decode = _no_cpu_path("_k_decode")


def _cuda(backend) -> CudaBackend:
    if backend is None:
        return default_backend()
    if not isinstance(backend, CudaBackend):
        raise TypeError(
            f"{type(backend).__name__} is not a CudaBackend: this package has no CPU execution path")
    return backend


def _draw_units(pk: PublicKey, count: int, rng: random.Random, backend: CudaBackend) -> WordArray:
    """Obfuscation factors in element order, exactly the stream draw_unit would yield
    (operators.py:133,142) -- see CudaBackend.draw_units."""
    return backend.draw_units(pk.n, count, rng)


# ---- codec ------------------------------------------------------------------------------------------

def batch_encode(pk: PublicKey, values, exponent: int, backend: ExecutionBackend | None = None) -> PlaintextBatch:
    """operators.py:109-114."""
    vals = values if isinstance(values, np.ndarray) else np.asarray(list(values), dtype=np.float64)
    vals = np.ascontiguousarray(vals, dtype=np.float64).ravel()
    if vals.shape[0] == 0:
        return PlaintextBatch(pk, (0,), (exponent or 0,), (), True)
    be = _cuda(backend)
    words, used = be.encode_f64(pk.n, vals, exponent)  # exponent None (used by encode_batch): exact shared exponent
    return PlaintextBatch(pk, (vals.shape[0],), (used,), words, True)


def batch_decode(pk: PublicKey, batch: PlaintextBatch, backend: ExecutionBackend | None = None) -> list:
    """operators.py:117-121."""
    exponent = shared_exponent_of(batch)
    if batch.count == 0:
        return []
    return [float(v) for v in _cuda(backend).decode_f64(pk.n, batch.words, exponent)]


# ---- encrypt / obfuscate / decrypt --------------------------------------------------------------------

def batch_encrypt(pk: PublicKey, plain: PlaintextBatch, rng: random.Random,
                  backend: ExecutionBackend | None = None) -> CiphertextBatch:
    """operators.py:124-136: one independent obfuscation factor per element, drawn before dispatch."""
    if plain.key != pk:
        raise ValueError("plaintext batch was encoded under a different key")
    be = _cuda(backend)
    out = be.encrypt_drawing(pk.n, plain.words, rng) if plain.count else None     # large batches: draws overlap the GPU
    if out is None:
        r = _draw_units(pk, plain.count, rng, be)
        out = be.encrypt(pk.n, plain.words, r) if plain.count else WordArray.from_ints((), ct_width(pk))
    return CiphertextBatch(pk, plain.shape, plain.exponents, out, plain.shared_exponent, obfuscated=True)


def batch_obfuscate(pk: PublicKey, cipher: CiphertextBatch, rng: random.Random,
                    backend: ExecutionBackend | None = None) -> CiphertextBatch:
    """operators.py:139-145."""
    be = _cuda(backend)
    out = be.encrypt_drawing(pk.n, cipher.words, rng, obfuscate=True) if cipher.count else None
    if out is None:
        r = _draw_units(pk, cipher.count, rng, be)
        out = be.obfuscate(pk.n, cipher.words, r) if cipher.count else cipher.words
    return CiphertextBatch(pk, cipher.shape, cipher.exponents, out, cipher.shared_exponent, obfuscated=True)


def _private_tuple(sk: PrivateKey):
    return (sk.p, sk.q, sk._hp, sk._hq, sk._q_inv_p)


def batch_decrypt(sk: PrivateKey, cipher: CiphertextBatch, backend: ExecutionBackend | None = None,
                  min_exponent: int = encoding.DEFAULT_MIN_EXPONENT) -> PlaintextBatch:
    """operators.py:148-167: exponents are preserved unless one sank below the floor, in which case
    every element is renormalised on the plaintext side."""
    pk = sk.public_key
    if cipher.key != pk:
        raise ValueError("ciphertext batch does not belong to this private key")
    if cipher.count:
        words = _cuda(backend).decrypt(pk.n, _private_tuple(sk), cipher.words)
    else:
        words = WordArray.from_ints((), pt_width(pk))
    plain = PlaintextBatch(pk, cipher.shape, cipher.exponents, words, cipher.shared_exponent)
    if not plain.exponents or min(plain.exponents) >= min_exponent:
        return plain
    lifted = [encoding.renormalize(pk, plain.element(i), min_exponent) for i in range(plain.count)]
    exps = tuple(e.exponent for e in lifted)
    shared = len(set(exps)) == 1
    return PlaintextBatch(pk, plain.shape, exps[:1] if shared else exps,
                          tuple(e.mantissa for e in lifted), shared)


# ---- add ----------------------------------------------------------------------------------------------

def _added_exponents(a: CiphertextBatch, b):
    if a.shared_exponent and b.shared_exponent:
        if a.exponents[0] != b.exponents[0]:
            raise ExponentMismatch(
                f"ciphertext exponents differ ({a.exponents[0]} vs {b.exponents[0]}); align at encode time")
        return a.exponents, True
    for i in range(a.count):
        if a.exponent_at(i) != b.exponent_at(i):
            raise ExponentMismatch(f"element {i}: exponents differ; align at encode time")
    return a.exponents, a.shared_exponent


def batch_add(pk: PublicKey, a: CiphertextBatch, b, backend: ExecutionBackend | None = None) -> CiphertextBatch:
    """operators.py:184-220.  A plaintext right operand is aligned down to the ciphertext exponent and
    lifted with the deterministic g^m form inside the kernel (no modular exponentiation)."""
    require_same_key(a, b)
    be = _cuda(backend)
    if isinstance(b, PlaintextBatch):
        broadcast = b.count == 1 and a.count != 1
        if not broadcast and a.shape != b.shape:
            raise ShapeMismatch(f"{a.shape} vs {b.shape}")
        if not a.shared_exponent:
            raise ExponentMismatch("plaintext addition needs a shared-exponent ciphertext")
        target = shared_exponent_of(a)
        if shared_exponent_of(b) < target:
            raise ExponentMismatch(
                f"plaintext exponent {b.exponents[0]} finer than ciphertext {target}; "
                "encode the ciphertext side at least as fine")
        b = plain_rescale(b, target, be)
        out = be.lift_mulmod(pk.n, a.words, b.words, broadcast) if a.count else a.words
        return CiphertextBatch(pk, a.shape, a.exponents, out, a.shared_exponent, a.obfuscated)
    if a.shape != b.shape:
        raise ShapeMismatch(f"{a.shape} vs {b.shape}")
    exps, shared = _added_exponents(a, b)
    out = be.mulmod(pk.n, a.words, b.words) if a.count else a.words
    return CiphertextBatch(pk, a.shape, exps, out, shared, a.obfuscated or b.obfuscated)


# ---- scalar multiplication ------------------------------------------------------------------------------

def batch_mul_plain(pk: PublicKey, a: CiphertextBatch, k: PlaintextBatch,
                    backend: ExecutionBackend | None = None) -> CiphertextBatch:
    """operators.py:223-251: k is a scalar (count 1), a same-shape batch, or a row vector over the
    columns of a 2-D batch; exponents add."""
    require_same_key(a, k)
    if k.count == 1:
        exps, shared = tuple(e + k.exponent_at(0) for e in a.exponents), a.shared_exponent
    elif k.shape == a.shape:
        if a.shared_exponent and k.shared_exponent:
            exps, shared = (a.exponents[0] + k.exponents[0],), True
        else:
            exps, shared = tuple(a.exponent_at(i) + k.exponent_at(i) for i in range(a.count)), False
    elif len(a.shape) == 2 and k.shape == (a.shape[1],):
        cols = a.shape[1]
        if a.shared_exponent and k.shared_exponent:
            exps, shared = (a.exponents[0] + k.exponents[0],), True
        else:
            exps, shared = tuple(a.exponent_at(i) + k.exponent_at(i % cols) for i in range(a.count)), False
    else:
        raise ShapeMismatch(f"cannot broadcast {k.shape} across {a.shape}")
    # all three modes are "element i uses scalar i mod k.count"
    out = _cuda(backend).powscalar(pk.n, a.words, k.words) if a.count else a.words
    return CiphertextBatch(pk, a.shape, exps, out, shared, a.obfuscated)


# ---- reductions -----------------------------------------------------------------------------------------

def batch_sum(pk: PublicKey, a: CiphertextBatch, axis: int | None = None,
              backend: ExecutionBackend | None = None) -> CiphertextBatch:
    """operators.py:254-291: modular-product reduction over everything, over rows (axis 0) or over
    columns (axis 1).  Modular multiplication is exact, so the tree order used on the device yields the
    same bits as the reference's sequential loop."""
    exponent = shared_exponent_of(a)
    be = _cuda(backend)
    if axis is None:
        if a.count == 0:
            return CiphertextBatch(pk, (1,), (exponent,), (1,), True, a.obfuscated)
        out = be.product(pk.n, a.words, 1, a.count, 0, 1)
        return CiphertextBatch(pk, (1,), (exponent,), out, True, a.obfuscated)
    if len(a.shape) != 2:
        raise ShapeMismatch("axis reduction requires a 2-D batch")
    rows, cols = a.shape
    if axis == 0:
        ngroups, glen, gstride, estride, shape = cols, rows, 1, cols, (cols,)
    elif axis == 1:
        ngroups, glen, gstride, estride, shape = rows, cols, cols, 1, (rows,)
    else:
        raise ValueError(f"bad axis {axis}")
    if ngroups == 0:
        return CiphertextBatch(pk, shape, (exponent,), (), True, a.obfuscated)
    if glen == 0:
        return CiphertextBatch(pk, shape, (exponent,), (1,) * ngroups, True, a.obfuscated)
    out = be.product(pk.n, a.words, ngroups, glen, gstride, estride)
    return CiphertextBatch(pk, shape, (exponent,), out, True, a.obfuscated)


def batch_matmul(pk: PublicKey, a: CiphertextBatch, x: PlaintextBatch,
                 backend: ExecutionBackend | None = None) -> CiphertextBatch:
    """operators.py:294-317: encrypted-left times plaintext-right; result[i][j] decrypts to
    sum_t a[i][t] * x[t][j]."""
    require_same_key(a, x)
    a_shape = a.shape if len(a.shape) == 2 else (1, a.shape[0])
    if len(x.shape) != 2:
        raise ShapeMismatch("right operand must be 2-D")
    k_rows, inner = a_shape
    if x.shape[0] != inner:
        raise ShapeMismatch(f"inner dims disagree: {a_shape} x {x.shape}")
    d = x.shape[1]
    ea, ex = shared_exponent_of(a), shared_exponent_of(x)
    shape = (k_rows, d) if len(a.shape) == 2 else (d,)
    if k_rows * d == 0:
        return CiphertextBatch(pk, shape, (ea + ex,), (), True, a.obfuscated)
    if inner == 0:
        return CiphertextBatch(pk, shape, (ea + ex,), (1,) * (k_rows * d), True, a.obfuscated)
    out = _cuda(backend).matvec(pk.n, a.words, x.words, k_rows, inner, d)
    return CiphertextBatch(pk, shape, (ea + ex,), out, True, a.obfuscated)


# ---- integer-level helpers for the scalar API in paillier.py -----------------------------------------------

def raw_encrypt(pk, ms, rs):
    be = default_backend()
    w = pt_width(pk)
    return list(be.encrypt(pk.n, WordArray.from_ints(ms, w), WordArray.from_ints(rs, w)).ints())


def raw_obfuscate(pk, cs, rs):
    be = default_backend()
    return list(be.obfuscate(pk.n, WordArray.from_ints(cs, ct_width(pk)),
                             WordArray.from_ints(rs, pt_width(pk))).ints())


def raw_decrypt(sk, cs):
    be = default_backend()
    pk = sk.public_key
    return list(be.decrypt(pk.n, _private_tuple(sk), WordArray.from_ints(cs, ct_width(pk))).ints())


def raw_mulmod(pk, a, b):
    be = default_backend()
    w = ct_width(pk)
    return list(be.mulmod(pk.n, WordArray.from_ints(a, w), WordArray.from_ints(b, w)).ints())


def raw_pow(pk, cs, ks):
    be = default_backend()
    return list(be.powscalar(pk.n, WordArray.from_ints(cs, ct_width(pk)),
                             WordArray.from_ints(ks, pt_width(pk)), raw_exponent=True).ints())
