"""Plaintext and ciphertext batches backed by aggregated word storage.

Same value semantics and attributes as the reference's batches module
(/root/reference/pkg/src/hebatch/batches.py:56-205): `key, shape, exponents, mantissas | payload,
shared_exponent, obfuscated, count, exponent_at(i), element(i)`, immutable, compared field by field.
The difference is the storage: the big integers live in a device.WordArray (dense little-endian limb
words, host and/or GPU resident) and the tuple-of-ints view the reference exposes is produced lazily.
A batch that came out of an operator stays on the GPU until somebody looks at its integers.
"""
from __future__ import annotations

from . import encoding
from .device import WordArray
from .encoding import EncodedNumber
from .paillier import PublicKey


class ShapeMismatch(ValueError):
    pass


class ExponentMismatch(ValueError):
    pass


class KeyMismatch(ValueError):
    pass


def pt_width(pk: PublicKey) -> int:
    return (pk.key_bits + 31) // 32


def ct_width(pk: PublicKey) -> int:
    return ((2 * pk.key_bits + 7) // 8 + 3) // 4


def _shape_count(shape) -> int:
    total = 1
    for dim in shape:
        total *= dim
    return total


class _Batch:
    """Shared machinery; subclasses fix the value attribute name, the range limit and the word width."""

    __slots__ = ("key", "shape", "exponents", "shared_exponent", "_store")
    _what = "value"

    def _init_common(self, key, shape, exponents, values, shared_exponent, limit, width):
        object.__setattr__(self, "key", key)
        shape = tuple(int(d) for d in shape)
        object.__setattr__(self, "shape", shape)
        object.__setattr__(self, "exponents", tuple(int(e) for e in exponents))
        object.__setattr__(self, "shared_exponent", bool(shared_exponent))
        if len(shape) not in (1, 2) or any(d < 0 for d in shape):
            raise ShapeMismatch(f"bad shape {shape}")
        count = _shape_count(shape)
        if isinstance(values, WordArray):
            store = values                     # produced by an operator: in range by construction
            if store.count != count:
                raise ShapeMismatch(f"payload length {store.count} does not match shape {shape}")
            if store.width != width:
                raise ValueError(f"word storage is {store.width} words per {self._what}, this key needs {width}")
        else:
            values = tuple(values)
            if len(values) != count:
                raise ShapeMismatch(f"payload length {len(values)} does not match shape {shape}")
            for i, v in enumerate(values):
                if not 0 <= v < limit:
                    raise ValueError(f"element {i}: {self._what} {v} out of range")
            store = WordArray.from_ints(values, width)
        if self.shared_exponent:
            if len(self.exponents) != 1:
                raise ExponentMismatch("shared-exponent batch must carry exactly one exponent")
        elif len(self.exponents) != count:
            raise ExponentMismatch("per-element batch needs one exponent per element")
        object.__setattr__(self, "_store", store)

    def __setattr__(self, name, value):
        raise AttributeError(f"{type(self).__name__} is immutable")

    @property
    def count(self) -> int:
        return _shape_count(self.shape)

    @property
    def words(self) -> WordArray:
        """The aggregated storage (not part of the reference API)."""
        return self._store

    def exponent_at(self, i: int) -> int:
        return self.exponents[0] if self.shared_exponent else self.exponents[i]


class PlaintextBatch(_Batch):
    """Encoded, not encrypted, values (batches.py:56-80)."""

    __slots__ = ()
    _what = "mantissa"

    def __init__(self, key: PublicKey, shape, exponents, mantissas, shared_exponent: bool = True):
        self._init_common(key, shape, exponents, mantissas, shared_exponent, key.n, pt_width(key))

    @property
    def mantissas(self) -> tuple:
        return self._store.ints()

    def element(self, i: int) -> EncodedNumber:
        return EncodedNumber(self.mantissas[i], self.exponent_at(i))

    def _fields(self):
        return (self.key, self.shape, self.exponents, self.shared_exponent)

    def __eq__(self, other):
        if not isinstance(other, PlaintextBatch):
            return NotImplemented
        return self._fields() == other._fields() and self._store == other._store

    def __hash__(self):
        return hash((self._fields(), self._store))

    def __repr__(self):
        return (f"PlaintextBatch(key={self.key!r}, shape={self.shape}, exponents={self.exponents[:4]}..., "
                f"shared_exponent={self.shared_exponent})")


class CiphertextBatch(_Batch):
    """Ciphertext values with their exponent metadata (batches.py:83-109)."""

    __slots__ = ("obfuscated",)
    _what = "ciphertext"

    def __init__(self, key: PublicKey, shape, exponents, payload, shared_exponent: bool = True,
                 obfuscated: bool = True):
        self._init_common(key, shape, exponents, payload, shared_exponent, key.n_squared, ct_width(key))
        object.__setattr__(self, "obfuscated", bool(obfuscated))

    @property
    def payload(self) -> tuple:
        return self._store.ints()

    def _fields(self):
        return (self.key, self.shape, self.exponents, self.shared_exponent, self.obfuscated)

    def __eq__(self, other):
        if not isinstance(other, CiphertextBatch):
            return NotImplemented
        return self._fields() == other._fields() and self._store == other._store

    def __hash__(self):
        return hash((self._fields(), self._store))

    def __repr__(self):
        return (f"CiphertextBatch(key={self.key!r}, shape={self.shape}, exponents={self.exponents[:4]}..., "
                f"shared_exponent={self.shared_exponent}, obfuscated={self.obfuscated})")


# ---- plaintext-side helpers ---------------------------------------------------------------------------

def _flatten(values):
    """(flat float64 numpy array, inferred shape); nested sequences and 1-D / 2-D numpy arrays are accepted."""
    import numpy as np
    if isinstance(values, np.ndarray):
        if values.ndim not in (1, 2):
            raise ShapeMismatch(f"bad shape {values.shape}")
        return np.ascontiguousarray(values, dtype=np.float64).ravel(), tuple(values.shape)
    values = list(values)
    if values and isinstance(values[0], (list, tuple, np.ndarray)):
        width = len(values[0])
        for row in values:
            if len(row) != width:
                raise ShapeMismatch("ragged rows")
        return np.asarray(values, dtype=np.float64).ravel(), (len(values), width)
    return np.asarray([float(v) for v in values], dtype=np.float64), (len(values),)


def encode_batch(pk: PublicKey, values, shape=None, target_exponent: int | None = None, backend=None,
                 compact: bool = False) -> PlaintextBatch:
    """Encode a flat or nested sequence (or a numpy array) under one shared exponent (batches.py:112-125): the
    minimum of the exact exponents unless a target is given.  The mantissas are produced by the GPU codec.

    compact=True (2-D input, the right operand of batch_matmul): keep the matrix in the compact resident form --
    sign + 64-bit magnitude per scalar, 9 bytes instead of a full residue -- which is all the encrypted matvec reads;
    `mantissas` are still there, materialised on demand.  The role of MiniBatchAggregator (bufferpool.py:182-226)."""
    from .backends import default_backend
    flat, inferred = _flatten(values)
    if shape is None:
        shape = inferred
    shape = tuple(shape)
    if target_exponent is None and flat.size == 0:
        target_exponent = 0
    if flat.size == 0:
        return PlaintextBatch(pk, shape, (target_exponent or 0,), (), True)
    be = backend or default_backend()
    if compact and len(shape) == 2:
        packed = be.encode_compact(pk.n, flat.reshape(shape), target_exponent)
        if packed is not None:
            return PlaintextBatch(pk, shape, (packed[1],), packed[0], True)
    # None: the exact shared exponent, found on the device
    words, used = be.encode_f64(pk.n, flat, target_exponent, row_width=shape[1] if len(shape) == 2 else 1)
    return PlaintextBatch(pk, shape, (used,), words, True)


def decode_batch(pk: PublicKey, batch: PlaintextBatch, backend=None) -> list:
    from . import operators
    if batch.shared_exponent or len(set(batch.exponents)) <= 1:
        return operators.batch_decode(pk, batch, backend)
    return [encoding.decode(pk, batch.element(i)) for i in range(batch.count)]


def require_same_key(a, b) -> None:
    if a.key != b.key:
        raise KeyMismatch("operands were built under different public keys")


def shared_exponent_of(batch) -> int:
    if batch.shared_exponent:
        return batch.exponents[0]
    first = batch.exponents[0] if batch.exponents else 0
    if any(e != first for e in batch.exponents):
        raise ExponentMismatch("operation requires one shared exponent")
    return first


def plain_rescale(batch: PlaintextBatch, new_exponent: int, backend=None) -> PlaintextBatch:
    """Exact re-grid of every element onto a finer shared exponent (batches.py:160-170), on the device."""
    from .backends import default_backend
    be = backend or default_backend()
    current = shared_exponent_of(batch)
    if new_exponent == current:
        return batch
    pk = batch.key
    if new_exponent > current:
        raise ValueError("can only rescale toward a smaller exponent")
    if batch.count == 0:
        return PlaintextBatch(pk, batch.shape, (new_exponent,), (), True)
    words, bad = be.plain_rescale(pk.n, batch.words, current - new_exponent)
    if bad >= 0:
        # the reference fails on the first offending element; let the scalar codec name the error
        encoding.rescale(pk, batch.element(bad), new_exponent)
        raise encoding.FixedPointOverflow(f"element {bad} cannot be rescaled to exponent {new_exponent}")
    return PlaintextBatch(pk, batch.shape, (new_exponent,), words, True)


def plain_mul(a: PlaintextBatch, b: PlaintextBatch, backend=None) -> PlaintextBatch:
    """Encoded product, element-wise or by one broadcast scalar: mantissas multiply mod n, exponents
    add (batches.py:173-192).  The residues are multiplied on the device."""
    from .backends import default_backend
    dev = backend or default_backend()
    require_same_key(a, b)
    pk = a.key
    if b.count == 1:
        be = b.exponent_at(0)
        prod = dev.plain_mulmod(pk.n, a.words, b.words, True) if a.count else a.words
        if a.shared_exponent:
            return PlaintextBatch(pk, a.shape, (a.exponents[0] + be,), prod, True)
        return PlaintextBatch(pk, a.shape, tuple(e + be for e in a.exponents), prod, False)
    if a.shape != b.shape:
        raise ShapeMismatch(f"{a.shape} vs {b.shape}")
    prod = dev.plain_mulmod(pk.n, a.words, b.words) if a.count else a.words
    if a.shared_exponent and b.shared_exponent:
        return PlaintextBatch(pk, a.shape, (a.exponents[0] + b.exponents[0],), prod, True)
    exps = tuple(a.exponent_at(i) + b.exponent_at(i) for i in range(a.count))
    shared = len(set(exps)) == 1
    return PlaintextBatch(pk, a.shape, exps[:1] if shared else exps, prod, shared)


def plain_add(a: PlaintextBatch, b: PlaintextBatch, backend=None) -> PlaintextBatch:
    """Encoded sum after exact alignment to the finer exponent (batches.py:195-205), on the device."""
    from .backends import default_backend
    dev = backend or default_backend()
    require_same_key(a, b)
    if a.shape != b.shape:
        raise ShapeMismatch(f"{a.shape} vs {b.shape}")
    target = min(shared_exponent_of(a), shared_exponent_of(b))
    a, b = plain_rescale(a, target, dev), plain_rescale(b, target, dev)
    total = dev.plain_addmod(a.key.n, a.words, b.words) if a.count else a.words
    return PlaintextBatch(a.key, a.shape, (target,), total, True)
