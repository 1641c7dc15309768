"""Host-side logic that needs no GPU: keys, scalar codec, batch value semantics, buffer pool, HAFB."""
import random
import struct

import pytest

import hebatch_oracle as ho
from golden_util import ints, load
from paper_2107_13797_b200 import bufferpool, encoding, paillier
from paper_2107_13797_b200.batches import (CiphertextBatch, ExponentMismatch, PlaintextBatch, ShapeMismatch,
                                           plain_add, plain_mul, plain_rescale)
from paper_2107_13797_b200.backends import get_backend
from paper_2107_13797_b200.device import WordArray, ints_to_words, words_to_ints

GOLD = load()


def test_keygen_same_stream_as_reference():
    for name, spec in GOLD["keys"].items():
        if spec["bits"] is None or spec["bits"] > 1024:
            continue
        kp = paillier.keygen(spec["bits"], paillier.default_rng(spec["seed"]), allow_insecure=True)
        assert (kp.private.p, kp.private.q) == (int(spec["p"], 16), int(spec["q"], 16))


def test_key_objects():
    kp = paillier.keypair_from_primes(5, 7)
    pk, sk = kp
    assert (pk.n, pk.n_squared, pk.g, pk.key_bits, pk.max_int) == (35, 1225, 36, 6, 11)
    assert sk.lam == 12 and pk == paillier.PublicKey(35) and hash(pk) == hash(paillier.PublicKey(35))
    ok = ho.Key(35, 5, 7)
    assert (sk._hp, sk._hq, sk._q_inv_p, sk.mu) == (ok.hp, ok.hq, ok.q_inv, ok.mu)
    with pytest.raises(ValueError):
        paillier.PrivateKey(pk, 5, 5)
    with pytest.raises(ValueError):
        paillier.keygen(512, random.Random(1))
    with pytest.raises(ValueError):
        paillier.keygen(17, random.Random(1), allow_insecure=True)
    data = paillier.export_key(kp)
    assert paillier.import_key(data).private == sk
    assert paillier.import_key(paillier.export_key(pk)) == pk
    with pytest.raises(ValueError):
        paillier.import_key({**data, "version": 2})
    assert paillier.lift_raw(pk, 3).value == 106 and paillier.lift_raw(pk, 3).obfuscated is False


def test_draw_unit_stream():
    rng_a, rng_b = random.Random(2), random.Random(2)
    assert [paillier.draw_unit(35, rng_a) for _ in range(50)] == [ho.draw_unit(35, rng_b) for _ in range(50)]


def test_scalar_codec_matches_oracle():
    ok = ho.keygen(128, random.Random(1234))
    pk = paillier.PublicKey(ok.n)
    rng = random.Random(4)
    for _ in range(200):
        v = rng.uniform(-1000, 1000) * 10 ** rng.randint(-8, 3)
        for target in (None, -8, -20, 2):
            try:
                want = ho.encode(ok, v, target)
            except ho.Overflow:
                with pytest.raises(encoding.FixedPointOverflow):
                    encoding.encode(pk, v, target)
                continue
            got = encoding.encode(pk, v, target)
            assert (got.mantissa, got.exponent) == want
            assert encoding.decode(pk, got) == ho.decode(ok, *want)
    e = encoding.encode(pk, 0.5)
    assert (e.mantissa, e.exponent) == (8, -1)
    assert encoding.rescale(pk, e, -3).mantissa == 8 * 256
    with pytest.raises(ValueError):
        encoding.rescale(pk, e, 0)
    a, b = encoding.align(pk, encoding.encode(pk, 1.0), e)
    assert a.exponent == b.exponent == -1
    tiny = paillier.PublicKey(35)
    for m in range(11, 25):
        with pytest.raises(encoding.FixedPointOverflow):
            encoding.signed_mantissa(tiny, encoding.EncodedNumber(m, 0))
    with pytest.raises(ValueError):
        encoding.encode(pk, float("nan"))
    low = encoding.EncodedNumber(3 * 16 ** 10, -50)
    r = encoding.renormalize(pk, low, -32)
    assert (r.mantissa, r.exponent) == ho.renormalize(ok, low.mantissa, -50, -32)


def test_batch_value_semantics():
    pk = paillier.PublicKey(35)
    a = CiphertextBatch(pk, (2, 2), (-1,), (1, 2, 3, 683), True)
    assert a.count == 4 and a.payload == (1, 2, 3, 683) and a.exponent_at(3) == -1 and a.obfuscated
    assert a == CiphertextBatch(pk, [2, 2], [-1], [1, 2, 3, 683], True, True)
    assert a != CiphertextBatch(pk, (2, 2), (-1,), (1, 2, 3, 683), True, False)
    assert hash(a) == hash(CiphertextBatch(pk, (2, 2), (-1,), (1, 2, 3, 683)))
    with pytest.raises(ValueError, match="element 2"):
        CiphertextBatch(pk, (3,), (0,), (1, 2, 1225), True)
    with pytest.raises(ShapeMismatch):
        CiphertextBatch(pk, (3,), (0,), (1, 2), True)
    with pytest.raises(ExponentMismatch):
        PlaintextBatch(pk, (2,), (0, 1), (1, 2), True)
    with pytest.raises(ExponentMismatch):
        PlaintextBatch(pk, (2,), (0,), (1, 2), False)
    with pytest.raises(AttributeError):
        a.shape = (4,)
    p = PlaintextBatch(pk, (2,), (0, -1), (3, 34), False)
    assert p.element(1) == encoding.EncodedNumber(34, -1) and p.mantissas == (3, 34)
    w = WordArray.from_numpy(ints_to_words([5, 6], 1))
    assert PlaintextBatch(pk, (2,), (0,), w, True).mantissas == (5, 6)
    assert words_to_ints(ints_to_words([2 ** 70 + 3, 0], 3)) == (2 ** 70 + 3, 0)


def test_backend_registry():
    with pytest.raises(ValueError):
        get_backend("naive")
    with pytest.raises(ValueError):
        get_backend("bogus")
    assert get_backend("cuda").name == "cuda"


def test_buffer_pool_reuse_and_gc():
    pool = bufferpool.BufferPool(capacity_bytes=1000)
    a = pool.alloc(400)
    b = pool.alloc(400)
    assert pool.stats.fresh_allocations == 2 and pool.retained_bytes == 800
    pool.free(a)
    again = pool.alloc(400)
    assert again is a and a.reuses == 1 and pool.stats.reuse_hits == 1
    with pytest.raises(bufferpool.PoolError):
        pool.free(bufferpool.BufferHandle(99, 8))
    pool.free(a)
    with pytest.raises(bufferpool.PoolError):
        pool.free(a)
    c = pool.alloc(500)                 # 1300 retained > 1000: the free 400-byte buffer goes
    assert pool.stats.evictions == 1 and pool.retained_bytes == 900 and not c.available
    pool.free(b)
    pool.free(c)
    assert pool.gc() == []
    with pytest.raises(ValueError):
        pool.alloc(0)
    # random alloc/free interleaving keeps the books straight (tests/test_bufferpool.py:63-75)
    rng = random.Random(0)
    pool = bufferpool.BufferPool(capacity_bytes=4096)
    out = []
    for _ in range(2000):
        if out and rng.random() < 0.5:
            pool.free(out.pop(rng.randrange(len(out))))
        else:
            out.append(pool.alloc(rng.choice((64, 128, 256))))
        assert pool.retained_bytes == sum(h.size_bytes for h in pool._all.values())


def test_hafb_golden_bytes_and_errors():
    pk = paillier.PublicKey(35)
    one = CiphertextBatch(pk, (1,), (-3,), (683,), True)
    blob = bufferpool.serialize_to_bytes(one)
    assert blob == ho.hafb_serialize(6, (1,), (-3,), [683], True)
    assert blob[-2:] == bytes([0xab, 0x02]) and len(blob) == 38                     # test_bufferpool.py:195-206
    assert len(bufferpool.serialize_to_bytes(CiphertextBatch(pk, (0,), (0,), (), True))) == 36
    assert bufferpool.deserialize(blob, pk) == one
    assert bufferpool.serialized_size(1, 6, True) == 38 and bufferpool.word_size(2048) == 512
    with pytest.raises(bufferpool.CorruptHeader):
        bufferpool.deserialize(b"XXXX" + blob[4:], pk)
    with pytest.raises(bufferpool.VersionMismatch):
        bufferpool.deserialize(blob[:4] + struct.pack("<I", 2) + blob[8:], pk)
    with pytest.raises(bufferpool.TruncatedPayload):
        bufferpool.deserialize(blob[:-1], pk)
    with pytest.raises(bufferpool.CorruptHeader):
        bufferpool.deserialize(blob[:10], pk)
    with pytest.raises(bufferpool.SerializationError):
        bufferpool.deserialize(blob, paillier.PublicKey(143))
    with pytest.raises(ValueError, match="element 0"):
        bufferpool.deserialize(blob[:-2] + struct.pack("<H", 1225), pk)
    pool = bufferpool.BufferPool()
    with pytest.raises(bufferpool.UndersizedBuffer):
        bufferpool.serialize(one, pool.alloc(10))
    buf = pool.alloc(64)
    ser = bufferpool.serialize(one, buf)
    assert ser.length == 38 and ser.to_bytes() == blob and ser.header == (1, 6, (1,), True)
    assert bufferpool.deserialize(ser, pk, pool) == one and buf.available
    with pytest.raises(ShapeMismatch):
        bufferpool.serialize_to_bytes(CiphertextBatch(pk, (2, 0), (0,), (), True))


def test_hafb_roundtrips_and_reference_bytes():
    rng = random.Random(5)
    for case in GOLD["cases"]:
        if case["op"] != "hafb":
            continue
        k = GOLD["keys"][case["key"]]
        pk = paillier.PublicKey(int(k["n"], 16))
        batch = CiphertextBatch(pk, tuple(case["shape"]), case["exponents"], ints(case["payload"]), True)
        assert bufferpool.serialize_to_bytes(batch).hex() == case["bytes"]
    pk = paillier.PublicKey(ho.keygen(128, random.Random(1234)).n)
    for _ in range(100):
        count = rng.randrange(0, 9)
        shared = rng.random() < 0.5
        shape = (count,) if rng.random() < 0.5 or count == 0 else (1, count)
        exps = (rng.randrange(-40, 5),) if shared else tuple(rng.randrange(-40, 5) for _ in range(count))
        batch = CiphertextBatch(pk, shape, exps, [rng.randrange(pk.n_squared) for _ in range(count)], shared,
                                obfuscated=True)
        blob = bufferpool.serialize_to_bytes(batch)
        assert blob == ho.hafb_serialize(pk.key_bits, shape, exps, batch.payload, shared)
        assert bufferpool.deserialize(blob, pk) == batch


def test_full_batch_row_selection_skips_the_copy():
    """flr.HeteroFederation._take: X[idx] without the gather when idx is every row in order, a copy otherwise."""
    import numpy as np
    from paper_2107_13797_b200.flr import HeteroFederation
    X = np.arange(12.0).reshape(6, 2)
    assert HeteroFederation._take(X, np.arange(6)) is X
    for idx in (np.array([0, 1, 2, 3, 5, 4]), np.arange(5), np.array([0, 2, 4]), np.array([5, 4, 3, 2, 1, 0]),
                np.array([0, 1, 2, 2, 4, 5])):
        got = HeteroFederation._take(X, idx)
        assert got is not X and np.array_equal(got, X[idx])
    y = np.arange(6.0)
    assert HeteroFederation._take(y, np.arange(6)) is y


def test_native_draw_stream_equals_cpython_without_a_gpu():
    """hb_mt19937_randrange1 is host code: CPython's randrange(1, n) stream reproduced word for word from getstate(),
    across state refills, for moduli whose bit length is and is not a multiple of 32, and the generator state handed
    back equals CPython's own after the same draws.  hb_secure_randrange1 (OS entropy): values in [1, n)."""
    import ctypes
    import random

    import numpy as np
    from paper_2107_13797_b200 import _native
    lib = _native.lib()
    for n in (35, 3, 2 ** 61 - 1, (1 << 100) + 7, (1 << 255) + 95, (1 << 2047) + 12345, (1 << 2048) - 159):
        wn = (n.bit_length() + 31) // 32
        n_words = np.frombuffer(n.to_bytes(4 * wn, "little"), dtype=np.uint32).copy()
        rng = random.Random(n % 1000)
        rng.random()                                              # start somewhere inside the state
        saved = rng.getstate()
        state = np.array(saved[1][:624], dtype=np.uint32)
        index = ctypes.c_int(saved[1][624])
        count = 700                                               # 700 x 64 words: dozens of refills
        out = np.empty((count, wn), np.uint32)
        _native.check(lib.hb_mt19937_randrange1(state.ctypes.data, ctypes.byref(index), n_words.ctypes.data, wn,
                                                count, out.ctypes.data))
        want = [rng.randrange(1, n) for _ in range(count)]
        assert [int.from_bytes(r.tobytes(), "little") for r in out] == want
        after = rng.getstate()[1]
        assert tuple(int(v) for v in state) == after[:624] and index.value == after[624]
        _native.check(lib.hb_secure_randrange1(n_words.ctypes.data, wn, count, out.ctypes.data))
        got = [int.from_bytes(r.tobytes(), "little") for r in out]
        assert all(1 <= v < n for v in got)
        assert n < 100 or len(set(got)) > count // 2


def test_compact_scalars_materialise_the_reference_residues():
    """device.CompactScalars.numpy(): sign + 64-bit magnitude, stored by column, back to the residues the reference
    keeps (n - |k| for negatives) -- including moduli whose zero words make the borrow run (host logic, no GPU)."""
    import random

    import numpy as np
    import torch
    from paper_2107_13797_b200.device import CompactScalars
    rng = random.Random(1)
    for n in ((1 << 2047) + 12345, (1 << 127) + (1 << 70) + 5, rng.getrandbits(2048) | (1 << 2047) | 1,
              (1 << 200) + 3, (1 << 255) + (1 << 64) + 1):
        rows, cols = 31, 5
        mags = [rng.getrandbits(rng.choice((1, 20, 52, 63, 64))) for _ in range(rows * cols)]
        mags[:4] = [0, 1, 2 ** 64 - 1, 2 ** 63]
        negs = [rng.random() < 0.5 and m != 0 for m in mags]
        by_col = np.array(mags, dtype=np.uint64).reshape(rows, cols).T.reshape(-1).copy()
        neg_col = np.array(negs, dtype=np.uint8).reshape(rows, cols).T.reshape(-1).copy()
        cs = CompactScalars(n, rows, cols, torch.from_numpy(by_col.view(np.int64)), torch.from_numpy(neg_col), 64,
                            int(sum(negs)))
        got = [int.from_bytes(r.tobytes(), "little") for r in cs.numpy()]
        assert got == [(n - m) % n if s else m for m, s in zip(mags, negs)]
