"""GPU parity: every operator of paper_2107_13797_b200.operators against the CPU oracle, bit for bit.

Mirrors the reference's tests/test_operators.py (golden 683, round trips, commutation, negative scalars,
reduction-order independence, matmul == mul + sum, seed determinism, decrypt renormalisation) with the
oracle in the role of the naive backend.
"""
import random

import pytest

import hebatch_oracle as ho
from paper_2107_13797_b200 import operators as ops
from paper_2107_13797_b200 import paillier
from paper_2107_13797_b200.backends import CudaBackend
from paper_2107_13797_b200.batches import (CiphertextBatch, ExponentMismatch, PlaintextBatch, ShapeMismatch,
                                           encode_batch)

pytestmark = pytest.mark.gpu

KEYS = ["tiny", "k128", "k512", "k1024", "k2048", "k3072"]
COUNT = {"tiny": 12, "k128": 37, "k512": 21, "k1024": 13, "k2048": 9, "k3072": 5}


class SequenceRng(random.Random):
    """Feeds fixed obfuscation factors (the reference's test double, tests/test_operators.py:30-37)."""

    def __init__(self, seq):
        super().__init__(0)
        self._seq = list(seq)

    def randrange(self, a, b=None, step=1):
        return self._seq.pop(0)


def product_keys(ok):
    kp = paillier.keypair_from_primes(ok.p, ok.q)
    return kp.public, kp.private


def rand_plain(ok, pk, count, rng, shape=None, exponent=-8):
    ms = [rng.randrange(ok.n) for _ in range(count)]
    return PlaintextBatch(pk, shape or (count,), (exponent,), ms, True), ms


def encrypt_oracle(ok, ms, seed):
    rng = random.Random(seed)
    rs = [ho.draw_unit(ok.n, rng) for _ in ms]
    return ho.k_encrypt(ok, list(zip(ms, rs)))


def test_golden_683(okeys):
    ok = okeys("tiny")
    pk, sk = product_keys(ok)
    plain = PlaintextBatch(pk, (1,), (0,), (3,), True)
    out = ops.batch_encrypt(pk, plain, SequenceRng([2]))
    assert out.payload == (683,)                      # tests/test_operators.py:63-70
    assert out.obfuscated is True
    assert ops.batch_decrypt(sk, out).mantissas == (3,)
    assert paillier.encrypt_raw(pk, 3, 2).value == 683    # tests/test_paillier.py:79-84
    assert paillier.encrypt_raw(pk, 0, 1).value == 1
    assert paillier.decrypt_raw(sk, paillier.RawCiphertext(683)) == 3
    assert paillier.decrypt_raw(sk, paillier.RawCiphertext(1)) == 0


def test_tiny_key_exhaustive(okeys):
    """Every plaintext and every unit r of n = 35 (tests/test_paillier.py:152-167)."""
    ok = okeys("tiny")
    pk, sk = product_keys(ok)
    units = [r for r in range(1, 35) if r % 5 and r % 7]
    ms = [m for m in range(35) for _ in units]
    rs = [r for _ in range(35) for r in units]
    got = ops.raw_encrypt(pk, ms, rs)
    assert got == ho.k_encrypt(ok, list(zip(ms, rs)))
    assert ops.raw_decrypt(sk, got) == ms
    # all of Z_{n^2}, units or not, through the CRT decryption
    allc = list(range(35 * 35))
    assert ops.raw_decrypt(sk, allc) == ho.k_decrypt(ok, allc)


@pytest.mark.parametrize("name", KEYS)
def test_encrypt_decrypt_obfuscate(okeys, name):
    ok = okeys(name)
    pk, sk = product_keys(ok)
    rng = random.Random(5)
    count = COUNT[name]
    plain, ms = rand_plain(ok, pk, count, rng)
    ms[0] = 0
    ms[-1] = ok.n - 1
    plain = PlaintextBatch(pk, (count,), (-8,), ms, True)
    enc = ops.batch_encrypt(pk, plain, random.Random(77))
    want = encrypt_oracle(ok, ms, 77)
    assert list(enc.payload) == want
    assert enc.shape == (count,) and enc.exponents == (-8,) and enc.obfuscated
    dec = ops.batch_decrypt(sk, enc)
    assert list(dec.mantissas) == ms
    assert list(dec.mantissas) == ho.k_decrypt(ok, want)
    assert [ho.decrypt_textbook(ok, c) for c in want[:4]] == ms[:4]
    ob = ops.batch_obfuscate(pk, enc, random.Random(78))
    rng2 = random.Random(78)
    rs = [ho.draw_unit(ok.n, rng2) for _ in ms]
    assert list(ob.payload) == ho.k_obfuscate(ok, list(zip(want, rs)))
    assert list(ops.batch_decrypt(sk, ob).mantissas) == ms
    # same seed, same bits (tests/test_operators.py:299-307)
    assert ops.batch_encrypt(pk, plain, random.Random(77)) == enc


@pytest.mark.parametrize("name", KEYS)
def test_add(okeys, name):
    ok = okeys(name)
    pk, sk = product_keys(ok)
    rng = random.Random(6)
    count = COUNT[name]
    pa, ma = rand_plain(ok, pk, count, rng)
    pb, mb = rand_plain(ok, pk, count, rng)
    ca = ops.batch_encrypt(pk, pa, random.Random(1))
    cb = ops.batch_encrypt(pk, pb, random.Random(2))
    s = ops.batch_add(pk, ca, cb)
    assert list(s.payload) == ho.k_add(ok, list(zip(ca.payload, cb.payload)))
    assert ops.batch_add(pk, cb, ca).payload == s.payload          # commutes bit-exactly
    assert list(ops.batch_decrypt(sk, s).mantissas) == [(x + y) % ok.n for x, y in zip(ma, mb)]
    # plaintext operand: lifted (1 + m n), flag copied from a (operators.py:209-214)
    unob = CiphertextBatch(pk, ca.shape, ca.exponents, ca.payload, True, obfuscated=False)
    sp = ops.batch_add(pk, unob, pb)
    assert list(sp.payload) == ho.k_add(ok, [(c, ho.lift(ok, m)) for c, m in zip(ca.payload, mb)])
    assert sp.obfuscated is False
    # scalar plaintext broadcast
    one = PlaintextBatch(pk, (1,), (-8,), (mb[0],), True)
    sb = ops.batch_add(pk, ca, one)
    assert list(sb.payload) == ho.k_add(ok, [(c, ho.lift(ok, mb[0])) for c in ca.payload])
    with pytest.raises(ExponentMismatch):
        ops.batch_add(pk, ca, CiphertextBatch(pk, cb.shape, (-9,), cb.payload, True))
    with pytest.raises(ShapeMismatch):
        ops.batch_add(pk, ca, CiphertextBatch(pk, (count, 1), cb.exponents, cb.payload, True))


def small_scalars(ok, count, rng, bits=40):
    """Residues of signed magnitudes, about half negative (n - |k|)."""
    out = []
    for i in range(count):
        mag = rng.getrandbits(min(bits, ok.max_int.bit_length() - 1))
        out.append(mag if i % 2 == 0 else (ok.n - mag) % ok.n)
    return out


@pytest.mark.parametrize("name", KEYS)
def test_mul_plain(okeys, name):
    ok = okeys(name)
    pk, sk = product_keys(ok)
    rng = random.Random(8)
    rows, cols = 3, max(2, COUNT[name] // 3)
    count = rows * cols
    pa, ma = rand_plain(ok, pk, count, rng, shape=(rows, cols))
    ca = ops.batch_encrypt(pk, pa, random.Random(3))
    cpay = list(ca.payload)
    # same-shape, mixed signs
    ks = small_scalars(ok, count, rng)
    kb = PlaintextBatch(pk, (rows, cols), (-3,), ks, True)
    out = ops.batch_mul_plain(pk, ca, kb)
    assert list(out.payload) == ho.k_mul(ok, list(zip(cpay, ks)))
    assert out.exponents == (-11,) and out.shape == (rows, cols)
    assert list(ops.batch_decrypt(sk, out).mantissas) == [m * k % ok.n for m, k in zip(ma, ks)]
    # scalar broadcast: positive, negative, zero, the band edge (positive branch), an overflow-band residue
    for k in (4 % ok.n, (ok.n - 8) % ok.n, 0, ok.n - ok.max_int, ok.n // 2):
        sc = PlaintextBatch(pk, (1,), (-1,), (k,), True)
        out = ops.batch_mul_plain(pk, ca, sc)
        assert list(out.payload) == ho.k_mul(ok, [(c, k) for c in cpay]), k
    # row vector over the columns
    kr = small_scalars(ok, cols, rng, bits=17)
    out = ops.batch_mul_plain(pk, ca, PlaintextBatch(pk, (cols,), (0,), kr, True))
    assert list(out.payload) == ho.k_mul(ok, [(c, kr[i % cols]) for i, c in enumerate(cpay)])
    # full-width random residues as scalars (acceptance criterion 3 does this on n = 35)
    kf = [rng.randrange(ok.n) for _ in range(count)]
    out = ops.batch_mul_plain(pk, ca, PlaintextBatch(pk, (rows, cols), (0,), kf, True))
    assert list(out.payload) == ho.k_mul(ok, list(zip(cpay, kf)))
    with pytest.raises(ShapeMismatch):
        ops.batch_mul_plain(pk, ca, PlaintextBatch(pk, (cols + 1,), (0,), [1] * (cols + 1), True))
    # hmul_raw exponentiates by the residue itself
    k = ok.n - 5
    assert paillier.hmul_raw(pk, paillier.RawCiphertext(cpay[0]), k).value == ho.gmp.powmod(cpay[0], k, ok.n2)


def test_mul_plain_non_unit_raises(okeys):
    ok = okeys("k128")
    pk, _ = product_keys(ok)
    bad = CiphertextBatch(pk, (2,), (0,), (ok.p * 3, 5), True)
    with pytest.raises(ZeroDivisionError):
        ops.batch_mul_plain(pk, bad, PlaintextBatch(pk, (1,), (0,), (ok.n - 2,), True))


@pytest.mark.parametrize("name", KEYS)
def test_sum(okeys, name):
    ok = okeys(name)
    pk, sk = product_keys(ok)
    rng = random.Random(9)
    rows, cols = 5, max(2, COUNT[name] // 4)
    count = rows * cols
    pa, ma = rand_plain(ok, pk, count, rng, shape=(rows, cols))
    ca = ops.batch_encrypt(pk, pa, random.Random(4))
    cpay = list(ca.payload)
    tot = ops.batch_sum(pk, ca)
    assert tot.payload == tuple(ho.k_product(ok, [cpay])) and tot.shape == (1,)
    s0 = ops.batch_sum(pk, ca, axis=0)
    assert list(s0.payload) == ho.k_product(ok, [[cpay[r * cols + c] for r in range(rows)] for c in range(cols)])
    assert s0.shape == (cols,)
    s1 = ops.batch_sum(pk, ca, axis=1)
    assert list(s1.payload) == ho.k_product(ok, [[cpay[r * cols + c] for c in range(cols)] for r in range(rows)])
    assert list(ops.batch_decrypt(sk, tot).mantissas) == [sum(ma) % ok.n]
    # order independence (tests/test_operators.py:199-205)
    perm = list(range(count))
    random.Random(1).shuffle(perm)
    shuffled = CiphertextBatch(pk, (count,), ca.exponents, [cpay[i] for i in perm], True)
    assert ops.batch_sum(pk, shuffled).payload == tot.payload
    with pytest.raises(ShapeMismatch):
        ops.batch_sum(pk, shuffled, axis=0)


def test_sum_long(okeys):
    """Multi-pass reduction (more than one chunk level) at 1024 bits, ciphertexts tiled from a pool."""
    ok = okeys("k1024")
    pk, _ = product_keys(ok)
    rng = random.Random(10)
    pool = encrypt_oracle(ok, [rng.randrange(ok.n) for _ in range(16)], 5)
    n_el = 5000
    pay = [pool[(i * 7) % 16] for i in range(n_el)]
    ca = CiphertextBatch(pk, (n_el,), (0,), pay, True)
    assert ops.batch_sum(pk, ca).payload == tuple(ho.k_product(ok, [pay]))
    ca2 = CiphertextBatch(pk, (1250, 4), (0,), pay, True)
    assert list(ops.batch_sum(pk, ca2, axis=0).payload) == ho.k_product(
        ok, [[pay[r * 4 + c] for r in range(1250)] for c in range(4)])


@pytest.mark.parametrize("name", KEYS)
def test_matmul(okeys, name):
    ok = okeys(name)
    pk, sk = product_keys(ok)
    rng = random.Random(11)
    inner, d = max(4, COUNT[name]), 3
    pa, ma = rand_plain(ok, pk, inner, rng, exponent=-4)
    ca = ops.batch_encrypt(pk, pa, random.Random(6))
    cpay = list(ca.payload)
    ks = small_scalars(ok, inner * d, rng, bits=52)
    x = PlaintextBatch(pk, (inner, d), (-13,), ks, True)
    out = ops.batch_matmul(pk, ca, x)
    rows = (tuple(cpay),)
    cols = tuple(tuple(ks[t * d + j] for t in range(inner)) for j in range(d))
    assert list(out.payload) == ho.k_dot(ok, rows, cols, [(0, j) for j in range(d)])
    assert out.shape == (d,) and out.exponents == (-17,)
    # matmul == mul then sum, bit for bit (tests/test_operators.py:236-246)
    tiled = CiphertextBatch(pk, (inner, d), ca.exponents, [c for c in cpay for _ in range(d)], True)
    via = ops.batch_sum(pk, ops.batch_mul_plain(pk, tiled, x), axis=0)
    assert via.payload == out.payload
    want = [sum(ma[t] * ks[t * d + j] for t in range(inner)) % ok.n for j in range(d)]
    assert list(ops.batch_decrypt(sk, out).mantissas) == want
    # 2-D left operand and full-width scalars (general path)
    a2 = CiphertextBatch(pk, (2, inner // 2), ca.exponents, cpay[:2 * (inner // 2)], True)
    kf = [rng.randrange(ok.n) for _ in range((inner // 2) * 2)]
    x2 = PlaintextBatch(pk, (inner // 2, 2), (0,), kf, True)
    out2 = ops.batch_matmul(pk, a2, x2)
    rows2 = tuple(tuple(cpay[i * (inner // 2) + t] for t in range(inner // 2)) for i in range(2))
    cols2 = tuple(tuple(kf[t * 2 + j] for t in range(inner // 2)) for j in range(2))
    assert list(out2.payload) == ho.k_dot(ok, rows2, cols2, [(i, j) for i in range(2) for j in range(2)])
    assert out2.shape == (2, 2)


def test_matmul_wide(okeys):
    """Bucket path with several segments, windows and both signs: 700 x 5 at 512 bits."""
    ok = okeys("k512")
    pk, _ = product_keys(ok)
    rng = random.Random(12)
    pool = encrypt_oracle(ok, [rng.randrange(ok.n) for _ in range(32)], 7)
    inner, d = 700, 5
    cpay = [pool[rng.randrange(32)] for _ in range(inner)]
    ca = CiphertextBatch(pk, (inner,), (0,), cpay, True)
    ks = small_scalars(ok, inner * d, rng, bits=61)
    ks[3] = 0
    x = PlaintextBatch(pk, (inner, d), (0,), ks, True)
    out = ops.batch_matmul(pk, ca, x)
    cols = tuple(tuple(ks[t * d + j] for t in range(inner)) for j in range(d))
    assert list(out.payload) == ho.k_dot(ok, (tuple(cpay),), cols, [(0, j) for j in range(d)])


def test_codec(okeys):
    ok = okeys("k1024")
    pk, _ = product_keys(ok)
    rng = random.Random(13)
    vals = [rng.uniform(-100.0, 100.0) for _ in range(300)] + [0.0, -0.0, 0.5, -0.5, 1e-30, 2.0 ** 60, -3.75,
                                                                 0.03125 * 3, 5e-324, 1.5 * 2 ** -8, 2.5 * 2 ** -8]
    for exponent in (-8, -16, 0, 3, -40):
        got = ops.batch_encode(pk, vals, exponent)
        want = [ho.encode(ok, v, exponent)[0] for v in vals]
        assert list(got.mantissas) == want, exponent
        back = ops.batch_decode(pk, got)
        assert back == [ho.decode(ok, m, exponent) for m in want]
    # default exponent = min exact exponent: exact round trip (tests/test_encoding.py:83-89)
    eb = encode_batch(pk, vals[:50])
    assert ops.batch_decode(pk, eb) == vals[:50]
    assert eb.exponents[0] == min(ho.exact_exponent(v) for v in vals[:50])
    # big mantissas: correct rounding of > 53-bit magnitudes, both signs
    big = [rng.randrange(ok.max_int) for _ in range(64)] + [ok.n - rng.randrange(1, ok.max_int) for _ in range(64)]
    pb = PlaintextBatch(pk, (128,), (-200,), big, True)
    assert ops.batch_decode(pk, pb) == [ho.decode(ok, m, -200) for m in big]
    from paper_2107_13797_b200.encoding import FixedPointOverflow
    with pytest.raises(FixedPointOverflow):
        ops.batch_encode(pk, [1.0, 2.0 ** 1100 if False else 1e300], -200)
    with pytest.raises(FixedPointOverflow):
        ops.batch_decode(pk, PlaintextBatch(pk, (2,), (0,), (1, ok.n // 2), True))


def test_codec_tiny_band(okeys):
    """n = 35: max_int = 11, overflow band [11, 24] (tests/test_encoding.py:73-81)."""
    ok = okeys("tiny")
    pk, _ = product_keys(ok)
    from paper_2107_13797_b200.encoding import FixedPointOverflow
    assert list(ops.batch_encode(pk, [10.0, -10.0, 0.5], 0).mantissas) == [10, 25, 0]
    assert list(ops.batch_encode(pk, [0.5, 1.5, 2.5, -0.5, -1.5], 0).mantissas) == [0, 2, 2, 0, 33]
    with pytest.raises(FixedPointOverflow):
        ops.batch_encode(pk, [11.0], 0)
    assert ops.batch_decode(pk, PlaintextBatch(pk, (3,), (0,), (10, 25, 0), True)) == [10.0, -10.0, 0.0]
    for m in (11, 24):
        with pytest.raises(FixedPointOverflow):
            ops.batch_decode(pk, PlaintextBatch(pk, (1,), (0,), (m,), True))


def test_decrypt_renormalises(okeys):
    """Exponents below the floor are lifted after decryption (tests/test_operators.py:310-321)."""
    ok = okeys("k512")
    pk, sk = product_keys(ok)
    vals = [0.75, -1.5, 3.0]
    plain = encode_batch(pk, vals, target_exponent=-40)
    enc = ops.batch_encrypt(pk, plain, random.Random(1))
    dec = ops.batch_decrypt(sk, enc)
    want = [ho.renormalize(ok, m, -40) for m in plain.mantissas]
    assert [(e.mantissa, e.exponent) for e in (dec.element(i) for i in range(3))] == want
    assert ops.batch_decrypt(sk, enc, min_exponent=-64).exponents == (-40,)


def test_backend_run_contract(okeys):
    """Level-1 plug-in: CudaBackend.run(kernel, common, items) with the reference's common tuples."""
    ok = okeys("k512")
    pk, sk = product_keys(ok)
    be = CudaBackend()
    rng = random.Random(14)
    ms = [rng.randrange(ok.n) for _ in range(6)]
    rs = [ho.draw_unit(ok.n, rng) for _ in ms]
    cs = be.run(ops._k_encrypt, (ok.n, ok.n2), list(zip(ms, rs)))
    assert cs == ho.k_encrypt(ok, list(zip(ms, rs)))
    assert be.run(ops._k_obfuscate, (ok.n, ok.n2), list(zip(cs, rs))) == ho.k_obfuscate(ok, list(zip(cs, rs)))
    common = (ok.p, ok.q, ok.p2, ok.q2, ok.hp, ok.hq, ok.q_inv)
    assert be.run(ops._k_decrypt, common, cs) == ms
    ks = small_scalars(ok, 6, rng)
    assert be.run(ops._k_mul, (ok.n, ok.n2, ok.neg_band), list(zip(cs, ks))) == ho.k_mul(ok, list(zip(cs, ks)))
    assert be.run(ops._k_add, ok.n2, list(zip(cs, cs[::-1]))) == ho.k_add(ok, list(zip(cs, cs[::-1])))
    groups = [tuple(cs[:3]), tuple(cs[3:]), ()]
    assert be.run(ops._k_product, ok.n2, groups) == ho.k_product(ok, groups)
    rows = (tuple(cs[:3]), tuple(cs[3:]))
    cols = (tuple(ks[:3]), tuple(ks[3:]))
    items = [(0, 0), (1, 1), (0, 1)]
    assert be.run(ops._k_dot, (ok.n, ok.n2, ok.neg_band, rows, cols), items) == ho.k_dot(ok, rows, cols, items)
    assert be.run(ops._k_encode, (pk, -8), [1.5, -2.25]) == [ho.encode(ok, v, -8)[0] for v in (1.5, -2.25)]
    assert be.run(ops._k_decode, (pk, -8), [ho.encode(ok, v, -8)[0] for v in (1.5, -2.25)]) == [1.5, -2.25]
    assert be.run(ops._k_add, ok.n2, []) == []


def test_empty_batches(okeys):
    ok = okeys("k128")
    pk, sk = product_keys(ok)
    empty = PlaintextBatch(pk, (0,), (0,), (), True)
    enc = ops.batch_encrypt(pk, empty, random.Random(1))
    assert enc.count == 0 and enc.payload == ()
    assert ops.batch_decrypt(sk, enc).mantissas == ()
    assert ops.batch_sum(pk, enc).payload == (1,)
    assert ops.batch_add(pk, enc, enc).payload == ()


def test_native_unit_stream_matches_python(okeys):
    """The native MT19937 replay yields draw_unit's values and leaves the generator where Python would
    (paillier.py:173-178); generators that are not plain random.Random take the per-element path."""
    ok = okeys("k1024")
    pk, _ = product_keys(ok)
    be = CudaBackend()
    a, b = random.Random(99), random.Random(99)
    got = be.draw_units(pk.n, 300, a).ints()
    assert list(got) == [ho.draw_unit(ok.n, b) for _ in range(300)]
    assert a.getstate() == b.getstate() and a.random() == b.random()
    # a second call continues the same stream
    assert list(be.draw_units(pk.n, 5, a).ints()) == [ho.draw_unit(ok.n, b) for _ in range(5)]
    seq = SequenceRng([7, 11, 13, 17])
    assert be.draw_units(pk.n, 4, seq).ints() == (7, 11, 13, 17)
    tiny = okeys("tiny")
    c, d = random.Random(3), random.Random(3)
    assert list(be.draw_units(35, 40, c).ints()) == [ho.draw_unit(35, d) for _ in range(40)]
    assert c.getstate() == d.getstate()


# ---- plaintext-side residue algebra on the device (reference batches.py:160-205, encoding.py:104-113) -------

def test_plain_algebra_small(okeys):
    from paper_2107_13797_b200.batches import plain_add, plain_mul, plain_rescale
    ok = okeys("k128")
    pk = paillier.PublicKey(ok.n)
    a = PlaintextBatch(pk, (3,), (-2,), (5, ok.n - 7, 0), True)
    b = PlaintextBatch(pk, (3,), (-1,), (2, 3, ok.n - 1), True)
    r = plain_rescale(b, -2)
    assert r.mantissas == (32, 48, ok.n - 16) and r.exponents == (-2,)
    s = plain_add(a, b)
    assert s.mantissas == (37, 41, ok.n - 16) and s.exponents == (-2,)
    m = plain_mul(a, b)
    assert m.mantissas == (10, (ok.n - 21), 0) and m.exponents == (-3,) and m.shared_exponent
    k = PlaintextBatch(pk, (1,), (-1,), (4,), True)
    assert plain_mul(a, k).mantissas == (20, ok.n - 28, 0)
    with pytest.raises(ShapeMismatch):
        plain_add(a, PlaintextBatch(pk, (2,), (0,), (1, 2), True))
    with pytest.raises(ValueError):
        plain_rescale(a, -1)


@pytest.mark.parametrize("name", KEYS)
def test_plain_algebra_matches_oracle(okeys, name):
    from paper_2107_13797_b200.batches import plain_add, plain_mul, plain_rescale
    ok = okeys(name)
    pk = paillier.PublicKey(ok.n)
    rng = random.Random(sum(map(ord, name)))
    count = 67
    n, max_int = ok.n, ok.n // 3
    xs = [rng.randrange(n) for _ in range(count)]
    ys = [rng.randrange(n) for _ in range(count)]
    xs[:4] = [0, 1, n - 1, n // 2]
    ys[:4] = [n - 1, n - 1, n - 1, 2]
    a = PlaintextBatch(pk, (count,), (-3,), tuple(xs), True)
    b = PlaintextBatch(pk, (count,), (-5,), tuple(ys), True)
    prod = plain_mul(a, b)
    assert prod.mantissas == tuple(x * y % n for x, y in zip(xs, ys)) and prod.exponents == (-8,)
    k = PlaintextBatch(pk, (1,), (-1,), (ys[5],), True)
    assert plain_mul(a, k).mantissas == tuple(x * ys[5] % n for x in xs)
    same = PlaintextBatch(pk, (count,), (-3,), tuple(ys), True)
    assert plain_add(a, same).mantissas == tuple((x + y) % n for x, y in zip(xs, ys))
    # rescale: small signed magnitudes (what the protocols hold), every shift 0..40 digits that still fits
    bits = max(2, max_int.bit_length() - 1)
    for digits in (1, 2, 7, 8, 9, 16, 33):
        room = bits - 4 * digits
        if room < 2:
            continue
        mags = [rng.getrandbits(rng.randrange(1, room)) for _ in range(count)]
        mags[0], mags[1] = 0, (1 << (room - 1)) - 1
        res = [m if rng.random() < 0.5 else (n - m) % n for m in mags]
        pb = PlaintextBatch(pk, (count,), (-2,), tuple(res), True)
        got = plain_rescale(pb, -2 - digits)
        assert got.mantissas == tuple(ho.rescale(ok, m, -2, -2 - digits) for m in res), (name, digits)
        assert got.exponents == (-2 - digits,)


def test_plain_rescale_overflow(okeys):
    from paper_2107_13797_b200.batches import plain_rescale
    from paper_2107_13797_b200.encoding import FixedPointOverflow
    for name in ("tiny", "k128", "k1024"):
        ok = okeys(name)
        pk = paillier.PublicKey(ok.n)
        n, max_int = ok.n, ok.n // 3
        # scaled magnitude reaches max_int
        big = max_int // 16 + 1
        for bad in (big, n - big):
            pb = PlaintextBatch(pk, (3,), (0,), (1, bad, 2), True)
            with pytest.raises(FixedPointOverflow):
                plain_rescale(pb, -1)
            with pytest.raises(ho.Overflow):
                ho.rescale(ok, bad, 0, -1)
        # a residue inside the overflow band cannot be interpreted at all
        pb = PlaintextBatch(pk, (2,), (0,), (1, max_int + 1), True)
        with pytest.raises(FixedPointOverflow):
            plain_rescale(pb, -1)
        # the largest magnitudes that still fit do
        fit = (max_int - 1) // 16
        if fit:
            ok_batch = PlaintextBatch(pk, (2,), (0,), (fit, n - fit), True)
            assert plain_rescale(ok_batch, -1).mantissas == (fit * 16, n - fit * 16)


@pytest.mark.parametrize("bits", [256, 512, 1024, 2048, 3072])
def test_codec_wide_kernels_edges(bits):
    """The 16-byte-access codec kernels (hb_codec.cu, k_*_wide) on their edges: magnitudes around 2^96 (where decode
    hands over to the generic kernel), sparse moduli whose zero words make the n - |x| borrow run long, values next
    to max_int, both signs, mixed with ordinary values in one batch."""
    from paper_2107_13797_b200.encoding import FixedPointOverflow
    rng = random.Random(bits)
    moduli = [rng.getrandbits(bits) | (1 << (bits - 1)) | 1,
              (1 << (bits - 1)) + 12345,                               # words 1 .. wn-2 are zero
              (1 << (bits - 1)) + (1 << 160) + 1,                      # zero words between 0 and 5, and above 5
              (1 << bits) - 1 - (1 << 40)]
    for n in moduli:
        ok = ho.Key(n)
        pk = paillier.PublicKey(n)
        # encode: ordinary doubles, tiny and huge ones, exact ties; every exponent moves the three words elsewhere
        vals = [rng.uniform(-100.0, 100.0) for _ in range(70)] + [0.0, -0.0, 1.0, -1.0, 2.0 ** -40, -2.0 ** -40,
                                                                  2.0 ** 52 + 1, -(2.0 ** 53 - 1), 1.5, -2.5, 3e15, -7e15]
        for exponent in (-8, 0, 5, -13, -24):
            want = [ho.encode(ok, v, exponent)[0] for v in vals]
            got = ops.batch_encode(pk, vals, exponent)
            assert list(got.mantissas) == want, (bits, hex(n)[:12], exponent)
            assert ops.batch_decode(pk, got) == [ho.decode(ok, m, exponent) for m in want]
        # decode: magnitudes around the 96-bit hand-over and up to max_int, both signs
        mags = [0, 1, 2 ** 53 - 1, 2 ** 53, 2 ** 53 + 1, 2 ** 64 - 1, 2 ** 64, 2 ** 95, 2 ** 96 - 1, 2 ** 96, 2 ** 96 + 1,
                2 ** 97 - 1, 3 * 2 ** 94 + 2 ** 41, 2 ** 96 - 2 ** 42 - 1, ok.max_int - 1, ok.max_int // 2 + 1]
        mags += [rng.getrandbits(rng.randrange(1, 130)) for _ in range(60)]
        mags = [m for m in mags if m < ok.max_int and m < 2 ** 900]      # beyond that the double overflows
        res = mags + [(n - m) % n for m in mags if m]
        rng.shuffle(res)
        for exponent in (-8, -30, 0):
            pb = PlaintextBatch(pk, (len(res),), (exponent,), tuple(res), True)
            assert ops.batch_decode(pk, pb) == [ho.decode(ok, m, exponent) for m in res], (bits, hex(n)[:12], exponent)
        # overflow band in the middle of a batch of fast-path elements
        band = res[:40] + [ok.max_int] + res[40:80]
        with pytest.raises(FixedPointOverflow):
            ops.batch_decode(pk, PlaintextBatch(pk, (len(band),), (0,), tuple(band), True))
        band[40] = n - ok.max_int
        with pytest.raises(FixedPointOverflow):
            ops.batch_decode(pk, PlaintextBatch(pk, (len(band),), (0,), tuple(band), True))
        # encode overflow exactly at max_int when it is representable as a double
        if bits == 256:
            edge = float(ok.max_int)
            if int(edge) >= ok.max_int:
                with pytest.raises(FixedPointOverflow):
                    ops.batch_encode(pk, [1.0, edge], 0)


def test_streamed_encrypt_equals_one_shot(okeys):
    """Large batches draw their obfuscation factors chunk by chunk while the GPU works (CudaBackend.encrypt_drawing):
    same ciphertexts, same generator state afterwards as the one-shot path; spot-checked against the oracle."""
    import numpy as np
    from paper_2107_13797_b200.device import WordArray
    ok = okeys("k512")
    pk, sk = product_keys(ok)
    be = CudaBackend()
    count = 2 * be.STREAM_CHUNK + 12345
    wn = (ok.n.bit_length() + 31) // 32
    m = np.zeros((count, wn), dtype=np.uint32)
    m[:, 0] = np.arange(count, dtype=np.uint32) * 2654435761 % (1 << 31)
    plain = PlaintextBatch(pk, (count,), (-8,), WordArray.from_numpy(m), True)
    rng_a, rng_b = random.Random(5), random.Random(5)
    streamed = ops.batch_encrypt(pk, plain, rng_a)                        # takes the streamed path
    r = be.draw_units(pk.n, count, rng_b)
    one_shot = be.encrypt(pk.n, plain.words, r)
    assert np.array_equal(streamed.words.numpy(), one_shot.numpy())
    assert rng_a.getstate() == rng_b.getstate()
    rng_c = random.Random(5)
    picks = [0, 1, be.STREAM_CHUNK - 1, be.STREAM_CHUNK, 2 * be.STREAM_CHUNK, count - 1]
    rs = [ho.draw_unit(ok.n, rng_c) for _ in range(count)] if count < 300000 else None
    assert rs is not None
    want = ho.k_encrypt(ok, [(int(m[i, 0]), rs[i]) for i in picks])
    got = WordArray.from_numpy(streamed.words.numpy()[picks]).ints()
    assert list(got) == want
    # obfuscate streams the same way
    rng_d, rng_e = random.Random(9), random.Random(9)
    again = ops.batch_obfuscate(pk, streamed, rng_d)
    r2 = be.draw_units(pk.n, count, rng_e)
    assert np.array_equal(again.words.numpy(), be.obfuscate(pk.n, streamed.words, r2).numpy())
    assert rng_d.getstate() == rng_e.getstate()
    dec = ops.batch_decrypt(sk, again)
    assert np.array_equal(dec.words.numpy()[:, 0], m[:, 0])


def test_wire_fast_paths(okeys):
    """HAFB bytes of a large device-resident batch (payload by DMA into pinned staging) equal the bytes of the same
    batch serialised from host words; deserialising them gives the batch back without a padding copy."""
    import numpy as np
    from paper_2107_13797_b200.bufferpool import deserialize, serialize_to_bytes
    from paper_2107_13797_b200.device import WordArray
    for name in ("k1024", "k2048"):
        ok = okeys(name)
        pk, _ = product_keys(ok)
        count = 5000
        wc = ((2 * ok.n.bit_length() + 7) // 8 + 3) // 4
        rng = np.random.default_rng(3)
        words = rng.integers(0, 1 << 32, size=(count, wc), dtype=np.uint64).astype(np.uint32)
        words[:, wc - 1] >>= 2                                     # below n^2
        host_batch = CiphertextBatch(pk, (count,), (-8,), WordArray.from_numpy(words), True, True)
        dev_batch = ops.batch_add(pk, host_batch, CiphertextBatch(pk, (count,), (-8,), (1,) * count, True, False))
        assert dev_batch.words.on_device and not dev_batch.words.on_host
        fast = serialize_to_bytes(dev_batch)
        assert not dev_batch.words.on_host                         # no host copy was cached on the way
        slow = serialize_to_bytes(CiphertextBatch(pk, (count,), (-8,), WordArray.from_numpy(words), True, True))
        assert fast == slow
        back = deserialize(fast, pk)
        assert back == host_batch and back.obfuscated
        assert ops.batch_add(pk, back, back) == ops.batch_add(pk, host_batch, host_batch)


def test_default_exponent_found_on_the_device(okeys):
    """encode_batch without a target exponent: min over the values of exact_exponent, zeros counting as 0
    (reference batches.py:122-123), computed by k_min_exact_exponent."""
    import numpy as np
    ok = okeys("k1024")
    pk, _ = product_keys(ok)
    rng = random.Random(21)
    cases = [[0.0, 4096.0], [4096.0, 65536.0], [0.0, 0.0, -0.0], [5e-324, 1.0], [2.0 ** -1074 * 3, 2.0 ** 40],
             [1.0], [0.5], [-0.75, 3.0], [16.0 ** 7, 16.0 ** 9 * 3], [1e-310, 2.5],
             [rng.uniform(-1, 1) for _ in range(1000)], [float(rng.randrange(1, 1 << 20)) * 16.0 ** 3 for _ in range(300)]]
    from paper_2107_13797_b200.encoding import FixedPointOverflow
    for vals in cases:
        want = min(ho.exact_exponent(v) for v in vals)
        try:
            mantissas = [ho.encode(ok, v, want)[0] for v in vals]
        except ho.Overflow:                      # a denormal next to 1.0 needs more bits than the key has
            with pytest.raises(FixedPointOverflow):
                encode_batch(pk, vals)
            continue
        got = encode_batch(pk, vals)
        assert got.exponents == (want,), vals[:4]
        assert list(got.mantissas) == mantissas
    big = np.random.default_rng(2).uniform(-1.0, 1.0, size=(3000, 7))
    eb = encode_batch(pk, big)
    assert eb.shape == (3000, 7) and eb.exponents == (min(ho.exact_exponent(float(v)) for v in big.ravel()),)
    assert encode_batch(pk, []).exponents == (0,)


@pytest.fixture
def forced_window(okeys):
    """hb_ctx_set_option(HB_OPT_MATVEC_WINDOW_BITS) on the contexts of the keys a test uses, reset afterwards."""
    from paper_2107_13797_b200.backends import default_backend
    touched = []

    def force(bits, names):
        for name in names:
            n = okeys(name).n
            default_backend().set_matvec_window(n, bits)
            touched.append(n)
    yield force
    for n in touched:
        default_backend().set_matvec_window(n, 0)


@pytest.mark.parametrize("width", ["9", "11", "13"])
def test_matmul_wide_windows(okeys, forced_window, width):
    """The bucket matvec with the window widths tall matrices use (9 bits from 32 k rows, 13 bits with the
    piecewise fold from 200 k rows), forced here on small problems: same bits as the oracle."""
    forced_window(int(width), ("k128", "k512", "k1024"))
    for name in ("k128", "k1024"):
        test_matmul(okeys, name)
    test_matmul_wide(okeys)
    ok = okeys("k512")
    pk, sk = product_keys(ok)
    rng = random.Random(int(width))
    inner, d = 700, 3
    pool = ho.k_encrypt(ok, [(rng.randrange(ok.n), ho.draw_unit(ok.n, rng)) for _ in range(6)])
    cs = [pool[rng.randrange(6)] for _ in range(inner)]
    ks = []
    for i in range(inner * d):
        mag = rng.getrandbits(rng.choice((1, 13, 26, 52, 53, 60)))
        ks.append(mag if rng.random() < 0.5 else (ok.n - mag) % ok.n)
    a = CiphertextBatch(pk, (inner,), (-4,), cs, True)
    x = PlaintextBatch(pk, (inner, d), (-9,), ks, True)
    got = ops.batch_matmul(pk, a, x)
    cols = tuple(tuple(ks[t * d + j] for t in range(inner)) for j in range(d))
    assert list(got.payload) == ho.k_dot(ok, (tuple(cs),), cols, [(0, j) for j in range(d)])


def test_large_batch_properties():
    """Size-independent properties at a batch size in the range of BASELINE's configs (200 k elements, Paillier-2048,
    where every kernel runs in its throughput shape): decrypt(encrypt) round trip, additivity of hadd, scalar
    multiplication by positive and negative constants, the sum reduction against its two halves and against the
    plaintext sum, and the encrypted matvec against integer arithmetic."""
    import numpy as np
    from paper_2107_13797_b200.device import WordArray
    keys = paillier.keygen(2048, paillier.default_rng(7), allow_insecure=True)
    pk, sk = keys.public, keys.private
    n = pk.n
    count, wn = 200_000, 64
    rs = np.random.default_rng(11)
    m = np.zeros((count, wn), dtype=np.uint32)
    m[:, 0] = rs.integers(0, 1 << 32, size=count, dtype=np.uint64).astype(np.uint32)
    m[:, 1] = rs.integers(0, 1 << 20, size=count, dtype=np.uint64).astype(np.uint32)          # 52-bit values
    vals = m[:, 0].astype(object) + (m[:, 1].astype(object) << 32)
    plain = PlaintextBatch(pk, (count,), (-8,), WordArray.from_numpy(m), True)
    c = ops.batch_encrypt(pk, plain, random.Random(1))
    assert np.array_equal(ops.batch_decrypt(sk, c).words.numpy(), m)
    # hadd: Dec(c_i * c_(count-1-i)) = m_i + m_(count-1-i)
    rev = CiphertextBatch(pk, (count,), (-8,), WordArray.from_numpy(c.words.numpy()[::-1].copy()), True, True)
    both = ops.batch_decrypt(sk, ops.batch_add(pk, c, rev)).words.numpy()
    want = vals + vals[::-1]
    got = both[:, 0].astype(object) + (both[:, 1].astype(object) << 32)
    assert (got == want).all() and not both[:, 2:].any()
    # hmul by 3 and by -2 (the inverse-base branch)
    three = PlaintextBatch(pk, (1,), (0,), (3,), True)
    t3 = ops.batch_decrypt(sk, ops.batch_mul_plain(pk, c, three)).words.numpy()
    assert ((t3[:, 0].astype(object) + (t3[:, 1].astype(object) << 32)) == 3 * vals).all()
    minus2 = PlaintextBatch(pk, (1,), (0,), (n - 2,), True)
    neg = ops.batch_decrypt(sk, ops.batch_mul_plain(pk, c, minus2))
    sample = [0, 1, 777, count // 2, count - 1]
    assert [neg.mantissas[i] for i in sample] == [(n - 2 * int(vals[i])) % n for i in sample]
    # hsum: whole == product of the halves, decrypts to the plaintext sum
    total = ops.batch_sum(pk, c)
    half = count // 2
    lo = CiphertextBatch(pk, (half,), (-8,), WordArray.from_numpy(c.words.numpy()[:half]), True, True)
    hi = CiphertextBatch(pk, (count - half,), (-8,), WordArray.from_numpy(c.words.numpy()[half:]), True, True)
    assert ops.batch_add(pk, ops.batch_sum(pk, lo), ops.batch_sum(pk, hi)).payload == total.payload
    assert ops.batch_decrypt(sk, total).mantissas[0] == int(vals.sum()) % n
    # matvec (13-bit windows at this height): 200 k x 3 signed 40-bit scalars
    d = 3
    mag = rs.integers(0, 1 << 40, size=(count, d), dtype=np.int64)
    sgn = rs.integers(0, 2, size=(count, d), dtype=np.int64) * 2 - 1
    x = (mag * sgn).astype(np.float64)
    xb = encode_batch(pk, x, target_exponent=0)
    out = ops.batch_decrypt(sk, ops.batch_matmul(pk, c, xb))
    signed = (mag * sgn).astype(object)
    for j in range(d):
        assert out.mantissas[j] == int((vals * signed[:, j]).sum()) % n
