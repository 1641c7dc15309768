"""GPU parity for what round 2 added: Montgomery-form residency between chained operators, the fused
fore-gradient kernel, compact resident scalar matrices, the bulk secure obfuscator draw, the single-process
multi-device backend (exercised with several workers on one GPU), blocked matvec for tall matrices, and
oracle comparisons at the shapes the benchmark runs (Paillier-2048 throughput kernels, 2 000 x 100 matvec).

Every comparison is bit for bit against the CPU oracle (oracle/hebatch_oracle.py, oracle/cpu_ref.c) or against the
plain single-device path.
"""
import ctypes
import math
import random

import numpy as np
import pytest

import cpuref
import hebatch_oracle as ho
from paper_2107_13797_b200 import _native, device, operators as ops, paillier
from paper_2107_13797_b200.arena import Arena
from paper_2107_13797_b200.backends import CudaBackend, MultiDeviceBackend, default_backend
from paper_2107_13797_b200.batches import CiphertextBatch, PlaintextBatch, decode_batch, encode_batch
from paper_2107_13797_b200.device import CompactScalars, WordArray

pytestmark = pytest.mark.gpu


def product_keys(ok):
    kp = paillier.keypair_from_primes(ok.p, ok.q)
    return kp.public, kp.private


def enc_oracle(ok, ms, seed):
    rng = random.Random(seed)
    rs = [ho.draw_unit(ok.n, rng) for _ in ms]
    return ho.k_encrypt(ok, list(zip(ms, rs)))


def signed_scalars(ok, count, rng, bits=40):
    out = []
    for _ in range(count):
        mag = rng.getrandbits(bits)
        out.append(mag if rng.random() < 0.5 else (ok.n - mag) % ok.n)
    return out


# ---- Montgomery residency ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["tiny", "k128", "k512", "k1024", "k2048", "k3072"])
def test_resident_chain_equals_plain_chain(okeys, name):
    """encrypt -> obfuscate -> add -> add(plain) -> mul -> sum -> matmul -> decrypt with every intermediate in
    Montgomery digit form, against the same chain through plain words and against the oracle."""
    ok = okeys(name)
    pk, sk = product_keys(ok)
    count = 24 if name != "k3072" else 8
    rng = random.Random(5)
    ms = [rng.randrange(ok.n) for _ in range(count)]
    plain = PlaintextBatch(pk, (count,), (-4,), ms, True)
    results = {}
    for label, be in (("mont", CudaBackend(True)), ("plain", CudaBackend(False))):
        c = ops.batch_encrypt(pk, plain, random.Random(11), be)
        assert (c.words.mont() is not None) == (label == "mont")
        o = ops.batch_obfuscate(pk, c, random.Random(12), be)
        s = ops.batch_add(pk, c, o, be)
        addend = PlaintextBatch(pk, (count,), (-4,), [rng2 % ok.n for rng2 in range(3, 3 + count)], True)
        s2 = ops.batch_add(pk, s, addend, be)
        k = PlaintextBatch(pk, (count,), (0,), signed_scalars(ok, count, random.Random(13), 20) if ok.n > 2 ** 60
                           else [random.Random(13).randrange(1, ok.n // 3) for _ in range(count)], True)
        units = all(math.gcd(v, ok.n) == 1 for v in s2.payload)
        m = ops.batch_mul_plain(pk, s2, k, be) if units else s2
        tot = ops.batch_sum(pk, m, None, be)
        x = PlaintextBatch(pk, (count, 2), (0,), [(i * 7 + 1) % (ok.n // 3) for i in range(2 * count)], True)
        mv = ops.batch_matmul(pk, m, x, be)
        dec = ops.batch_decrypt(sk, m, be)
        results[label] = (c.payload, o.payload, s.payload, s2.payload, m.payload, tot.payload, mv.payload,
                          dec.mantissas)
    assert results["mont"] == results["plain"]
    c_want = enc_oracle(ok, ms, 11)
    assert list(results["mont"][0]) == c_want
    assert list(results["mont"][2]) == ho.k_add(ok, list(zip(c_want, results["mont"][1])))
    assert list(results["mont"][7]) == ho.k_decrypt(ok, list(results["mont"][4]))


@pytest.mark.parametrize("name", ["k128", "k1024", "k2048"])
def test_mulmod_rep_every_flag_combination(okeys, name):
    """hb_mulmod_rep / hb_lift_mulmod_rep / hb_ct_convert through the C ABI for all eight representation triples."""
    ok = okeys(name)
    lib = _native.lib()
    ctx = device.context_for(ok.n)
    t = device.torch()
    rng = random.Random(3)
    count = 10
    a_int = enc_oracle(ok, [rng.randrange(ok.n) for _ in range(count)], 1)
    b_int = enc_oracle(ok, [rng.randrange(ok.n) for _ in range(count)], 2)
    m_int = [rng.randrange(ok.n) for _ in range(count)]
    stream = device.current_stream_ptr()

    def plain(v, w):
        return WordArray.from_ints(v, w).device()

    def to_mont(x):
        out = t.empty((count, ctx.limbs), dtype=t.int32, device="cuda")
        _native.check(lib.hb_ct_convert(ctx.handle, x.data_ptr(), out.data_ptr(), count, 1, stream))
        return out

    def back(x, is_mont):
        if not is_mont:
            return WordArray.from_device(x).ints()
        out = t.empty((count, ctx.wc), dtype=t.int32, device="cuda")
        _native.check(lib.hb_ct_convert(ctx.handle, x.data_ptr(), out.data_ptr(), count, 0, stream))
        return WordArray.from_device(out).ints()

    a_p, b_p, m_p = plain(a_int, ctx.wc), plain(b_int, ctx.wc), plain(m_int, ctx.wn)
    a_m, b_m = to_mont(a_p), to_mont(b_p)
    assert list(back(a_m, True)) == a_int
    want_mul = ho.k_add(ok, list(zip(a_int, b_int)))
    want_lift = ho.k_add(ok, [(a, (1 + m * ok.n) % ok.n2) for a, m in zip(a_int, m_int)])
    for am in (0, 1):
        for bm in (0, 1):
            for om in (0, 1):
                flags = (_native.HB_A_MONT if am else 0) | (_native.HB_B_MONT if bm else 0) | \
                        (_native.HB_OUT_MONT if om else 0)
                out = t.empty((count, ctx.limbs if om else ctx.wc), dtype=t.int32, device="cuda")
                _native.check(lib.hb_mulmod_rep(ctx.handle, (a_m if am else a_p).data_ptr(),
                                                (b_m if bm else b_p).data_ptr(), out.data_ptr(), count, 0, flags,
                                                stream))
                assert list(back(out, om)) == want_mul, (am, bm, om)
                if not bm:
                    _native.check(lib.hb_lift_mulmod_rep(ctx.handle, (a_m if am else a_p).data_ptr(), m_p.data_ptr(),
                                                         out.data_ptr(), count, 0, flags, stream))
                    assert list(back(out, om)) == want_lift, ("lift", am, om)


def test_decrypt_accepts_both_forms_at_throughput_shape(okeys):
    """hb_decrypt_rep on Montgomery input at a count that runs the (16, 4) throughput shape, and at a small count
    (the (8, 8) shape): same plaintexts as the plain-word path and the oracle."""
    ok = okeys("k2048")
    pk, sk = product_keys(ok)
    for count in (16, 20_000):
        rs = np.random.default_rng(count)
        m = np.zeros((count, 64), np.uint32)
        m[:, :2] = rs.integers(0, 2 ** 32, size=(count, 2), dtype=np.uint64).astype(np.uint32)
        plain = PlaintextBatch(pk, (count,), (0,), WordArray.from_numpy(m), True)
        be = CudaBackend(True)
        c = ops.batch_encrypt(pk, plain, random.Random(1), be)
        assert c.words.mont() is not None
        got = ops.batch_decrypt(sk, c, be).words.numpy()
        assert np.array_equal(got, m)
        c_plain = CiphertextBatch(pk, (count,), (0,), WordArray.from_numpy(c.words.numpy().copy()), True)
        assert np.array_equal(ops.batch_decrypt(sk, c_plain, be).words.numpy(), m)
        chk = min(count, 256)
        assert np.array_equal(cpuref.decrypt_words(ok, c.words.numpy()[:chk]), m[:chk])


# ---- throughput-shape parity against the oracle (the shapes bench.py times) -----------------------------------------

def test_throughput_kernels_match_oracle_on_4096_strided_elements(okeys):
    """k_encrypt<32,4> / k_decrypt<16,4> at a batch that fills the persistent grid (40 000 elements, Paillier-2048),
    compared ciphertext for ciphertext with GMP on 4 096 elements taken with a stride over the whole batch
    (the reference verifies at min(count, 4096), cli.py:204)."""
    ok = okeys("k2048")
    lib = _native.lib()
    ctx = device.context_for(ok.n)
    ctx.set_private(ok.p, ok.q, ok.hp, ok.hq, ok.q_inv)
    t = device.torch()
    count = 40_000
    rs = np.random.default_rng(99)
    m = rs.integers(0, 2 ** 32, size=(count, ctx.wn), dtype=np.uint64).astype(np.uint32)
    m[:, -1] &= 0x0fffffff                                # below n
    r = rs.integers(0, 2 ** 32, size=(count, ctx.wn), dtype=np.uint64).astype(np.uint32)
    r[:, -1] = 1
    dm, dr = t.from_numpy(m.view(np.int32)).cuda(), t.from_numpy(r.view(np.int32)).cuda()
    c = t.empty((count, ctx.wc), dtype=t.int32, device="cuda")
    back = t.empty((count, ctx.wn), dtype=t.int32, device="cuda")
    s = device.current_stream_ptr()
    _native.check(lib.hb_encrypt(ctx.handle, dm.data_ptr(), dr.data_ptr(), c.data_ptr(), count, s))
    _native.check(lib.hb_decrypt(ctx.handle, c.data_ptr(), back.data_ptr(), count, s))
    hc = c.cpu().numpy().view(np.uint32)
    assert np.array_equal(back.cpu().numpy().view(np.uint32), m)
    idx = np.arange(0, count, count // 4096)[:4096]
    assert np.array_equal(cpuref.encrypt_words(ok.n, m[idx], r[idx]), hc[idx])
    assert np.array_equal(cpuref.decrypt_words(ok, hc[idx]), m[idx])


def test_matvec_2000_x_100_at_2048_bits_matches_oracle(okeys):
    """BASELINE configs[2] on a reduced instance: 2 000 ciphertexts x 100 columns of
    uniform(-1, 1) features under their exact shared exponent, ciphertext bits == GMP -- for the residue form and for
    the compact resident form of the feature matrix."""
    ok = okeys("k2048")
    pk, _ = product_keys(ok)
    inner, d = 2000, 100
    vals = np.random.default_rng(1).uniform(-10, 10, inner)
    a = ops.batch_encrypt(pk, encode_batch(pk, vals, target_exponent=-16), random.Random(1))
    X = np.random.default_rng(0).uniform(-1, 1, (inner, d))
    x_res = encode_batch(pk, X)
    x_cmp = encode_batch(pk, X, compact=True)
    assert isinstance(x_cmp.words, CompactScalars) and x_cmp.exponents == x_res.exponents
    assert x_cmp.words.maxbits <= 53 and x_cmp.words.nneg > 0
    want = cpuref.matvec_words(ok.n, a.words.numpy(), x_res.words.numpy(), inner, d)
    got_res = ops.batch_matmul(pk, a, x_res)
    got_cmp = ops.batch_matmul(pk, a, x_cmp)
    assert np.array_equal(got_res.words.numpy(), want)
    assert np.array_equal(got_cmp.words.numpy(), want)
    assert got_cmp.exponents == got_res.exponents == (a.exponents[0] + x_res.exponents[0],)


# ---- compact scalars -------------------------------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["k128", "k1024"])
def test_compact_encoding_equals_residue_encoding(okeys, name):
    ok = okeys(name)
    pk, _ = product_keys(ok)
    rng = np.random.default_rng(4)
    X = rng.uniform(-1, 1, (37, 5))
    X[3, 2] = 0.0
    X[4, 1] = -0.0
    X[5, 0] = 0.5
    for exponent in (None, -13, -8, -3):
        res = encode_batch(pk, X, target_exponent=exponent)
        cmp_ = encode_batch(pk, X, target_exponent=exponent, compact=True)
        assert isinstance(cmp_.words, CompactScalars)
        assert cmp_ == res and cmp_.mantissas == res.mantissas
    # magnitudes beyond 64 bits have no compact form: the residue encoding is returned instead
    wide = encode_batch(pk, np.array([[1e30, 1.0]]), target_exponent=-2, compact=True) if name != "k128" else None
    if wide is not None:
        assert not isinstance(wide.words, CompactScalars)
        assert wide == encode_batch(pk, np.array([[1e30, 1.0]]), target_exponent=-2)
    # residues -> compact on the device
    k = PlaintextBatch(pk, (20, 3), (0,), signed_scalars(ok, 60, random.Random(1), 60), True)
    packed = default_backend().compact_scalars(pk.n, k.words, 20, 3)
    assert packed.maxbits <= 60 and np.array_equal(packed.numpy(), k.words.numpy())


def test_matvec_in_row_blocks(okeys):
    """Tall matrices are reduced block by block (HB_OPT_MATVEC_BLOCK_ROWS, 2^21 rows by default): forced to 64-row
    blocks here, same bits as one pass and as the oracle."""
    ok = okeys("k512")
    pk, _ = product_keys(ok)
    rng = random.Random(21)
    inner, d = 300, 4
    pool = enc_oracle(ok, [rng.randrange(ok.n) for _ in range(8)], 3)
    cs = [pool[rng.randrange(8)] for _ in range(inner)]
    ks = signed_scalars(ok, inner * d, rng, 52)
    a = CiphertextBatch(pk, (inner,), (0,), cs, True)
    x = PlaintextBatch(pk, (inner, d), (0,), ks, True)
    cols = tuple(tuple(ks[t * d + j] for t in range(inner)) for j in range(d))
    want = ho.k_dot(ok, (tuple(cs),), cols, [(0, j) for j in range(d)])
    ctx = device.context_for(ok.n)
    try:
        ctx.set_option(_native.HB_OPT_MATVEC_BLOCK_ROWS, 64)
        assert list(ops.batch_matmul(pk, a, x).payload) == want
    finally:
        ctx.set_option(_native.HB_OPT_MATVEC_BLOCK_ROWS, 0)
    assert list(ops.batch_matmul(pk, a, x).payload) == want


def test_non_unit_under_non_negative_scalar_is_a_value(okeys):
    """_pow_scalar inverts element by element (operators.py:60-61): a ciphertext without an inverse only raises when
    ITS scalar is negative."""
    ok = okeys("k128")
    pk, _ = product_keys(ok)
    good = enc_oracle(ok, [5, 6, 7], 1)
    cs = [good[0], ok.p, good[1], 0, good[2]]
    ks = [ok.n - 3, 2, ok.n - 5, 7, 4]
    a = CiphertextBatch(pk, (5,), (0,), cs, True)
    k = PlaintextBatch(pk, (5,), (0,), ks, True)
    out = ops.batch_mul_plain(pk, a, k)
    assert list(out.payload) == ho.k_mul(ok, list(zip(cs, ks)))
    with pytest.raises(ZeroDivisionError):
        ops.batch_mul_plain(pk, a, PlaintextBatch(pk, (5,), (0,), [1, ok.n - 2, 1, 1, 1], True))


# ---- fused fore-gradient pipeline --------------------------------------------------------------------------------

@pytest.mark.parametrize("name,count", [("k128", 9), ("k1024", 33), ("k2048", 150_000)])
def test_fused_fore_gradient_equals_six_operators(okeys, name, count):
    """Arena.run_fore_gradient_pipeline as one kernel: same ciphertexts, same ledger, same conservation state and the
    same generator state afterwards as the six-operator form (arena.py:345-366 of the reference)."""
    ok = okeys(name)
    pk, sk = product_keys(ok)
    rs = np.random.default_rng(8)
    lh = rs.uniform(-4, 4, count).round(6)
    lg = rs.uniform(-4, 4, count).round(6)
    y = np.where(rs.uniform(size=count) > 0.5, 1.0, -1.0)
    c_lh = ops.batch_encrypt(pk, encode_batch(pk, lh, target_exponent=-8), random.Random(2))
    lg_plain = encode_batch(pk, lg, target_exponent=-8)
    y_plain = encode_batch(pk, y, target_exponent=0)
    outs = {}
    for fused in (True, False):
        arena = Arena(pk, rng=random.Random(100), fused=fused)
        h = arena.upload(CiphertextBatch(pk, c_lh.shape, c_lh.exponents, WordArray.from_numpy(c_lh.words.numpy().copy()),
                                         True, True))
        h_fore = arena.run_fore_gradient_pipeline(h, lg_plain, y_plain)
        fore = arena.download(h_fore)
        outs[fused] = (fore, arena.ledger.to_json(), arena.resident_bytes, arena.produced_bytes, arena.released_bytes,
                       arena.check_conservation(), arena.rng.getstate(), h_fore.id)
    assert outs[True][0] == outs[False][0]
    assert outs[True][1:] == outs[False][1:]
    assert outs[True][5] is True
    dec = np.asarray(decode_batch(pk, ops.batch_decrypt(sk, outs[True][0])))
    grid = lambda v, e: np.round(v * 16.0 ** -e) * 16.0 ** e          # noqa: E731
    assert np.allclose(dec, 0.25 * (grid(lh, -8) + grid(lg, -8)) - 0.5 * y, atol=1e-12)
    # immediate (non-handle) host logits: the pipeline uploads and releases them itself
    a1, a2 = Arena(pk, rng=random.Random(5), fused=True), Arena(pk, rng=random.Random(5), fused=False)
    f1 = a1.download(a1.run_fore_gradient_pipeline(c_lh, lg_plain, y_plain))
    f2 = a2.download(a2.run_fore_gradient_pipeline(c_lh, lg_plain, y_plain))
    assert f1 == f2 and a1.ledger.to_json() == a2.ledger.to_json() and a1.check_conservation()
    assert (a1.resident_bytes, a1.released_bytes) == (a2.resident_bytes, a2.released_bytes)


# ---- bulk secure obfuscator draw -----------------------------------------------------------------------------------

def test_secure_draw_is_bulk_and_valid(okeys):
    ok = okeys("k1024")
    pk, sk = product_keys(ok)
    be = default_backend()
    for rng in (None, random.SystemRandom()):
        r = be.draw_units(ok.n, 3000, rng)
        vals = r.ints()
        assert all(1 <= v < ok.n for v in vals) and len(set(vals)) == 3000
        assert all(math.gcd(v, ok.n) == 1 for v in vals[:50])
        assert sum(v.bit_length() == ok.n.bit_length() for v in vals) > 500       # not truncated
    plain = encode_batch(pk, [0.5 * i for i in range(64)], target_exponent=-4)
    c1 = ops.batch_encrypt(pk, plain, paillier.default_rng())
    c2 = ops.batch_encrypt(pk, plain, paillier.default_rng())
    assert c1.payload != c2.payload
    assert ops.batch_decrypt(sk, c1).mantissas == ops.batch_decrypt(sk, c2).mantissas == plain.mantissas
    # the native generator itself: values below a bound that is not a power of two, uniform top word
    lib = _native.lib()
    n = 3 * 2 ** 70 + 1
    words = device.ints_to_words([n], 3)
    out = np.empty((20000, 3), np.uint32)
    _native.check(lib.hb_secure_randrange1(words.ctypes.data, 3, 20000, out.ctypes.data))
    vals = device.words_to_ints(out)
    assert all(1 <= v < n for v in vals) and max(vals) > 2.9 * 2 ** 70 and min(vals) < 0.1 * 2 ** 70


def test_private_key_is_checked_and_droppable(okeys):
    ok, other = okeys("k128"), okeys("k512")
    pk, sk = product_keys(ok)
    c = ops.batch_encrypt(pk, encode_batch(pk, [1.5, -2.0], target_exponent=-4), random.Random(1))
    assert ops.batch_decode(pk, ops.batch_decrypt(sk, c)) == [1.5, -2.0]
    ctx = device.context_for(ok.n)
    with pytest.raises(ValueError):
        ctx.set_private(ok.p, ok.q, ok.hp, ok.hq, (ok.q_inv + 1) % ok.p)
    with pytest.raises(ValueError):
        default_backend().decrypt(ok.n, (other.p, other.q, other.hp, other.hq, other.q_inv), c.words)
    device.drop_private(ok.n)
    assert not device.context_for(ok.n).has_private
    assert ops.batch_decode(pk, ops.batch_decrypt(sk, c)) == [1.5, -2.0]      # re-installed from the real key


# ---- single-process multi-device backend (several workers on this GPU) ------------------------------------------

@pytest.fixture(scope="module")
def multi():
    t = device.torch()
    devs = list(range(t.cuda.device_count())) if t.cuda.device_count() > 1 else [0, 0, 0]
    be = MultiDeviceBackend(devs)
    yield be
    be.close()


@pytest.mark.parametrize("name", ["k128", "k1024"])
def test_multi_device_operators_equal_single_device(okeys, multi, name):
    """Every operator through MultiDeviceBackend (element ranges of ceil(count / workers), partials + combine for the
    reductions) against the single-device backend: identical batches, identical generator state."""
    ok = okeys(name)
    pk, sk = product_keys(ok)
    one = CudaBackend()
    rng = np.random.default_rng(6)
    count = 41                                          # not a multiple of the worker count
    vals = rng.uniform(-50, 50, count)
    res = {}
    for label, be in (("one", one), ("multi", multi)):
        g = random.Random(77)
        plain = encode_batch(pk, vals, target_exponent=-8, backend=be)
        c = ops.batch_encrypt(pk, plain, g, be)
        o = ops.batch_obfuscate(pk, c, g, be)
        s = ops.batch_add(pk, c, o, be)
        s2 = ops.batch_add(pk, s, encode_batch(pk, vals * 0.5, target_exponent=-6, backend=be), be)
        s3 = ops.batch_add(pk, s2, encode_batch(pk, [3.0], target_exponent=0, backend=be), be)
        k_el = encode_batch(pk, rng.integers(-1000, 1000, count).astype(float), target_exponent=0, backend=be)
        m1 = ops.batch_mul_plain(pk, s3, k_el, be)
        m2 = ops.batch_mul_plain(pk, m1, encode_batch(pk, [-0.25], backend=be), be)
        tot = ops.batch_sum(pk, m2, None, be)
        X = np.random.default_rng(2).uniform(-1, 1, (count, 7))
        mv = ops.batch_matmul(pk, m2, encode_batch(pk, X, backend=be), be)
        mvc = ops.batch_matmul(pk, m2, encode_batch(pk, X, backend=be, compact=True), be)
        dec = ops.batch_decrypt(sk, m2, be)
        back = ops.batch_decode(pk, ops.batch_decrypt(sk, c, be), be)
        res[label] = (plain, c, o, s, s2, s3, m1, m2, tot, mv, mvc, dec, back, g.getstate())
        rng = np.random.default_rng(6)
        rng.uniform(-50, 50, count)
    for a, b in zip(res["one"], res["multi"]):
        assert a == b
    assert res["multi"][1].words.shards is not None and len(res["multi"][1].words.shards.parts) == multi.worker_count
    # 2-D reductions and row-vector broadcast fall back to one device: same bits
    grid = ops.batch_encrypt(pk, encode_batch(pk, np.arange(24.0).reshape(6, 4), target_exponent=0, backend=multi),
                             random.Random(3), multi)
    grid1 = ops.batch_encrypt(pk, encode_batch(pk, np.arange(24.0).reshape(6, 4), target_exponent=0),
                              random.Random(3), one)
    assert grid == grid1
    row = encode_batch(pk, [1.0, -2.0, 3.0, -4.0], target_exponent=0)
    assert ops.batch_mul_plain(pk, grid, row, multi) == ops.batch_mul_plain(pk, grid1, row, one)
    for axis in (0, 1):
        assert ops.batch_sum(pk, grid, axis, multi) == ops.batch_sum(pk, grid1, axis, one)


def test_multi_device_streamed_encrypt_and_wire(okeys, multi):
    """A batch large enough for the streamed draw: the sharded, chunk-dispatched form yields the ciphertexts and the
    generator state of the one-shot single-device form (MT19937 replay in global element order), and serialises
    shard by shard to the same bytes."""
    from paper_2107_13797_b200.bufferpool import deserialize, serialize_to_bytes
    ok = okeys("k1024")
    pk, sk = product_keys(ok)
    count = 9001
    rs = np.random.default_rng(3)
    m = np.zeros((count, 32), np.uint32)
    m[:, 0] = rs.integers(0, 2 ** 32, size=count, dtype=np.uint64).astype(np.uint32)
    plain = PlaintextBatch(pk, (count,), (-8,), WordArray.from_numpy(m), True)
    g1, g2 = random.Random(9), random.Random(9)
    c_multi = ops.batch_encrypt(pk, plain, g1, multi)
    c_one = ops.batch_encrypt(pk, plain, g2, CudaBackend())
    assert c_multi == c_one and g1.getstate() == g2.getstate()
    wire = serialize_to_bytes(c_multi)
    assert wire == serialize_to_bytes(c_one)
    assert np.array_equal(ops.batch_decrypt(sk, deserialize(wire, pk), multi).words.numpy(), m)
    o_multi = ops.batch_obfuscate(pk, c_multi, g1, multi)
    assert o_multi == ops.batch_obfuscate(pk, c_one, g2, CudaBackend()) and g1.getstate() == g2.getstate()
    # OS entropy: every worker draws its own chunks
    c_sys = ops.batch_encrypt(pk, plain, paillier.default_rng(), multi)
    assert c_sys.payload[:3] != c_multi.payload[:3]
    assert np.array_equal(ops.batch_decrypt(sk, c_sys, multi).words.numpy(), m)


def test_multi_device_flr_epoch_equals_single_device(multi):
    """The FLR driver unchanged, with the multi-device backend passed in: same decrypted gradients, loss and model as
    the single-device run (and the ledger of the arena)."""
    from paper_2107_13797_b200 import flr
    keys = paillier.keygen(512, paillier.default_rng(5), allow_insecure=True)
    ids, X, y = flr.make_synthetic(60, 6, seed=1)
    runs = {}
    for label, be in (("one", CudaBackend()), ("multi", multi)):
        guest, host = flr.vertical_split(ids, X, y, 2)
        fed = flr.HeteroFederation(guest, host, flr.make_minibatches(60, 25, seed=1), np.arange(60), keys,
                                   flr.FlrConfig(0.15, 25, seed=3), backend=be)
        out = fed.run(2)
        runs[label] = ([r.loss for r in out], fed.combined_theta().tolist(), fed.decrypted, out[-1].ledger)
    assert runs["one"] == runs["multi"]


@pytest.mark.parametrize("name", ["k1024", "k2048", "k3072"])
def test_codec_sector_paths_far_from_word_zero(okeys, name):
    """The 32-byte-sector codec kernels with the magnitude words far above word 0: at exponents -70 ... -127 the
    three words of uniform(-100, 100) values sit in sectors 1 to 2 -- warps whose 32 elements agree on the sector take
    the write-once path with a shifted sector, the others the background-and-patch path; negative residues borrow
    against words of n that are not the low ones.  Encode against the oracle, decode (generic kernel: magnitudes
    beyond 2^96) back to the same doubles."""
    ok = okeys(name)
    pk, _sk = product_keys(ok)
    rng = random.Random(5)
    vals = [rng.uniform(-100.0, 100.0) for _ in range(150)] + [0.0, -0.0, 64.0, -64.0, 2.0 ** -20, -3.0 * 2.0 ** -18]
    same_word = [float(rng.randrange(2 ** 20, 2 ** 21)) * (1 if i % 2 else -1) for i in range(96)]   # one ws for all
    for exponent in (-70, -81, -100, -127):
        for batch in (vals, same_word):
            want = [ho.encode(ok, v, exponent)[0] for v in batch]
            got = ops.batch_encode(pk, batch, exponent)
            assert list(got.mantissas) == want, (name, exponent)
            assert ops.batch_decode(pk, got) == [ho.decode(ok, m, exponent) for m in want]


@pytest.mark.parametrize("name", ["k128", "k1024"])
def test_matmul_2d_left_operand_bucket_path(okeys, name):
    """A 2-D encrypted left operand (3 x inner) times signed 40-bit scalars: every output row goes through the bucket
    kernels, enqueued one behind the other with ONE inversion flag read after the last row.  Against the oracle; a
    non-unit ciphertext in the LAST row under a negative scalar still raises ZeroDivisionError, under a non-negative
    one it is a value."""
    ok = okeys(name)
    pk, _sk = product_keys(ok)
    rng = random.Random(21)
    rows, inner, d = 3, 37, 4
    ms = [rng.randrange(ok.n) for _ in range(rows * inner)]
    cpay = enc_oracle(ok, ms, 8)
    ks = signed_scalars(ok, inner * d, rng)
    a = CiphertextBatch(pk, (rows, inner), (-3,), cpay, True)
    x = PlaintextBatch(pk, (inner, d), (-2,), ks, True)
    out = ops.batch_matmul(pk, a, x)
    rws = tuple(tuple(cpay[i * inner + t] for t in range(inner)) for i in range(rows))
    cols = tuple(tuple(ks[t * d + j] for t in range(inner)) for j in range(d))
    assert list(out.payload) == ho.k_dot(ok, rws, cols, [(i, j) for i in range(rows) for j in range(d)])
    assert out.shape == (rows, d) and out.exponents == (-5,)
    bad = list(cpay)
    bad[-1] = ok.p                                              # not a unit mod n^2, last row, last term
    neg_last = list(ks)
    neg_last[(inner - 1) * d] = ok.n - 5                        # its scalar in column 0 is negative
    with pytest.raises(ZeroDivisionError):
        ops.batch_matmul(pk, CiphertextBatch(pk, (rows, inner), (-3,), bad, True),
                         PlaintextBatch(pk, (inner, d), (-2,), neg_last, True))
    pos = [k if k < ok.max_int else ok.n - k for k in ks]       # magnitudes only: nothing is inverted
    got = ops.batch_matmul(pk, CiphertextBatch(pk, (rows, inner), (-3,), bad, True),
                           PlaintextBatch(pk, (inner, d), (-2,), pos, True))
    rws_bad = tuple(tuple(bad[i * inner + t] for t in range(inner)) for i in range(rows))
    cols_pos = tuple(tuple(pos[t * d + j] for t in range(inner)) for j in range(d))
    assert list(got.payload) == ho.k_dot(ok, rws_bad, cols_pos, [(i, j) for i in range(rows) for j in range(d)])


def test_multi_device_homo_aggregation_equals_single_device(multi):
    """The horizontal protocol (BASELINE configs[4] shape, reduced) with the multi-device backend passed in: same
    aggregated gradients, model and loss as the single-device run."""
    from paper_2107_13797_b200 import flr
    keys = paillier.keygen(512, paillier.default_rng(5), allow_insecure=True)
    ids, X, y = flr.make_synthetic(90, 40, seed=2)
    runs = {}
    for label, be in (("one", CudaBackend()), ("multi", multi)):
        parts = flr.horizontal_split(ids, X, y, 3)
        fed = flr.HomoFederation(parts, keys, flr.FlrConfig(learning_rate=0.15, seed=6), backend=be)
        out = fed.run(2)
        runs[label] = ([r.loss for r in out], fed.theta.tolist(), [g.tolist() for g in fed.aggregated_gradients])
    assert runs["one"] == runs["multi"]


def test_misaligned_digit_form_pointer_is_rejected(okeys):
    """Montgomery digit-form arrays are moved 16 bytes at a time: a base pointer that is not 16-byte aligned is an
    argument error, not a fault; plain-word arrays of any alignment still work (word path)."""
    t = device.torch()
    ok = okeys("k512")
    pk, sk = product_keys(ok)
    ctx = device.context_for(ok.n)
    lib = _native.lib()
    count = 5
    c = ops.batch_encrypt(pk, encode_batch(pk, [1.0, -2.0, 3.5, 0.25, -7.0], target_exponent=-4), random.Random(4),
                          CudaBackend(resident_montgomery=False))
    plain = c.words.device()
    buf = t.zeros((count * ctx.limbs + 4,), dtype=t.int32, device="cuda")
    stream = device.current_stream_ptr()
    with pytest.raises(ValueError):
        _native.check(lib.hb_ct_convert(ctx.handle, plain.data_ptr(), buf.data_ptr() + 4, count, 1, stream))
    _native.check(lib.hb_ct_convert(ctx.handle, plain.data_ptr(), buf.data_ptr(), count, 1, stream))
    with pytest.raises(ValueError):
        _native.check(lib.hb_mulmod_rep(ctx.handle, buf.data_ptr() + 4, buf.data_ptr(), buf.data_ptr(), count, 0,
                                        _native.HB_A_MONT | _native.HB_B_MONT | _native.HB_OUT_MONT, stream))
    # plain words at a 4-byte offset: accepted, same bits as the aligned call
    shifted = t.zeros((count * ctx.wc + 1,), dtype=t.int32, device="cuda")
    shifted[1:] = plain.reshape(-1)
    out_a = t.empty((count, ctx.wc), dtype=t.int32, device="cuda")
    out_b = t.empty((count, ctx.wc), dtype=t.int32, device="cuda")
    _native.check(lib.hb_mulmod(ctx.handle, plain.data_ptr(), plain.data_ptr(), out_a.data_ptr(), count, 0, stream))
    _native.check(lib.hb_mulmod(ctx.handle, shifted.data_ptr() + 4, shifted.data_ptr() + 4, out_b.data_ptr(), count, 0,
                                stream))
    assert t.equal(out_a, out_b)
