"""Pins the oracle (oracle/hebatch_oracle.py, oracle/cpu_ref.c) to the reference:

  (a) known-answer values held by the reference's own tests, cited per assertion;
  (b) tests/golden/hebatch_golden.json -- transcripts of the unmodified reference's operators.

CPU only."""
import random
import struct

import numpy as np
import pytest

import cpuref
import hebatch_oracle as ho
from golden_util import ints, load

GOLD = load()


def key_of(name):
    k = GOLD["keys"][name]
    return ho.Key(int(k["n"], 16), int(k["p"], 16), int(k["q"], 16))


# ---- (a) known answers from /root/reference/pkg/tests --------------------------------------------------

def test_kat_n35():
    k = ho.Key(35, 5, 7)
    assert k.lam == 12                                              # test_paillier.py:48-54
    assert ho.k_encrypt(k, [(3, 2)]) == [683]                       # test_paillier.py:79-84, test_operators.py:63-70
    assert ho.k_encrypt(k, [(0, 1)]) == [1]                         # test_paillier.py:85-88
    assert ho.k_decrypt(k, [683, 1]) == [3, 0]                      # test_paillier.py:101-104
    for c in (683, 1, 36, 1224):
        assert ho.k_decrypt(k, [c])[0] == ho.decrypt_textbook(k, c)  # test_paillier.py:108-113
    for m in range(35):                                             # test_paillier.py:152-167
        for r in (1, 2, 3, 4, 6, 8, 9, 11):
            c = ho.k_encrypt(k, [(m, r)])[0]
            assert ho.k_decrypt(k, [c]) == [m]


def test_kat_codec():
    k = ho.Key(35, 5, 7)
    big = ho.keygen(128, random.Random(1234))
    assert ho.encode(big, 0.5) == (8, -1)                           # test_encoding.py:25-29
    assert k.max_int == 11
    for m in range(11, 25):                                         # overflow band [11, 24], test_encoding.py:73-81
        with pytest.raises(ho.Overflow):
            ho.signed_mantissa(k, m)
    assert ho.signed_mantissa(k, 10) == 10 and ho.signed_mantissa(k, 25) == -10
    table = {1.0: 0, 16.0: 1, 0.5: -1, 0.0625: -1, 0.03125: -2, 256.0: 2, 3.0: 0, 48.0: 1, 0.0: 0}
    for v, e in table.items():                                      # test_encoding.py:152-158
        assert ho.exact_exponent(v) == e, v
    for v in (0.1, -123.456, 2.0 ** -40, 1e10, -7.25):              # exact round trip, test_encoding.py:83-89
        m, e = ho.encode(big, v)
        assert ho.decode(big, m, e) == v


def test_kat_hafb():
    # 32-byte header, shared exponent, 2-byte words for the 6-bit key: ... ab 02 (test_bufferpool.py:195-206)
    blob = ho.hafb_serialize(6, (1,), (-3,), [683], True)
    assert blob[:4] == b"HAFB" and len(blob) == 32 + 4 + 2
    assert blob[-2:] == bytes([0xab, 0x02])
    assert struct.unpack_from("<I", blob, 4)[0] == 1
    assert ho.hafb_serialize(6, (0,), (0,), [], True).__len__() == 36   # empty batch, test_acceptance.py:209-217
    assert ho.hafb_deserialize(blob) == (6, (1,), (-3,), [683], True)


def test_seeded_key_is_the_references():
    # keygen(1024, default_rng(7)) of the reference: n = 0xdeea09d1f2963929e0...69d9dcb1
    k = ho.keygen(1024, random.Random(7))
    h = format(k.n, "x")
    assert h.startswith("deea09d1f2963929e0") and h.endswith("69d9dcb1")


# ---- (b) transcripts of the unmodified reference ------------------------------------------------------------

@pytest.mark.parametrize("name", list(GOLD["keys"]))
def test_keygen_matches(name):
    spec = GOLD["keys"][name]
    if spec["bits"] is None:
        return
    k = ho.keygen(spec["bits"], random.Random(spec["seed"]))
    assert (k.p, k.q) == (int(spec["p"], 16), int(spec["q"], 16))


@pytest.mark.parametrize("idx", range(len(GOLD["cases"])))
def test_case(idx):
    case = GOLD["cases"][idx]
    k = key_of(case["key"])
    op = case["op"]
    if op == "encode":
        assert [ho.encode(k, v, case["exponent"])[0] for v in case["values"]] == ints(case["mantissas"])
    elif op == "decode":
        assert [ho.decode(k, m, case["exponent"]) for m in ints(case["mantissas"])] == case["values"]
    elif op == "encode_batch_default":
        ms, e = ho.encode_batch(k, case["values"])
        assert e == case["exponent"] and ms == ints(case["mantissas"])
    elif op == "encrypt":
        rng = random.Random(case["seed"])
        rs = [ho.draw_unit(k.n, rng) for _ in case["mantissas"]]
        assert rs == ints(case["r"])
        assert ho.k_encrypt(k, list(zip(ints(case["mantissas"]), rs))) == ints(case["payload"])
    elif op == "decrypt":
        assert ho.k_decrypt(k, ints(case["payload"])) == ints(case["mantissas"])
    elif op == "obfuscate":
        rng = random.Random(case["seed"])
        rs = [ho.draw_unit(k.n, rng) for _ in case["payload_in"]]
        assert ho.k_obfuscate(k, list(zip(ints(case["payload_in"]), rs))) == ints(case["payload"])
    elif op == "add":
        assert ho.k_add(k, list(zip(ints(case["a"]), ints(case["b"])))) == ints(case["payload"])
    elif op == "add_plain":
        assert ho.k_add(k, [(a, ho.lift(k, m)) for a, m in zip(ints(case["a"]), ints(case["m"]))]) == ints(case["payload"])
    elif op == "mul":
        assert ho.k_mul(k, list(zip(ints(case["c"]), ints(case["k"])))) == ints(case["payload"])
    elif op == "sum":
        pay = ints(case["payload_in"])
        rows, cols = case["shape"]
        if case["axis"] is None:
            groups = [pay]
        elif case["axis"] == 0:
            groups = [[pay[r * cols + c] for r in range(rows)] for c in range(cols)]
        else:
            groups = [[pay[r * cols + c] for c in range(cols)] for r in range(rows)]
        assert ho.k_product(k, groups) == ints(case["payload"])
    elif op == "matmul":
        a, x, d = ints(case["a"]), ints(case["x"]), case["d"]
        cols = tuple(tuple(x[t * d + j] for t in range(len(a))) for j in range(d))
        assert ho.k_dot(k, (tuple(a),), cols, [(0, j) for j in range(d)]) == ints(case["payload"])
    elif op == "hafb":
        blob = ho.hafb_serialize(case["key_bits"], tuple(case["shape"]), case["exponents"], ints(case["payload"]),
                                 case["shared"])
        assert blob.hex() == case["bytes"]
        assert ho.hafb_deserialize(blob)[3] == ints(case["payload"])
    else:
        raise AssertionError(op)


# ---- the C / GMP / OpenMP checker agrees with the Python oracle --------------------------------------------------

def _rows(arr):
    return [int.from_bytes(r.tobytes(), "little") for r in arr]


@pytest.mark.parametrize("name", ["k128", "k1024", "k2048", "k3072"])
def test_cpuref_matches_oracle(name):
    k = key_of(name)
    rng = random.Random(3)
    wn, wc = cpuref.widths(k.n)
    cnt = 6
    ms = [rng.randrange(k.n) for _ in range(cnt)]
    rs = [ho.draw_unit(k.n, rng) for _ in ms]
    want = ho.k_encrypt(k, list(zip(ms, rs)))
    c = cpuref.encrypt_words(k.n, cpuref._w(ms, wn), cpuref._w(rs, wn))
    assert _rows(c) == want
    assert _rows(cpuref.obfuscate_words(k.n, c, cpuref._w(rs[::-1], wn))) == ho.k_obfuscate(k, list(zip(want, rs[::-1])))
    assert _rows(cpuref.decrypt_words(k, c)) == ms
    assert _rows(cpuref.mulmod_words(k.n, c, c[::-1].copy())) == ho.k_add(k, list(zip(want, want[::-1])))
    ks = [rng.getrandbits(40) if i % 2 else k.n - rng.getrandbits(40) for i in range(cnt)]
    assert _rows(cpuref.powscalar_words(k.n, c, cpuref._w(ks, wn))) == ho.k_mul(k, list(zip(want, ks)))
    d = 2
    cols = tuple(tuple(ks[t * d + j] for t in range(3)) for j in range(d))
    mv = cpuref.matvec_words(k.n, c[:3].copy(), cpuref._w(ks, wn), 3, d)
    assert _rows(mv) == ho.k_dot(k, (tuple(want[:3]),), cols, [(0, j) for j in range(d)])
