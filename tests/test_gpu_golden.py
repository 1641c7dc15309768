"""GPU parity against tests/golden/hebatch_golden.json: the transcripts of the UNMODIFIED reference's
operators, replayed through this package's operator API on the B200."""
import random

import pytest

from golden_util import ints, load
from paper_2107_13797_b200 import bufferpool, operators as ops, paillier
from paper_2107_13797_b200.batches import CiphertextBatch, PlaintextBatch, encode_batch

pytestmark = pytest.mark.gpu
GOLD = load()
_keys = {}


def keys_of(name):
    if name not in _keys:
        k = GOLD["keys"][name]
        _keys[name] = paillier.keypair_from_primes(int(k["p"], 16), int(k["q"], 16))
    return _keys[name]


@pytest.mark.parametrize("name", [k for k, v in GOLD["keys"].items() if v["bits"]])
def test_keygen_matches(name):
    spec = GOLD["keys"][name]
    kp = paillier.keygen(spec["bits"], paillier.default_rng(spec["seed"]), allow_insecure=True)
    assert (kp.private.p, kp.private.q) == (int(spec["p"], 16), int(spec["q"], 16))


@pytest.mark.parametrize("idx", range(len(GOLD["cases"])))
def test_case(idx):
    case = GOLD["cases"][idx]
    pk, sk = keys_of(case["key"])
    op = case["op"]
    if op == "encode":
        assert list(ops.batch_encode(pk, case["values"], case["exponent"]).mantissas) == ints(case["mantissas"])
    elif op == "decode":
        ms = ints(case["mantissas"])
        plain = PlaintextBatch(pk, (len(ms),), (case["exponent"],), ms, True)
        got = ops.batch_decode(pk, plain)
        assert got == case["values"]
        assert [str(v) for v in got] == [str(v) for v in case["values"]]      # -0.0 vs 0.0
    elif op == "encode_batch_default":
        eb = encode_batch(pk, case["values"])
        assert eb.exponents == (case["exponent"],) and list(eb.mantissas) == ints(case["mantissas"])
    elif op == "encrypt":
        ms = ints(case["mantissas"])
        plain = PlaintextBatch(pk, (len(ms),), (-8,), ms, True)
        assert list(ops.batch_encrypt(pk, plain, random.Random(case["seed"])).payload) == ints(case["payload"])
    elif op == "decrypt":
        pay = ints(case["payload"])
        got = ops.batch_decrypt(sk, CiphertextBatch(pk, (len(pay),), (0,), pay, True))
        assert list(got.mantissas) == ints(case["mantissas"])
    elif op == "obfuscate":
        pay = ints(case["payload_in"])
        got = ops.batch_obfuscate(pk, CiphertextBatch(pk, (len(pay),), (0,), pay, True), random.Random(case["seed"]))
        assert list(got.payload) == ints(case["payload"])
    elif op == "add":
        a, b = ints(case["a"]), ints(case["b"])
        ca = CiphertextBatch(pk, (len(a),), (0,), a, True)
        cb = CiphertextBatch(pk, (len(b),), (0,), b, True)
        assert list(ops.batch_add(pk, ca, cb).payload) == ints(case["payload"])
    elif op == "add_plain":
        a, m = ints(case["a"]), ints(case["m"])
        ca = CiphertextBatch(pk, (len(a),), (0,), a, True)
        assert list(ops.batch_add(pk, ca, PlaintextBatch(pk, (len(m),), (0,), m, True)).payload) == ints(case["payload"])
    elif op == "mul":
        c, k = ints(case["c"]), ints(case["k"])
        ca = CiphertextBatch(pk, (len(c),), (-8,), c, True)
        got = ops.batch_mul_plain(pk, ca, PlaintextBatch(pk, (len(k),), (0,), k, True))
        assert list(got.payload) == ints(case["payload"])
    elif op == "sum":
        pay = ints(case["payload_in"])
        got = ops.batch_sum(pk, CiphertextBatch(pk, tuple(case["shape"]), (0,), pay, True), case["axis"])
        assert list(got.payload) == ints(case["payload"]) and list(got.shape) == case["out_shape"]
    elif op == "matmul":
        a, x, d = ints(case["a"]), ints(case["x"]), case["d"]
        ca = CiphertextBatch(pk, (len(a),), (0,), a, True)
        got = ops.batch_matmul(pk, ca, PlaintextBatch(pk, (len(a), d), (-3,), x, True))
        assert list(got.payload) == ints(case["payload"])
    elif op == "hafb":
        batch = CiphertextBatch(pk, tuple(case["shape"]), case["exponents"], ints(case["payload"]), case["shared"])
        blob = bufferpool.serialize_to_bytes(batch)
        assert blob.hex() == case["bytes"]
        assert bufferpool.deserialize(blob, pk) == CiphertextBatch(pk, batch.shape, batch.exponents, batch.payload, True, True)
    else:
        raise AssertionError(op)
