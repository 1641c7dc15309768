"""Generates tests/golden/hebatch_golden.json by running the UNMODIFIED reference package.

Run in the build container only (needs /root/reference and the gmpy2 stand-in over libgmp):

    python tools/make_golden.py

The reference's own operators (NaiveBackend) produce every expected value; nothing from this
repository's oracle or CUDA code is involved, so the fixture pins both of them to the reference.
Big integers are stored as hex strings.
"""
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle", "gmpy2_shim"))
sys.path.insert(0, "/root/reference/pkg/src")

from hebatch import bufferpool, operators  # noqa: E402
from hebatch.backends import NaiveBackend  # noqa: E402
from hebatch.batches import CiphertextBatch, PlaintextBatch, encode_batch  # noqa: E402
from hebatch.paillier import default_rng, draw_unit, keygen, keypair_from_primes  # noqa: E402

KEYS = {"tiny": None, "k128": (128, 1234), "k512": (512, 99), "k1024": (1024, 7), "k2048": (2048, 7),
        "k3072": (3072, 7)}
COUNT = {"tiny": 6, "k128": 8, "k512": 6, "k1024": 5, "k2048": 4, "k3072": 3}


def hx(v):
    return format(int(v), "x")


def hxl(vs):
    return [hx(v) for v in vs]


def main():
    naive = NaiveBackend()
    out = {"generator": "tools/make_golden.py", "reference": "hebatch 0.1.0 (unmodified), gmpy2 stand-in over libgmp 6.3.0",
           "keys": {}, "cases": []}
    cases = out["cases"]
    for name, spec in KEYS.items():
        kp = keypair_from_primes(5, 7) if spec is None else keygen(spec[0], default_rng(spec[1]), allow_insecure=True)
        pk, sk = kp.public, kp.private
        out["keys"][name] = {"bits": None if spec is None else spec[0], "seed": None if spec is None else spec[1],
                             "p": hx(sk.p), "q": hx(sk.q), "n": hx(pk.n)}
        rng = random.Random(hash(name) & 0xffff if False else len(name) * 7919)
        cnt = COUNT[name]
        tiny = spec is None
        # codec
        vals = [0.5, -0.5, 1.0, -2.0, 2.5, 3.5, -10.0] if tiny else [rng.uniform(-100, 100) for _ in range(cnt)] + [0.0, -0.0, 1.5]
        exp = 0 if tiny else -8
        enc_plain = operators.batch_encode(pk, vals, exp, naive)
        cases.append({"key": name, "op": "encode", "values": vals, "exponent": exp, "mantissas": hxl(enc_plain.mantissas)})
        cases.append({"key": name, "op": "decode", "mantissas": hxl(enc_plain.mantissas), "exponent": exp,
                      "values": operators.batch_decode(pk, enc_plain, naive)})
        if not tiny:
            eb = encode_batch(pk, vals)
            cases.append({"key": name, "op": "encode_batch_default", "values": vals, "exponent": eb.exponents[0],
                          "mantissas": hxl(eb.mantissas)})
        # encrypt / decrypt / obfuscate
        ms = [rng.randrange(pk.n) for _ in range(cnt)]
        plain = PlaintextBatch(pk, (cnt,), (exp,), tuple(ms), True)
        seed = 100 + cnt
        ca = operators.batch_encrypt(pk, plain, default_rng(seed), naive)
        r_rng = default_rng(seed)
        rs = [draw_unit(pk.n, r_rng) for _ in ms]
        cases.append({"key": name, "op": "encrypt", "mantissas": hxl(ms), "seed": seed, "r": hxl(rs),
                      "payload": hxl(ca.payload)})
        cases.append({"key": name, "op": "decrypt", "payload": hxl(ca.payload),
                      "mantissas": hxl(operators.batch_decrypt(sk, ca, naive).mantissas)})
        ob = operators.batch_obfuscate(pk, ca, default_rng(seed + 1), naive)
        cases.append({"key": name, "op": "obfuscate", "payload_in": hxl(ca.payload), "seed": seed + 1,
                      "payload": hxl(ob.payload)})
        # add
        ms2 = [rng.randrange(pk.n) for _ in range(cnt)]
        cb = operators.batch_encrypt(pk, PlaintextBatch(pk, (cnt,), (exp,), tuple(ms2), True), default_rng(seed + 2), naive)
        cases.append({"key": name, "op": "add", "a": hxl(ca.payload), "b": hxl(cb.payload),
                      "payload": hxl(operators.batch_add(pk, ca, cb, naive).payload)})
        small = [rng.randrange(pk.max_int // 4 + 1) for _ in range(cnt)]
        pb = PlaintextBatch(pk, (cnt,), (exp,), tuple(small), True)
        cases.append({"key": name, "op": "add_plain", "a": hxl(ca.payload), "m": hxl(small),
                      "payload": hxl(operators.batch_add(pk, ca, pb, naive).payload)})
        # scalar multiplication: paired scalars, mixed signs, plus band edge and an overflow-band residue
        mag_bits = max(1, min(40, pk.max_int.bit_length() - 1))
        ks = []
        for i in range(cnt):
            mag = rng.getrandbits(mag_bits) % pk.max_int
            ks.append(mag if i % 2 == 0 else (pk.n - mag) % pk.n)
        ks[-1] = pk.n - pk.max_int
        if cnt > 2:
            ks[-2] = pk.n // 2
        kb = PlaintextBatch(pk, (cnt,), (0,), tuple(ks), True)
        mul = operators.batch_mul_plain(pk, ca, kb, naive)
        cases.append({"key": name, "op": "mul", "c": hxl(ca.payload), "k": hxl(ks), "payload": hxl(mul.payload),
                      "exponents": list(mul.exponents)})
        # reductions on a 2 x (cnt // 2) view
        cols = cnt // 2
        two = CiphertextBatch(pk, (2, cols), (exp,), ca.payload[:2 * cols], True)
        for axis in (None, 0, 1):
            s = operators.batch_sum(pk, two, axis, naive)
            cases.append({"key": name, "op": "sum", "payload_in": hxl(two.payload), "shape": [2, cols], "axis": axis,
                          "payload": hxl(s.payload), "out_shape": list(s.shape)})
        # matmul: 1 x cnt encrypted row times cnt x 2 scalars
        xs = []
        for i in range(cnt * 2):
            mag = rng.getrandbits(min(52, mag_bits)) % pk.max_int
            xs.append(mag if i % 3 else (pk.n - mag) % pk.n)
        x = PlaintextBatch(pk, (cnt, 2), (-3,), tuple(xs), True)
        mm = operators.batch_matmul(pk, ca, x, naive)
        cases.append({"key": name, "op": "matmul", "a": hxl(ca.payload), "x": hxl(xs), "d": 2,
                      "payload": hxl(mm.payload), "exponent": mm.exponents[0]})
        # wire format
        blob = bufferpool.serialize_to_bytes(two)
        cases.append({"key": name, "op": "hafb", "key_bits": pk.key_bits, "shape": [2, cols], "exponents": [exp],
                      "shared": True, "payload": hxl(two.payload), "bytes": blob.hex()})
    path = os.path.join(ROOT, "tests", "golden", "hebatch_golden.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as fh:
        json.dump(out, fh, indent=0, separators=(",", ":"))
    print(path, os.path.getsize(path), "bytes,", len(cases), "cases")


if __name__ == "__main__":
    main()
