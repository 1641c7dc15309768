"""The dedicated Montgomery squaring (csrc/mont32.cuh, Mont::sqr) against Python integers, for every limb shape
that has one -- (8,4), (16,4), (24,4), (32,4) -- forced through `throughput_shape`, plus the large-batch shapes
of encrypt / decrypt end to end (the small-count launches of the other tests pick other shapes)."""
import random

import numpy as np
import pytest

from paper_2107_13797_b200 import paillier
from paper_2107_13797_b200.backends import default_backend
from paper_2107_13797_b200.device import WordArray

pytestmark = pytest.mark.gpu


def _odd_modulus_key(bits, rng):
    """Any odd n works for the modular kernels (no primality needed): n^2 is the modulus under test."""
    return rng.getrandbits(bits) | (1 << (bits - 1)) | 1


@pytest.mark.parametrize("key_bits", [500, 512, 1000, 1024, 1500, 1536, 2040, 2048])
def test_squaring_matches_integers(key_bits):
    rng = random.Random(key_bits)
    n = _odd_modulus_key(key_bits, rng)
    n2 = n * n
    be = default_backend()
    wc = ((2 * key_bits + 7) // 8 + 3) // 4
    vals = [rng.randrange(n2) for _ in range(61)]
    vals += [0, 1, 2, n2 - 1, n2 - 2, n, n - 1, (1 << (n2.bit_length() - 1)) - 1, 1 << (n2.bit_length() - 1),
             (1 << (n2.bit_length() - 1)) + 1, n2 // 2, n2 // 3, int("f" * (n2.bit_length() // 4 - 1), 16)]
    # limbs of all ones / alternating patterns below the modulus: every carry path of the column sums
    top = n2.bit_length() - 8
    vals += [(1 << top) - 1, ((1 << top) - 1) // 3, ((1 << top) - 1) // 5 * 4, (1 << top) - (1 << 31)]
    arr = WordArray.from_ints(vals, wc)
    for reps in (1, 2, 7):
        got = be.sqrmod(n, arr, reps, throughput_shape=True).ints()
        want = [pow(v, 1 << reps, n2) for v in vals]
        assert list(got) == want, f"key {key_bits} reps {reps}"


def test_squaring_all_ones_modulus():
    """Modulus with every limb 0xffffffff except the lowest: the reduction's carries run the whole width."""
    be = default_backend()
    for bits in (512, 1024, 2048):
        n = (1 << bits) - 1 - 2 * 77
        n2 = n * n
        wc = (2 * bits) // 32
        rng = random.Random(bits)
        vals = [n2 - 1, n2 - 3, rng.randrange(n2), (1 << (2 * bits - 2)) - 1]
        got = be.sqrmod(n, WordArray.from_ints(vals, wc), 3, throughput_shape=True).ints()
        assert list(got) == [pow(v, 8, n2) for v in vals]


@pytest.mark.parametrize("key_bits,count", [(1024, 20000), (2048, 19200), (3072, 15000)])
def test_large_batch_shapes_round_trip(key_bits, count):
    """Encrypt / decrypt at counts that select the throughput shapes ((16,4)/(32,4) at 2048 bits), checked by
    the size-independent round trip and, on a prefix, bit for bit against Python integers."""
    keys = paillier.keygen(key_bits, paillier.default_rng(7), allow_insecure=True)
    pk, sk = keys.public, keys.private
    be = default_backend()
    rng = np.random.default_rng(5)
    wn = (key_bits + 31) // 32
    m = np.zeros((count, wn), dtype=np.uint32)
    m[:, :2] = rng.integers(0, 1 << 32, size=(count, 2), dtype=np.uint64).astype(np.uint32)
    r = rng.integers(0, 1 << 32, size=(count, wn), dtype=np.uint64).astype(np.uint32)
    r[:, wn - 1] >>= 8                       # below n
    r[:, 0] |= 1
    enc = be.encrypt(pk.n, WordArray.from_numpy(m), WordArray.from_numpy(r))
    dec = be.decrypt(pk.n, (sk.p, sk.q, sk._hp, sk._hq, sk._q_inv_p), enc)
    assert np.array_equal(dec.numpy(), m)
    k = 24
    ms = WordArray.from_numpy(m[:k]).ints()
    rs = WordArray.from_numpy(r[:k]).ints()
    want = [(1 + mi * pk.n) * pow(ri, pk.n, pk.n_squared) % pk.n_squared for mi, ri in zip(ms, rs)]
    assert list(WordArray.from_numpy(enc.numpy()[:k]).ints()) == want
