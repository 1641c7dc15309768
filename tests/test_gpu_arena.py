"""Device-memory arena on the B200: residency, ledger arithmetic, LRU spill, the fore-gradient pipeline.
Follows the assertions of the reference's tests/test_arena.py (cited inline)."""
import random

import pytest

from paper_2107_13797_b200 import operators as ops, paillier
from paper_2107_13797_b200.arena import Arena, ArenaCapacityError, DeadHandle, TransferLedger
from paper_2107_13797_b200.batches import decode_batch, encode_batch
from paper_2107_13797_b200.bufferpool import serialized_size

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def keys():
    return paillier.keygen(128, paillier.default_rng(1234), allow_insecure=True)


def make_arena(keys, **kw):
    return Arena(keys.public, rng=paillier.default_rng(100), **kw)


def cipher_of(keys, values, seed=0, exponent=-8):
    plain = encode_batch(keys.public, values, target_exponent=exponent)
    return ops.batch_encrypt(keys.public, plain, paillier.default_rng(seed))


def test_round_trip_and_ledger(keys):
    arena = make_arena(keys)
    batch = cipher_of(keys, [1.0, -2.0, 3.0])
    h = arena.upload(batch)
    assert batch.words.on_device
    assert arena.download(h) == batch
    size = serialized_size(3, keys.public.key_bits, True)
    assert arena.ledger.to_json() == {"uploads": {"count": 1, "bytes": size}, "downloads": {"count": 1, "bytes": size},
                                      "serializations": 1, "deserializations": 1}
    assert h.live and h.kind == "cipher" and h.shape == (3,)
    assert arena.upload(batch).id != h.id
    with pytest.raises(ValueError):
        arena.upload(cipher_of(paillier.keygen(64, paillier.default_rng(1), allow_insecure=True), [1.0]))


def test_release_semantics(keys):
    arena = make_arena(keys)
    h = arena.upload(cipher_of(keys, [5.0]))
    arena.release(h)
    assert not h.live
    with pytest.raises(DeadHandle):
        arena.download(h)
    with pytest.raises(DeadHandle):
        arena.release(h)
    assert arena.check_conservation()


def test_exec_op_matches_direct_operators(keys):
    pk = keys.public
    arena = make_arena(keys)
    ca, cb = cipher_of(keys, [1.5, -2.0], seed=3), cipher_of(keys, [0.25, 8.0], seed=4)
    ha, hb = arena.upload(ca), arena.upload(cb)
    before = arena.ledger.downloads.count
    h_sum = arena.exec_op("add", [ha, hb])
    assert arena.ledger.downloads.count == before            # cached: nothing came back (test_arena.py:86-94)
    assert arena.download(h_sum) == ops.batch_add(pk, ca, cb)
    k = encode_batch(pk, [0.25])
    assert arena.download(arena.exec_op("mul", [ha, k])) == ops.batch_mul_plain(pk, ca, k)
    x = encode_batch(pk, [[1.0], [2.0]], target_exponent=-8)
    assert arena.download(arena.exec_op("matmul", [ha, x])) == ops.batch_matmul(pk, ca, x)
    two = cipher_of(keys, [[1.0, 2.0], [3.0, 4.0]], seed=9)
    assert arena.exec_op("sum", [two], cache_result=False, axis=0) == ops.batch_sum(pk, two, 0)
    out = arena.exec_op("add", [ha, hb], cache_result=False)
    assert decode_batch(pk, ops.batch_decrypt(keys.private, out)) == [1.75, 6.0]
    with pytest.raises(ValueError):
        arena.exec_op("nope", [ha])
    assert arena.check_conservation()


def test_lru_spill_and_restore(keys):
    """Capacity for two batches: the third upload spills the least recently used one to the host; touching it
    brings it back (test_arena.py:142-180)."""
    size = serialized_size(2, keys.public.key_bits, True)
    arena = make_arena(keys, capacity_bytes=2 * size)
    b1, b2, b3 = (cipher_of(keys, [float(i), -float(i)], seed=i) for i in (1, 2, 3))
    h1, h2 = arena.upload(b1), arena.upload(b2)
    arena.download(h1)                                      # h1 is now the most recently used
    h3 = arena.upload(b3)
    assert arena.state_of(h2) == "evicted" and arena.state_of(h1) == "live" and arena.state_of(h3) == "live"
    assert not b2.words.on_device and b1.words.on_device
    assert arena.evicted_bytes == size and arena.resident_bytes == 2 * size
    ups = arena.ledger.uploads.count
    assert arena.download(h2) == b2                         # transparent restore, counted as an upload
    assert arena.ledger.uploads.count == ups + 1 and arena.state_of(h2) == "live"
    assert arena.check_conservation()
    # pinned inputs cannot be evicted
    tight = make_arena(keys, capacity_bytes=2 * size)
    ha, hb = tight.upload(b1), tight.upload(b2)
    with pytest.raises(ArenaCapacityError):
        tight.exec_op("add", [ha, hb])


def test_dag_under_eviction_equals_direct(keys):
    """A chain of operators under forced eviction gives the bits of direct execution (test_arena.py:203-224)."""
    pk = keys.public
    size = serialized_size(4, pk.key_bits, True)
    arena = make_arena(keys, capacity_bytes=3 * size)
    cs = [cipher_of(keys, [i + 0.5, -i, 2.0 * i, 1.0], seed=10 + i) for i in range(4)]
    hs = [arena.upload(c) for c in cs]
    k = encode_batch(pk, [-0.5])
    t1 = arena.exec_op("add", [hs[0], hs[1]])
    t2 = arena.exec_op("mul", [hs[2], k])
    t3 = arena.exec_op("add", [t1, hs[3]])
    direct = ops.batch_add(pk, ops.batch_add(pk, cs[0], cs[1]), cs[3])
    assert arena.download(t3) == direct
    assert arena.download(t2) == ops.batch_mul_plain(pk, cs[2], k)
    assert arena.ledger.downloads.count > 2                 # spills happened
    assert arena.check_conservation()


@pytest.mark.parametrize("caching", [True, False])
def test_fore_gradient_pipeline(keys, caching):
    """fore(lh = 0.4, lg = 0.6, y = 1) = 0.25 * (0.4 + 0.6) - 0.5 = -0.25 (test_arena.py:228-237)."""
    pk, sk = keys
    arena = make_arena(keys, caching_enabled=caching)
    lh = cipher_of(keys, [0.4, -1.0, 2.5], seed=1, exponent=-10)
    lg = encode_batch(pk, [0.6, 0.5, -0.5], target_exponent=-10)
    y = encode_batch(pk, [1.0, 0.0, 1.0], target_exponent=0)
    out = arena.run_fore_gradient_pipeline(lh, lg, y)
    batch = arena.download(out) if caching else out
    got = decode_batch(pk, ops.batch_decrypt(sk, batch))
    want = [0.25 * (a + b) - 0.5 * c for a, b, c in zip([0.4, -1.0, 2.5], [0.6, 0.5, -0.5], [1.0, 0.0, 1.0])]
    assert all(abs(g - w) < 1e-9 for g, w in zip(got, want)) and abs(got[0] + 0.25) < 1e-9
    if caching:
        assert arena.ledger.downloads.count == 1            # only the final result crossed back
    else:
        assert arena.ledger.downloads.count >= 6
    with pytest.raises(ValueError):
        arena.run_fore_gradient_pipeline(lh, encode_batch(pk, [0.6, 0.5, -0.5], target_exponent=-9), y)
    assert arena.check_conservation()


def test_shared_ledger(keys):
    ledger = TransferLedger()
    a1, a2 = make_arena(keys, ledger=ledger), make_arena(keys, ledger=ledger)
    a1.upload(cipher_of(keys, [1.0]))
    a2.upload(cipher_of(keys, [2.0]))
    assert ledger.uploads.count == 2 and ledger.snapshot()[0] == 2
