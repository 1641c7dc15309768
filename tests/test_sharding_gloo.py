"""Host-side logic of the multi-GPU path with a 2-rank gloo group on CPU (no GPU needed):
slice arithmetic, batch sharding, the all-gather of partials and its combine order.  The device kernels
behind sharded_matmul / sharded_sum are covered by tests/test_gpu_sharding.py with a single-rank group."""
import os
import random
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

import hebatch_oracle as ho
from paper_2107_13797_b200 import paillier, sharding
from paper_2107_13797_b200.batches import CiphertextBatch, PlaintextBatch
from paper_2107_13797_b200.device import WordArray

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_shard_range_is_the_reference_schedule():
    # contiguous chunks of ceil(count / workers), order preserving (reference backends.py:64-73)
    for count in (0, 1, 7, 8, 9, 100, 1001):
        for world in (1, 2, 3, 4, 8):
            chunk = -(-count // world) if count else 0
            want = [(min(i * chunk, count), min(i * chunk + chunk, count)) for i in range(world)]
            got = [sharding.shard_range(count, r, world) for r in range(world)]
            assert got == want
            assert sum(hi - lo for lo, hi in got) == count
            assert all(got[i][1] == got[i + 1][0] for i in range(world - 1))
    with pytest.raises(ValueError):
        sharding.shard_range(4, 2, 2)


def test_shard_rows_keeps_metadata():
    pk = paillier.PublicKey(35)
    c = CiphertextBatch(pk, (5,), (-2,), (1, 2, 3, 4, 5), True, obfuscated=False)
    parts = [sharding.shard_rows(c, r, 2) for r in range(2)]
    assert [p.payload for p in parts] == [(1, 2, 3), (4, 5)]
    assert all(p.exponents == (-2,) and p.obfuscated is False for p in parts)
    x = PlaintextBatch(pk, (3, 2), (0, 1, 2, 3, 4, 5), (1, 2, 3, 4, 5, 6), False)
    parts = [sharding.shard_rows(x, r, 2) for r in range(2)]
    assert [p.mantissas for p in parts] == [(1, 2, 3, 4), (5, 6)]
    assert [p.exponents for p in parts] == [(0, 1, 2, 3), (4, 5)] and parts[1].shape == (1, 2)


class IntBackend:
    """Stands in for the device kernels behind sharding.sharded_matmul / sharded_sum with the oracle's integer
    arithmetic, so that the REAL gather / combine code of sharding.py runs with two processes on CPU."""

    def __init__(self, ok):
        self.ok = ok
        self.wc = ((2 * ok.key_bits + 7) // 8 + 3) // 4

    def matvec_partial(self, n, c, k, inner, d):
        ok = self.ok
        cs, ks = c.ints(), k.ints()
        pairs = []
        for j in range(d):
            a = b = 1
            for t in range(inner):
                kk = ks[t * d + j]
                if kk > ok.neg_band:
                    b = b * pow(cs[t], ok.n - kk, ok.n2) % ok.n2
                else:
                    a = a * pow(cs[t], kk, ok.n2) % ok.n2
            pairs += [a, b]
        return WordArray.from_ints(pairs, self.wc)

    def matvec_combine(self, n, ab_all, nranks, d):
        flat = ab_all.ints()
        blocks = [[(flat[(r * d + j) * 2], flat[(r * d + j) * 2 + 1]) for j in range(d)] for r in range(nranks)]
        return WordArray.from_ints(sharding.combine_partials_reference(self.ok.n2, blocks), self.wc)

    def product(self, n, c, ngroups, glen, gstride, estride):
        assert ngroups == 1 and estride == 1
        tot = 1
        for v in c.ints()[:glen]:
            tot = tot * v % self.ok.n2
        return WordArray.from_ints([tot], self.wc)


def _worker(rank, world, port, ret):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist
    from paper_2107_13797_b200 import operators
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ok = ho.keygen(128, random.Random(1234))
        pk = paillier.PublicKey(ok.n)
        be = IntBackend(ok)
        operators._cuda = lambda backend: backend          # the stub is not a CudaBackend; nothing else changes
        rng = random.Random(7)
        inner, d = 11, 3
        ms = [rng.randrange(ok.n) for _ in range(inner)]
        rs = [ho.draw_unit(ok.n, rng) for _ in ms]
        cs = ho.k_encrypt(ok, list(zip(ms, rs)))
        ks = [rng.getrandbits(30) if i % 2 else ok.n - rng.getrandbits(30) for i in range(inner * d)]
        a = CiphertextBatch(pk, (inner,), (-3,), cs, True, obfuscated=True)
        x = PlaintextBatch(pk, (inner, d), (-2,), ks, True)
        # the product's own sharding helpers, then the product's own gather + combine
        a_loc, x_loc = sharding.shard_rows(a, rank, world), sharding.shard_rows(x, rank, world)
        got = sharding.sharded_matmul(pk, a_loc, x_loc, be)
        cols = tuple(tuple(ks[t * d + j] for t in range(inner)) for j in range(d))
        want = ho.k_dot(ok, (tuple(cs),), cols, [(0, j) for j in range(d)])
        ok_mat = (list(got.payload) == want and got.exponents == (-5,) and got.shape == (d,) and got.obfuscated)
        total = sharding.sharded_sum(pk, a_loc, be)
        ok_sum = list(total.payload) == ho.k_product(ok, [cs]) and total.exponents == (-3,)
        ret[rank] = (ok_mat, ok_sum, (a_loc.count, x_loc.shape))
    finally:
        dist.destroy_process_group()


def test_two_rank_gather_and_combine():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(2, port, ret), nprocs=2, join=True)
    assert ret[0][:2] == (True, True) and ret[1][:2] == (True, True)
    assert ret[0][2] == (6, (6, 3)) and ret[1][2] == (5, (5, 3))
