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
from paper_2107_13797_b200.device import WordArray, words_to_ints

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


def _worker(rank, world, port, ret):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ok = ho.keygen(128, random.Random(1234))
        rng = random.Random(7)
        inner, d = 11, 3
        ms = [rng.randrange(ok.n) for _ in range(inner)]
        rs = [ho.draw_unit(ok.n, rng) for _ in ms]
        cs = ho.k_encrypt(ok, list(zip(ms, rs)))
        ks = [rng.getrandbits(30) if i % 2 else ok.n - rng.getrandbits(30) for i in range(inner * d)]
        lo, hi = sharding.shard_range(inner, rank, world)
        # this rank's partial pairs (A_j, B_j), computed on integers in place of hb_matvec_partial
        pairs = []
        for j in range(d):
            a = b = 1
            for t in range(lo, hi):
                k = ks[t * d + j]
                if k > ok.neg_band:
                    b = b * pow(cs[t], ok.n - k, ok.n2) % ok.n2
                else:
                    a = a * pow(cs[t], k, ok.n2) % ok.n2
            pairs += [a, b]
        wc = ((2 * ok.key_bits + 7) // 8 + 3) // 4
        local = WordArray.from_ints(pairs, wc)
        gathered = sharding.all_gather_words(sharding._comm_tensor(local, None))
        assert tuple(gathered.shape) == (world, 2 * d, wc)
        flat = words_to_ints(gathered.reshape(world * 2 * d, wc).numpy().view(np.uint32))
        blocks = [[(flat[(r * d + j) * 2], flat[(r * d + j) * 2 + 1]) for j in range(d)] for r in range(world)]
        got = sharding.combine_partials_reference(ok.n2, blocks)
        cols = tuple(tuple(ks[t * d + j] for t in range(inner)) for j in range(d))
        want = ho.k_dot(ok, (tuple(cs),), cols, [(0, j) for j in range(d)])
        # the sum: per-rank partial products, gathered, multiplied
        part = 1
        for c in cs[lo:hi]:
            part = part * c % ok.n2
        g2 = sharding.all_gather_words(sharding._comm_tensor(WordArray.from_ints([part], wc), None))
        tot = 1
        for v in words_to_ints(g2.reshape(world, wc).numpy().view(np.uint32)):
            tot = tot * v % ok.n2
        ret[rank] = (got == want, tot == ho.k_product(ok, [cs])[0], (lo, hi))
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
    assert ret[0][2] == (0, 6) and ret[1][2] == (6, 11)
