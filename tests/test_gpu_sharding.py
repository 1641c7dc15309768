"""Row-sharded matvec / sum on the GPU: partial + combine kernels against the single-call result, with the
gather done in-process (one GPU here; the collective itself is covered by tests/test_sharding_gloo.py) and
through a 1-rank NCCL group."""
import os
import random

import numpy as np
import pytest

import hebatch_oracle as ho
from paper_2107_13797_b200 import operators as ops, paillier, sharding
from paper_2107_13797_b200.backends import CudaBackend
from paper_2107_13797_b200.batches import CiphertextBatch, PlaintextBatch
from paper_2107_13797_b200.device import WordArray

pytestmark = pytest.mark.gpu


def setup_problem(okeys, name, inner, d, bits, seed=3):
    ok = okeys(name)
    kp = paillier.keypair_from_primes(ok.p, ok.q)
    rng = random.Random(seed)
    pool = ho.k_encrypt(ok, [(rng.randrange(ok.n), ho.draw_unit(ok.n, rng)) for _ in range(8)])
    cs = [pool[rng.randrange(8)] for _ in range(inner)]
    ks = []
    for i in range(inner * d):
        mag = rng.getrandbits(bits) % ok.max_int
        ks.append(mag if i % 2 else (ok.n - mag) % ok.n)
    a = CiphertextBatch(kp.public, (inner,), (-4,), cs, True)
    x = PlaintextBatch(kp.public, (inner, d), (-9,), ks, True)
    return ok, kp.public, a, x


@pytest.mark.parametrize("name,bits", [("k512", 52), ("k1024", 40), ("k128", 100)])
@pytest.mark.parametrize("world", [1, 2, 3])
def test_partials_combine_to_the_single_call(okeys, name, bits, world):
    ok, pk, a, x = setup_problem(okeys, name, 37, 4, bits)
    be = CudaBackend()
    want = ops.batch_matmul(pk, a, x)
    blocks = []
    for r in range(world):
        ar, xr = sharding.shard_rows(a, r, world), sharding.shard_rows(x, r, world)
        blocks.append(be.matvec_partial(pk.n, ar.words, xr.words, ar.shape[0], 4).numpy())
    allw = WordArray.from_numpy(np.concatenate(blocks, axis=0))
    got = be.matvec_combine(pk.n, allw, world, 4)
    assert got.ints() == want.payload


def test_sharded_ops_through_a_process_group(okeys):
    import torch
    import torch.distributed as dist
    ok, pk, a, x = setup_problem(okeys, "k512", 50, 3, 52)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        be = CudaBackend()
        out = sharding.sharded_matmul(pk, a, x, be)
        assert out == ops.batch_matmul(pk, a, x)
        tot = sharding.sharded_sum(pk, a, be)
        assert tot == ops.batch_sum(pk, a)
    finally:
        dist.destroy_process_group()
