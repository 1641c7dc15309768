"""End-to-end heterogeneous FLR on the B200 against the UNMODIFIED reference's run of the same configuration
(tests/golden/flr_config1.json, tools/make_golden_flr.py): BASELINE configs[0] -- synthetic 1000 x 10, Paillier
1024-bit, one epoch -- plus a small two-epoch run with caching off.  Same data, key and seeds give the same
ciphertexts, so the decrypted masked gradients, the model and the loss must be EQUAL, not close."""
import json
import os
import time

import numpy as np
import pytest

from paper_2107_13797_b200 import flr, paillier

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "flr_config1.json")))["cases"]


def run_case(case):
    ids, X, y = flr.make_synthetic(case["rows"], case["features"], seed=case["seed"])
    guest, host = flr.vertical_split(ids, X, y, 2)
    batches = flr.make_minibatches(case["rows"], case["batch_size"], seed=case["seed"])
    keys = paillier.keygen(case["key_bits"], paillier.default_rng(case["key_seed"]), allow_insecure=True)
    assert format(keys.public.n, "x") == case["n"]
    fed = flr.HeteroFederation(guest, host, batches, list(range(case["rows"])), keys,
                               flr.FlrConfig(0.15, case["batch_size"], seed=case["seed"],
                                             caching_enabled=case["caching"]))
    t0 = time.time()
    results = fed.run(case["epochs"])
    return fed, results, time.time() - t0


@pytest.mark.parametrize("name", ["small_uncached", "config1", "full_batch_2048x200"])
def test_hetero_flr_equals_reference(name):
    case = GOLD[name]
    fed, results, secs = run_case(case)
    assert [r.loss.hex() for r in results] == case["loss"]
    assert [r.grad_norm.hex() for r in results] == case["grad_norm"]
    assert [float(v).hex() for v in fed.combined_theta()] == case["theta"]
    grads = [vec for vec in fed.decrypted if len(vec) > 1]
    assert len(grads) == case["masked_gradients_count"]
    assert [[float(v).hex() for v in vec] for vec in grads[:4]] == case["masked_gradients_first4"]
    assert results[-1].ledger == case["ledger"]
    assert fed.arena.check_conservation()
    print(f"{name}: {secs:.2f}s on the GPU vs {case['reference_seconds']:.2f}s reference CPU")


@pytest.mark.parametrize("name", ["homo_1024", "homo_8party_512"])
def test_homo_flr_equals_reference(name):
    """Horizontal mode (BASELINE configs[4] shape, reduced): encrypted gradient vectors weighted by row count,
    added and decrypted only in aggregate -- aggregated gradients, model and loss equal the reference's."""
    case = GOLD[name]
    ids, X, y = flr.make_synthetic(case["rows"], case["features"], seed=case["seed"])
    parts = flr.horizontal_split(ids, X, y, case["parties"])
    keys = paillier.keygen(case["key_bits"], paillier.default_rng(case["key_seed"]), allow_insecure=True)
    assert format(keys.public.n, "x") == case["n"]
    fed = flr.HomoFederation(parts, keys, flr.FlrConfig(learning_rate=0.15, seed=case["seed"]))
    results = fed.run(case["epochs"])
    assert [r.loss.hex() for r in results] == case["loss"]
    assert [r.grad_norm.hex() for r in results] == case["grad_norm"]
    assert [float(v).hex() for v in fed.theta] == case["theta"]
    assert [[float(v).hex() for v in g] for g in fed.aggregated_gradients] == case["aggregated_gradients"]


def test_full_batch_iteration_equals_cpu_oracle_iteration():
    """The check bench.py makes beside its FLR timing, as a test: full-batch iterations (idx = every row in order, the
    path that skips the row gather) on the GPU against oracle/flr_cpu.py (GMP) with the same data, key and seeds --
    every decrypted masked gradient and the loss equal, float for float."""
    import random

    import flr_cpu
    import hebatch_oracle as ho
    rows, features = 48, 12
    ids, X, y = flr.make_synthetic(rows, features, seed=11)
    guest, host = flr.vertical_split(ids, X, y, 2)
    keys = paillier.keygen(1024, paillier.default_rng(7), allow_insecure=True)
    fed = flr.HeteroFederation(guest, host, [np.arange(rows)], np.arange(rows), keys, flr.FlrConfig(0.15, rows, seed=4))
    okey = ho.Key(keys.public.n, keys.private.p, keys.private.q)
    ref = flr_cpu.CpuHeteroFlr(okey, guest.X, guest.y, host.X, 0.15, 4)
    for _ in range(3):
        assert fed.run_epoch().loss == ref.run_iteration()
    assert fed.decrypted == ref.decrypted
    assert fed.combined_theta().tolist() == np.concatenate([ref.guest_theta, ref.host_theta]).tolist()
