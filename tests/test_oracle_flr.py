"""Pins oracle/flr_cpu.py (the host-CPU FLR iteration bench.py times beside the GPU) to the UNMODIFIED reference's
runs recorded in tests/golden/flr_config1.json (tools/make_golden_flr.py): same data, key and seeds must give the
same loss, model and decrypted masked gradients, float for float.  CPU only."""
import json
import os
import random

import numpy as np
import pytest

import flr_cpu
import hebatch_oracle as ho

GOLD = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "flr_config1.json")))["cases"]


def synthetic(rows, features, seed, noise=0.25):
    """flr/data.py:195-206 of the reference."""
    rng = np.random.default_rng(seed)
    w = rng.normal(size=features)
    w /= np.linalg.norm(w)
    X = rng.uniform(-1.0, 1.0, size=(rows, features))
    y = np.where(X @ w + noise * rng.normal(size=rows) > 0, 1.0, -1.0)
    return X, y


def minibatches(rows, size, seed):
    """flr/data.py:163-171."""
    order = list(range(rows))
    random.Random(seed).shuffle(order)
    return [np.asarray(order[i:i + size], dtype=np.intp) for i in range(0, rows, size)]


@pytest.mark.parametrize("name", ["small_uncached", "config1", "full_batch_2048x200"])
def test_cpu_flr_equals_reference(name):
    if name not in GOLD:
        pytest.skip("golden case not generated")
    case = GOLD[name]
    key = ho.keygen(case["key_bits"], random.Random(case["key_seed"]))
    assert format(key.n, "x") == case["n"]
    X, y = synthetic(case["rows"], case["features"], case["seed"])
    cut = round(case["features"] / 2)                                   # vertical_split, flr/data.py:104-122
    fed = flr_cpu.CpuHeteroFlr(key, X[:, :cut], y, X[:, cut:], 0.15, case["seed"])
    batches = minibatches(case["rows"], case["batch_size"], case["seed"])
    losses = [fed.run_iteration(batches, np.arange(case["rows"])) for _ in range(case["epochs"])]
    assert [v.hex() for v in losses] == case["loss"]
    theta = np.concatenate([fed.guest_theta, fed.host_theta])
    assert [float(v).hex() for v in theta] == case["theta"]
    grads = [vec for vec in fed.decrypted if len(vec) > 1]
    assert len(grads) == case["masked_gradients_count"]
    assert [[float(v).hex() for v in vec] for vec in grads[:4]] == case["masked_gradients_first4"]
