"""Generates tests/golden/flr_config1.json: BASELINE configs[0] -- hetero LR, synthetic 1000 x 10, Paillier
1024-bit, one epoch -- run with the UNMODIFIED reference (NaiveBackend) in the build container.

    python tools/make_golden_flr.py

Floats are stored with float.hex() so the comparison on the GPU box is exact.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle", "gmpy2_shim"))
sys.path.insert(0, "/root/reference/pkg/src")

from hebatch.backends import NaiveBackend  # noqa: E402
from hebatch.flr.data import horizontal_split, make_minibatches, make_synthetic, vertical_split  # noqa: E402
from hebatch.flr.parties import DecryptEvent, FlrConfig, HeteroFederation, HomoFederation, Message  # noqa: E402
from hebatch.paillier import default_rng, keygen  # noqa: E402


def run(rows, features, key_bits, batch_size, epochs, seed=42, key_seed=7, caching=True):
    table = make_synthetic(rows, features, seed=seed)
    guest, host = vertical_split(table, 2)
    batches = make_minibatches(rows, batch_size, seed=seed)
    keys = keygen(key_bits, default_rng(key_seed), allow_insecure=True)
    fed = HeteroFederation(guest, host, batches, list(range(rows)), keys,
                           FlrConfig(0.15, batch_size, seed=seed, caching_enabled=caching), NaiveBackend())
    t0 = time.time()
    results = fed.run(epochs)
    secs = time.time() - t0
    masked = [m.payload for m in fed.hub.trace if isinstance(m, Message) and m.kind == "masked_gradient"]
    return {
        "rows": rows, "features": features, "key_bits": key_bits, "batch_size": batch_size, "epochs": epochs,
        "seed": seed, "key_seed": key_seed, "caching": caching, "reference_seconds": secs,
        "loss": [r.loss.hex() for r in results], "grad_norm": [r.grad_norm.hex() for r in results],
        "theta": [float(v).hex() for v in fed.combined_theta()],
        "masked_gradients_first4": [[float(v).hex() for v in vec] for vec in masked[:4]],
        "masked_gradients_count": len(masked), "ledger": results[-1].ledger,
        "n": format(keys.public.n, "x"),
    }


def run_homo(rows, features, key_bits, parties, epochs, seed=43, key_seed=7):
    """Horizontal mode (BASELINE configs[4] shape, reduced): aggregated gradients, model and loss per epoch."""
    table = make_synthetic(rows, features, seed=seed)
    parts = horizontal_split(table, parties)
    keys = keygen(key_bits, default_rng(key_seed), allow_insecure=True)
    fed = HomoFederation(parts, keys, FlrConfig(learning_rate=0.15, seed=seed), NaiveBackend())
    t0 = time.time()
    results = fed.run(epochs)
    secs = time.time() - t0
    return {
        "rows": rows, "features": features, "key_bits": key_bits, "parties": parties, "epochs": epochs,
        "seed": seed, "key_seed": key_seed, "reference_seconds": secs,
        "loss": [r.loss.hex() for r in results], "grad_norm": [r.grad_norm.hex() for r in results],
        "theta": [float(v).hex() for v in fed.theta],
        "aggregated_gradients": [[float(v).hex() for v in g] for g in fed.aggregated_gradients],
        "n": format(keys.public.n, "x"),
    }


if __name__ == "__main__":
    out = {"generator": "tools/make_golden_flr.py", "cases": {
        "config1": run(1000, 10, 1024, 32, 1),
        "small_uncached": run(96, 6, 512, 16, 2, seed=5, key_seed=99, caching=False),
        "homo_1024": run_homo(1000, 8, 1024, 2, 3),
        "homo_8party_512": run_homo(400, 24, 512, 8, 2, seed=9, key_seed=99),
        # BASELINE configs[3] shape (Paillier-2048, 200 features, full-batch steps) at 256 rows, two iterations
        "full_batch_2048x200": run(256, 200, 2048, 256, 2),
    }}
    path = os.path.join(ROOT, "tests", "golden", "flr_config1.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(path, {k: (v["reference_seconds"], v["loss"]) for k, v in out["cases"].items()})
