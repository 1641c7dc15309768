"""Scaled heterogeneous-FLR iteration on the GPU (BASELINE configs[3] shape: 2 parties, 200 features,
Paillier-2048, full-batch steps) with a per-operator wall-clock breakdown.

    python tools/flr_scale.py --rows 100000 --features 200 --iters 2 [--key-bits 2048] [--profile]

One iteration = one full-batch gradient step + the loss over all rows.  Prints a
JSON line: seconds per iteration, the loss per iteration, and the time spent inside each operator / codec /
wire-format function (host wall clock, device-synchronised after every call).
"""
from __future__ import annotations

import argparse
import collections
import functools
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2107_13797_b200 import batches, bufferpool, flr, operators, paillier  # noqa: E402

SPENT = collections.defaultdict(float)
CALLS = collections.defaultdict(int)
_depth = [0]


def _sync():
    import torch
    torch.cuda.synchronize()


def timed(mod, name):
    fn = getattr(mod, name)

    @functools.wraps(fn)
    def wrapper(*a, **kw):
        outer = _depth[0] == 0
        _depth[0] += 1
        t0 = time.perf_counter()
        try:
            return fn(*a, **kw)
        finally:
            _depth[0] -= 1
            if outer:
                _sync()
                SPENT[name] += time.perf_counter() - t0
                CALLS[name] += 1
    setattr(mod, name, wrapper)
    return wrapper


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=100_000)
    ap.add_argument("--features", type=int, default=200)
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--key-bits", type=int, default=2048)
    ap.add_argument("--pool-keep-gib", type=float, default=0.0, help="HB_OPT_POOL_KEEP_BYTES for the key's context")
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--profile-first", action="store_true", help="cProfile the FIRST iteration instead of the last")
    args = ap.parse_args()

    for name in ("batch_encrypt", "batch_obfuscate", "batch_decrypt", "batch_add", "batch_mul_plain", "batch_sum",
                 "batch_matmul", "batch_encode", "batch_decode"):
        timed(operators, name)
    for name in ("plain_mul", "plain_add", "plain_rescale"):
        w = timed(batches, name)
        for mod in (operators, flr):
            if hasattr(mod, name):
                setattr(mod, name, w)
        from paper_2107_13797_b200 import arena as arena_mod
        if hasattr(arena_mod, name):
            setattr(arena_mod, name, w)
    from paper_2107_13797_b200 import arena as arena_mod
    timed(arena_mod.Arena, "run_fore_gradient_pipeline")        # the fused chain (one kernel) or its six operators
    for name in ("serialize_to_bytes", "deserialize"):
        w = timed(bufferpool, name)
        setattr(flr, name, w)

    t0 = time.perf_counter()
    ids, X, y = flr.make_synthetic(args.rows, args.features, seed=42)
    guest, host = flr.vertical_split(ids, X, y, 2)
    keys = paillier.keygen(args.key_bits, paillier.default_rng(7), allow_insecure=True)
    if args.pool_keep_gib:
        from paper_2107_13797_b200 import _native, device
        device.context_for(keys.public.n).set_option(_native.HB_OPT_POOL_KEEP_BYTES, int(args.pool_keep_gib * 2 ** 30))
    full = [np.arange(args.rows)]
    fed = flr.HeteroFederation(guest, host, full, np.arange(args.rows), keys,
                               flr.FlrConfig(0.15, args.rows, seed=42))
    setup = time.perf_counter() - t0
    per_iter, losses = [], []
    prof = None
    for it in range(args.iters):
        if it == 0 and args.profile_first:
            import cProfile
            prof = cProfile.Profile()
            prof.enable()
        if it == 1 and args.profile_first and prof is not None:
            prof.disable()
            import pstats
            pstats.Stats(prof).sort_stats("tottime").print_stats(30)
            prof = None
        if it == args.iters - 1:          # the breakdown reports the last (steady-state) iteration only
            SPENT.clear()
            CALLS.clear()
            if args.profile:
                import cProfile
                prof = cProfile.Profile()
                prof.enable()
        t0 = time.perf_counter()
        res = fed.run_epoch()
        _sync()
        per_iter.append(time.perf_counter() - t0)
        losses.append(res.loss)
    if prof is not None:
        prof.disable()
        import pstats
        pstats.Stats(prof).sort_stats("cumulative").print_stats(35)
    inside = sum(SPENT.values())
    print(json.dumps({
        "rows": args.rows, "features": args.features, "key_bits": args.key_bits, "iters": args.iters,
        "setup_s": round(setup, 2), "s_per_iter": [round(t, 3) for t in per_iter], "loss": losses,
        "breakdown_s": {k: round(v, 3) for k, v in sorted(SPENT.items(), key=lambda kv: -kv[1])},
        "calls": dict(CALLS), "outside_ops_s": round(per_iter[-1] - inside, 3),
        "ledger": fed.ledger.to_json(),
    }))


if __name__ == "__main__":
    main()
