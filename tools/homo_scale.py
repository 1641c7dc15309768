"""Homogeneous-FLR encrypted model aggregation at scale (BASELINE configs[4]: 8 parties x 1M-parameter vectors,
Paillier-3072), through the operator API, with per-operator device-synchronised timings.

    python tools/homo_scale.py --params 1000000 --parties 8 --key-bits 3072

Per aggregation (reference flr/parties.py:416-432): 8 x batch_encrypt, 8 x batch_mul_plain (weight = the party's
row count), 7 x batch_add, 1 x batch_decrypt.  The result is checked with a size-independent property: the
decrypted aggregate must equal sum_i rows_i * m_i mod n over the encoded gradient mantissas, computed exactly on
the device-independent integers of a strided sample of positions.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2107_13797_b200 import operators, paillier  # noqa: E402
from paper_2107_13797_b200.batches import encode_batch  # noqa: E402
from paper_2107_13797_b200.device import WordArray  # noqa: E402

HOMO_GRADIENT_EXPONENT = -12


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--params", type=int, default=100_000)
    ap.add_argument("--parties", type=int, default=8)
    ap.add_argument("--key-bits", type=int, default=3072)
    ap.add_argument("--sample", type=int, default=64, help="positions checked exactly")
    args = ap.parse_args()
    import torch

    keys = paillier.keygen(args.key_bits, paillier.default_rng(7), allow_insecure=True)
    pk, sk = keys.public, keys.private
    spent = {"encrypt": 0.0, "mul_plain": 0.0, "add": 0.0, "decrypt": 0.0, "encode": 0.0}

    def timed(name, fn, *a):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn(*a)
        torch.cuda.synchronize()
        spent[name] += time.perf_counter() - t0
        return out

    rows = [100_000 + 7_919 * i for i in range(args.parties)]           # 17-bit weights, like row counts
    step = max(1, args.params // args.sample)
    picks = np.arange(0, args.params, step)[:args.sample]
    expect = [0] * len(picks)
    acc = None
    t_all = time.perf_counter()
    for i in range(args.parties):
        grad = np.random.default_rng(100 + i).normal(0.0, 1e-2, size=args.params)
        plain = timed("encode", encode_batch, pk, grad, None, HOMO_GRADIENT_EXPONENT)
        sample = WordArray.from_numpy(plain.words.numpy()[picks]).ints()
        for k, m in enumerate(sample):
            expect[k] = (expect[k] + rows[i] * m) % pk.n
        cipher = timed("encrypt", operators.batch_encrypt, pk, plain, paillier.default_rng(1000 + i))
        weight = encode_batch(pk, [float(rows[i])], target_exponent=0)
        weighted = timed("mul_plain", operators.batch_mul_plain, pk, cipher, weight)
        acc = weighted if acc is None else timed("add", operators.batch_add, pk, acc, weighted)
        del cipher, weighted
    out = timed("decrypt", operators.batch_decrypt, sk, acc)
    total = time.perf_counter() - t_all
    got = WordArray.from_numpy(out.words.numpy()[picks]).ints()
    assert list(got) == expect, "aggregate differs from sum_i rows_i * m_i mod n"
    n = args.params
    print(json.dumps({
        "params": n, "parties": args.parties, "key_bits": args.key_bits, "total_s": round(total, 3),
        "seconds": {k: round(v, 3) for k, v in spent.items()},
        "rates_per_s": {"encrypt": round(args.parties * n / spent["encrypt"]),
                        "mul_plain": round(args.parties * n / spent["mul_plain"]),
                        "add": round((args.parties - 1) * n / max(spent["add"], 1e-9)),
                        "decrypt": round(n / spent["decrypt"])},
        "checked_positions": len(picks),
    }))


if __name__ == "__main__":
    main()
