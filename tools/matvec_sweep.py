"""Encrypted-matvec time against the bucket window width and the row count (development tool, GPU box).

    python tools/matvec_sweep.py --rows 100000,200000,400000,1000000 --bits 9,11,13 [--d 100]

Ciphertext operands are random residues below n^2 (units with overwhelming probability; the arithmetic does not
care), scalars are uniform(-1, 1) features at their exact shared exponent (52-bit magnitudes, half negative) in
the compact resident form.  Every width must give the same bits: checked against the first width per row count.
"""
import argparse
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    sys.path.insert(0, p)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", default="100000,200000,400000,1000000")
    ap.add_argument("--bits", default="0,9,11,13")
    ap.add_argument("--d", type=int, default=100)
    ap.add_argument("--key-bits", type=int, default=2048)
    ap.add_argument("--pool-keep-gib", type=float, default=0.0, help="HB_OPT_POOL_KEEP_BYTES (0: library default)")
    ap.add_argument("--sync", action="store_true", help="synchronise the device between the timed calls")
    args = ap.parse_args()
    import torch
    import hebatch_oracle as ho
    from paper_2107_13797_b200 import device
    from paper_2107_13797_b200.backends import CudaBackend
    from paper_2107_13797_b200.device import WordArray

    key = ho.keygen(args.key_bits, random.Random(7))
    be = CudaBackend()
    ctx = device.context_for(key.n)
    if args.pool_keep_gib:
        ctx.set_option(2, int(args.pool_keep_gib * 2 ** 30))
    g = torch.Generator(device="cuda"); g.manual_seed(3)
    out = {}
    for rows in (int(v) for v in args.rows.split(",")):
        c = torch.randint(-2 ** 31, 2 ** 31 - 1, (rows, ctx.wc), generator=g, device="cuda", dtype=torch.int32)
        c[:, -1] = 1
        cw = WordArray.from_device(c)
        X = np.random.default_rng(0).uniform(-1, 1, (rows, args.d))
        k, _ = be.encode_compact(key.n, X, None)
        first = None
        for bits in (int(v) for v in args.bits.split(",")):
            be.set_matvec_window(key.n, bits)
            res = be.matvec(key.n, cw, k, 1, rows, args.d)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            import time
            t0 = time.perf_counter()
            a.record()
            for _ in range(2):
                res = be.matvec(key.n, cw, k, 1, rows, args.d)
                if args.sync:
                    torch.cuda.synchronize()
            b.record()
            b.synchronize()
            out[f"{rows}x{args.d}@{bits}_wall"] = round((time.perf_counter() - t0) * 500, 1)
            got = res.numpy().copy()
            if first is None:
                first = got
            elif not np.array_equal(first, got):
                raise SystemExit(f"window {bits} gives different bits at {rows} rows")
            out[f"{rows}x{args.d}@{bits}"] = round(a.elapsed_time(b) / 2, 1)
        be.set_matvec_window(key.n, 0)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
