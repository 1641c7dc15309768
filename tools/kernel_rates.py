"""Encrypt / obfuscate / decrypt rates of the C ABI at one key size, with a strided check against the CPU oracle and
the fraction of the integer-multiply roofline in canonical limb products.  Development and
profiling tool (run on a GPU box); the records it prints are kept under profiles/.

    python tools/kernel_rates.py --key-bits 3072 --count 200000 [--check 256] [--reps 2] [--only encrypt]
"""
from __future__ import annotations

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
    ap.add_argument("--key-bits", type=int, default=3072)
    ap.add_argument("--count", type=int, default=200_000)
    ap.add_argument("--check", type=int, default=256)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--only", default="", help="encrypt | decrypt | obfuscate (default: all three)")
    ap.add_argument("--lib", default="", help="alternative build of the library to load (A/B comparisons)")
    ap.add_argument("--peak", type=float, default=0.0, help="IMAD peak in LP/s (0: profiles/r01_imad_peak2.json)")
    args = ap.parse_args()
    import torch
    import cpuref
    import hebatch_oracle as ho
    from paper_2107_13797_b200 import _native, device
    if args.lib:
        _native.LIB_PATH = os.path.abspath(args.lib)

    key = ho.keygen(args.key_bits, random.Random(7))
    lib = _native.lib()
    ctx = device.context_for(key.n)
    ctx.set_private(key.p, key.q, key.hp, key.hq, key.q_inv)
    wn, wc = ctx.wn, ctx.wc
    count = args.count
    stream = device.current_stream_ptr()
    g = torch.Generator(device="cuda"); g.manual_seed(5)
    vals = torch.rand(count, generator=g, device="cuda", dtype=torch.float64) * 200.0 - 100.0
    m = torch.empty((count, wn), dtype=torch.int32, device="cuda")
    bad = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    _native.check(lib.hb_encode_f64(ctx.handle, vals.data_ptr(), -8, m.data_ptr(), count, bad.data_ptr(), stream))
    r = torch.randint(-2 ** 31, 2 ** 31 - 1, (count, wn), generator=g, device="cuda", dtype=torch.int32)
    r[:, -1] = 1
    c = torch.empty((count, wc), dtype=torch.int32, device="cuda")
    c2 = torch.empty((count, wc), dtype=torch.int32, device="cuda")
    back = torch.empty((count, wn), dtype=torch.int32, device="cuda")

    def timed(fn):
        fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(args.reps):
            fn()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) * 1e-3 / args.reps

    L2 = -(-2 * args.key_bits // 32)          # limbs of n^2
    L1 = -(-args.key_bits // 32)              # limbs of p^2
    modmul = lambda L: 2 * L * L + L          # noqa: E731
    lp = {"encrypt": (1.25 * args.key_bits + 3) * modmul(L2) + (L2 // 2) ** 2,
          "obfuscate": (1.25 * args.key_bits + 3) * modmul(L2),
          "decrypt": 2 * (1.25 * args.key_bits / 2 + 3) * modmul(L1)}
    peak = args.peak
    if not peak:
        with open(os.path.join(ROOT, "profiles", "r01_imad_peak2.json")) as fh:
            peak = json.load(fh)["lp_per_s_wide_carry"]
    out = {"key_bits": args.key_bits, "count": count, "imad_peak_lp_per_s": peak}
    want = lambda name: not args.only or args.only == name      # noqa: E731
    _native.check(lib.hb_encrypt(ctx.handle, m.data_ptr(), r.data_ptr(), c.data_ptr(), count, stream))
    if want("encrypt"):
        t = timed(lambda: _native.check(lib.hb_encrypt(ctx.handle, m.data_ptr(), r.data_ptr(), c.data_ptr(), count, stream)))
        out["encrypt_per_s"] = count / t
        out["encrypt_frac"] = lp["encrypt"] * count / t / peak
    if want("obfuscate"):
        t = timed(lambda: _native.check(lib.hb_obfuscate(ctx.handle, c.data_ptr(), r.data_ptr(), c2.data_ptr(), count, stream)))
        out["obfuscate_per_s"] = count / t
        out["obfuscate_frac"] = lp["obfuscate"] * count / t / peak
    if want("decrypt"):
        t = timed(lambda: _native.check(lib.hb_decrypt(ctx.handle, c.data_ptr(), back.data_ptr(), count, stream)))
        out["decrypt_per_s"] = count / t
        out["decrypt_frac"] = lp["decrypt"] * count / t / peak
        if not torch.equal(back, m):
            raise SystemExit("round trip failed")
    # strided check against the CPU oracle
    nchk = min(args.check, count)
    idx = torch.arange(nchk, device="cuda", dtype=torch.int64) * (count // nchk)
    hm, hr = m[idx].cpu().numpy().view(np.uint32), r[idx].cpu().numpy().view(np.uint32)
    ref = cpuref.encrypt_words(key.n, hm, hr)
    if not np.array_equal(ref, c[idx].cpu().numpy().view(np.uint32)):
        raise SystemExit("ciphertexts differ from the CPU oracle")
    if want("obfuscate"):
        if not np.array_equal(cpuref.obfuscate_words(key.n, ref, hr), c2[idx].cpu().numpy().view(np.uint32)):
            raise SystemExit("obfuscated ciphertexts differ from the CPU oracle")
    if not np.array_equal(cpuref.decrypt_words(key, ref), hm):
        raise SystemExit("oracle decrypt mismatch")
    out["oracle_check"] = f"{nchk} strided elements bit-identical"
    print(json.dumps(out))


if __name__ == "__main__":
    main()
