"""Parity soak at the THROUGHPUT kernel shapes (GPU box): tens of thousands of random and adversarial operands per key
size through the C ABI, every result compared bit for bit with oracle/cpu_ref.c (GMP).  The unit tests cover the
small-launch shapes exhaustively; this covers the shapes the benchmark runs in ((16,4) / (32,4) / (48,4) encrypt,
(8,4) / (16,4) / (24,4) decrypt, the Montgomery-resident forms, the bucket matvec with wide windows).

    python tools/soak.py --key-bits 1024,2048,3072 --count 40000 --seed 1 > profiles/r02_soak.json
"""
from __future__ import annotations

import argparse
import json
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    sys.path.insert(0, p)

import numpy as np  # noqa: E402


def adversarial(limit: int, width: int, rng: random.Random, unit_of=None):
    """Values below `limit` that stress carries: 0, 1, limit - 1, all-ones words, single high bits, sparse words."""
    bits = limit.bit_length()
    vals = [0, 1, 2, limit - 1, limit - 2, limit // 2, limit // 3, (1 << (bits - 1)) - 1, 1 << (bits - 1)]
    for k in range(32, bits, 32):
        vals += [(1 << k) - 1, 1 << k, (1 << k) + 1, limit - (1 << k)]
    for _ in range(64):
        words = [rng.choice((0, 0xffffffff, 0xfffffffe, 1, 0x80000000, rng.getrandbits(32))) for _ in range(width)]
        vals.append(int.from_bytes(np.array(words, dtype=np.uint32).tobytes(), "little"))
    vals = [v % limit for v in vals]
    if unit_of is not None:
        import math
        vals = [v if v and math.gcd(v, unit_of) == 1 else 1 for v in vals]
    return vals


def words(vals, width):
    return np.frombuffer(b"".join(int(v).to_bytes(4 * width, "little") for v in vals), dtype=np.uint32).reshape(-1, width).copy()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--key-bits", default="1024,2048,3072")
    ap.add_argument("--count", type=int, default=40000)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    import torch
    import cpuref
    import hebatch_oracle as ho
    from paper_2107_13797_b200 import _native, device
    lib = _native.lib()
    A, B, O = 0x10, 0x20, 0x40
    report = {"count": args.count, "seed": args.seed, "keys": {}}
    for bits in (int(v) for v in args.key_bits.split(",")):
        t_start = time.perf_counter()
        rng = random.Random(args.seed * 1000 + bits)
        key = ho.keygen(bits, random.Random(7))
        n, n2 = key.n, key.n2
        ctx = device.context_for(n)
        ctx.set_private(key.p, key.q, key.hp, key.hq, key.q_inv)
        wn, wc, lc = ctx.wn, ctx.wc, ctx.limbs
        stream = device.current_stream_ptr()
        count = args.count
        nprng = np.random.default_rng(args.seed + bits)

        def rand_words(limit, width, cnt):
            arr = nprng.integers(0, 2 ** 32, size=(cnt, width), dtype=np.uint32)
            top = limit.bit_length() - 1                       # clear the top bit: value < 2^(bits-1) <= limit
            arr[:, top // 32] &= np.uint32((1 << (top % 32)) - 1)
            arr[:, top // 32 + 1:] = 0
            return arr

        adv_m = adversarial(n, wn, rng)
        adv_r = adversarial(n, wn, rng, unit_of=n)
        m = rand_words(n, wn, count); m[:len(adv_m)] = words(adv_m, wn)
        r = rand_words(n, wn, count); r[:, 0] |= 1; r[:len(adv_r)] = words(adv_r[:len(adv_r)], wn)
        r[(r == 0).all(axis=1), 0] = 1
        dm, dr = torch.from_numpy(m.view(np.int32)).cuda(), torch.from_numpy(r.view(np.int32)).cuda()
        c = torch.empty((count, wc), dtype=torch.int32, device="cuda")
        cm = torch.empty((count, lc), dtype=torch.int32, device="cuda")
        checks = {}

        def dev_u32(t):
            return t.cpu().numpy().view(np.uint32)

        # encrypt: plain and Montgomery-resident results
        _native.check(lib.hb_encrypt(ctx.handle, dm.data_ptr(), dr.data_ptr(), c.data_ptr(), count, stream))
        want_c = cpuref.encrypt_words(n, m, r)
        checks["encrypt"] = bool(np.array_equal(want_c, dev_u32(c)))
        _native.check(lib.hb_encrypt_rep(ctx.handle, dm.data_ptr(), dr.data_ptr(), cm.data_ptr(), count, O, stream))
        back_plain = torch.empty_like(c)
        _native.check(lib.hb_ct_convert(ctx.handle, cm.data_ptr(), back_plain.data_ptr(), count, 0, stream))
        checks["encrypt_resident"] = bool(torch.equal(back_plain, c))
        # obfuscate (adversarial ciphertext operands: arbitrary residues below n^2, not only real ciphertexts)
        adv_c = adversarial(n2, wc, rng)
        cx = want_c.copy(); cx[:len(adv_c)] = words(adv_c, wc)
        dcx = torch.from_numpy(cx.view(np.int32)).cuda()
        ob = torch.empty_like(c)
        _native.check(lib.hb_obfuscate(ctx.handle, dcx.data_ptr(), dr.data_ptr(), ob.data_ptr(), count, stream))
        checks["obfuscate"] = bool(np.array_equal(cpuref.obfuscate_words(n, cx, r), dev_u32(ob)))
        # decrypt: both operand forms (arbitrary residues decrypt to *something*: the CRT formula is total)
        pm = torch.empty((count, wn), dtype=torch.int32, device="cuda")
        _native.check(lib.hb_decrypt(ctx.handle, dcx.data_ptr(), pm.data_ptr(), count, stream))
        want_m = cpuref.decrypt_words(key, cx)
        checks["decrypt"] = bool(np.array_equal(want_m, dev_u32(pm)))
        _native.check(lib.hb_decrypt_rep(ctx.handle, cm.data_ptr(), pm.data_ptr(), count, A, stream))
        checks["decrypt_resident_round_trip"] = bool(np.array_equal(m, dev_u32(pm)))
        # hadd: plain x plain, resident x resident
        perm = torch.randperm(count, device="cuda")
        dcy = dcx[perm].contiguous()
        s1 = torch.empty_like(c)
        _native.check(lib.hb_mulmod(ctx.handle, dcx.data_ptr(), dcy.data_ptr(), s1.data_ptr(), count, 0, stream))
        want_s = cpuref.mulmod_words(n, cx, dev_u32(dcy).copy())
        checks["hadd"] = bool(np.array_equal(want_s, dev_u32(s1)))
        xm, ym, sm = torch.empty_like(cm), torch.empty_like(cm), torch.empty_like(cm)
        _native.check(lib.hb_ct_convert(ctx.handle, dcx.data_ptr(), xm.data_ptr(), count, 1, stream))
        _native.check(lib.hb_ct_convert(ctx.handle, dcy.data_ptr(), ym.data_ptr(), count, 1, stream))
        _native.check(lib.hb_mulmod_rep(ctx.handle, xm.data_ptr(), ym.data_ptr(), sm.data_ptr(), count, 0, A | B | O, stream))
        _native.check(lib.hb_ct_convert(ctx.handle, sm.data_ptr(), s1.data_ptr(), count, 0, stream))
        checks["hadd_resident"] = bool(np.array_equal(want_s, dev_u32(s1)))
        # hmul: signed 64-bit scalars (fast path) on real ciphertexts, both forms
        mags = nprng.integers(0, 2 ** 63, size=count, dtype=np.uint64)
        ks = [int(v) if i % 2 else (n - int(v)) % n for i, v in enumerate(mags)]
        ks[:5] = [0, 1, n - 1, 2 ** 64 - 1, n - (2 ** 64 - 1)]
        kw = words(ks, wn)
        dk = torch.from_numpy(kw.view(np.int32)).cuda()
        pw = torch.empty_like(c)
        _native.check(lib.hb_powscalar(ctx.handle, c.data_ptr(), dk.data_ptr(), pw.data_ptr(), count, count, 0, stream))
        want_p = cpuref.powscalar_words(n, want_c, kw)
        checks["hmul"] = bool(np.array_equal(want_p, dev_u32(pw)))
        _native.check(lib.hb_powscalar(ctx.handle, cm.data_ptr(), dk.data_ptr(), sm.data_ptr(), count, count, A | O, stream))
        _native.check(lib.hb_ct_convert(ctx.handle, sm.data_ptr(), pw.data_ptr(), count, 0, stream))
        checks["hmul_resident"] = bool(np.array_equal(want_p, dev_u32(pw)))
        # hmul, full-width path: band edges and arbitrary residues as scalars (operators.py:60: k == n - max_int takes
        # the positive branch with the residue itself as the exponent)
        nw = 1500
        kf = [rng.randrange(n) for _ in range(nw)]
        kf[:6] = [key.neg_band, key.neg_band + 1, key.neg_band - 1, key.max_int, n - 1, 0]
        kfw = words(kf, wn)
        dkf = torch.from_numpy(kfw.view(np.int32)).cuda()
        pf = torch.empty((nw, wc), dtype=torch.int32, device="cuda")
        _native.check(lib.hb_powscalar(ctx.handle, c.data_ptr(), dkf.data_ptr(), pf.data_ptr(), nw, nw, 0, stream))
        checks["hmul_full_width"] = bool(np.array_equal(cpuref.powscalar_words(n, want_c[:nw].copy(), kfw), dev_u32(pf)))
        # fused fore-gradient chain (arena.py:345-366 in one kernel) against its six-operator composition on the CPU:
        # (1 + (lg kg mod n) n) r^n  *  c^kh  *  (1 + yl n), plain and resident operand / result forms
        nf = min(count, 24000)
        kg_int, kh = 4, 4
        lg_ints = [int.from_bytes(row.tobytes(), "little") for row in m[:nf]]
        glog = words([(v * kg_int) % n for v in lg_ints], wn)
        yl = rand_words(n, wn, nf); yl[:len(adv_m)] = words(adv_m, wn)[:nf]
        genc = cpuref.encrypt_words(n, glog, r[:nf].copy())
        hpow = cpuref.powscalar_words(n, want_c[:nf].copy(), words([kh], wn))
        ones = np.zeros((nf, wn), np.uint32); ones[:, 0] = 1
        lifted = cpuref.encrypt_words(n, yl, ones)                       # (1 + yl n) * 1^n
        want_f = cpuref.mulmod_words(n, cpuref.mulmod_words(n, genc, hpow), lifted)
        dyl = torch.from_numpy(yl.view(np.int32)).cuda()
        dkg = torch.from_numpy(words([kg_int], wn).view(np.int32)).cuda()
        fo = torch.empty((nf, wc), dtype=torch.int32, device="cuda")
        _native.check(lib.hb_fore_gradient(ctx.handle, c.data_ptr(), dm.data_ptr(), dkg.data_ptr(), kh, dyl.data_ptr(),
                                           dr.data_ptr(), fo.data_ptr(), nf, 0, stream))
        checks["fore_gradient"] = bool(np.array_equal(want_f, dev_u32(fo)))
        fm = torch.empty((nf, lc), dtype=torch.int32, device="cuda")
        _native.check(lib.hb_fore_gradient(ctx.handle, cm.data_ptr(), dm.data_ptr(), dkg.data_ptr(), kh, dyl.data_ptr(),
                                           dr.data_ptr(), fm.data_ptr(), nf, A | O, stream))
        _native.check(lib.hb_ct_convert(ctx.handle, fm.data_ptr(), fo.data_ptr(), nf, 0, stream))
        checks["fore_gradient_resident"] = bool(np.array_equal(want_f, dev_u32(fo)))
        # hsum of everything
        one = torch.empty((1, wc), dtype=torch.int32, device="cuda")
        _native.check(lib.hb_product(ctx.handle, c.data_ptr(), one.data_ptr(), 1, count, 0, 1, stream))
        acc = want_c
        while acc.shape[0] > 1:
            half = acc.shape[0] // 2
            head = cpuref.mulmod_words(n, np.ascontiguousarray(acc[:half]), np.ascontiguousarray(acc[half:2 * half]))
            acc = np.vstack([head, acc[2 * half:]]) if acc.shape[0] % 2 else head
        checks["hsum"] = bool(np.array_equal(acc, dev_u32(one)))
        # matvec: wide windows forced (11 and 13 bits) on a problem the CPU finishes, 52-bit signed scalars
        inner, d = min(count, 6000), 12
        xm52 = nprng.integers(0, 2 ** 52, size=inner * d, dtype=np.uint64)
        xs = [int(v) if (i * 7) % 3 else (n - int(v)) % n for i, v in enumerate(xm52)]
        xw = words(xs, wn)
        dx = torch.from_numpy(xw.view(np.int32)).cuda()
        want_mv = cpuref.matvec_words(n, want_c[:inner].copy(), xw, inner, d)
        mv = torch.empty((d, wc), dtype=torch.int32, device="cuda")
        for cb in (0, 11, 13):
            ctx.set_option(_native.HB_OPT_MATVEC_WINDOW_BITS, cb)
            _native.check(lib.hb_matvec(ctx.handle, c.data_ptr(), dx.data_ptr(), mv.data_ptr(), 1, inner, d, stream))
            checks[f"matvec_window_{cb}"] = bool(np.array_equal(want_mv, dev_u32(mv)))
        ctx.set_option(_native.HB_OPT_MATVEC_WINDOW_BITS, 0)
        report["keys"][str(bits)] = {"checks": checks, "all_equal": all(checks.values()),
                                     "seconds": round(time.perf_counter() - t_start, 1)}
        del c, cm, dm, dr, dcx, dcy, ob, pm, s1, xm, ym, sm, pw, dk, dx
        torch.cuda.empty_cache()
    report["all_equal"] = all(v["all_equal"] for v in report["keys"].values())
    print(json.dumps(report))
    if not report["all_equal"]:
        raise SystemExit(1)


if __name__ == "__main__":
    main()
