"""First-light GPU check of the C ABI against Python integers (development tool, not a test).

Usage (on a GPU box):  python tools/gpu_check.py [--time]
"""
import ctypes
import json
import random
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2107_13797_b200 import _native  # noqa: E402


def is_probable_prime(n, rng, rounds=24):
    if n < 2:
        return False
    for sp in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if n % sp == 0:
            return n == sp
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for _ in range(rounds):
        a = rng.randrange(2, n - 1)
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def gen_prime(bits, rng):
    while True:
        c = rng.getrandbits(bits) | (3 << (bits - 2)) | 1
        if is_probable_prime(c, rng):
            return c


def to_words(vals, w):
    buf = b"".join(int(v).to_bytes(4 * w, "little") for v in vals)
    return np.frombuffer(buf, dtype=np.uint32).reshape(len(vals), w).copy()


def from_words(arr):
    arr = np.ascontiguousarray(arr)
    w = arr.shape[1]
    raw = arr.tobytes()
    return [int.from_bytes(raw[i * 4 * w:(i + 1) * 4 * w], "little") for i in range(arr.shape[0])]


class Ctx:
    def __init__(self, p, q):
        L = _native.lib()
        self.L = L
        self.p, self.q = p, q
        self.n = p * q
        self.n2 = self.n * self.n
        kb = self.n.bit_length()
        wn = (kb + 31) // 32
        nw = to_words([self.n], wn)
        h = ctypes.c_void_p()
        _native.check(L.hb_ctx_create(ctypes.byref(h), nw.ctypes.data, wn, 0))
        self.h = h
        self.wn = L.hb_pt_words(h)
        self.wc = L.hb_ct_words(h)
        n = self.n
        g = n + 1
        hp = pow((pow(g, p - 1, p * p) - 1) // p, -1, p)
        hq = pow((pow(g, q - 1, q * q) - 1) // q, -1, q)
        qinv = pow(q, -1, p)
        self.hp, self.hq, self.qinv = hp, hq, qinv
        hw = (max(p, q).bit_length() + 31) // 32
        arrs = [to_words([v], hw) for v in (p, q, hp, hq, qinv)]
        _native.check(L.hb_ctx_set_private(h, *[a.ctypes.data for a in arrs], hw))

    def dev(self, arr):
        return torch.from_numpy(arr.view(np.int32)).cuda()

    def encrypt(self, ms, rs):
        m = self.dev(to_words(ms, self.wn))
        r = self.dev(to_words(rs, self.wn))
        out = torch.empty((len(ms), self.wc), dtype=torch.int32, device="cuda")
        _native.check(self.L.hb_encrypt(self.h, m.data_ptr(), r.data_ptr(), out.data_ptr(), len(ms), None))
        torch.cuda.synchronize()
        return from_words(out.cpu().numpy().view(np.uint32))

    def obfuscate(self, cs, rs):
        c = self.dev(to_words(cs, self.wc))
        r = self.dev(to_words(rs, self.wn))
        out = torch.empty((len(cs), self.wc), dtype=torch.int32, device="cuda")
        _native.check(self.L.hb_obfuscate(self.h, c.data_ptr(), r.data_ptr(), out.data_ptr(), len(cs), None))
        torch.cuda.synchronize()
        return from_words(out.cpu().numpy().view(np.uint32))

    def decrypt(self, cs):
        c = self.dev(to_words(cs, self.wc))
        out = torch.empty((len(cs), self.wn), dtype=torch.int32, device="cuda")
        _native.check(self.L.hb_decrypt(self.h, c.data_ptr(), out.data_ptr(), len(cs), None))
        torch.cuda.synchronize()
        return from_words(out.cpu().numpy().view(np.uint32))

    def mulmod(self, a, b, lift=False):
        A = self.dev(to_words(a, self.wc))
        B = self.dev(to_words(b, self.wn if lift else self.wc))
        out = torch.empty((len(a), self.wc), dtype=torch.int32, device="cuda")
        fn = self.L.hb_lift_mulmod if lift else self.L.hb_mulmod
        _native.check(fn(self.h, A.data_ptr(), B.data_ptr(), out.data_ptr(), len(a), 0, None))
        torch.cuda.synchronize()
        return from_words(out.cpu().numpy().view(np.uint32))

    def ref_decrypt(self, c):
        p, q = self.p, self.q
        mp = (pow(c, p - 1, p * p) - 1) // p * self.hp % p
        mq = (pow(c, q - 1, q * q) - 1) // q * self.hq % q
        return mq + q * ((mp - mq) * self.qinv % p)


def check_key(p, q, count, rng, label):
    t0 = time.time()
    cx = Ctx(p, q)
    n, n2 = cx.n, cx.n2
    ms = [rng.randrange(n) for _ in range(count)]
    ms[0] = 0
    if count > 1:
        ms[1] = n - 1
    rs = []
    while len(rs) < count:
        r = rng.randrange(1, n)
        if r % p and r % q:
            rs.append(r)
    want = [(1 + m * n) * pow(r, n, n2) % n2 for m, r in zip(ms, rs)]
    got = cx.encrypt(ms, rs)
    ok_e = got == want
    back = cx.decrypt(want)
    ok_d = back == ms
    ref_d = [cx.ref_decrypt(c) for c in want[:8]]
    ok_d2 = back[:8] == ref_d
    ob = cx.obfuscate(want, rs[::-1])
    ok_o = ob == [c * pow(r, n, n2) % n2 for c, r in zip(want, rs[::-1])]
    prod = cx.mulmod(want, want[::-1])
    ok_a = prod == [a * b % n2 for a, b in zip(want, want[::-1])]
    lifted = cx.mulmod(want, ms[::-1], lift=True)
    ok_l = lifted == [a * (1 + m * n) % n2 for a, m in zip(want, ms[::-1])]
    # arbitrary (also non-unit) ciphertext values through decrypt
    arb = [rng.randrange(n2) for _ in range(min(count, 16))] + [0, 1, p, q * q % n2]
    ok_arb = cx.decrypt(arb) == [cx.ref_decrypt(c) for c in arb]
    res = dict(key=label, count=count, encrypt=ok_e, decrypt=ok_d, decrypt_ref=ok_d2, obfuscate=ok_o,
               mulmod=ok_a, lift=ok_l, decrypt_arbitrary=ok_arb, secs=round(time.time() - t0, 2))
    print(json.dumps(res), flush=True)
    return all([ok_e, ok_d, ok_d2, ok_o, ok_a, ok_l, ok_arb])


def timing(bits, count, rng):
    p, q = gen_prime(bits // 2, rng), gen_prime(bits // 2, rng)
    cx = Ctx(p, q)
    L = cx.L
    m = torch.randint(0, 2**31 - 1, (count, cx.wn), dtype=torch.int32, device="cuda")
    m[:, -1] = 0   # < n
    r = torch.randint(0, 2**31 - 1, (count, cx.wn), dtype=torch.int32, device="cuda")
    r[:, -1] = 1
    out = torch.empty((count, cx.wc), dtype=torch.int32, device="cuda")
    dec = torch.empty((count, cx.wn), dtype=torch.int32, device="cuda")
    res = {"key_bits": bits, "count": count}
    for name, fn in (
        ("encrypt", lambda: L.hb_encrypt(cx.h, m.data_ptr(), r.data_ptr(), out.data_ptr(), count, None)),
        ("decrypt", lambda: L.hb_decrypt(cx.h, out.data_ptr(), dec.data_ptr(), count, None)),
        ("mulmod", lambda: L.hb_mulmod(cx.h, out.data_ptr(), out.data_ptr(), out.data_ptr(), count, 0, None)),
    ):
        _native.check(fn())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _native.check(fn())
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        res[name + "_ms"] = round(ms, 3)
        res[name + "_per_s"] = round(count / ms * 1e3, 1)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    rng = random.Random(11)
    ok = True
    ok &= check_key(5, 7, 12, rng, "n=35")
    ok &= check_key(gen_prime(32, rng), gen_prime(32, rng), 37, rng, "64")
    ok &= check_key(gen_prime(256, rng), gen_prime(256, rng), 33, rng, "512")
    ok &= check_key(gen_prime(512, rng), gen_prime(512, rng), 41, rng, "1024")
    ok &= check_key(gen_prime(768, rng), gen_prime(768, rng), 9, rng, "1536")
    ok &= check_key(gen_prime(1024, rng), gen_prime(1024, rng), 19, rng, "2048")
    ok &= check_key(gen_prime(1536, rng), gen_prime(1536, rng), 7, rng, "3072")
    print("ALL OK" if ok else "MISMATCH", flush=True)
    if "--time" in sys.argv:
        timing(2048, 148 * 64 * 4, rng)
        timing(1024, 148 * 128 * 4, rng)
        timing(3072, 148 * 48 * 2, rng)
    sys.exit(0 if ok else 1)
