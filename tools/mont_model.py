"""Lane-level Python model of the warp-cooperative, carry-free Montgomery
multiplication implemented in paper_2107_13797_b200/csrc/mont.cuh.

Design-validation tool only: it is not shipped, not an oracle and not imported by
the package.  It mirrors the CUDA data flow one-to-one so that the carry logic
and the 64-bit overflow bounds can be checked with Python integers.

Numbers are held as RB=29-bit digits, LPT digits per lane, TPI lanes per
instance.  Every limb product is one IMAD.WIDE.U32 into a 64-bit column
accumulator with *no carry chain* (B200 issues the carry form, IMAD.WIDE.U32.X,
at half rate - profiles/r01_imad_peak.json).  After each row the frame moves
down one digit; every LPT rows a carry-save pass pulls the accumulators back
below 2^31 so they never overflow 64 bits.
"""
import random

RB = 29
MASK = (1 << RB) - 1
M64 = (1 << 64) - 1


def to_digits(v, L):
    return [(v >> (RB * i)) & MASK for i in range(L)]


def from_digits(d):
    return sum(x << (RB * i) for i, x in enumerate(d))


def carry_save_pass(acc, ovf, LPT, TPI):
    """acc[t][i] (any 64-bit) -> d + e(prev) + f(prev-1); returns new acc (< 2^31) and ovf."""
    d = [[x & MASK for x in lane] for lane in acc]
    e = [[(x >> RB) & MASK for x in lane] for lane in acc]
    f = [[x >> (2 * RB) for x in lane] for lane in acc]
    new = [[0] * LPT for _ in range(TPI)]
    for t in range(TPI):
        v0 = e[t][LPT - 1] + f[t][LPT - 2]      # to column 0 of lane t+1
        v1 = f[t][LPT - 1]                      # to column 1 of lane t+1
        for i in range(LPT):
            s = d[t][i]
            if i >= 1:
                s += e[t][i - 1]
            if i >= 2:
                s += f[t][i - 2]
            new[t][i] = s
        if t + 1 < TPI:
            new[t + 1][0] += 0  # placeholder (added below, after the lane loop)
        else:
            ovf = ovf + v0 + (v1 << RB)
    for t in range(1, TPI):
        new[t][0] += e[t - 1][LPT - 1] + f[t - 1][LPT - 2]
        new[t][1] += f[t - 1][LPT - 1]
    for lane in new:
        for x in lane:
            assert x < (1 << 31)
    assert ovf <= M64
    return new, ovf


def mont_mul(a, b, n, np, LPT, TPI, stats=None):
    """a, b: digit lists (digits may be slightly above 2^29); n exact digits.
    Returns almost-normalised digits (< 2^29 + 2) of a*b/R mod-ish n, value < a*b/R + N."""
    L = LPT * TPI
    A = [a[t * LPT:(t + 1) * LPT] for t in range(TPI)]
    N = [n[t * LPT:(t + 1) * LPT] for t in range(TPI)]
    acc = [[0] * LPT for _ in range(TPI)]
    ovf = 0
    for s in range(TPI):
        for i in range(LPT):
            bj = b[s * LPT + i]
            for t in range(TPI):
                for k in range(LPT):
                    acc[t][k] += A[t][k] * bj
            q = ((acc[0][0] & 0xFFFFFFFF) * np) & MASK
            for t in range(TPI):
                for k in range(LPT):
                    acc[t][k] += N[t][k] * q
                    assert acc[t][k] <= M64, "64-bit accumulator overflow"
                    if stats is not None:
                        stats[0] = max(stats[0], acc[t][k])
            assert acc[0][0] & MASK == 0
            out = [acc[t][0] for t in range(TPI)]
            for t in range(TPI):
                recv = out[t + 1] if t + 1 < TPI else ovf
                acc[t] = acc[t][1:] + [recv]
            ovf = 0
            acc[0][0] += out[0] >> RB
            assert acc[0][0] <= M64
        acc, ovf = carry_save_pass(acc, ovf, LPT, TPI)
    # second (32-bit) pass: digits < 2^29 + 2
    assert ovf == 0, ovf
    res = [[0] * LPT for _ in range(TPI)]
    for t in range(TPI):
        for i in range(LPT):
            if i >= 1:
                c = acc[t][i - 1] >> RB
            elif t >= 1:
                c = acc[t - 1][LPT - 1] >> RB
            else:
                c = 0
            res[t][i] = (acc[t][i] & MASK) + c
    assert acc[TPI - 1][LPT - 1] >> RB == 0
    return [x for lane in res for x in lane]


def check(bits, LPT, TPI, trials, rng, stats):
    L = LPT * TPI
    R = 1 << (RB * L)
    assert bits + 2 <= RB * L
    for _ in range(trials):
        n = rng.getrandbits(bits) | 1 | (1 << (bits - 1))
        np = (-pow(n, -1, 1 << RB)) & MASK
        nd = to_digits(n, L)
        x = rng.randrange(2 * n)
        y = rng.randrange(2 * n)
        xd, yd = to_digits(x, L), to_digits(y, L)
        # chain of multiplications feeding almost-normalised outputs back in
        for step in range(4):
            zd = mont_mul(xd, yd, nd, np, LPT, TPI, stats)
            z = from_digits(zd)
            assert (z * R - from_digits(xd) * from_digits(yd)) % n == 0
            assert z < 2 * n
            assert max(zd) < (1 << RB) + 2
            xd, yd = zd, (zd if step % 2 else yd)


if __name__ == "__main__":
    rng = random.Random(5)
    stats = [0]
    check(100, 4, 2, 100, rng, stats)
    check(1024, 9, 4, 10, rng, stats)
    check(2048, 18, 4, 4, rng, stats)
    check(4096, 18, 8, 2, rng, stats)
    check(3072, 27, 4, 2, rng, stats)
    check(6144, 27, 8, 1, rng, stats)
    print("mont model ok; max accumulator = 2^%.2f" % (len(bin(stats[0])) - 2))
