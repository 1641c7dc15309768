"""Lane-level Python model of the dedicated Montgomery SQUARING for TPI = 4 (mont32.cuh, Mont::sqr).

Design-validation tool only (not shipped, not an oracle).  a^2 is split into

  * four lane-local squares  a_t^2                     (columns [2 LPT t, 2 LPT (t+1)), not doubled), and
  * six off-diagonal blocks a_i a_j (i < j), doubled, computed as five lane-local operand-scanning
    "pieces" of 1.5 LPT rows per lane (one block and a half each -- the balanced schedule):

        lane 0: a_0 x limbs [LPT, 2.5 LPT)          at column     LPT
        lane 3: a_0 x limbs [2.5 LPT, 4 LPT)        at column 2.5 LPT
        lane 1: a_3 x limbs [LPT, 2.5 LPT)          at column 4   LPT
        lane 2: a_2 x limbs [LPT, 2 LPT)            at column 3   LPT      (phase alpha, LPT rows)
                a_3 x limbs [2.5 LPT, 3 LPT)        at column 5.5 LPT      (phase beta, LPT/2 rows)

Each piece is accumulated in the lane's own E/O carry-chain frame (one IMAD.WIDE.U32.X per limb product),
one column retiring per row.  The pieces meet in a scratch area (shared memory on the GPU): lane t sums the
columns [2 LPT t, 2 LPT (t+1)), doubles, adds its local square, and the four lanes settle the carries between
them.  The 2L-limb square T is then Montgomery-reduced row by row in the distributed frame of the ordinary
multiplication, the high half of T entering one limb per row at the top lane.

Multiplies per lane: LPT^2 (local square, LPT (LPT+1) / 2 with the triangle trick) + 1.5 LPT^2 (pieces)
+ 4 LPT^2 (reduction) against 8 LPT^2 for the generic multiplication.
"""
import random

from mont32_model import Lane, M32, limbs

TPI = 4


def piece(v, xs, lpt):
    """Operand-scanning product of the LPT-limb v with the limb sequence xs; returns len(xs) + LPT words."""
    ln = Lane(lpt)
    out = []
    for x in xs:
        ln.mac(v, x)
        out.append((ln.E[0] + ln.pend) & M32)
        ln.shift(0)
    rest = ln.value()
    assert rest < 1 << (32 * lpt)
    out += limbs(rest, lpt)
    return out


def schedule(lpt):
    """(owner lane, v lane, first x limb, rows, column offset) of the five off-diagonal pieces."""
    h = lpt // 2
    return [
        (0, 0, lpt, 3 * h, lpt),
        (3, 0, 5 * h, 3 * h, 5 * h),
        (1, 3, lpt, 3 * h, 4 * lpt),
        (2, 2, lpt, lpt, 3 * lpt),
        (2, 3, 5 * h, h, 11 * h),
    ]


def square_words(a, lpt):
    """T = a^2 as 2L words, following the lane-level data flow."""
    L = lpt * TPI
    A = [a[t * lpt:(t + 1) * lpt] for t in range(TPI)]
    pieces = []
    for owner, vl, x0, rows, off in schedule(lpt):
        assert off == vl * lpt + x0
        pieces.append((off, piece(A[vl], a[x0:x0 + rows], lpt)))
    local = [piece(A[t], A[t], lpt) for t in range(TPI)]            # a_t^2, 2 LPT words each
    W = 2 * lpt
    accs, tops = [], []
    for t in range(TPI):
        acc, top = [0] * W, 0
        for off, words in pieces:
            c = 0
            for k in range(W):
                idx = W * t + k - off
                w = words[idx] if 0 <= idx < len(words) else 0
                s = acc[k] + w + c
                acc[k], c = s & M32, s >> 32
            top += c
        # double
        msb = acc[W - 1] >> 31
        for k in range(W - 1, 0, -1):
            acc[k] = ((acc[k] << 1) | (acc[k - 1] >> 31)) & M32
        acc[0] = (acc[0] << 1) & M32
        top = 2 * top + msb
        # add the local square
        c = 0
        for k in range(W):
            s = acc[k] + local[t][k] + c
            acc[k], c = s & M32, s >> 32
        top += c
        accs.append(acc)
        tops.append(top)
    # carries between lanes: the small multi-bit value first, then single bits with propagate detection
    g = [0] * TPI
    for t in range(TPI - 1, 0, -1):
        c = tops[t - 1]
        for k in range(W):
            s = accs[t][k] + c
            accs[t][k], c = s & M32, s >> 32
        g[t] = c
        assert c <= 1
    assert tops[TPI - 1] == 0
    carry = 0
    for t in range(TPI):
        if carry:
            for k in range(W):
                s = accs[t][k] + carry
                accs[t][k], carry = s & M32, s >> 32
                if not carry:
                    break
        carry += g[t]                                   # g[t]: what left lane t when tops[t - 1] came in
        assert carry <= 1
    assert carry == 0
    return [w for acc in accs for w in acc]


def redc_words(T, n, np, lpt):
    """Montgomery reduction of the 2L-word T in the distributed frame; high words enter at the top lane."""
    L = lpt * TPI
    lanes = [Lane(lpt) for _ in range(TPI)]
    for t, ln in enumerate(lanes):
        for i in range(ln.H):
            ln.E[i] = T[t * lpt + 2 * i] | (T[t * lpt + 2 * i + 1] << 32)
    N = [n[t * lpt:(t + 1) * lpt] for t in range(TPI)]
    for j in range(L):
        q = (((lanes[0].E[0] + lanes[0].pend) & M32) * np) & M32
        for t in range(TPI):
            lanes[t].mac(N[t], q)
        assert (lanes[0].E[0] + lanes[0].pend) & M32 == 0
        send = [(ln.E[0] + ln.pend) & M32 for ln in lanes]
        for t in range(TPI):
            lanes[t].shift(send[t + 1] if t + 1 < TPI else T[L + j])
    total = sum(ln.value() << (32 * lpt * t) for t, ln in enumerate(lanes))
    nn = sum(x << (32 * i) for i, x in enumerate(n))
    assert total < 2 * nn
    return total - nn if total >= nn else total


def check(bits, lpt, trials, rng):
    L = lpt * TPI
    R = 1 << (32 * L)
    cases = []
    for _ in range(trials):
        n = rng.getrandbits(bits) | 1 | (1 << (bits - 1))
        cases.append((n, rng.randrange(n)))
    n = (1 << bits) - 1 - 2 * rng.getrandbits(8)
    cases += [(n, n - 1), (n, 0), (n, 1), (n, (1 << (bits - 1)) - 1)]
    full = (1 << (32 * L)) - 1 if bits == 32 * L else None
    for n, x in cases:
        np = (-pow(n, -1, 1 << 32)) & M32
        T = square_words(limbs(x, L), lpt)
        assert sum(w << (32 * i) for i, w in enumerate(T)) == x * x
        assert redc_words(T, limbs(n, L), np, lpt) == x * x * pow(R, -1, n) % n
    if full:
        T = square_words(limbs(full, L), lpt)      # all-ones operand: every carry path
        assert sum(w << (32 * i) for i, w in enumerate(T)) == full * full


if __name__ == "__main__":
    rng = random.Random(11)
    check(512, 4, 20, rng)
    check(1024, 8, 10, rng)
    check(2048, 16, 4, rng)
    check(3072, 24, 2, rng)
    check(4096, 32, 2, rng)
    print("mont32 squaring model ok")
