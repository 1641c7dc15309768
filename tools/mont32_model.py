"""Lane-level Python model of the radix-2^32, carry-chain Montgomery multiplication (mont32.cuh).

Design-validation tool only (not shipped, not an oracle).  It mirrors the CUDA data flow: TPI lanes per
number, LPT 32-bit limbs per lane, and per lane two arrays of 64-bit accumulators -- E[i] sits on lane
columns (2i, 2i+1), O[i] on (2i+1, 2i+2) -- so that every limb product a*b is ONE 64-bit multiply-add
(IMAD.WIDE.U32.X) in a carry chain, the form the B200 integer pipe issues at its full (quarter) rate.
One extra element per array (E[H], O[H]) holds what spills past the lane's top column; it is passed
to the lane above only once, after the last row.
"""
import random

M32 = (1 << 32) - 1
M64 = (1 << 64) - 1


class Lane:
    def __init__(self, lpt):
        self.H = lpt // 2
        self.E = [0] * (self.H + 1)
        self.O = [0] * (self.H + 1)
        self.pend = 0

    def mac(self, v, x):
        """E, O += v * x with one carry chain per array."""
        H = self.H
        c = 0
        for i in range(H):
            s = self.E[i] + v[2 * i] * x + c
            self.E[i], c = s & M64, s >> 64
        self.E[H] += c
        assert self.E[H] <= M64
        c = 0
        for i in range(H):
            s = self.O[i] + v[2 * i + 1] * x + c
            self.O[i], c = s & M64, s >> 64
        self.O[H] += c
        assert self.O[H] <= M64

    def shift(self, recv):
        """Divide the lane value by 2^32.  The low word of column 0 (E[0] + pend) has been eliminated (lane 0)
        or sent to the lane below; what is left of that column becomes the pending value of the new column 0,
        so the accumulators themselves never see a ripple add."""
        H = self.H
        v = self.E[0] + self.pend
        self.pend = v >> 32                       # up to 33 bits
        newE = list(self.O)
        newO = self.E[1:] + [0]
        s = newO[H - 1] + recv
        newO[H - 1], c = s & M64, s >> 64
        newO[H] += c
        self.E, self.O = newE, newO

    def value(self):
        return self.pend + sum(e << (64 * i) for i, e in enumerate(self.E)) + sum(o << (64 * i + 32) for i, o in enumerate(self.O))


def mont_mul(a, b, n, np, lpt, tpi):
    """a, b, n: limb lists of length lpt*tpi (a, b < n).  Returns (a*b/R mod n) limbs, canonical."""
    L = lpt * tpi
    lanes = [Lane(lpt) for _ in range(tpi)]
    A = [a[t * lpt:(t + 1) * lpt] for t in range(tpi)]
    N = [n[t * lpt:(t + 1) * lpt] for t in range(tpi)]
    for j in range(L):
        bj = b[j]
        for t in range(tpi):
            lanes[t].mac(A[t], bj)
        q = (((lanes[0].E[0] + lanes[0].pend) & M32) * np) & M32
        for t in range(tpi):
            lanes[t].mac(N[t], q)
        assert (lanes[0].E[0] + lanes[0].pend) & M32 == 0
        send = [(ln.E[0] + ln.pend) & M32 for ln in lanes]
        for t in range(tpi):
            lanes[t].shift(send[t + 1] if t + 1 < tpi else 0)
    total = sum(ln.value() << (32 * lpt * t) for t, ln in enumerate(lanes))
    nn = sum(x << (32 * i) for i, x in enumerate(n))
    assert total < 2 * nn
    if total >= nn:
        total -= nn
    return total


def limbs(v, L):
    return [(v >> (32 * i)) & M32 for i in range(L)]


def check(bits, lpt, tpi, trials, rng):
    L = lpt * tpi
    R = 1 << (32 * L)
    for _ in range(trials):
        n = rng.getrandbits(bits) | 1 | (1 << (bits - 1))
        np = (-pow(n, -1, 1 << 32)) & M32
        x, y = rng.randrange(n), rng.randrange(n)
        z = mont_mul(limbs(x, L), limbs(y, L), limbs(n, L), np, lpt, tpi)
        assert z == x * y * pow(R, -1, n) % n
    # worst case operands
    n = (1 << bits) - 1 - 2 * rng.getrandbits(8)
    np = (-pow(n, -1, 1 << 32)) & M32
    z = mont_mul(limbs(n - 1, L), limbs(n - 1, L), limbs(n, L), np, lpt, tpi)
    assert z == (n - 1) * (n - 1) * pow(R, -1, n) % n


if __name__ == "__main__":
    rng = random.Random(9)
    check(64, 2, 1, 50, rng)
    check(256, 4, 2, 50, rng)
    check(1024, 8, 4, 10, rng)
    check(2048, 16, 4, 4, rng)
    check(4096, 16, 8, 2, rng)
    check(4096, 32, 4, 2, rng)
    check(6144, 24, 8, 1, rng)
    print("mont32 model ok")
