"""TEST INFRASTRUCTURE ONLY -- the reference's heterogeneous-FLR iteration on the host CPU.

One full-batch iteration (gradient step over `rows` rows, then the loss over the same rows) of the 2-party
protocol of /root/reference/pkg/src/hebatch/flr/parties.py: HeteroHost.send_logits :249-254, HeteroGuest
.fore_gradient :161-179 (through Arena.run_fore_gradient_pipeline, arena.py:316-375), .gradient :181-191,
_mask_and_ship :122-132, HeteroHost.gradient :256-262, Arbiter.decrypt_gradient :289-298, the loss path
:199-225 / :267-276 / :300-305 and the epoch loop :330-346.  Every modular power, product and inverse runs in
oracle/cpu_ref.c (GMP under OpenMP on all host threads -- the arithmetic the reference reaches through gmpy2,
without the interpreter); the per-element glue (codec, lifts, exponent rules) is oracle/hebatch_oracle.py.

Two uses, both on the checker side: (1) bench.py's cpu_baseline leg times it on a row subsample to put a
MEASURED host-CPU FLR iteration beside the GPU one (BASELINE north_star: "FLR iteration speedup over the host-CPU
reference"); (2) tests compare everything the arbiter decrypts with the CUDA path on the same data, key and seed.
Random streams as in the reference: guest seed*4+1, guest arena seed*4+2, host seed*4+3.
"""
from __future__ import annotations

import math
import random
import time

import numpy as np

import cpuref
import hebatch_oracle as ho

LOGIT_EXPONENT_CAP = -8      # parties.py:39
MASK_RANGE = 8.0             # parties.py:41
LOG2 = math.log(2.0)


def _protocol_exponent(values, cap=LOGIT_EXPONENT_CAP) -> int:
    """parties.py:91-96."""
    exact = min((ho.exact_exponent(float(v)) for v in values), default=0)
    return min(exact, cap)


class CpuHeteroFlr:
    """State of guest, host and arbiter for full-batch steps on one key; `seconds` accumulates per-operator
    wall time of the last iteration (feature encoding is one-off and cached, as MiniBatchAggregator does)."""

    def __init__(self, key: ho.Key, guest_X, guest_y, host_X, learning_rate: float, seed: int, threads=None):
        self.key = key
        self.wn, self.wc = cpuref.widths(key.n)
        self.threads = threads or cpuref.threads()
        self.guest_X = np.hstack([guest_X, np.ones((len(guest_X), 1))])
        self.guest_y = np.asarray(guest_y, dtype=np.float64)
        self.host_X = np.asarray(host_X, dtype=np.float64)
        self.lr = learning_rate
        self.guest_rng = random.Random(seed * 4 + 1)
        self.arena_rng = random.Random(seed * 4 + 2)
        self.host_rng = random.Random(seed * 4 + 3)
        self.guest_theta = np.zeros(self.guest_X.shape[1])
        self.host_theta = np.zeros(self.host_X.shape[1])
        self.decrypted = []
        self.seconds = {}
        self._features = {}

    # ---- word-array helpers ------------------------------------------------------------------------------
    def _pt(self, ints):
        return cpuref._w(ints, self.wn)

    def _ct(self, ints):
        return cpuref._w(ints, self.wc)

    def _ints(self, words):
        return [int.from_bytes(row.tobytes(), "little") for row in words]

    def _tick(self, label, t0):
        self.seconds[label] = self.seconds.get(label, 0.0) + time.perf_counter() - t0

    def _draw(self, rng, count):
        t0 = time.perf_counter()
        out = self._pt([ho.draw_unit(self.key.n, rng) for _ in range(count)])
        self._tick("draw_unit", t0)
        return out

    def _encode(self, values, exponent):
        t0 = time.perf_counter()
        out = [ho.encode(self.key, float(v), exponent)[0] for v in values]
        self._tick("codec", t0)
        return out

    def _encrypt(self, mantissas, rng):
        r = self._draw(rng, len(mantissas))
        t0 = time.perf_counter()
        out = cpuref.encrypt_words(self.key.n, self._pt(mantissas), r, self.threads)
        self._tick("encrypt", t0)
        return out

    def _obfuscate(self, c, rng):
        r = self._draw(rng, c.shape[0])
        t0 = time.perf_counter()
        out = cpuref.obfuscate_words(self.key.n, c, r, self.threads)
        self._tick("obfuscate", t0)
        return out

    def _add(self, a, b):
        t0 = time.perf_counter()
        out = cpuref.mulmod_words(self.key.n, a, b, self.threads)
        self._tick("hadd", t0)
        return out

    def _add_plain(self, c, mantissas):
        """batch_add with a plaintext already on the ciphertext's grid: lift, then multiply (operators.py:209-212)."""
        t0 = time.perf_counter()
        lifted = self._ct([ho.lift(self.key, m) for m in mantissas])
        self._tick("lift", t0)
        return self._add(c, lifted)

    def _mul(self, c, scalars):
        t0 = time.perf_counter()
        out = cpuref.powscalar_words(self.key.n, c, self._pt(scalars), self.threads)
        self._tick("hmul", t0)
        return out

    def _matvec(self, c, feats, d):
        t0 = time.perf_counter()
        out = cpuref.matvec_words(self.key.n, c, feats, c.shape[0], d, self.threads)
        self._tick("matvec", t0)
        return out

    def _sum(self, c):
        t0 = time.perf_counter()
        while c.shape[0] > 1:                               # exact and commutative: any order gives the same bits
            half = c.shape[0] // 2
            head = cpuref.mulmod_words(self.key.n, np.ascontiguousarray(c[:half]),
                                       np.ascontiguousarray(c[half:2 * half]), self.threads)
            c = np.vstack([head, c[2 * half:]]) if c.shape[0] % 2 else head
        self._tick("hsum", t0)
        return c

    def _decrypt_decode(self, c, exponent):
        """Arbiter: CRT decrypt, renormalise below exponent -32 (operators.py:160-167), decode."""
        t0 = time.perf_counter()
        plain = self._ints(cpuref.decrypt_words(self.key, c, self.threads))
        self._tick("decrypt", t0)
        out = []
        for m in plain:
            m2, e2 = ho.renormalize(self.key, m, exponent)
            out.append(ho.decode(self.key, m2, e2))
        return out

    def _feature_words(self, name, X, batch_id, idx):
        hit = self._features.get((name, batch_id))
        if hit is None:
            mant, e = ho.encode_batch(self.key, X[idx].reshape(-1))
            hit = self._features[(name, batch_id)] = (self._pt(mant), e)
        return hit

    def _mask_and_ship(self, grad, exponent, rng):
        raw = [rng.uniform(0.0, MASK_RANGE) for _ in range(grad.shape[0])]
        mask_m = self._encode(raw, exponent)
        mask = np.asarray([ho.decode(self.key, m, exponent) for m in mask_m])
        return mask, self._obfuscate(self._add_plain(grad, mask_m), rng)

    # ---- one mini-batch (parties.py:330-340); idx = all rows for a full-batch step -----------------------------
    def step(self, batch_id=0, idx=None):
        key, n = self.key, self.key.n
        idx = np.arange(self.guest_X.shape[0]) if idx is None else np.asarray(idx)
        s = len(idx)
        logits_h = self.host_X[idx] @ self.host_theta
        e = _protocol_exponent(logits_h)
        c_lh = self._encrypt(self._encode(logits_h, e), self.host_rng)
        # guest: [[0.25 (lh + lg) - 0.5 y]] -- arena.py:337-366
        q_m, q_e = ho.encode(key, 0.25)
        h_m, h_e = ho.encode(key, -0.5)
        lg = self._encode(self.guest_X[idx] @ self.guest_theta, e)
        lab = self._encode(self.guest_y[idx], 0)
        genc = self._encrypt([m * q_m % n for m in lg], self.arena_rng)
        hlog = self._mul(c_lh, [q_m])
        total = self._add(genc, hlog)
        target = e + q_e
        ylab = [ho.rescale(key, m * h_m % n, 0 + h_e, target) for m in lab]
        fore = self._add_plain(total, ylab)
        fore_sent = self._obfuscate(fore, self.guest_rng)
        feats_g, ex_g = self._feature_words("guest", self.guest_X, batch_id, idx)
        grad_g = self._matvec(fore, feats_g, self.guest_X.shape[1])
        mask_g, wire_g = self._mask_and_ship(grad_g, target + ex_g, self.guest_rng)
        feats_h, ex_h = self._feature_words("host", self.host_X, batch_id, idx)
        grad_h = self._matvec(fore_sent, feats_h, self.host_X.shape[1])
        mask_h, wire_h = self._mask_and_ship(grad_h, target + ex_h, self.host_rng)
        dec_g = self._decrypt_decode(wire_g, target + ex_g)
        self.decrypted.append(dec_g)
        dec_h = self._decrypt_decode(wire_h, target + ex_h)
        self.decrypted.append(dec_h)
        g_guest = (np.asarray(dec_g) - mask_g) / s
        g_host = (np.asarray(dec_h) - mask_h) / s
        self.guest_theta = self.guest_theta - self.lr * g_guest
        self.host_theta = self.host_theta - self.lr * g_host

    # ---- loss over all rows (parties.py:199-225, 267-276, 300-305) ---------------------------------------------
    def loss(self, idx=None) -> float:
        key = self.key
        idx = np.arange(self.guest_X.shape[0]) if idx is None else np.asarray(idx)
        z_h = self.host_X[idx] @ self.host_theta
        sq = z_h * z_h
        e1, e2 = _protocol_exponent(z_h), _protocol_exponent(sq)
        c1 = self._encrypt(self._encode(z_h, e1), self.host_rng)
        c2 = self._encrypt(self._encode(sq, e2), self.host_rng)
        lg = self.guest_X[idx] @ self.guest_theta
        y = self.guest_y[idx]
        k1 = 0.25 * lg - 0.5 * y
        plain_part = LOG2 - 0.5 * y * lg + 0.125 * lg * lg
        target = min(e1 + _protocol_exponent(k1), e2 + ho.exact_exponent(0.125), _protocol_exponent(plain_part))
        t1 = self._mul(c1, self._encode(k1, target - e1))
        t2 = self._mul(c2, self._encode([0.125], target - e2))
        total = self._add_plain(self._add(t1, t2), self._encode(plain_part, target))
        sent = self._obfuscate(self._sum(total), self.guest_rng)
        value = self._decrypt_decode(sent, target)[0]
        self.decrypted.append([value])
        return value / len(y)

    def run_iteration(self, batches=None, loss_indices=None) -> float:
        """One epoch: every mini-batch in order, then the loss (parties.py:330-346).  Default: one full batch."""
        self.seconds = {}
        t0 = time.perf_counter()
        for batch_id, idx in enumerate(batches if batches is not None else [None]):
            self.step(batch_id, idx)
        loss = self.loss(loss_indices)
        self.seconds["total"] = time.perf_counter() - t0
        return loss
