"""Federated logistic regression on the B200 operators: heterogeneous (vertical) and homogeneous (horizontal).

This is the caller of the hot path: the per-mini-batch message flow of the reference's
flr/parties.py (HeteroGuest :135-225, HeteroHost :228-276, Arbiter :279-305, HeteroFederation :308-354),
driven through this package's operators, arena and wire format.  It keeps the reference's operator
sequence, exponent choices, random-stream layout (guest: seed*4+1, guest arena: seed*4+2, host: seed*4+3) and
hop-by-hop serialisation, so with the same data, key and seed every ciphertext -- and therefore every
decrypted masked gradient, the model and the loss -- equals the reference's run.  HomoFederation does the same for the
horizontal mode (parties.py:357-454).  What is not carried over is the reference's control plane (ChannelHub
message audit, CLI): messages are passed as HAFB bytes between the roles inside one object.

Second-order Taylor objective (reference flr/objective.py): fore gradient 0.25 * theta.x - 0.5 * y, loss
log 2 - 0.5 y z + 0.125 z^2 with z = theta.x.
"""
from __future__ import annotations

import math
import random
from dataclasses import dataclass

import numpy as np

from . import encoding, operators
from .arena import Arena, TransferLedger
from .backends import default_backend
from .batches import PlaintextBatch, decode_batch, encode_batch
from .bufferpool import deserialize, serialize_to_bytes
from .paillier import KeyPair, default_rng

LOGIT_EXPONENT_CAP = -8       # parties.py:39
HOMO_GRADIENT_EXPONENT = -12  # parties.py:40
MASK_RANGE = 8.0              # parties.py:41
LOG2 = math.log(2.0)


@dataclass
class FlrConfig:
    learning_rate: float = 0.15
    batch_size: int = 32
    seed: int = 0
    caching_enabled: bool = True


@dataclass
class EpochResult:
    epoch: int
    loss: float
    grad_norm: float
    ledger: dict


@dataclass
class PartyData:
    name: str
    ids: tuple
    X: np.ndarray
    y: np.ndarray | None = None

    @property
    def rows(self) -> int:
        return len(self.ids)


def make_synthetic(rows: int, features: int, seed: int, noise: float = 0.25):
    """The reference's synthetic task (flr/data.py:195-206): X ~ U(-1, 1), unit-norm normal weights, noisy margin.
    Returns (ids, X, y)."""
    rng = np.random.default_rng(seed)
    w = rng.normal(size=features)
    w /= np.linalg.norm(w)
    X = rng.uniform(-1.0, 1.0, size=(rows, features))
    y = np.where(X @ w + noise * rng.normal(size=rows) > 0, 1.0, -1.0)
    return tuple(str(i) for i in range(rows)), X, y


def vertical_split(ids, X, y, parties: int = 2):
    """Contiguous column groups, labels stay with party 0 (flr/data.py:104-122)."""
    d = X.shape[1]
    cuts = [round(i * d / parties) for i in range(parties + 1)]
    return [PartyData("guest" if i == 0 else "host", ids, X[:, cuts[i]:cuts[i + 1]].copy(), y.copy() if i == 0 else None)
            for i in range(parties)]


def horizontal_split(ids, X, y, parties: int):
    """Round-robin row assignment, every party keeps all columns (flr/data.py:125-136)."""
    if parties < 1:
        raise ValueError("need at least one party")
    out = []
    for i in range(parties):
        take = np.arange(i, len(ids), parties)
        out.append(PartyData(f"party{i}", tuple(ids[j] for j in take), X[take].copy(), y[take].copy()))
    return out


def make_minibatches(n_rows: int, batch_size: int, seed: int):
    """Seeded permutation in fixed chunks (flr/data.py:163-171)."""
    order = list(range(n_rows))
    default_rng(seed).shuffle(order)
    return [np.asarray(order[i:i + batch_size], dtype=np.intp) for i in range(0, n_rows, batch_size)]


def protocol_exponent(values, cap: int = LOGIT_EXPONENT_CAP, pk=None, backend=None) -> int:
    """Exact shared exponent of the values, never coarser than the cap (parties.py:91-96).  With a key the minimum
    is taken on the device (large vectors); the value is the same."""
    values = np.asarray(values, dtype=np.float64)
    if pk is not None and values.size >= 4096:
        exact = (backend or default_backend()).min_exact_exponent(pk.n, values)
    else:
        exact = int(encoding.exact_exponents(values).min()) if values.size else 0
    return min(exact, cap)


def _encode(pk, values, exponent, backend=None) -> PlaintextBatch:
    return encode_batch(pk, np.asarray(values, dtype=np.float64), target_exponent=exponent, backend=backend)


class HeteroFederation:
    """Guest (labels + bias column), host (features only) and arbiter (private key) for one training run."""

    def __init__(self, guest_data, host_data, batches, loss_indices, keys: KeyPair, config: FlrConfig,
                 backend=None):
        if tuple(guest_data.ids) != tuple(host_data.ids):
            raise ValueError("vertical parties must hold identical id sets")
        self.keys = keys
        self.pk = keys.public
        self.config = config
        self.backend = backend or default_backend()
        self.batches = list(batches)
        self.loss_indices = np.asarray(loss_indices)
        self.epoch = 0
        s = config.seed
        self.guest_rng, self.host_rng = default_rng(s * 4 + 1), default_rng(s * 4 + 3)
        self.arena = Arena(self.pk, backend=self.backend, rng=default_rng(s * 4 + 2),
                           caching_enabled=config.caching_enabled)
        self.guest_X = np.hstack([guest_data.X, np.ones((len(guest_data.ids), 1))])   # bias on the guest side
        self.guest_y = guest_data.y
        self.host_X = host_data.X.copy()
        self.guest_theta = np.zeros(self.guest_X.shape[1])
        self.host_theta = np.zeros(self.host_X.shape[1])
        self._guest_features, self._host_features = {}, {}
        self.decrypted = []          # what the arbiter saw, in order (masked gradients, loss sums)

    @property
    def ledger(self) -> TransferLedger:
        return self.arena.ledger

    # ---- building blocks -----------------------------------------------------------------------------
    @staticmethod
    def _take(X, idx):
        """X[idx] -- without the copy when idx selects every row in order (full-batch steps: 800 MB per call at
        1M x 100, four calls per iteration)."""
        idx = np.asarray(idx)
        n = X.shape[0]
        if idx.shape == (n,) and n and idx[0] == 0 and idx[-1] == n - 1 and bool((np.diff(idx) == 1).all()):
            return X
        return X[idx]

    def _mask_and_ship(self, grad_cipher, rng: random.Random):
        """Additive mask on the codec grid, re-randomise, serialise (parties.py:122-132)."""
        pk, be = self.pk, self.backend
        exponent = grad_cipher.exponents[0]
        raw = [rng.uniform(0.0, MASK_RANGE) for _ in range(grad_cipher.count)]
        mask_plain = _encode(pk, raw, exponent, be)
        mask = np.asarray(decode_batch(pk, mask_plain, be))
        masked = operators.batch_obfuscate(pk, operators.batch_add(pk, grad_cipher, mask_plain, be), rng, be)
        return mask, serialize_to_bytes(masked)

    def _arbiter_gradient(self, wire: bytes):
        cipher = deserialize(wire, self.pk)
        plain = operators.batch_decrypt(self.keys.private, cipher, self.backend)
        values = decode_batch(self.pk, plain, self.backend)
        self.decrypted.append(values)
        return np.asarray(values)

    def _features(self, cache, X, batch_id, idx):
        """The mini-batch's feature matrix, packed once and kept device-resident for later epochs (the role of
        MiniBatchAggregator, bufferpool.py:182-226): the compact form -- sign + 64-bit magnitude per scalar, 9 bytes
        instead of a 256-byte residue -- which is what the encrypted matvec reads."""
        hit = cache.get(batch_id)
        if hit is None:
            hit = cache[batch_id] = encode_batch(self.pk, self._take(X, idx), backend=self.backend, compact=True)
        return hit

    # ---- one mini-batch (parties.py:330-340) -------------------------------------------------------------
    def step(self, batch_id: int, idx: np.ndarray):
        pk, be = self.pk, self.backend
        s = len(idx)
        # host -> guest: encrypted logits
        logits_h = self._take(self.host_X, idx) @ self.host_theta
        wire = serialize_to_bytes(operators.batch_encrypt(
            pk, _encode(pk, logits_h, protocol_exponent(logits_h, pk=pk, backend=be), be), self.host_rng, be))
        # guest: fore gradient through the arena pipeline, then its gradient slice
        c_lh = deserialize(wire, pk)
        exponent = c_lh.exponents[0]
        lg_plain = _encode(pk, self._take(self.guest_X, idx) @ self.guest_theta, exponent, be)
        label_plain = _encode(pk, self._take(self.guest_y, idx), 0, be)
        if self.arena.caching_enabled:
            h_lh = self.arena.upload(c_lh)
            h_fore = self.arena.run_fore_gradient_pipeline(h_lh, lg_plain, label_plain)
            fore = self.arena.download(h_fore)
        else:
            fore = self.arena.run_fore_gradient_pipeline(c_lh, lg_plain, label_plain)
            h_fore = h_lh = None
        wire_fore = serialize_to_bytes(operators.batch_obfuscate(pk, fore, self.guest_rng, be))
        feats_g = self._features(self._guest_features, self.guest_X, batch_id, idx)
        if h_fore is not None:
            h_grad = self.arena.exec_op("matmul", [h_fore, feats_g])
            grad_g = self.arena.download(h_grad)
            for h in (h_grad, h_fore, h_lh):
                self.arena.release(h)
        else:
            grad_g = operators.batch_matmul(pk, fore, feats_g, be)
        mask_g, wire_g = self._mask_and_ship(grad_g, self.guest_rng)
        # host: its gradient slice from the re-randomised fore gradient
        fore_h = deserialize(wire_fore, pk)
        feats_h = self._features(self._host_features, self.host_X, batch_id, idx)
        mask_h, wire_h = self._mask_and_ship(operators.batch_matmul(pk, fore_h, feats_h, be), self.host_rng)
        # arbiter decrypts; owners unmask, scale and step
        g_guest = (self._arbiter_gradient(wire_g) - mask_g) / s
        g_host = (self._arbiter_gradient(wire_h) - mask_h) / s
        self.guest_theta = self.guest_theta - self.config.learning_rate * g_guest
        self.host_theta = self.host_theta - self.config.learning_rate * g_host
        return g_guest, g_host

    # ---- loss over the loss set (parties.py:199-225, 267-276, 300-305) ---------------------------------------
    def loss(self) -> float:
        pk, be = self.pk, self.backend
        idx = self.loss_indices
        z_h = self._take(self.host_X, idx) @ self.host_theta
        sq = z_h * z_h
        c1 = operators.batch_encrypt(pk, _encode(pk, z_h, protocol_exponent(z_h, pk=pk, backend=be), be),
                                     self.host_rng, be)
        c2 = operators.batch_encrypt(pk, _encode(pk, sq, protocol_exponent(sq, pk=pk, backend=be), be),
                                     self.host_rng, be)
        c_lh, c_lh2 = deserialize(serialize_to_bytes(c1), pk), deserialize(serialize_to_bytes(c2), pk)
        lg = self._take(self.guest_X, idx) @ self.guest_theta
        y = self._take(self.guest_y, idx)
        k1 = 0.25 * lg - 0.5 * y
        plain_part = LOG2 - 0.5 * y * lg + 0.125 * lg * lg
        e1, e2 = c_lh.exponents[0], c_lh2.exponents[0]
        target = min(e1 + protocol_exponent(k1, pk=pk, backend=be), e2 + encoding.exact_exponent(0.125),
                     protocol_exponent(plain_part, pk=pk, backend=be))
        total = operators.batch_add(
            pk,
            operators.batch_mul_plain(pk, c_lh, _encode(pk, k1, target - e1, be), be),
            operators.batch_mul_plain(pk, c_lh2, _encode(pk, [0.125], target - e2, be), be), be)
        total = operators.batch_add(pk, total, _encode(pk, plain_part, target, be), be)
        loss_sum = operators.batch_obfuscate(pk, operators.batch_sum(pk, total, None, be), self.guest_rng, be)
        cipher = deserialize(serialize_to_bytes(loss_sum), pk)
        value = decode_batch(pk, operators.batch_decrypt(self.keys.private, cipher, be), be)[0]
        self.decrypted.append([value])
        return value / len(idx)

    def run_epoch(self) -> EpochResult:
        last = (np.zeros_like(self.guest_theta), np.zeros_like(self.host_theta))
        for batch_id, idx in enumerate(self.batches):
            last = self.step(batch_id, idx)
        loss = self.loss()
        self.epoch += 1
        return EpochResult(self.epoch, loss, float(np.linalg.norm(np.concatenate(last))), self.ledger.to_json())

    def run(self, epochs: int):
        return [self.run_epoch() for _ in range(epochs)]

    def combined_theta(self) -> np.ndarray:
        return np.concatenate([self.guest_theta, self.host_theta])


class HomoFederation:
    """Horizontal federation (reference flr/parties.py:357-454): every party encrypts its full-batch Taylor
    gradient at exponent -12, the arbiter weights each vector by the party's row count (a scalar power), adds
    them homomorphically and decrypts only the aggregate; the epoch loss travels the same way as one encrypted
    sum per party.  Random streams as in the reference (party i: (seed + 13) * 31 + i), so with the same data, key
    and seed the aggregated gradients, the model and the loss equal the reference's."""

    def __init__(self, party_data, keys: KeyPair, config: FlrConfig, backend=None):
        if len({p.X.shape[1] for p in party_data}) != 1:
            raise ValueError("horizontal parties must share one feature schema")
        self.keys = keys
        self.pk = keys.public
        self.config = config
        self.backend = backend or default_backend()
        self.parties = [{"name": p.name, "rng": default_rng((config.seed + 13) * 31 + i),
                         "X": np.hstack([p.X, np.ones((p.rows, 1))]), "y": p.y}
                        for i, p in enumerate(party_data)]
        self.theta = np.zeros(self.parties[0]["X"].shape[1])
        self.epoch = 0
        self.aggregated_gradients = []

    def _send(self, party, values) -> tuple:
        """Encode at the protocol exponent, encrypt with the party's stream, ship as HAFB bytes."""
        plain = _encode(self.pk, [float(v) for v in values], HOMO_GRADIENT_EXPONENT, self.backend)
        cipher = operators.batch_encrypt(self.pk, plain, party["rng"], self.backend)
        return serialize_to_bytes(cipher), len(party["X"])

    def run_epoch(self) -> EpochResult:
        pk, be = self.pk, self.backend
        wires = []
        for party in self.parties:                                        # parties.py:373-381
            X, y = party["X"], party["y"]
            grad = (0.25 * (X @ self.theta) - 0.5 * y) @ X / len(y)
            wires.append(self._send(party, grad))
        total_rows = sum(rows for _, rows in wires)
        acc = None
        for wire, rows in wires:                                          # parties.py:422-428
            cipher = deserialize(wire, pk)
            weight = encode_batch(pk, [float(rows)], target_exponent=0, backend=be)
            weighted = operators.batch_mul_plain(pk, cipher, weight, be)
            acc = weighted if acc is None else operators.batch_add(pk, acc, weighted, be)
        aggregated = np.asarray(decode_batch(pk, operators.batch_decrypt(self.keys.private, acc, be), be)) / total_rows
        self.aggregated_gradients.append(aggregated)
        self.theta = self.theta - self.config.learning_rate * aggregated
        loss_acc = None
        for party in self.parties:                                        # parties.py:383-389, 439-446
            z = party["X"] @ self.theta
            total = float(np.sum(LOG2 - 0.5 * party["y"] * z + 0.125 * z * z))
            cipher = deserialize(self._send(party, [total])[0], pk)
            loss_acc = cipher if loss_acc is None else operators.batch_add(pk, loss_acc, cipher, be)
        loss = decode_batch(pk, operators.batch_decrypt(self.keys.private, loss_acc, be), be)[0] / total_rows
        self.epoch += 1
        return EpochResult(self.epoch, loss, float(np.linalg.norm(aggregated)), TransferLedger().to_json())

    def run(self, epochs: int):
        return [self.run_epoch() for _ in range(epochs)]
