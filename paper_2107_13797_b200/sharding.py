"""Multi-GPU execution of the operators, SPMD form: one process per GPU, `torch.distributed` for the plumbing.
(The single-process form -- one backend driving every device of the box, which is what the sequential FLR parties
need -- is backends.MultiDeviceBackend; both use the same partial / combine kernels.)

Element-wise operators (encrypt, obfuscate, decrypt, add, mul) shard by contiguous element ranges of
ceil(count / world) -- the reference's own schedule (backends.py:64-73 of the reference) -- and need no
collective: every rank works on its slice and the results stay sharded.  Reductions shard the reduced axis:

  * batch_sum(axis=None): each rank multiplies its slice down to one ciphertext, the world all-gathers
    `world` ciphertexts and multiplies them (same shape as operators.py:263-275);
  * batch_matmul: rows are sharded, each rank emits d pairs (A_j, B_j), the world all-gathers
    world x d x 2 ciphertexts (d KiB-sized messages: latency bound) and combines them, one batch inversion
    at the end.

Modular multiplication is exact and commutative, so the bits equal the single-GPU result whatever the world
size.  The gather is `torch.distributed.all_gather` on whatever backend the process group has: NCCL over
NVLink on the GPU box, gloo in the CPU tests of the host logic.
"""
from __future__ import annotations

import numpy as np

from .backends import shard_range      # noqa: F401  (the reference's ceil(count / workers) schedule)
from .batches import CiphertextBatch, PlaintextBatch, ShapeMismatch, ct_width, shared_exponent_of
from .device import WordArray


def shard_rows(batch, rank: int, world: int):
    """The rank's contiguous block of rows (axis 0) of a 1-D or 2-D batch, exponent metadata included."""
    rows = batch.shape[0]
    lo, hi = shard_range(rows, rank, world)
    width = batch.shape[1] if len(batch.shape) == 2 else 1
    words = batch.words.numpy()[lo * width:hi * width]
    shape = (hi - lo,) if len(batch.shape) == 1 else (hi - lo, width)
    exps = batch.exponents if batch.shared_exponent else batch.exponents[lo * width:hi * width]
    store = WordArray.from_numpy(words.copy())
    if isinstance(batch, CiphertextBatch):
        return CiphertextBatch(batch.key, shape, exps, store, batch.shared_exponent, batch.obfuscated)
    return PlaintextBatch(batch.key, shape, exps, store, batch.shared_exponent)


def all_gather_words(local, group=None):
    """local: torch tensor [k, w] (any device the group's backend accepts) -> tensor [world, k, w]."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local.contiguous(), group=group)
    return torch.stack(parts, dim=0)


def _comm_tensor(words: WordArray, group):
    """The word array as a tensor on the device the process group communicates on."""
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        return words.device()
    return torch.from_numpy(words.numpy().view(np.int32).copy())


def sharded_sum(pk, local: CiphertextBatch, backend, group=None) -> CiphertextBatch:
    """batch_sum(axis=None) over a batch whose elements are spread across the ranks of `group`."""
    from . import operators
    import torch.distributed as dist
    part = operators.batch_sum(pk, local, None, backend)          # (1,) ciphertext, 1 for an empty slice
    gathered = all_gather_words(_comm_tensor(part.words, group), group)       # [world, 1, wc]
    world = dist.get_world_size(group)
    store = _as_wordarray(gathered.reshape(world, -1))
    total = backend.product(pk.n, store, 1, world, 0, 1)
    return CiphertextBatch(pk, (1,), part.exponents, total, True, local.obfuscated)


def sharded_matmul(pk, a_local: CiphertextBatch, x_local: PlaintextBatch, backend, group=None) -> CiphertextBatch:
    """batch_matmul of a 1-D encrypted vector with a 2-D plaintext matrix, both sharded by rows."""
    import torch.distributed as dist
    if len(a_local.shape) != 1 or len(x_local.shape) != 2 or x_local.shape[0] != a_local.shape[0]:
        raise ShapeMismatch(f"row shards disagree: {a_local.shape} x {x_local.shape}")
    d = x_local.shape[1]
    ea, ex = shared_exponent_of(a_local), shared_exponent_of(x_local)
    world = dist.get_world_size(group)
    partial = backend.matvec_partial(pk.n, a_local.words, x_local.words, a_local.shape[0], d)   # [2d, wc]
    gathered = all_gather_words(_comm_tensor(partial, group), group)                           # [world, 2d, wc]
    out = backend.matvec_combine(pk.n, _as_wordarray(gathered.reshape(world * 2 * d, -1)), world, d)
    return CiphertextBatch(pk, (d,), (ea + ex,), out, True, a_local.obfuscated)


def _as_wordarray(tensor) -> WordArray:
    if tensor.is_cuda:
        return WordArray.from_device(tensor.contiguous())
    return WordArray.from_numpy(tensor.contiguous().numpy().view(np.uint32))


def combine_partials_reference(n2: int, blocks) -> list:
    """What matvec_combine computes, on Python integers: blocks[r][j] = (A_rj, B_rj).  Used by the CPU tests
    of the gather logic; never on the product path."""
    d = len(blocks[0])
    out = []
    for j in range(d):
        num = den = 1
        for blk in blocks:
            num = num * blk[j][0] % n2
            den = den * blk[j][1] % n2
        out.append(num * pow(den, -1, n2) % n2)
    return out
