"""B200-native homomorphic operators for federated logistic regression (HAFLO, arXiv 2107.13797).

Module layout mirrors the reference package `hebatch` so that its hot path is a drop-in:

    paillier    keys, scalar operations              (reference: paillier.py)
    encoding    fixed-point codec for single numbers (encoding.py)
    batches     PlaintextBatch / CiphertextBatch      (batches.py)      -- device-resident word storage
    backends    ExecutionBackend, CudaBackend         (backends.py)     -- the plug-in boundary
    operators   batch_* operators                     (operators.py)    -- the hot path, CUDA only
    bufferpool  pinned pool, HAFB wire format         (bufferpool.py)
    arena       device-memory arena                   (arena.py)
    device      key contexts and word arrays          (no counterpart: the reference has no device)
    csrc/       sm_100a kernels and the C ABI (include/hebatch_b200.h)

Importing the package never touches CUDA; the first operator call loads
paper_2107_13797_b200/_lib/libhebatch_b200.so and fails loudly if it (or a GPU) is missing.
"""

__version__ = "0.1.0"

__all__ = ["paillier", "encoding", "batches", "backends", "operators", "bufferpool", "arena", "device"]
