"""Device plumbing: key contexts, word arrays and their residency.

WordArray is the aggregated storage of the operators: `count` big integers as a dense
[count, width] array of little-endian 32-bit words (byte-identical to the HAFB payload for the usual
key sizes), living on the host (numpy), on the GPU (torch tensor) or both.  Operators take and
return WordArrays, so chained operators never leave the device; Python integers are materialised
only when somebody asks for them (`.ints()`), which is what the reference API's `payload` /
`mantissas` attributes do lazily.

torch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _native

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as _t
        _torch = _t
    return _torch


def require_cuda() -> None:
    t = torch()
    if not t.cuda.is_available():
        raise _native.NativeLibraryError(
            "no CUDA device is visible: the homomorphic operators have no CPU path")


def ints_to_words(values, width: int) -> np.ndarray:
    """Python ints -> [count, width] uint32 little-endian words.  Raises OverflowError if one does not fit."""
    nbytes = 4 * width
    buf = b"".join(int(v).to_bytes(nbytes, "little") for v in values)
    return np.frombuffer(buf, dtype=np.uint32).reshape(-1, width).copy() if buf else np.zeros((0, width), np.uint32)


def words_to_ints(arr: np.ndarray) -> tuple:
    arr = np.ascontiguousarray(arr, dtype=np.uint32)
    count, width = arr.shape
    raw = arr.tobytes()
    nbytes = 4 * width
    return tuple(int.from_bytes(raw[i * nbytes:(i + 1) * nbytes], "little") for i in range(count))


class WordArray:
    """count x width little-endian 32-bit words; host and/or device resident."""

    __slots__ = ("count", "width", "_np", "_dev", "_ints")

    def __init__(self, count: int, width: int, np_words=None, dev_words=None, ints=None):
        self.count = count
        self.width = width
        self._np = np_words
        self._dev = dev_words
        self._ints = ints

    # -- constructors
    @classmethod
    def from_ints(cls, values, width: int) -> "WordArray":
        values = tuple(values)
        return cls(len(values), width, ints_to_words(values, width), None, values)

    @classmethod
    def from_numpy(cls, arr: np.ndarray) -> "WordArray":
        arr = np.ascontiguousarray(arr, dtype=np.uint32)
        return cls(arr.shape[0], arr.shape[1], arr, None, None)

    @classmethod
    def from_device(cls, tensor) -> "WordArray":
        return cls(tensor.shape[0], tensor.shape[1], None, tensor, None)

    @classmethod
    def empty_device(cls, count: int, width: int) -> "WordArray":
        require_cuda()
        t = torch()
        return cls(count, width, None, t.empty((count, width), dtype=t.int32, device="cuda"), None)

    # -- views
    @property
    def on_device(self) -> bool:
        return self._dev is not None

    @property
    def on_host(self) -> bool:
        return self._np is not None or self._ints is not None

    def device(self):
        """torch int32 tensor [count, width] on the current CUDA device (uploaded once, then cached)."""
        if self._dev is None:
            require_cuda()
            t = torch()
            arr = self.numpy().view(np.int32)
            if arr.flags.writeable:
                host = t.from_numpy(arr)
            else:                                  # a view of received wire bytes: read-only is what we want
                import warnings
                with warnings.catch_warnings():
                    warnings.simplefilter("ignore")
                    host = t.from_numpy(arr)
            self._dev = host.cuda(non_blocking=False)
        return self._dev

    def ptr(self) -> int:
        return self.device().data_ptr() if self.count else 0

    def numpy(self) -> np.ndarray:
        if self._np is None:
            if self._dev is not None:
                self._np = self._dev.cpu().numpy().view(np.uint32)
            else:
                self._np = ints_to_words(self._ints, self.width)
        return self._np

    def ints(self) -> tuple:
        if self._ints is None:
            self._ints = words_to_ints(self.numpy())
        return self._ints

    def drop_device(self) -> None:
        """Keep a host copy and release the device tensor (Arena spill)."""
        self.numpy()
        self._dev = None

    def __len__(self):
        return self.count

    def __eq__(self, other):
        if not isinstance(other, WordArray):
            return NotImplemented
        if self.count != other.count:
            return False
        if self._ints is not None and other._ints is not None:
            return self._ints == other._ints
        if self.width == other.width:
            return bool(np.array_equal(self.numpy(), other.numpy()))
        return self.ints() == other.ints()

    def __hash__(self):
        return hash(self.ints())


class KeyContext:
    """One hb_ctx per (modulus, device); owns the native handle."""

    def __init__(self, n: int, device_index: int = 0):
        require_cuda()
        lib = _native.lib()
        self.n = int(n)
        self.key_bits = self.n.bit_length()
        wn = (self.key_bits + 31) // 32
        words = ints_to_words([self.n], wn)
        handle = ctypes.c_void_p()
        _native.check(lib.hb_ctx_create(ctypes.byref(handle), words.ctypes.data, wn, device_index))
        self.handle = handle
        self.wn = lib.hb_pt_words(handle)
        self.wc = lib.hb_ct_words(handle)
        self.has_private = False
        self._lib = lib

    def set_private(self, p: int, q: int, hp: int, hq: int, q_inv: int) -> None:
        if self.has_private:
            return
        hw = (max(p, q).bit_length() + 31) // 32
        arrs = [ints_to_words([v], hw) for v in (p, q, hp, hq, q_inv)]
        _native.check(self._lib.hb_ctx_set_private(self.handle, *[a.ctypes.data for a in arrs], hw))
        self.has_private = True

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self._lib.hb_ctx_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


_contexts: dict = {}
_ctx_lock = threading.Lock()


def context_for(n: int) -> KeyContext:
    """Cached key context for modulus n on the current CUDA device."""
    require_cuda()
    dev = torch().cuda.current_device()
    key = (int(n), dev)
    with _ctx_lock:
        ctx = _contexts.get(key)
        if ctx is None:
            ctx = KeyContext(n, dev)
            _contexts[key] = ctx
        return ctx


def current_stream_ptr() -> int:
    return torch().cuda.current_stream().cuda_stream


def launch_count() -> int:
    return int(_native.lib().hb_launch_count())
