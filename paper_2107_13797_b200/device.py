"""Device plumbing: key contexts, word arrays and their residency.

WordArray is the aggregated storage of the operators: `count` big integers as a dense
[count, width] array of little-endian 32-bit words (byte-identical to the HAFB payload for the usual
key sizes), living on the host (numpy), on the GPU (torch tensor) or both.  Operators take and
return WordArrays, so chained operators never leave the device; Python integers are materialised
only when somebody asks for them (`.ints()`), which is what the reference API's `payload` /
`mantissas` attributes do lazily.

Two more resident forms exist next to the plain device tensor:

  * Montgomery digit form (`from_mont`): what the ciphertext operators hand each other, x * R mod n^2 in
    hb_ct_limbs words per element.  An addition of two resident ciphertexts is then ONE modular multiplication and
    no operator converts in and out; plain words are produced (one kernel) only when somebody needs them -- a
    download, the wire format, a comparison.
  * Shards (`from_shards`): contiguous element ranges living on several devices (backends.MultiDeviceBackend).

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


class Shards:
    """Element ranges [lo, hi) of one array and the WordArray holding each, part i resident on `devices[i]`."""

    __slots__ = ("ranges", "parts", "devices")

    def __init__(self, ranges, parts, devices):
        self.ranges = tuple((int(lo), int(hi)) for lo, hi in ranges)
        self.parts = list(parts)
        self.devices = tuple(devices)


class WordArray:
    """count x width little-endian 32-bit words; host and/or device resident."""

    __slots__ = ("count", "width", "_np", "_dev", "_ints", "_mont", "_n", "_shards")

    def __init__(self, count: int, width: int, np_words=None, dev_words=None, ints=None):
        self.count = count
        self.width = width
        self._np = np_words
        self._dev = dev_words
        self._ints = ints
        self._mont = None       # torch tensor [count, limbs]: Montgomery digit form mod _n^2
        self._n = None
        self._shards = None

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
    def from_mont(cls, tensor, n: int, width: int) -> "WordArray":
        """Ciphertexts in Montgomery digit form (tensor [count, hb_ct_limbs]); `width` = plain words per element."""
        out = cls(tensor.shape[0], width)
        out._mont = tensor
        out._n = int(n)
        return out

    @classmethod
    def from_shards(cls, shards: Shards, width: int) -> "WordArray":
        out = cls(shards.ranges[-1][1] if shards.ranges else 0, width)
        out._shards = shards
        return out

    @classmethod
    def empty_device(cls, count: int, width: int) -> "WordArray":
        require_cuda()
        t = torch()
        return cls(count, width, None, t.empty((count, width), dtype=t.int32, device="cuda"), None)

    # -- views
    @property
    def on_device(self) -> bool:
        return self._dev is not None or self._mont is not None or self._shards is not None

    @property
    def on_host(self) -> bool:
        return self._np is not None or self._ints is not None

    @property
    def shards(self):
        return self._shards

    def mont(self):
        """The Montgomery digit-form tensor if this array is resident in that form, else None."""
        return self._mont

    def device(self):
        """torch int32 tensor [count, width] of plain words on the current CUDA device (produced once, then cached):
        converted from the Montgomery form, gathered from the shards, or uploaded from the host."""
        if self._dev is None:
            require_cuda()
            t = torch()
            if self._mont is not None:
                self._dev = _from_mont(self._mont, self._n, self.width)
            elif self._shards is not None and self._np is None and self._ints is None:
                cur = t.cuda.current_device()
                parts = [p.device().to(f"cuda:{cur}", non_blocking=True) for p in self._shards.parts if p.count]
                for dev in set(self._shards.devices):            # the copies were issued on the sources' streams
                    t.cuda.synchronize(dev)
                self._dev = (t.cat(parts, dim=0) if parts
                             else t.empty((0, self.width), dtype=t.int32, device=f"cuda:{cur}"))
            else:
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

    def make_resident(self) -> None:
        """Have the array in HBM in a form the kernels read (Arena.upload / restore after a spill)."""
        if self.count and not self.on_device:
            self.device()

    def ptr(self) -> int:
        return self.device().data_ptr() if self.count else 0

    def ct_operand(self):
        """(device pointer, is_montgomery) of a ciphertext operand, in whichever form is already resident."""
        if not self.count:
            return 0, False
        if self._mont is not None and self._mont.device.index == torch().cuda.current_device():
            return self._mont.data_ptr(), True
        return self.device().data_ptr(), False

    def numpy(self) -> np.ndarray:
        if self._np is None:
            if self._ints is not None:
                self._np = ints_to_words(self._ints, self.width)
            elif self._dev is not None or self._mont is not None:
                self._np = self.device().cpu().numpy().view(np.uint32)
            elif self._shards is not None:
                parts = [p.numpy() for p in self._shards.parts]
                self._np = (np.concatenate(parts, axis=0) if parts else np.zeros((0, self.width), np.uint32))
            else:
                self._np = np.zeros((0, self.width), np.uint32)
        return self._np

    def ints(self) -> tuple:
        if self._ints is None:
            self._ints = words_to_ints(self.numpy())
        return self._ints

    def drop_device(self) -> None:
        """Keep a host copy and release every device-resident form (Arena spill)."""
        self.numpy()
        self._dev = None
        self._mont = None
        self._shards = None

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


def _from_mont(mont, n: int, width: int):
    """Plain words [count, width] of a Montgomery digit-form tensor, on the tensor's device."""
    t = torch()
    with t.cuda.device(mont.device):
        ctx = context_for(n)
        out = t.empty((mont.shape[0], width), dtype=t.int32, device=mont.device)
        if mont.shape[0]:
            _native.check(_native.lib().hb_ct_convert(ctx.handle, mont.data_ptr(), out.data_ptr(), mont.shape[0], 0,
                                                      current_stream_ptr()))
    return out


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
        self.device_index = device_index
        self.wn = lib.hb_pt_words(handle)
        self.wc = lib.hb_ct_words(handle)
        self.limbs = lib.hb_ct_limbs(handle)
        self.has_private = False
        self._private = None
        self._lock = threading.Lock()
        self._lib = lib

    def set_private(self, p: int, q: int, hp: int, hq: int, q_inv: int) -> None:
        """Install the CRT constants (once).  A later call must name the same factorisation: a caller that only
        knows n cannot decrypt with somebody else's cached key."""
        given = (int(p), int(q), int(hp), int(hq), int(q_inv))
        with self._lock:
            if self.has_private:
                if given != self._private:
                    raise ValueError("private key does not match the one installed for this modulus")
                return
            hw = (max(p, q).bit_length() + 31) // 32
            arrs = [ints_to_words([v], hw) for v in given]
            _native.check(self._lib.hb_ctx_set_private(self.handle, *[a.ctypes.data for a in arrs], hw))
            self._private = given
            self.has_private = True

    def set_option(self, option: int, value: int) -> None:
        _native.check(self._lib.hb_ctx_set_option(self.handle, int(option), int(value)))

    def close(self) -> None:
        """Destroy the native context (the device copy of the private constants is freed with it)."""
        with self._lock:
            if getattr(self, "handle", None):
                self._lib.hb_ctx_destroy(self.handle)
                self.handle = None
            self._private = None
            self.has_private = False

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_contexts: dict = {}
_ctx_lock = threading.Lock()
MAX_CONTEXTS = 64          # least recently created contexts beyond this are destroyed


def context_for(n: int) -> KeyContext:
    """Cached key context for modulus n on the current CUDA device."""
    require_cuda()
    dev = torch().cuda.current_device()
    key = (int(n), dev)
    with _ctx_lock:
        ctx = _contexts.get(key)
        if ctx is None:
            while len(_contexts) >= MAX_CONTEXTS:
                _contexts.pop(next(iter(_contexts)))       # its __del__ destroys the native context
            ctx = KeyContext(n, dev)
            _contexts[key] = ctx
        return ctx


def drop_private(n: int) -> None:
    """Forget the private part installed for modulus n on every device: the contexts are destroyed (their device
    memory, private constants included, is freed) and rebuilt public-only on next use."""
    with _ctx_lock:
        for key in [k for k in _contexts if k[0] == int(n)]:
            _contexts.pop(key).close()


def clear_contexts() -> None:
    with _ctx_lock:
        while _contexts:
            _contexts.popitem()[1].close()


def current_stream_ptr() -> int:
    return torch().cuda.current_stream().cuda_stream


def launch_count() -> int:
    return int(_native.lib().hb_launch_count())


class CompactScalars(WordArray):
    """A rows x cols matrix of encoded plaintext scalars kept as sign + 64-bit magnitude, stored by column
    (mag[j * rows + t], neg[j * rows + t]) -- all the encrypted matvec reads; 9 bytes per scalar instead of a full
    residue (256 B at 2048 bits).  The role of the reference's MiniBatchAggregator (bufferpool.py:182-226): a
    mini-batch's feature block is packed once and reused every epoch.  Presents the WordArray interface: the residues
    (n - magnitude for negatives) are materialised on the host only if somebody asks for them."""

    __slots__ = ("rows", "cols", "mag", "neg", "maxbits", "nneg", "modulus")

    def __init__(self, n: int, rows: int, cols: int, mag, neg, maxbits: int, nneg: int):
        wn = (int(n).bit_length() + 31) // 32
        super().__init__(rows * cols, wn)
        self.modulus = int(n)
        self.rows, self.cols = rows, cols
        self.mag, self.neg = mag, neg            # torch tensors: int64 [cols * rows], uint8 [cols * rows]
        self.maxbits, self.nneg = int(maxbits), int(nneg)

    @property
    def on_device(self) -> bool:
        return self.mag is not None

    def make_resident(self) -> None:
        """The compact form IS the resident form: nothing to upload while it is there (materialising 256-byte
        residues for a 1M x 101 feature block would be 26 GB and minutes of host work)."""
        if not self.on_device:
            super().make_resident()

    def numpy(self) -> np.ndarray:
        """Residues [rows * cols, wn] in row-major element order.  Negative scalars are n - magnitude: the low 64 bits
        are a two-word subtraction, and its borrow runs up through n only while n's words are zero -- vectorised over
        the elements, one pass per word the borrow actually reaches (normally one)."""
        if self._np is None:
            mag = np.ascontiguousarray(self.mag.cpu().numpy().view(np.uint64).reshape(self.cols, self.rows).T).reshape(-1)
            neg = np.ascontiguousarray(self.neg.cpu().numpy().reshape(self.cols, self.rows).T).reshape(-1).astype(bool)
            width = self.width
            out = np.zeros((self.count, width), np.uint32)
            pos = ~neg
            out[pos, 0] = (mag[pos] & np.uint64(0xffffffff)).astype(np.uint32)
            if width > 1:
                out[pos, 1] = (mag[pos] >> np.uint64(32)).astype(np.uint32)
            if neg.any():
                nw = ints_to_words([self.modulus], width)[0]
                m = mag[neg]
                n_lo = np.uint64(int(nw[0]) | ((int(nw[1]) << 32) if width > 1 else 0))
                lo = n_lo - m                                      # wraps mod 2^64 exactly when a borrow leaves
                res = np.broadcast_to(nw, (m.shape[0], width)).copy()
                res[:, 0] = (lo & np.uint64(0xffffffff)).astype(np.uint32)
                if width > 1:
                    res[:, 1] = (lo >> np.uint64(32)).astype(np.uint32)
                else:
                    res[:, 0] = ((int(nw[0]) - m.astype(np.int64)) & 0xffffffff).astype(np.uint32)
                borrow = np.nonzero(m > n_lo)[0]                   # rows whose subtraction borrows from word 2 up
                i = 2
                while borrow.size and i < width:
                    word = res[borrow, i]
                    res[borrow, i] = word - np.uint32(1)           # wraps to 0xffffffff when the word was zero
                    borrow = borrow[word == 0]
                    i += 1
                out[neg] = res
            self._np = out
        return self._np

    def drop_device(self) -> None:
        self.numpy()
        self.mag = self.neg = None
        self._dev = None
