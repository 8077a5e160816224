"""L0 bit primitives on the GPU — drop-in for the reference ``formats.py``.

Layouts are fixed by the reference (``formats.py:1-19``):

* BF16 word x:  e = (x >> 7) & 0xFF,  a = ((x >> 8) & 0x80) | (x & 0x7F)
* E5M2 word x:  e = (x >> 2) & 0x1F,  a = ((x >> 7) << 2)   | (x & 0x03)
* E4M3 word x:  e = (x >> 3) & 0x0F,  a = ((x >> 7) << 3)   | (x & 0x07)
* packed symbols: LSB-first bit stream, symbol i at bits [i*w, (i+1)*w);
  unused trailing bits are zero.

Array arguments run through the sm_100a kernels in ``libsz_b200.so``.  A numpy
array in gives numpy out (copied through the device); a CUDA tensor in gives
a CUDA tensor out.  Plain Python integers (single words) are split with
integer arithmetic on the host — the same two shifts the kernels do.
"""

from __future__ import annotations

import enum
from typing import Any, NamedTuple

import numpy as np
import torch

from . import _native as N
from .errors import CodeRangeError, ConfigError, MalformedStreamError

__all__ = [
    "ElementFormat", "SplitFields", "RawTensorStream", "split_fields", "reconstruct",
    "pack_codes", "unpack_codes", "packed_nbytes", "trailing_bits_zero",
]


class ElementFormat(enum.Enum):
    """Element word layouts: (cli name, word bits, exponent bits, sign|mantissa
    bits) — the same members and attributes as the reference (formats.py:42-79)."""

    BF16 = ("bf16", 16, 8, 8)
    FP8_E5M2 = ("e5m2", 8, 5, 3)
    FP8_E4M3 = ("e4m3", 8, 4, 4)

    def __init__(self, cli_name: str, word_bits: int, exp_bits: int, sm_bits: int):
        self.cli_name = cli_name
        self.word_bits = word_bits
        self.exp_bits = exp_bits
        self.sm_bits = sm_bits

    @property
    def code(self) -> int:
        """Format byte of the container and of the C ABI (sz_format)."""
        return {"bf16": 0, "e5m2": 1, "e4m3": 2}[self.cli_name]

    @property
    def exp_bins(self) -> int:
        return 1 << self.exp_bits

    @property
    def word_dtype(self) -> np.dtype:
        return np.dtype(np.uint16 if self.word_bits == 16 else np.uint8)

    @property
    def torch_dtype(self) -> torch.dtype:
        return torch.uint16 if self.word_bits == 16 else torch.uint8

    @property
    def word_nbytes(self) -> int:
        return self.word_bits // 8

    @classmethod
    def from_name(cls, name: str) -> "ElementFormat":
        for fmt in cls:
            if fmt.cli_name == name.lower():
                return fmt
        raise ConfigError(f"unknown element format {name!r}; choose from "
                          f"{[f.cli_name for f in cls]}")


class SplitFields(NamedTuple):
    exponent: Any
    sign_mantissa: Any


# ------------------------------------------------------------ host <-> device
def is_device(x) -> bool:
    return isinstance(x, torch.Tensor) and x.device.type == "cuda"


def to_numpy(x) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    if isinstance(x, (bytes, bytearray, memoryview)):
        return np.frombuffer(bytes(x), dtype=np.uint8)
    return np.asarray(x)


def to_device(x, dtype: torch.dtype, align: int = 32) -> torch.Tensor:
    """Any array-like/bytes -> aligned contiguous CUDA tensor of ``dtype``."""
    if isinstance(x, torch.Tensor):
        t = x.reshape(-1)
        if t.dtype != dtype:
            if t.element_size() == torch.empty(0, dtype=dtype).element_size():
                t = t.view(dtype)
            else:
                t = t.to(dtype)
        return N.aligned_device_copy(t, align)
    if isinstance(x, (bytes, bytearray, memoryview)):
        arr = np.frombuffer(bytes(x), dtype=np.uint8)
    else:
        arr = np.asarray(x)
    np_dtype = {torch.uint8: np.uint8, torch.uint16: np.uint16, torch.uint32: np.uint32,
                torch.int64: np.int64}[dtype]
    arr = np.ascontiguousarray(arr.reshape(-1), dtype=np_dtype)
    if not arr.flags.writeable:
        arr = arr.copy()
    return N.aligned_device_copy(torch.from_numpy(arr), align)


class RawTensorStream(NamedTuple):
    """A flat run of element words plus its format (formats.py:89-110).

    ``words`` may be a numpy array (host) or a torch tensor (CUDA or CPU).
    """

    fmt: ElementFormat
    words: Any

    @property
    def n_elements(self) -> int:
        w = self.words
        return int(w.numel() if isinstance(w, torch.Tensor) else np.asarray(w).size)

    @property
    def raw_bytes(self) -> int:
        return self.n_elements * self.fmt.word_nbytes

    @property
    def on_device(self) -> bool:
        return is_device(self.words)

    def to_bytes(self) -> bytes:
        return np.ascontiguousarray(to_numpy(self.words).reshape(-1),
                                    dtype=self.fmt.word_dtype).tobytes()

    def device_words(self) -> torch.Tensor:
        return to_device(self.words, self.fmt.torch_dtype)

    @classmethod
    def from_words(cls, fmt: ElementFormat, words) -> "RawTensorStream":
        if isinstance(words, torch.Tensor):
            return cls(fmt, words.reshape(-1))
        return cls(fmt, np.ascontiguousarray(words, dtype=fmt.word_dtype).ravel())


# ------------------------------------------------------------ split / join
def _split_int(x: int, fmt: ElementFormat) -> tuple[int, int]:
    mb = fmt.sm_bits - 1
    x &= (1 << fmt.word_bits) - 1
    return (x >> mb) & (fmt.exp_bins - 1), ((x >> (fmt.word_bits - 1)) << mb) | (x & ((1 << mb) - 1))


def _join_int(e: int, a: int, fmt: ElementFormat) -> int:
    mb = fmt.sm_bits - 1
    return (((a >> mb) & 1) << (fmt.word_bits - 1)) | ((e & (fmt.exp_bins - 1)) << mb) | (a & ((1 << mb) - 1))


def split_fields(word, fmt: ElementFormat) -> SplitFields:
    """(exponent, sign_mantissa) of every word — formats.py:113-133."""
    if isinstance(word, (int, np.integer)) or (not isinstance(word, torch.Tensor)
                                               and np.ndim(word) == 0):
        return SplitFields(*_split_int(int(word), fmt))
    lib = N.load_library()
    words = to_device(word, fmt.torch_dtype)
    n = words.numel()
    exp = torch.empty(n, dtype=torch.uint8, device=words.device)
    sm = torch.empty(n, dtype=torch.uint8, device=words.device)
    N.check(lib.sz_split_fields(N.ptr(words), n, fmt.code, N.ptr(exp), N.ptr(sm),
                                N.stream_handle()), "split_fields")
    if is_device(word):
        return SplitFields(exp, sm)
    shape = np.shape(word)
    return SplitFields(exp.cpu().numpy().reshape(shape), sm.cpu().numpy().reshape(shape))


def reconstruct(fields: SplitFields, fmt: ElementFormat):
    """Exact inverse of :func:`split_fields` — formats.py:136-155."""
    e, a = fields
    if isinstance(e, (int, np.integer)) or (not isinstance(e, torch.Tensor) and np.ndim(e) == 0):
        return _join_int(int(e), int(a), fmt)
    lib = N.load_library()
    ed = to_device(e, torch.uint8)
    ad = to_device(a, torch.uint8)
    n = ed.numel()
    if ad.numel() != n:
        raise ConfigError("exponent and sign-mantissa planes differ in length")
    out = torch.empty(n, dtype=fmt.torch_dtype, device=ed.device)
    N.check(lib.sz_reconstruct(N.ptr(ed), N.ptr(ad), n, fmt.code, N.ptr(out),
                               N.stream_handle()), "reconstruct")
    if is_device(e):
        return out
    return out.cpu().numpy().reshape(np.shape(e))


# ------------------------------------------------------------ bit packing
def packed_nbytes(n: int, code_bits: int) -> int:
    return (n * code_bits + 7) // 8


def _device_max(t: torch.Tensor) -> int:
    lib = N.load_library()
    out = torch.empty(1, dtype=torch.uint32, device=t.device)
    N.check(lib.sz_max_u8(N.ptr(t), t.numel(), N.ptr(out), N.stream_handle()), "max")
    return int(out.cpu().numpy()[0])


def pack_bits_device(sym: torch.Tensor, width: int) -> torch.Tensor:
    """uint8 CUDA symbols -> packed CUDA bytes (no range check)."""
    lib = N.load_library()
    n = sym.numel()
    out = torch.empty(packed_nbytes(n, width), dtype=torch.uint8, device=sym.device)
    if n:
        N.check(lib.sz_pack_bits(N.ptr(sym), n, width, N.ptr(out), N.stream_handle()),
                "pack_bits")
    return out


def unpack_bits_device(packed: torch.Tensor, n: int, width: int) -> tuple[torch.Tensor, bool]:
    lib = N.load_library()
    sym = torch.empty(max(n, 1), dtype=torch.uint8, device=packed.device)[:n]
    flag = torch.empty(1, dtype=torch.uint32, device=packed.device)
    N.check(lib.sz_unpack_bits(N.ptr(packed), n, width, N.ptr(sym), N.ptr(flag),
                               N.stream_handle()), "unpack_bits")
    return sym, bool(flag.cpu().numpy()[0])


def pack_codes(codes, code_bits: int):
    """Dense LSB-first packing of 3/4-bit symbols — formats.py:167-189."""
    if code_bits not in (3, 4):
        raise ConfigError(f"code_bits must be 3 or 4, got {code_bits}")
    dev = is_device(codes)
    if not dev:
        arr = np.asarray(codes)
        if arr.size == 0:
            return b""
        if arr.min() < 0 or arr.max() > 255:
            bad = int(np.argmax((arr < 0) | (arr > 255)))
            raise CodeRangeError(f"code {int(arr.ravel()[bad])} at index {bad} does not fit "
                                 f"in {code_bits} bits")
    sym = to_device(codes, torch.uint8, align=16)
    if sym.numel() == 0:
        return torch.empty(0, dtype=torch.uint8, device=sym.device) if dev else b""
    if _device_max(sym) >= 1 << code_bits:
        bad = int((sym >= (1 << code_bits)).nonzero()[0, 0])
        raise CodeRangeError(f"code {int(sym[bad])} at index {bad} does not fit in "
                             f"{code_bits} bits")
    out = pack_bits_device(sym, code_bits)
    return out if dev else out.cpu().numpy().tobytes()


def unpack_codes(data, n: int, code_bits: int):
    """Exact inverse of :func:`pack_codes` — formats.py:197-220."""
    if code_bits not in (3, 4):
        raise ConfigError(f"code_bits must be 3 or 4, got {code_bits}")
    dev = is_device(data)
    size = data.numel() if isinstance(data, torch.Tensor) else len(data)
    if size != packed_nbytes(n, code_bits):
        raise MalformedStreamError(f"packed stream is {size} bytes, expected "
                                   f"{packed_nbytes(n, code_bits)} for {n} codes of "
                                   f"{code_bits} bits")
    if n == 0:
        return torch.empty(0, dtype=torch.uint8, device=N.device()) if dev else \
            np.zeros(0, dtype=np.uint8)
    sym, _ = unpack_bits_device(to_device(data, torch.uint8, align=16), n, code_bits)
    return sym if dev else sym.cpu().numpy()


def trailing_bits_zero(data, n: int, code_bits: int) -> bool:
    """True when every pad bit after n*code_bits is zero (formats.py:223-231).

    The pad bits all live in the final byte, so this is a one-byte check.
    """
    size = data.numel() if isinstance(data, torch.Tensor) else len(data)
    used = n * code_bits
    if used == size * 8:
        return True
    if used > size * 8:
        return False
    if size * 8 - used >= 8:  # whole spare bytes: all must be zero
        tail = to_numpy(data[used // 8 + (1 if used % 8 else 0):])
        if np.any(tail):
            return False
    if used % 8 == 0:
        return True
    last = int(to_numpy(data[used // 8: used // 8 + 1])[0])
    return (last >> (used % 8)) == 0
