"""SPLZ container framing — reference ``container.py``.

Same names, byte layout and error classes as the reference
(``/root/reference/pkg/src/splitzip/container.py``; ``docs/FORMATS.md:65-105``):

* ``container_to_bytes`` (container.py:201-215) — device-resident sections
  are framed **on the GPU** (``sz_frame_container``: header, SZCB codebook
  record and the five sections assembled in one contiguous HBM buffer, the
  escape count read from device memory) and copied out once; host sections
  are concatenated.
* ``encode_container`` — GPU-native: encode + frame, the container stays in
  HBM (one buffer for a file write or a single NCCL send).
* ``container_from_bytes`` (container.py:225-296) — parses bytes or a CUDA
  ``uint8`` tensor with the reference's checks, in the reference's order, and
  raises the same classes (``BadMagicError``, ``UnsupportedVersionError``,
  ``ContainerError``, ``TruncatedError(section=...)``,
  ``LengthMismatchError``, ``CorruptionError``).  Sections of a device
  container are sliced out in HBM; only the <= 292-byte header travels to the
  host.
* ``decode_container`` — parse + decode (the decode kernels).
* Codebook records (container.py:128-176) and raw ``.szrw`` dumps
  (container.py:305-339) for file interop.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np
import torch

from . import _native as N
from .calibration import CodebookMode, ExponentCodebook
from .codec import (CodecConfig, EncodedStreams, PositionMode, _config_params, decode,
                    encode)
from .errors import (BadMagicError, ConfigError, ContainerError, CorruptionError,
                     LengthMismatchError, TruncatedError, UnsupportedVersionError)
from .formats import (ElementFormat, RawTensorStream, is_device, packed_nbytes,
                      trailing_bits_zero, unpack_bits_device)

__all__ = [
    "CONTAINER_MAGIC", "RAW_MAGIC", "CODEBOOK_MAGIC", "FORMAT_VERSION",
    "codebook_record_bytes", "codebook_from_bytes", "write_codebook", "read_codebook",
    "container_to_bytes", "container_from_bytes", "write_container", "read_container",
    "encode_container", "decode_container", "frame_device",
    "raw_tensor_to_bytes", "raw_tensor_from_bytes", "write_raw_tensor", "read_raw_tensor",
]

CONTAINER_MAGIC = b"SPLZ"
RAW_MAGIC = b"SZRW"
CODEBOOK_MAGIC = b"SZCB"
FORMAT_VERSION = 1
_HEADER = struct.Struct("<BBBBIQQ")        # container.py:203-211
_FMT_CODES = {ElementFormat.BF16: 0, ElementFormat.FP8_E5M2: 1, ElementFormat.FP8_E4M3: 2}
_FMT_FROM_CODE = {v: k for k, v in _FMT_CODES.items()}
_MODE_CHUNKED, _MODE_SENTINEL, _MODE_ABS32 = 0, 1, 2


def _mode_byte(config: CodecConfig) -> int:
    if config.sentinel:
        return _MODE_SENTINEL
    return _MODE_ABS32 if config.abs32 else _MODE_CHUNKED


# ------------------------------------------------------------ codebook record
def codebook_record_bytes(codebook: ExponentCodebook) -> bytes:
    """``SZCB | 1 | fmt | code_bits | mode | k | entries`` (container.py:128-137)."""
    return (CODEBOOK_MAGIC
            + bytes([FORMAT_VERSION, _FMT_CODES[codebook.fmt], codebook.code_bits,
                     0 if codebook.mode is CodebookMode.TOPK_EXPLICIT else 1,
                     len(codebook.entries)])
            + bytes(codebook.entries))


class _Cursor:
    """Sequential reader raising TruncatedError(section=...) on short reads
    (container.py:92-115).  ``fetch(lo, hi)`` returns bytes of the source."""

    def __init__(self, total: int, fetch):
        self.total, self.fetch, self.offset = total, fetch, 0

    def skip(self, n: int, section: str) -> int:
        if self.offset + n > self.total:
            raise TruncatedError(f"file ends at byte {self.total} while reading {n} bytes at "
                                 f"offset {self.offset}", section=section)
        lo = self.offset
        self.offset += n
        return lo

    def take(self, n: int, section: str) -> bytes:
        lo = self.skip(n, section)
        return self.fetch(lo, lo + n)

    def u8(self, section: str) -> int:
        return self.take(1, section)[0]

    def u32(self, section: str) -> int:
        return struct.unpack("<I", self.take(4, section))[0]

    def u64(self, section: str) -> int:
        return struct.unpack("<Q", self.take(8, section))[0]


def _parse_codebook_record(cur: _Cursor) -> ExponentCodebook:
    magic = cur.take(4, "codebook")
    if magic != CODEBOOK_MAGIC:
        raise BadMagicError(f"bad codebook magic {magic!r}")
    version = cur.u8("codebook")
    if version != FORMAT_VERSION:
        raise UnsupportedVersionError(f"unsupported codebook version {version}")
    fmt_code = cur.u8("codebook")
    if fmt_code not in _FMT_FROM_CODE:
        raise ContainerError(f"unknown element format code {fmt_code}")
    code_bits = cur.u8("codebook")
    mode_code = cur.u8("codebook")
    if mode_code not in (0, 1):
        raise ContainerError(f"unknown codebook mode code {mode_code}")
    count = cur.u8("codebook")
    entries = cur.take(count, "codebook")
    try:
        return ExponentCodebook(_FMT_FROM_CODE[fmt_code], tuple(entries), code_bits,
                                CodebookMode.TOPK_EXPLICIT if mode_code == 0
                                else CodebookMode.TOP15_SENTINEL)
    except ConfigError as exc:
        raise CorruptionError(f"inconsistent codebook record: {exc}") from exc


def codebook_from_bytes(data: bytes) -> ExponentCodebook:
    data = bytes(data)
    cur = _Cursor(len(data), lambda lo, hi: data[lo:hi])
    book = _parse_codebook_record(cur)
    if cur.offset != len(data):
        raise LengthMismatchError(f"{len(data) - cur.offset} unexpected bytes after the "
                                  "codebook record")
    return book


def write_codebook(codebook: ExponentCodebook, sink) -> int:
    data = codebook_record_bytes(codebook)
    Path(sink).write_bytes(data)
    return len(data)


def read_codebook(source) -> ExponentCodebook:
    return codebook_from_bytes(Path(source).read_bytes())


# ------------------------------------------------------------ device framing
def _encoded_struct(streams: EncodedStreams, m_dev: torch.Tensor) -> N.SzEncoded:
    s = N.SzEncoded()
    s.d_codes = N.ptr(streams.packed_codes)
    s.d_sm = N.ptr(streams.sign_mantissa)
    counts = streams.chunk_counts
    s.d_counts = N.ptr(counts) if isinstance(counts, torch.Tensor) and counts.numel() else None
    pos = streams.escape_positions
    s.d_positions = N.ptr(pos) if isinstance(pos, torch.Tensor) and pos.numel() else None
    s.d_values = N.ptr(streams.escape_values) if streams.n_escapes else None
    s.d_values_packed = N.ptr(streams.values_packed) if streams.values_packed is not None \
        else None
    s.d_n_escapes = N.ptr(m_dev)
    s.escape_capacity = int(streams.n_escapes)
    s.d_escape_base = None
    return s


def frame_device(params: N.SzParams, n: int, enc: N.SzEncoded, out: torch.Tensor,
                 nbytes_dev: torch.Tensor, stream=None) -> None:
    """Enqueue ``sz_frame_container``: no host synchronisation."""
    lib = N.load_library()
    N.check(lib.sz_frame_container(params, n, enc, N.ptr(out), out.numel(), N.ptr(nbytes_dev),
                                   N.stream_handle(stream)), "frame_container")


def _frame_streams(streams: EncodedStreams, config: CodecConfig,
                   codebook: ExponentCodebook) -> torch.Tensor:
    lib = N.load_library()
    params = _config_params(config, codebook)
    n, m = int(streams.n_elements), int(streams.n_escapes)
    dev = streams.packed_codes.device
    if config.fmt.exp_bits != 8 and m and streams.values_packed is None:
        from .formats import pack_bits_device
        streams.values_packed = pack_bits_device(streams.escape_values[:m], config.fmt.exp_bits)
    total = lib.sz_container_bytes(n, m, params)
    out = torch.empty(total, dtype=torch.uint8, device=dev)
    m_dev = torch.tensor([m], dtype=torch.int64, device=dev)
    nb = torch.empty(1, dtype=torch.int64, device=dev)
    frame_device(params, n, _encoded_struct(streams, m_dev), out, nb)
    return out


def container_to_bytes(streams: EncodedStreams, config: CodecConfig,
                       codebook: ExponentCodebook) -> bytes:
    """The SPLZ file image (container.py:201-215), byte-identical."""
    if streams.on_device:
        return _frame_streams(streams, config, codebook).cpu().numpy().tobytes()
    header = CONTAINER_MAGIC + _HEADER.pack(FORMAT_VERSION, _FMT_CODES[config.fmt],
                                            _mode_byte(config), config.code_bits,
                                            config.chunk_size, int(streams.n_elements),
                                            int(streams.n_escapes))
    parts = [header, codebook_record_bytes(codebook)]
    parts.extend(data for _, data in streams.section_bytes())
    return b"".join(parts)


def encode_container(stream: RawTensorStream, config: CodecConfig) -> torch.Tensor:
    """Encode a device stream straight into an HBM-resident SPLZ container
    (a CUDA uint8 tensor, exactly the file's bytes)."""
    enc = encode(stream, config)
    if not enc.on_device:
        raise ConfigError("encode_container needs a CUDA stream (RawTensorStream on the GPU)")
    return _frame_streams(enc, config, enc.codebook)


def write_container(streams: EncodedStreams, config: CodecConfig,
                    codebook: ExponentCodebook, sink) -> int:
    data = container_to_bytes(streams, config, codebook)
    Path(sink).write_bytes(data)
    return len(data)


# ------------------------------------------------------------ parsing
_VALUE_PAD_MSG = "nonzero padding bits in escape-value stream"


def _unpack_values_np(raw: bytes, m: int, exp_bits: int) -> np.ndarray:
    """Dense little-endian exp_bits stream -> raw values (codec.py:248-257),
    rejecting nonzero pad bits like the reference (codec.py:255-256)."""
    if exp_bits == 8:
        return np.frombuffer(raw, dtype=np.uint8).copy()
    if not trailing_bits_zero(raw, m, exp_bits):
        raise CorruptionError(_VALUE_PAD_MSG)
    bits = np.unpackbits(np.frombuffer(raw, dtype=np.uint8), bitorder="little")
    bits = bits[:m * exp_bits].reshape(m, exp_bits)
    return (bits.astype(np.uint8) << np.arange(exp_bits, dtype=np.uint8)).sum(
        axis=1, dtype=np.uint32).astype(np.uint8)


def container_from_bytes(data) -> tuple[EncodedStreams, CodecConfig, ExponentCodebook]:
    """Parse an SPLZ container (container.py:225-296): ``bytes``-like host data
    gives reference-typed sections; a CUDA ``uint8`` tensor gives device
    sections sliced in HBM (only the header is read by the host)."""
    on_dev = is_device(data)
    if on_dev:
        buf = data.reshape(-1)
        if buf.dtype != torch.uint8:
            buf = buf.view(torch.uint8)
        total = buf.numel()
        head = buf[:min(total, 28 + 9 + 255)].cpu().numpy().tobytes()

        def fetch(lo, hi):
            if hi <= len(head):
                return head[lo:hi]
            return buf[lo:hi].cpu().numpy().tobytes()
    else:
        raw = data.numpy().tobytes() if isinstance(data, torch.Tensor) else bytes(data)
        total = len(raw)

        def fetch(lo, hi):
            return raw[lo:hi]
    cur = _Cursor(total, fetch)
    magic = cur.take(4, "header")
    if magic != CONTAINER_MAGIC:
        raise BadMagicError(f"bad container magic {magic!r}")
    version = cur.u8("header")
    if version != FORMAT_VERSION:
        raise UnsupportedVersionError(f"unsupported container version {version}")
    fmt_code = cur.u8("header")
    if fmt_code not in _FMT_FROM_CODE:
        raise ContainerError(f"unknown element format code {fmt_code}")
    fmt = _FMT_FROM_CODE[fmt_code]
    mode_code = cur.u8("header")
    if mode_code not in (_MODE_CHUNKED, _MODE_SENTINEL, _MODE_ABS32):
        raise ContainerError(f"unknown container mode code {mode_code}")
    code_bits = cur.u8("header")
    chunk_size = cur.u32("header")
    n = cur.u64("header")
    m = cur.u64("header")
    codebook = _parse_codebook_record(cur)
    try:
        config = CodecConfig(
            fmt=fmt, code_bits=code_bits,
            mode=CodebookMode.TOP15_SENTINEL if mode_code == _MODE_SENTINEL
            else CodebookMode.TOPK_EXPLICIT,
            chunk_size=chunk_size,
            position_mode=PositionMode.ABSOLUTE_32 if mode_code == _MODE_ABS32
            else PositionMode.CHUNK_RELATIVE,
            codebook=codebook)
    except ConfigError as exc:
        raise CorruptionError(f"inconsistent container header: {exc}") from exc
    if n < 1:
        raise CorruptionError("container declares zero elements")
    if m > n:
        raise CorruptionError("container declares more escapes than elements")

    spans = {}
    spans["chunk_counts"] = (cur.skip(4 * config.n_chunks(n), "chunk_counts"),
                             4 * config.n_chunks(n))
    spans["packed_codes"] = (cur.skip(packed_nbytes(n, code_bits), "packed_codes"),
                             packed_nbytes(n, code_bits))
    sm_len = config.sm_nbytes(n)
    spans["sign_mantissa"] = (cur.skip(sm_len, "sign_mantissa"), sm_len)
    pos_len = m * config.position_nbytes if not config.sentinel else 0
    spans["escape_positions"] = (cur.skip(pos_len, "escape_positions"), pos_len)
    val_len = packed_nbytes(m, fmt.exp_bits)
    spans["escape_values"] = (cur.skip(val_len, "escape_values"), val_len)
    if cur.offset != total:
        raise LengthMismatchError(f"{total - cur.offset} unexpected trailing bytes after the "
                                  "escape values")

    if on_dev:
        def sect(name, dtype=torch.uint8):
            lo, ln = spans[name]
            t = torch.empty(ln, dtype=torch.uint8, device=buf.device)
            if ln:
                t.copy_(buf[lo:lo + ln])       # realigned copy in HBM
            return t.view(dtype) if ln else torch.empty(0, dtype=dtype, device=buf.device)
        vals_packed = sect("escape_values")
        if fmt.exp_bits == 8:
            values = vals_packed
        elif m:
            values, pad_nonzero = unpack_bits_device(vals_packed, m, fmt.exp_bits)
            if pad_nonzero:
                raise CorruptionError(_VALUE_PAD_MSG)
        else:
            values = torch.empty(0, dtype=torch.uint8, device=buf.device)
        streams = EncodedStreams(
            n, m, sect("packed_codes"), sect("sign_mantissa"),
            sect("chunk_counts", torch.uint32),
            sect("escape_positions", config.position_torch_dtype), values, codebook,
            None if fmt.exp_bits == 8 else vals_packed)
    else:
        def sect_b(name):
            lo, ln = spans[name]
            return fetch(lo, lo + ln)
        pos_raw = sect_b("escape_positions")
        streams = EncodedStreams(
            n, m, sect_b("packed_codes"), sect_b("sign_mantissa"),
            np.frombuffer(sect_b("chunk_counts"), dtype="<u4"),
            np.frombuffer(pos_raw, dtype=config.position_np_dtype.newbyteorder("<"))
            if pos_len else np.zeros(0, dtype=config.position_np_dtype),
            _unpack_values_np(sect_b("escape_values"), m, fmt.exp_bits), codebook)
    return streams, config, codebook


def read_container(source) -> tuple[EncodedStreams, CodecConfig, ExponentCodebook]:
    return container_from_bytes(Path(source).read_bytes())


def decode_container(data) -> RawTensorStream:
    """``container_from_bytes`` + ``decode`` (the K3+K4 kernels)."""
    streams, config, codebook = container_from_bytes(data)
    return decode(streams, config, codebook)


# ------------------------------------------------------------ raw dumps
def raw_tensor_to_bytes(stream: RawTensorStream) -> bytes:
    """``SZRW | 1 | fmt | N u64 | words`` (container.py:305-309)."""
    words = stream.words
    arr = words.detach().cpu().numpy() if isinstance(words, torch.Tensor) else np.asarray(words)
    header = RAW_MAGIC + struct.pack("<BBQ", FORMAT_VERSION, _FMT_CODES[stream.fmt], arr.size)
    return header + arr.astype(stream.fmt.word_dtype.newbyteorder("<")).tobytes()


def raw_tensor_from_bytes(data: bytes) -> RawTensorStream:
    data = bytes(data)
    cur = _Cursor(len(data), lambda lo, hi: data[lo:hi])
    magic = cur.take(4, "header")
    if magic != RAW_MAGIC:
        raise BadMagicError(f"bad raw-tensor magic {magic!r}")
    version = cur.u8("header")
    if version != FORMAT_VERSION:
        raise UnsupportedVersionError(f"unsupported raw-tensor version {version}")
    fmt_code = cur.u8("header")
    if fmt_code not in _FMT_FROM_CODE:
        raise ContainerError(f"unknown element format code {fmt_code}")
    fmt = _FMT_FROM_CODE[fmt_code]
    n = cur.u64("header")
    payload = cur.take(n * fmt.word_nbytes, "payload")
    if cur.offset != len(data):
        raise LengthMismatchError(f"{len(data) - cur.offset} unexpected bytes after the payload")
    words = np.frombuffer(payload, dtype=fmt.word_dtype.newbyteorder("<"))
    return RawTensorStream(fmt, words.astype(fmt.word_dtype))


def write_raw_tensor(stream: RawTensorStream, sink) -> int:
    data = raw_tensor_to_bytes(stream)
    Path(sink).write_bytes(data)
    return len(data)


def read_raw_tensor(source) -> RawTensorStream:
    return raw_tensor_from_bytes(Path(source).read_bytes())

