"""Lossless encode/decode on the B200 — drop-in for the reference ``codec.py``.

Same public names, signatures, section layout and exceptions as the
reference; the work runs in the sm_100a kernels of ``libsz_b200.so``:

* ``encode`` / ``encode_quad`` -> K2 (fused dense transform + ordered escape
  compaction), plus K6 for the FP8 5/4-bit escape-value stream;
* ``decode`` -> K3 (chunk offsets) + K4 (LUT unpack, merge, in-tile escape
  overwrite, corruption checks);
* ``compare_streams`` -> K7.

Host inputs (numpy / bytes) give host outputs with the reference's exact
types; CUDA-tensor inputs keep every section on the device
(``EncodedStreams.section_bytes()`` materialises host bytes on demand).
There is no CPU fallback: without the library or a GPU the calls raise
:class:`~paper_2605_01708_b200.errors.NativeError`.
"""

from __future__ import annotations

import functools
from dataclasses import dataclass, field
from typing import Any, Iterator

import numpy as np
import torch

from . import _native as N
from .calibration import (CodebookMode, ExponentCodebook, build_histogram_device,
                          CalibrationStats, select_codebook)
from .errors import ConfigError, CorruptionError, EmptyInputError, NativeError
from .formats import (ElementFormat, RawTensorStream, is_device, pack_bits_device,
                      packed_nbytes, to_device, to_numpy, trailing_bits_zero,
                      unpack_bits_device)

__all__ = [
    "PositionMode", "CodecConfig", "EscapeChunk", "EncodedStreams", "RoundtripReport",
    "resolve_codebook", "encode", "encode_quad", "decode", "compressed_payload_bytes",
    "compression_ratio", "verify_roundtrip", "compare_streams", "kernel_params",
    "DUMMY_CODE", "CHUNK_COUNT_NBYTES",
]

DUMMY_CODE = 0          # explicit-mode placeholder code (codec.py:67)
CHUNK_COUNT_NBYTES = 4  # per-chunk counts are u32 (codec.py:68)


class PositionMode:
    CHUNK_RELATIVE = "chunk"
    ABSOLUTE_32 = "abs32"
    _ALL = (CHUNK_RELATIVE, ABSOLUTE_32)

    @classmethod
    def validate(cls, value: str) -> str:
        if value not in cls._ALL:
            raise ConfigError(f"unknown position mode {value!r}")
        return value


@dataclass(frozen=True)
class CodecConfig:
    """Everything that fixes the compressed representation (codec.py:86-135).
    ``codebook=None`` selects dynamic calibration on every encode."""

    fmt: ElementFormat
    code_bits: int = 4
    mode: CodebookMode = CodebookMode.TOPK_EXPLICIT
    chunk_size: int = 1024
    position_mode: str = PositionMode.CHUNK_RELATIVE
    codebook: ExponentCodebook | None = None

    def __post_init__(self):
        if self.code_bits not in (3, 4):
            raise ConfigError(f"code_bits must be 3 or 4, got {self.code_bits}")
        PositionMode.validate(self.position_mode)
        if self.chunk_size < 1:
            raise ConfigError(f"chunk_size must be >= 1, got {self.chunk_size}")
        if self.position_mode == PositionMode.CHUNK_RELATIVE and self.chunk_size > 65536:
            raise ConfigError("chunk-relative positions require chunk_size <= 65536")
        if self.codebook is not None:
            if self.codebook.fmt is not self.fmt:
                raise ConfigError("codebook format does not match codec format")
            if self.codebook.code_bits != self.code_bits:
                raise ConfigError("codebook code width does not match codec")
            if self.codebook.mode is not self.mode:
                raise ConfigError("codebook mode does not match codec mode")

    @property
    def position_nbytes(self) -> int:
        if self.position_mode == PositionMode.ABSOLUTE_32:
            return 4
        return 1 if self.chunk_size <= 256 else 2

    @property
    def chunked(self) -> bool:
        return (self.mode is CodebookMode.TOPK_EXPLICIT
                and self.position_mode == PositionMode.CHUNK_RELATIVE)

    @property
    def sentinel(self) -> bool:
        return self.mode is CodebookMode.TOP15_SENTINEL

    @property
    def abs32(self) -> bool:
        return not self.sentinel and self.position_mode == PositionMode.ABSOLUTE_32

    def n_chunks(self, n_elements: int) -> int:
        return -(-n_elements // self.chunk_size) if self.chunked else 0

    def sm_nbytes(self, n: int) -> int:
        return n if self.fmt.sm_bits == 8 else packed_nbytes(n, self.fmt.sm_bits)

    @property
    def position_np_dtype(self) -> np.dtype:
        return np.dtype({1: np.uint8, 2: np.uint16, 4: np.uint32}[self.position_nbytes])

    @property
    def position_torch_dtype(self) -> torch.dtype:
        return {1: torch.uint8, 2: torch.uint16, 4: torch.uint32}[self.position_nbytes]


@functools.lru_cache(maxsize=256)
def _params_cached(fmt: ElementFormat, code_bits: int, mode: CodebookMode, chunk: int,
                   abs32: bool, codebook: ExponentCodebook) -> N.SzParams:
    p = N.SzParams()
    p.fmt = fmt.code
    p.code_bits = code_bits
    p.sentinel = int(mode is CodebookMode.TOP15_SENTINEL)
    p.abs32 = int(abs32 and mode is not CodebookMode.TOP15_SENTINEL)
    p.chunk_size = chunk
    p.n_entries = len(codebook.entries)
    lut = codebook.marked_lut()
    for i in range(256):
        p.enc_lut[i] = int(lut[i])
    for c, e in enumerate(codebook.entries):
        p.dec_lut[c] = e
    return p


def kernel_params(fmt, code_bits, mode, chunk, abs32, codebook) -> N.SzParams:
    """sz_params for the C ABI (cached per codebook and layout)."""
    return _params_cached(fmt, code_bits, mode, int(chunk), bool(abs32), codebook)


def _config_params(config: CodecConfig, codebook: ExponentCodebook) -> N.SzParams:
    return kernel_params(config.fmt, config.code_bits, config.mode, config.chunk_size,
                         config.abs32, codebook)


@dataclass(frozen=True)
class EscapeChunk:
    index: int
    positions: Any
    values: Any

    @property
    def count(self) -> int:
        return int(len(self.positions))


def _nbytes(x) -> int:
    if isinstance(x, torch.Tensor):
        return x.numel() * x.element_size()
    if isinstance(x, np.ndarray):
        return x.nbytes
    return len(x)


def _as_bytes(x, np_dtype=None) -> bytes:
    if isinstance(x, (bytes, bytearray)):
        return bytes(x)
    arr = to_numpy(x)
    if np_dtype is not None:
        arr = arr.astype(np.dtype(np_dtype).newbyteorder("<"), copy=False)
    return np.ascontiguousarray(arr).tobytes()


@dataclass
class EncodedStreams:
    """Compressed sections of one stream (codec.py:151-188).

    Fields are bytes/numpy (host encode) or CUDA tensors (device encode).
    ``escape_values`` always holds raw exponent bytes; FP8 formats serialise
    them as a dense little-endian ``exp_bits`` stream.
    """

    n_elements: int
    n_escapes: int
    packed_codes: Any
    sign_mantissa: Any
    chunk_counts: Any
    escape_positions: Any
    escape_values: Any
    codebook: ExponentCodebook = field(repr=False)
    values_packed: Any = field(default=None, repr=False, compare=False)

    @property
    def on_device(self) -> bool:
        return is_device(self.packed_codes)

    def escape_chunks(self) -> Iterator[EscapeChunk]:
        counts = to_numpy(self.chunk_counts)
        off = 0
        for k, c in enumerate(counts):
            c = int(c)
            yield EscapeChunk(k, self.escape_positions[off:off + c], self.escape_values[off:off + c])
            off += c

    def _values_section(self) -> bytes:
        fmt = self.codebook.fmt
        if fmt.exp_bits == 8:
            return _as_bytes(self.escape_values, np.uint8)
        if self.values_packed is not None:
            return _as_bytes(self.values_packed)
        if self.n_escapes == 0:
            return b""
        vals = to_device(self.escape_values, torch.uint8, align=16)
        return pack_bits_device(vals, fmt.exp_bits).cpu().numpy().tobytes()

    def section_bytes(self) -> list:
        return [
            ("chunk_counts", _as_bytes(self.chunk_counts, np.uint32)),
            ("packed_codes", _as_bytes(self.packed_codes)),
            ("sign_mantissa", _as_bytes(self.sign_mantissa)),
            ("escape_positions", _as_bytes(self.escape_positions)),
            ("escape_values", self._values_section()),
        ]

    @property
    def payload_nbytes(self) -> int:
        """Serialized size, from section lengths (no device->host copy)."""
        m = int(self.n_escapes)
        return (4 * len(self.chunk_counts) + _nbytes(self.packed_codes)
                + _nbytes(self.sign_mantissa) + _nbytes(self.escape_positions)
                + packed_nbytes(m, self.codebook.fmt.exp_bits))

    def to_host(self) -> "EncodedStreams":
        """Reference-typed copy (bytes planes, numpy arrays) of tensor sections."""
        if not isinstance(self.packed_codes, torch.Tensor):
            return self
        pos = to_numpy(self.escape_positions)
        return EncodedStreams(
            self.n_elements, self.n_escapes, _as_bytes(self.packed_codes),
            _as_bytes(self.sign_mantissa), to_numpy(self.chunk_counts).astype(np.uint32),
            pos, to_numpy(self.escape_values).astype(np.uint8), self.codebook,
            None if self.values_packed is None else _as_bytes(self.values_packed))


@dataclass(frozen=True)
class RoundtripReport:
    ok: bool
    n: int
    mismatch_count: int
    first_mismatch_index: int | None


def _check_stream(stream: RawTensorStream, config: CodecConfig) -> None:
    if stream.fmt is not config.fmt:
        raise ConfigError(f"stream format {stream.fmt.cli_name} does not match codec "
                          f"format {config.fmt.cli_name}")
    if stream.n_elements == 0:
        raise EmptyInputError("cannot encode an empty stream")
    if config.position_mode == PositionMode.ABSOLUTE_32 and stream.n_elements > 1 << 32:
        raise ConfigError("absolute 32-bit positions cap streams at 2^32 elements")


def _dynamic_codebook(words: torch.Tensor, config: CodecConfig) -> ExponentCodebook:
    counts = build_histogram_device(words, config.fmt).cpu().numpy()
    stats = CalibrationStats(config.fmt, counts, int(words.numel()))
    return select_codebook(stats, config.code_bits, config.mode)


def resolve_codebook(stream: RawTensorStream, config: CodecConfig) -> ExponentCodebook:
    """Pinned codebook, or one calibrated on the input (GPU histogram)."""
    if config.codebook is not None:
        return config.codebook
    return _dynamic_codebook(stream.device_words(), config)


# --------------------------------------------------------------- encode
class EncodeBuffers:
    """Device outputs of one encode call (allocated by the caller side)."""

    def __init__(self, n: int, config: CodecConfig, capacity: int, dev: torch.device):
        fmt = config.fmt
        self.n, self.capacity = n, capacity
        self.codes = torch.empty(packed_nbytes(n, config.code_bits), dtype=torch.uint8, device=dev)
        self.sm = torch.empty(config.sm_nbytes(n), dtype=torch.uint8, device=dev)
        self.counts = torch.empty(config.n_chunks(n), dtype=torch.uint32, device=dev)
        self.positions = (torch.empty(capacity, dtype=config.position_torch_dtype, device=dev)
                          if not config.sentinel else None)
        self.values = torch.empty(capacity, dtype=torch.uint8, device=dev)
        self.values_packed = (torch.empty(packed_nbytes(capacity, fmt.exp_bits),
                                          dtype=torch.uint8, device=dev)
                              if fmt.exp_bits != 8 else None)
        self.m = torch.empty(1, dtype=torch.int64, device=dev)

    def struct(self) -> N.SzEncoded:
        s = N.SzEncoded()
        s.d_codes = N.ptr(self.codes)
        s.d_sm = N.ptr(self.sm)
        s.d_counts = N.ptr(self.counts) if self.counts.numel() else None
        s.d_positions = N.ptr(self.positions)
        s.d_values = N.ptr(self.values)
        s.d_values_packed = N.ptr(self.values_packed)
        s.d_n_escapes = N.ptr(self.m)
        s.escape_capacity = self.capacity
        s.d_escape_base = None
        return s


def default_capacity(n: int) -> int:
    """Escape capacity before the overflow-retry protocol kicks in: 1/32 of
    the elements (3.1% escapes; realistic KV is 0.16-1.2%)."""
    return min(n, max(4096, n // 32))


def launch_encode(words: torch.Tensor, params: N.SzParams, bufs: EncodeBuffers,
                  workspace: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Enqueue K2 (+K6) on ``stream``; no host synchronisation.  Returns the
    workspace so callers can reuse it."""
    lib = N.load_library()
    n = words.numel()
    need = lib.sz_encode_workspace_bytes(n, params)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=words.device)
    out = bufs.struct()
    N.check(lib.sz_encode(N.ptr(words), n, params, out, N.ptr(workspace), workspace.numel(),
                          N.stream_handle(stream)), "encode")
    return workspace


def encode(stream: RawTensorStream, config: CodecConfig, *,
           capacity: int | None = None) -> EncodedStreams:
    """Compress a stream; :func:`decode` inverts it bit-exactly (codec.py:299-321)."""
    _check_stream(stream, config)
    if not stream.on_device and config.codebook is not None:
        from . import hostpipe
        if hostpipe.pipelinable(config, stream.n_elements):
            # host-resident stream: piecewise H2D / K2 / D2H overlap
            words_h = hostpipe.host_tensor(stream.words, config.fmt.torch_dtype)
            enc = hostpipe.encode_host(words_h, config, config.codebook, capacity)
            return enc if isinstance(stream.words, torch.Tensor) else enc.to_host()
    words = stream.device_words()
    codebook = config.codebook or _dynamic_codebook(words, config)
    params = _config_params(config, codebook)
    n = words.numel()
    cap = min(n, capacity if capacity is not None else default_capacity(n))
    bufs = EncodeBuffers(n, config, cap, words.device)
    ws = launch_encode(words, params, bufs)
    m = int(bufs.m.cpu().numpy()[0])
    if m > cap:  # overflow protocol: re-run with the exact escape count
        bufs = EncodeBuffers(n, config, m, words.device)
        launch_encode(words, params, bufs, ws)
    positions = (bufs.positions[:m] if bufs.positions is not None
                 else torch.empty(0, dtype=torch.uint8, device=words.device))
    vp = (bufs.values_packed[:packed_nbytes(m, config.fmt.exp_bits)]
          if bufs.values_packed is not None else None)
    enc = EncodedStreams(n, m, bufs.codes, bufs.sm, bufs.counts, positions, bufs.values[:m],
                         codebook, vp)
    return enc if stream.on_device else enc.to_host()


def encode_quad(stream: RawTensorStream, config: CodecConfig) -> EncodedStreams:
    """The reference's Quad64 variant (codec.py:324-401) is a restatement of
    the dense stage with wide loads; K2 already is the wide-load kernel (32 B
    per thread), so both entry points share it and are byte-identical."""
    return encode(stream, config)


# --------------------------------------------------------------- decode
def _chunk_of(counts_np: np.ndarray | None, config: CodecConfig, ordinal: int):
    """codec.py:483-488."""
    if not config.chunked or counts_np is None or counts_np.size == 0:
        return None
    return int(np.searchsorted(np.cumsum(counts_np.astype(np.int64)), ordinal, side="right"))


def _status_view(raw: np.ndarray):
    st = N.SzDecodeStatus.from_buffer_copy(raw.tobytes())
    first = [None if v == 0 else (~v) & 0xFFFFFFFFFFFFFFFF for v in st.first_inv]
    return st, first


def _raise_values(first, streams, config):
    if first[N.DEC_VALUE_DOMAIN] is not None:
        raise CorruptionError("escape value outside the exponent domain")
    if first[N.DEC_VALUE_IN_BOOK] is not None:
        raise CorruptionError("escape value is inside the codebook",
                              chunk=_chunk_of(_counts_np(streams), config,
                                              first[N.DEC_VALUE_IN_BOOK]))


def _fetch_int(arr, i: int) -> int:
    """One element of a host or device array (error messages only)."""
    return int(to_numpy(arr[i:i + 1])[0])


def _code_at(packed, el: int, code_bits: int) -> int:
    """Dense code ``el`` of an LSB-first packed stream (formats.py:197-218);
    reads the <= 2 bytes holding it, host or device."""
    bit = el * code_bits
    lo = bit >> 3
    raw = to_numpy(packed[lo:lo + 2]).view(np.uint8)
    word = int(raw[0]) | (int(raw[1]) << 8 if raw.size > 1 else 0)
    return (word >> (bit & 7)) & ((1 << code_bits) - 1)


def _counts_np(streams) -> np.ndarray | None:
    c = streams.chunk_counts
    return None if c is None else to_numpy(c).astype(np.int64)


def _check_values_device(values: torch.Tensor, m: int, config: CodecConfig,
                         codebook: ExponentCodebook) -> list:
    lib = N.load_library()
    status = torch.empty(N.STATUS_BYTES, dtype=torch.uint8, device=values.device)
    N.check(lib.sz_check_values(N.ptr(values), m, _config_params(config, codebook),
                                N.ptr(status), N.stream_handle()), "check_values")
    return _status_view(status.cpu().numpy())[1]


def _raise_from_status(raw: np.ndarray, streams: EncodedStreams, config: CodecConfig,
                       codebook: ExponentCodebook, values_dev: torch.Tensor | None) -> None:
    st, first = _status_view(raw)
    flags = st.flags
    if flags & (1 << N.DEC_CAPACITY):
        raise NativeError("escape count M read on the device exceeds the decoder's escape "
                          "capacity: re-run the encode with a larger capacity "
                          "(DeviceCodec.ensure_capacity)")
    inconsistent = ((config.chunked and flags & (1 << N.DEC_COUNTS_TOTAL)) or
                    (config.sentinel and flags & (1 << N.DEC_SENTINEL_COUNT)))
    if inconsistent and values_dev is not None and streams.n_escapes:
        # The fused kernel checks escape values only for ordinals its tiles
        # visit; with inconsistent counts (or sentinel marks) some are never
        # visited, and the reference checks values first (codec.py:446-457)
        # — complete them.
        full = _check_values_device(values_dev, int(streams.n_escapes), config, codebook)
        first[N.DEC_VALUE_DOMAIN] = full[N.DEC_VALUE_DOMAIN]
        first[N.DEC_VALUE_IN_BOOK] = full[N.DEC_VALUE_IN_BOOK]
    if first[N.DEC_CODE_PAD] is not None:
        raise CorruptionError("nonzero padding bits in code stream")
    if first[N.DEC_SM_PAD] is not None:
        raise CorruptionError("nonzero padding bits in sign-mantissa stream")
    _raise_values(first, streams, config)
    if config.sentinel:
        if flags & (1 << N.DEC_SENTINEL_COUNT):
            raise CorruptionError(f"dense stream marks {st.marks_total} escapes, header "
                                  f"declares {streams.n_escapes}")
    elif config.abs32:
        if first[N.DEC_ABS_PAST_END] is not None:
            raise CorruptionError("absolute escape position beyond the stream")
        if first[N.DEC_ABS_NOT_INC] is not None:
            raise CorruptionError("absolute escape positions not strictly increasing")
    else:
        if flags & (1 << N.DEC_COUNTS_TOTAL):
            raise CorruptionError("chunk escape counts do not add up to the header total")
        counts = _counts_np(streams)
        o = first[N.DEC_POS_OVER_CHUNK]
        if o is not None:
            pos = _fetch_int(streams.escape_positions, o)
            raise CorruptionError(f"escape position {pos} exceeds the chunk size",
                                  chunk=_chunk_of(counts, config, o))
        for chk, msg in ((N.DEC_POS_PAST_END, "escape position beyond the end of the stream"),
                         (N.DEC_POS_NOT_INC, "escape positions not strictly increasing")):
            if first[chk] is not None:
                raise CorruptionError(msg, chunk=_chunk_of(counts, config, first[chk]))
    if first[N.DEC_CODE_RANGE] is not None:
        el = first[N.DEC_CODE_RANGE]
        code = _code_at(streams.packed_codes, el, config.code_bits)
        raise CorruptionError(f"dense code {code} at element {el} exceeds the "
                              f"{len(codebook.entries)}-entry codebook")
    if not config.sentinel and first[N.DEC_NONDUMMY] is not None:
        el = first[N.DEC_NONDUMMY]
        raise CorruptionError("escaped element carries a non-dummy dense code",
                              chunk=(el // config.chunk_size) if config.chunked else None)


def _pending_length_error(streams, config, n, m):
    """First failing host length check among those the reference performs
    after the device-side pad/value checks (codec.py:444-514)."""
    fmt = config.fmt
    sm_len = _nbytes(streams.sign_mantissa)
    if sm_len != config.sm_nbytes(n):
        return 5, f"sign-mantissa stream is {sm_len} bytes, expected {config.sm_nbytes(n)}"
    if len(streams.escape_values) != m:
        return 6, f"{len(streams.escape_values)} escape values for {m} declared escapes"
    if not config.sentinel:
        if len(streams.escape_positions) != m:
            return 8, f"{len(streams.escape_positions)} escape positions for {m} declared escapes"
        if config.chunked and len(streams.chunk_counts) != config.n_chunks(n):
            return 9, f"{len(streams.chunk_counts)} chunk counts, expected {config.n_chunks(n)}"
    return None


def check_section_lengths(streams: EncodedStreams, config: CodecConfig,
                          codebook: ExponentCodebook) -> None:
    """The host-side checks ``decode`` performs before launching
    (codec.py:431-514): N >= 1, M <= N and every section length, raising
    ``CorruptionError`` in the reference's priority order (a pad bit or an
    escape value the reference checks before a failing length still wins).
    Every entry point that launches the decode kernels on caller sections
    calls this first, so the kernels never read past a short section."""
    fmt = config.fmt
    n, m = int(streams.n_elements), int(streams.n_escapes)
    if n < 1:
        raise CorruptionError("container declares zero elements")
    if m > n:
        raise CorruptionError(f"{m} escapes exceed {n} elements")
    clen = _nbytes(streams.packed_codes)
    if clen != packed_nbytes(n, config.code_bits):
        raise CorruptionError(f"code stream is {clen} bytes, expected "
                              f"{packed_nbytes(n, config.code_bits)}")
    pending = _pending_length_error(streams, config, n, m)
    if pending is not None:
        prio, msg = pending
        # Checks the reference performs before this one still take precedence.
        if not trailing_bits_zero(streams.packed_codes, n, config.code_bits):
            raise CorruptionError("nonzero padding bits in code stream")
        if prio >= 6 and fmt.sm_bits != 8 and \
                not trailing_bits_zero(streams.sign_mantissa, n, fmt.sm_bits):
            raise CorruptionError("nonzero padding bits in sign-mantissa stream")
        if prio >= 8 and m:
            lib = N.load_library()
            vals = to_device(streams.escape_values, torch.uint8, align=16)
            status = torch.empty(N.STATUS_BYTES, dtype=torch.uint8, device=vals.device)
            N.check(lib.sz_check_values(N.ptr(vals), m, _config_params(config, codebook),
                                        N.ptr(status), N.stream_handle()), "check_values")
            _, first = _status_view(status.cpu().numpy())
            _raise_values(first, streams, config)
        raise CorruptionError(msg)


def decode(streams: EncodedStreams, config: CodecConfig,
           codebook: ExponentCodebook) -> RawTensorStream:
    """Reconstruct the original words, validating every section
    (codec.py:421-536); raises CorruptionError like the reference."""
    fmt = config.fmt
    n, m = int(streams.n_elements), int(streams.n_escapes)
    check_section_lengths(streams, config, codebook)

    if not is_device(streams.packed_codes):
        from . import hostpipe
        if hostpipe.pipelinable(config, n):
            counts_np = to_numpy(streams.chunk_counts)
            if int(counts_np.sum(dtype=np.int64)) == m:
                out_h = hostpipe.decode_host(streams, config, codebook, counts_np)
                if out_h is not None:
                    keep_torch = isinstance(streams.packed_codes, torch.Tensor)
                    return RawTensorStream(fmt, out_h if keep_torch else out_h.numpy())
            # inconsistent or corrupt: the monolithic path below raises exactly
    lib = N.load_library()
    codes = to_device(streams.packed_codes, torch.uint8, align=16)
    sm = to_device(streams.sign_mantissa, torch.uint8, align=16)
    dev = codes.device
    counts = (to_device(streams.chunk_counts, torch.uint32, align=16) if config.chunked else None)
    positions = (to_device(streams.escape_positions, config.position_torch_dtype, align=16)
                 if (not config.sentinel and m) else None)
    values = to_device(streams.escape_values, torch.uint8, align=16) if m else None
    out = torch.empty(n, dtype=fmt.torch_dtype, device=dev)
    status = torch.empty(N.STATUS_BYTES, dtype=torch.uint8, device=dev)
    params = _config_params(config, codebook)
    ws = torch.empty(lib.sz_decode_workspace_bytes(n, m, params), dtype=torch.uint8, device=dev)
    src = N.SzEncodedIn()
    src.d_codes, src.d_sm = N.ptr(codes), N.ptr(sm)
    src.d_counts = N.ptr(counts) if counts is not None and counts.numel() else None
    src.d_positions, src.d_values = N.ptr(positions), N.ptr(values)
    src.n_elements, src.n_escapes = n, m
    src.n_counts = counts.numel() if counts is not None else 0
    src.d_n_escapes = None
    N.check(lib.sz_decode(src, params, N.ptr(out), N.ptr(status), N.ptr(ws), ws.numel(),
                          N.stream_handle()), "decode")
    raw = status.cpu().numpy()
    _raise_from_status(raw, streams, config, codebook, values)
    if streams.on_device or is_device(streams.packed_codes):
        return RawTensorStream(fmt, out)
    return RawTensorStream(fmt, out.cpu().numpy())


# --------------------------------------------------------------- sizes
def compressed_payload_bytes(n: int, m: int, config: CodecConfig) -> int:
    """Exact serialized payload size, header excluded (codec.py:539-550)."""
    if m > n:
        raise ConfigError(f"escape count {m} exceeds element count {n}")
    size = packed_nbytes(n, config.code_bits) + config.sm_nbytes(n)
    size += CHUNK_COUNT_NBYTES * config.n_chunks(n)
    if config.mode is CodebookMode.TOPK_EXPLICIT:
        size += m * config.position_nbytes
    return size + packed_nbytes(m, config.fmt.exp_bits)


def compression_ratio(n: int, m: int, config: CodecConfig) -> float:
    """Closed-form ratio without chunk-count overhead (codec.py:553-569)."""
    if n <= 0:
        raise ConfigError(f"element count must be positive, got {n}")
    if m > n:
        raise ConfigError(f"escape count {m} exceeds element count {n}")
    fmt = config.fmt
    per_escape = fmt.exp_bits + (8 * config.position_nbytes
                                 if config.mode is CodebookMode.TOPK_EXPLICIT else 0)
    return n * fmt.word_bits / (n * (fmt.sm_bits + config.code_bits) + m * per_escape)


# --------------------------------------------------------------- compare
def compare_streams(expected: RawTensorStream, actual: RawTensorStream) -> RoundtripReport:
    """Bitwise comparison on the GPU (K7); never raises on mismatch."""
    if expected.fmt is not actual.fmt or expected.n_elements != actual.n_elements:
        return RoundtripReport(False, expected.n_elements, expected.n_elements, 0)
    n = expected.n_elements
    if n == 0:
        return RoundtripReport(True, 0, 0, None)
    lib = N.load_library()
    a = expected.device_words()
    b = actual.device_words()
    res = torch.empty(2, dtype=torch.int64, device=a.device)
    N.check(lib.sz_compare(N.ptr(a), N.ptr(b), n, expected.fmt.word_nbytes, N.ptr(res),
                           N.stream_handle()), "compare")
    cnt, first_inv = (int(v) for v in res.cpu().numpy().view(np.uint64))
    first = None if first_inv == 0 else (~first_inv) & 0xFFFFFFFFFFFFFFFF
    return RoundtripReport(cnt == 0, n, cnt, first)


def verify_roundtrip(stream: RawTensorStream, config: CodecConfig) -> RoundtripReport:
    enc = encode(stream, config)
    return compare_streams(stream, decode(enc, config, enc.codebook))
