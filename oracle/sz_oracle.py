"""CPU oracle for the SplitZip codec hot path — TEST INFRASTRUCTURE ONLY.

This module is a from-scratch numpy restatement of the reference algorithm
(``/root/reference/pkg/src/splitzip``).  It exists to *check* the CUDA
product path, and to time the reference algorithm on host cores for the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
may import it.  The product package (``paper_2605_01708_b200``) never
imports, calls or falls back to anything in ``oracle/``.

Parity is pinned: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by running the real reference package in the
build container (``tests/golden/make_golden.py``), plus the reference's own
known-answer tests restated in ``tests/test_oracle_known_answers.py``.

Element formats are identified by small ints, like the container's format
byte (``container.py:278-279``): 0 = BF16, 1 = FP8-E5M2, 2 = FP8-E4M3.
"""

from __future__ import annotations

import numpy as np

# (word_bits, exp_bits, sm_bits) — formats.py:49-51
FORMATS = {0: (16, 8, 8), 1: (8, 5, 3), 2: (8, 4, 4)}
ESCAPE_MARK = 0xFF          # calibration.py:40 (non-member marker)
DUMMY = 0                   # codec.py:67 (explicit-mode placeholder code)


class OracleCorruption(Exception):
    """Decode-side inconsistency; ``kind`` names the failed check, ``chunk``
    mirrors ``CorruptionError.chunk`` (errors.py:46-57)."""

    def __init__(self, kind: str, chunk=None):
        super().__init__(kind if chunk is None else f"{kind} (chunk {chunk})")
        self.kind = kind
        self.chunk = chunk


def word_dtype(fmt: int):
    return np.uint16 if FORMATS[fmt][0] == 16 else np.uint8


# ---------------------------------------------------------------- L0 bits
def split(words: np.ndarray, fmt: int):
    """(exponent, sign|mantissa) planes — formats.py:113-133."""
    wb, eb, sb = FORMATS[fmt]
    if wb == 16:
        # byte-plane form of the same bit moves (u8 arithmetic only): for
        # w = hi:lo, exp = hi[6:0]:lo[7], sm = hi[7]:lo[6:0]
        b = np.ascontiguousarray(words, dtype=np.uint16).view(np.uint8)
        lo, hi = b[0::2], b[1::2]
        exp = (hi << np.uint8(1)) | (lo >> np.uint8(7))
        sm = (hi & np.uint8(0x80)) | (lo & np.uint8(0x7F))
        return exp, sm
    w = np.asarray(words, dtype=np.uint8)
    mant_bits = sb - 1
    exp = (w >> np.uint8(mant_bits)) & np.uint8((1 << eb) - 1)
    sm = ((w >> np.uint8(wb - 1)) << np.uint8(mant_bits)) | (w & np.uint8((1 << mant_bits) - 1))
    return exp, sm


def join(exp: np.ndarray, sm: np.ndarray, fmt: int) -> np.ndarray:
    """Inverse of :func:`split` — formats.py:136-155."""
    wb, eb, sb = FORMATS[fmt]
    e = np.asarray(exp, dtype=np.uint8)
    a = np.asarray(sm, dtype=np.uint8)
    if wb == 16:
        out = np.empty(2 * e.size, dtype=np.uint8)
        out[1::2] = (a & np.uint8(0x80)) | (e >> np.uint8(1))
        out[0::2] = (e << np.uint8(7)) | (a & np.uint8(0x7F))
        return out.view(np.uint16)
    mant_bits = sb - 1
    return (((a >> np.uint8(mant_bits)) << np.uint8(wb - 1)) | (e << np.uint8(mant_bits))
            | (a & np.uint8((1 << mant_bits) - 1)))


def packed_len(count: int, width: int) -> int:
    return (count * width + 7) // 8


def pack_le(symbols, width: int) -> bytes:
    """Dense LSB-first bit stream: symbol i occupies bits [i*w, (i+1)*w).

    Covers the nibble layout (formats.py:180-183), the 3-bit stream
    (formats.py:184-189) and the 5-bit escape-value stream (codec.py:260-266);
    width 8 is the plain byte plane.
    """
    s = np.asarray(symbols, dtype=np.uint8).ravel()
    if s.size == 0:
        return b""
    if width == 8:
        return s.tobytes()
    if width == 4:  # element 2i in the low nibble (formats.py:180-183)
        if s.size & 1:
            s = np.append(s, np.uint8(0))
        return (s[0::2] | (s[1::2] << np.uint8(4))).tobytes()
    bit_planes = (s[:, None] >> np.arange(width, dtype=np.uint8)) & 1
    return np.packbits(bit_planes.reshape(-1), bitorder="little").tobytes()


def unpack_le(data: bytes, count: int, width: int) -> np.ndarray:
    buf = np.frombuffer(data, dtype=np.uint8)
    if count == 0:
        return np.zeros(0, dtype=np.uint8)
    if width == 8:
        return buf[:count].copy()
    if width == 4:
        out = np.empty(2 * buf.size, dtype=np.uint8)
        out[0::2] = buf & np.uint8(0x0F)
        out[1::2] = buf >> np.uint8(4)
        return out[:count]
    bits = np.unpackbits(buf, bitorder="little", count=count * width)
    weights = (1 << np.arange(width)).astype(np.uint16)
    return (bits.reshape(count, width).astype(np.uint16) @ weights).astype(np.uint8)


def pad_bits_clear(data: bytes, count: int, width: int) -> bool:
    """formats.py:223-231: every bit past count*width is zero."""
    used = count * width
    buf = np.frombuffer(data, dtype=np.uint8)
    if used >= buf.size * 8:
        return True
    first = used // 8
    if int(buf[first]) >> (used % 8):
        return False
    return not buf[first + 1:].any()


# ---------------------------------------------------------- calibration
def histogram(words: np.ndarray, fmt: int) -> np.ndarray:
    """int64 exponent counts — calibration.py:79-85."""
    exp, _ = split(words, fmt)
    return np.bincount(exp, minlength=1 << FORMATS[fmt][1]).astype(np.int64)


def ranked(counts: np.ndarray) -> np.ndarray:
    """Exponents by (count desc, value asc) — calibration.py:107-110."""
    counts = np.asarray(counts, dtype=np.int64)
    keys = sorted(range(counts.size), key=lambda e: (-int(counts[e]), e))
    return np.array(keys, dtype=np.int64)


def choose_book(counts: np.ndarray, code_bits: int, sentinel: bool) -> tuple:
    """Top-k non-zero exponents — calibration.py:173-188."""
    cap = (1 << code_bits) - (1 if sentinel else 0)
    order = [int(e) for e in ranked(counts) if counts[e] > 0]
    return tuple(order[:cap])


def tables(book, fmt: int):
    """(encode LUT with 0xFF for non-members, decode LUT, membership) —
    calibration.py:149-158."""
    bins = 1 << FORMATS[fmt][1]
    enc = np.full(bins, ESCAPE_MARK, dtype=np.uint8)
    member = np.zeros(bins, dtype=bool)
    for code, e in enumerate(book):
        enc[e] = code
        member[e] = True
    dec = np.array(book, dtype=np.uint8)
    return enc, dec, member


# ---------------------------------------------------------------- codec
class Params:
    """Mirror of ``CodecConfig`` (codec.py:86-135) as plain fields."""

    def __init__(self, fmt=0, code_bits=4, sentinel=False, chunk=1024, abs32=False):
        self.fmt, self.code_bits, self.sentinel = fmt, code_bits, sentinel
        self.chunk, self.abs32 = chunk, abs32

    @property
    def pos_bytes(self) -> int:          # codec.py:119-124
        if self.abs32:
            return 4
        return 1 if self.chunk <= 256 else 2

    @property
    def chunked(self) -> bool:           # codec.py:126-130
        return not self.sentinel and not self.abs32

    def n_chunks(self, n: int) -> int:   # codec.py:132-135
        return -(-n // self.chunk) if self.chunked else 0


def encode(words: np.ndarray, p: Params, book) -> dict:
    """All payload sections for one stream — codec.py:299-321 (and the
    byte-identical encode_quad, codec.py:324-401)."""
    words = np.ascontiguousarray(words, dtype=word_dtype(p.fmt)).ravel()
    n = words.size
    exp, sm = split(words, p.fmt)
    enc, _, member = tables(book, p.fmt)
    fill = ((1 << p.code_bits) - 1) if p.sentinel else DUMMY
    # one gather through the encode table; non-members carry ESCAPE_MARK
    # (codec.py:303-309: member -> code, else the escape/dummy code)
    codes = enc[exp]
    where = np.flatnonzero(codes == ESCAPE_MARK)
    codes[where] = fill
    values = exp[where]
    if p.sentinel:
        counts = np.zeros(0, dtype=np.uint32)
        pos = np.zeros(0, dtype=np.uint8)
    elif p.abs32:
        counts = np.zeros(0, dtype=np.uint32)
        pos = where.astype(np.uint32)
    else:
        counts = np.bincount(where // p.chunk, minlength=p.n_chunks(n)).astype(np.uint32)
        pos = (where % p.chunk).astype(np.uint8 if p.pos_bytes == 1 else np.uint16)
    eb = FORMATS[p.fmt][1]
    sb = FORMATS[p.fmt][2]
    return {
        "n": n,
        "m": int(where.size),
        "chunk_counts": counts,
        "packed_codes": pack_le(codes, p.code_bits),
        "sign_mantissa": pack_le(sm, sb),
        "escape_positions": pos,
        "escape_values": values,
        "escape_values_packed": pack_le(values, eb),
    }


def section_bytes(sec: dict) -> list:
    """Serialization order — codec.py:176-184."""
    return [
        sec["chunk_counts"].astype("<u4").tobytes(),
        sec["packed_codes"],
        sec["sign_mantissa"],
        np.ascontiguousarray(sec["escape_positions"]).tobytes(),
        sec["escape_values_packed"],
    ]


def codebook_record(book, p: Params) -> bytes:
    """SZCB record — container.py:128-137."""
    return (b"SZCB" + bytes([1, p.fmt, p.code_bits, 1 if p.sentinel else 0, len(book)])
            + bytes(book))


def container_bytes(sec: dict, p: Params, book) -> bytes:
    """SPLZ container image — container.py:201-215 (header layout
    container.py:7-36: magic, version, format, mode, code bits, chunk u32,
    N u64, M u64), then the codebook record and the sections."""
    import struct
    mode = 1 if p.sentinel else (2 if p.abs32 else 0)
    header = b"SPLZ" + struct.pack("<BBBBIQQ", 1, p.fmt, mode, p.code_bits, p.chunk,
                                   sec["n"], sec["m"])
    return header + codebook_record(book, p) + b"".join(section_bytes(sec))


def payload_bytes(n: int, m: int, p: Params) -> int:
    """codec.py:539-550."""
    wb, eb, sb = FORMATS[p.fmt]
    total = packed_len(n, p.code_bits) + packed_len(n, sb) + 4 * p.n_chunks(n)
    if not p.sentinel:
        total += m * p.pos_bytes
    return total + packed_len(m, eb)


def formula_ratio(n: int, m: int, p: Params) -> float:
    """codec.py:553-569."""
    wb, eb, sb = FORMATS[p.fmt]
    esc = m * (eb if p.sentinel else 8 * p.pos_bytes + eb)
    return n * wb / (n * (sb + p.code_bits) + esc)


def _chunk_of(counts: np.ndarray, ordinal: int, p: Params):
    """codec.py:483-488."""
    if not p.chunked or counts.size == 0:
        return None
    return int(np.searchsorted(np.cumsum(counts.astype(np.int64)), ordinal, side="right"))


def decode(sec: dict, p: Params, book) -> np.ndarray:
    """Reconstruct words, raising OracleCorruption in the reference's check
    order — codec.py:421-536."""
    n, m = int(sec["n"]), int(sec["m"])
    wb, eb, sb = FORMATS[p.fmt]
    if n < 1:
        raise OracleCorruption("zero elements")
    if m > n:
        raise OracleCorruption("more escapes than elements")
    pc = bytes(sec["packed_codes"])
    if len(pc) != packed_len(n, p.code_bits):
        raise OracleCorruption("code stream length")
    if not pad_bits_clear(pc, n, p.code_bits):
        raise OracleCorruption("code stream padding")
    codes = unpack_le(pc, n, p.code_bits)
    smb = bytes(sec["sign_mantissa"])
    if len(smb) != packed_len(n, sb):
        raise OracleCorruption("sign-mantissa length")
    if sb != 8 and not pad_bits_clear(smb, n, sb):
        raise OracleCorruption("sign-mantissa padding")
    sm = unpack_le(smb, n, sb)
    values = np.asarray(sec["escape_values"], dtype=np.uint8)
    if values.size != m:
        raise OracleCorruption("escape value count")
    _, dec, member = tables(book, p.fmt)
    counts = np.asarray(sec["chunk_counts"], dtype=np.uint32)
    if m:
        if int(values.max()) >= (1 << eb):
            raise OracleCorruption("escape value domain")
        inbook = member[values]
        if inbook.any():
            raise OracleCorruption("escape value in codebook",
                                   _chunk_of(counts, int(np.argmax(inbook)), p))
    lut = np.zeros(1 << p.code_bits, dtype=np.uint8)
    lut[:len(book)] = dec
    if p.sentinel:
        marks = codes == (1 << p.code_bits) - 1
        if int(marks.sum()) != m:
            raise OracleCorruption("sentinel count")
        bad = (codes >= len(book)) & ~marks
        if bad.any():
            raise OracleCorruption("dense code range")
        exp = lut[codes]
        exp[marks] = values
        return join(exp, sm, p.fmt)
    pos = np.asarray(sec["escape_positions"])
    if pos.size != m:
        raise OracleCorruption("escape position count")
    if p.abs32:
        idx = pos.astype(np.int64)
        if idx.size and int(idx.max()) >= n:
            raise OracleCorruption("absolute position beyond stream")
        if idx.size > 1 and (np.diff(idx) <= 0).any():
            raise OracleCorruption("absolute positions not increasing")
    else:
        if counts.size != p.n_chunks(n):
            raise OracleCorruption("chunk count length")
        if int(counts.astype(np.int64).sum()) != m:
            raise OracleCorruption("chunk counts total")
        p64 = pos.astype(np.int64)
        over = p64 >= p.chunk
        if over.any():
            raise OracleCorruption("position beyond chunk",
                                   _chunk_of(counts, int(np.argmax(over)), p))
        base = np.repeat(np.arange(counts.size, dtype=np.int64) * p.chunk,
                         counts.astype(np.int64))
        idx = base + p64
        if idx.size:
            past = idx >= n
            if past.any():
                raise OracleCorruption("position beyond stream",
                                       _chunk_of(counts, int(np.argmax(past)), p))
            nonmono = np.diff(idx) <= 0
            if nonmono.any():
                raise OracleCorruption("positions not increasing",
                                       _chunk_of(counts, int(np.argmax(nonmono)) + 1, p))
    if (codes >= len(book)).any():
        raise OracleCorruption("dense code range")
    exp = lut[codes]
    if idx.size:
        nd = codes[idx] != DUMMY
        if nd.any():
            raise OracleCorruption("non-dummy code at escape",
                                   _chunk_of(counts, int(np.argmax(nd)), p))
        exp[idx] = values
    return join(exp, sm, p.fmt)


# ------------------------------------------------------ synthetic inputs
def _largest_remainder(total: int, weights: np.ndarray) -> np.ndarray:
    """datagen.py:80-95 (ties to the lowest index)."""
    if total == 0:
        return np.zeros(len(weights), dtype=np.int64)
    ideal = weights / weights.sum() * total
    out = np.floor(ideal).astype(np.int64)
    short = total - int(out.sum())
    if short:
        frac = ideal - out
        order = sorted(range(len(weights)), key=lambda i: (-frac[i], i))
        out[order[:short]] += 1
    return out


def exact_stream(fmt: int, count: int, rate: float, seed: int, book_w, escapes):
    """Byte-identical restatement of ``generate(ExponentSpec(...,
    exact_counts=True))`` — datagen.py:98-126."""
    rng = np.random.default_rng(seed)
    bex = np.array([e for e, _ in book_w], dtype=np.int64)
    bw = np.array([w for _, w in book_w], dtype=np.float64)
    esc = np.array(escapes, dtype=np.int64)
    m = int(round(rate * count))
    parts = [np.repeat(bex, _largest_remainder(count - m, bw))]
    if esc.size:
        parts.append(np.repeat(esc, _largest_remainder(m, np.ones(esc.size))))
    exps = np.concatenate(parts)
    rng.shuffle(exps)
    sm = rng.integers(0, 1 << FORMATS[fmt][2], size=count, dtype=np.uint8)
    return join(exps.astype(np.uint8), sm, fmt)


def random_words(fmt: int, count: int, seed: int) -> np.ndarray:
    """Uniform bit patterns — the reference conftest's universal stress."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, 1 << FORMATS[fmt][0], size=count).astype(word_dtype(fmt))


# The reference's synthetic exponent profiles (conftest.py:19-26,
# test_acceptance.py:70-80).
BF16_BOOK = tuple((0x70 + i, 0.72 ** i) for i in range(16))
BF16_ESC = tuple(range(0x10, 0x18))
E5M2_BOOK = tuple((8 + i, 0.72 ** i) for i in range(16))
E5M2_ESC = (0, 1, 2, 3, 28, 29, 30, 31)
E4M3_BOOK = tuple((4 + i, 0.72 ** i) for i in range(8))
E4M3_ESC = (0, 1, 2, 3, 12, 13, 14, 15)
