"""Escape-dense streams (top-8 3-bit books put ~7% of real KV exponents
outside the book; the handoff tests use 7.89%; all-escape chunks exist in
the reference's own matrix): the encoder's staged-record path (K2a writers,
K2b moves) and the decoder's K3e scatter + bitmap staging, checked against
the CPU oracle section for section, bit for bit, and verdict for verdict on
corrupted streams (exception class and chunk, codec.py:404-536).  Every
case runs the decoder both ways (SZ_DEC_MARKED forces the path): the K3e
pre-pass (escape bitmap + tile counts, sentinel-style staging) and the
stagers' own walk over positions (the path realistic rates take)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import sz_oracle as O

pytestmark = pytest.mark.gpu

BOOKS = {0: (O.BF16_BOOK, O.BF16_ESC), 1: (O.E5M2_BOOK, O.E5M2_ESC),
         2: (O.E4M3_BOOK, O.E4M3_ESC)}
TILE = {0: 8192, 1: 16384, 2: 16384}   # decode tile (K4 / K3e)


def sz():
    import paper_2605_01708_b200 as m
    return m


def dense_case(fmt_id, n, rate, cb, seed):
    bk, esc = BOOKS[fmt_id]
    book_w = bk[:8] if cb == 3 else bk
    words = O.exact_stream(fmt_id, n, rate, seed, book_w, esc)
    return words, tuple(e for e, _ in book_w)


def config(fmt_id, cb, chunk, book):
    m = sz()
    fmt = list(m.ElementFormat)[fmt_id]
    return fmt, m.CodecConfig(fmt, cb, chunk_size=chunk, codebook=m.ExponentCodebook(
        fmt, book, cb, m.CodebookMode.TOPK_EXPLICIT))


CASES = [  # fmt, chunk, rate, code bits, n
    (0, 1024, 0.0789, 4, 5 * 8192 + 333), (0, 1024, 0.0689, 3, 4 * 8192),
    (0, 64, 0.2, 4, 3 * 8192 + 17), (0, 256, 0.03, 3, 6 * 8192 + 1),
    (0, 8192, 0.5, 4, 2 * 8192 + 4095), (0, 4096, 0.009, 4, 8 * 8192 + 9),
    (0, 1000, 0.07, 4, 3 * 8192 + 5),          # chunk not dividing the tile
    (0, 48, 0.1, 3, 3 * 8192 + 100),           # chunk not a power of two, < a bitmap window word run
    (0, 16384, 0.07, 4, 5 * 8192),             # chunk larger than the decode tile
    (0, 65536, 0.07, 4, 3 * 65536 + 100),      # chunk spanning 4 K3e windows
    (1, 32, 0.1, 3, 2 * 16384 + 999),          # the smallest chunk K3e takes
    (1, 1024, 0.0789, 4, 3 * 16384 + 77), (1, 1024, 0.0689, 3, 4 * 16384),
    (1, 16384, 0.3, 4, 2 * 16384 + 1), (1, 128, 0.05, 3, 3 * 16384 + 3),
    (2, 1024, 0.07, 3, 3 * 16384 + 11), (2, 512, 1.0, 3, 16384 + 5),
    # 3-bit top-8 BF16 tiles past the encoder's staged-record capacity (K2c)
    (0, 1024, 0.16, 3, 4 * 16384 + 123),
]


@pytest.fixture(params=["0", "1"], ids=["stager", "k3e"])
def dec_path(request, monkeypatch):
    monkeypatch.setenv("SZ_DEC_MARKED", request.param)
    return request.param


@pytest.mark.parametrize("fmt_id,chunk,rate,cb,n", CASES)
def test_dense_roundtrip_matches_oracle(fmt_id, chunk, rate, cb, n, dec_path):
    m = sz()
    words, book = dense_case(fmt_id, n, rate, cb, 1000 + n % 97)
    fmt, cfg = config(fmt_id, cb, chunk, book)
    stream = m.RawTensorStream(fmt, torch.from_numpy(words).cuda())
    enc = m.encode(stream, cfg)
    ref = O.encode(words, O.Params(fmt_id, cb, False, chunk, False), book)
    assert enc.n_escapes == ref["m"]
    assert [b for _, b in enc.section_bytes()] == O.section_bytes(ref)
    dec = m.decode(enc, cfg, enc.codebook)
    assert torch.equal(dec.words, stream.words)
    # the engine path: M stays on the device (workspace sized for K3e by
    # ensure_capacity)
    from paper_2605_01708_b200.engine import DeviceCodec
    eng = DeviceCodec(cfg, enc.codebook, n)
    eng.ensure_capacity(stream.words)
    out = eng.decode()
    eng.check_status()
    assert torch.equal(out, stream.words)


def _mutations(sec, chunk, rng):
    """(name, mutated sections) on an escape-dense stream: positions,
    values and counts, at ordinals spread over the dense tiles."""
    m_ = int(sec["m"])
    pos, vals, counts = sec["escape_positions"], sec["escape_values"], sec["chunk_counts"]
    out = []
    for o in rng.choice(np.arange(1, m_), size=6, replace=False):
        o = int(o)
        p = pos.copy()
        p[o] = p[o - 1]                         # not strictly increasing (or chunk start)
        out.append((f"dup@{o}", dict(sec, escape_positions=p)))
        over = chunk if pos.dtype == np.uint16 else 255
        if over <= np.iinfo(pos.dtype).max:     # (a u16 position cannot reach chunk 65536)
            p = pos.copy()
            p[o] = over
            out.append((f"over@{o}", dict(sec, escape_positions=p)))
        v = vals.copy()
        v[o] = O.tables(sec["book"], sec["fmt"])[1][0]  # an in-book exponent
        out.append((f"inbook@{o}", dict(sec, escape_values=v,
                                        escape_values_packed=O.pack_le(v, O.FORMATS[sec["fmt"]][1]))))
    k = int(rng.integers(0, counts.size - 1))
    while counts[k] == 0:
        k += 1
    c = counts.copy()
    c[k] -= 1
    c[k + 1] += 1                               # an escape moved to the next chunk
    out.append((f"shift@{k}", dict(sec, chunk_counts=c)))
    p = pos.copy()
    p[-1] = chunk - 1                           # last escape past the stream end (ragged tail)
    out.append(("tail", dict(sec, escape_positions=p)))
    return out


@pytest.mark.parametrize("fmt_id,chunk,rate,cb,n", [
    (0, 1024, 0.0789, 4, 5 * 8192 + 333), (0, 256, 0.05, 3, 3 * 8192 + 7),
    (1, 1024, 0.0689, 3, 3 * 16384 + 77),
    # chunks longer than the decode tile: each tile checks only its share
    # of the chunk's ordinals (the split must still see every corruption)
    (0, 65536, 0.0016, 4, 4 * 65536 + 100), (1, 65536, 0.0123, 4, 3 * 65536 + 77),
    (0, 32768, 0.0123, 3, 2 * 32768 + 9), (1, 65536, 0.0016, 4, 2 * 65536),
])
def test_dense_corruption_verdicts_match_oracle(fmt_id, chunk, rate, cb, n, dec_path):
    m = sz()
    words, book = dense_case(fmt_id, n, rate, cb, 77 + n % 31)
    fmt, cfg = config(fmt_id, cb, chunk, book)
    p = O.Params(fmt_id, cb, False, chunk, False)
    ref = O.encode(words, p, book)
    ref = dict(ref, book=book, fmt=fmt_id)
    rng = np.random.default_rng(n)
    checked = 0
    for name, sec in _mutations(ref, chunk, rng):
        try:
            O.decode(sec, p, book)
            want = None
        except O.OracleCorruption as exc:
            want = exc.chunk
        cb_book = cfg.codebook
        streams = m.EncodedStreams(
            n, int(sec["m"]), sec["packed_codes"], sec["sign_mantissa"], sec["chunk_counts"],
            sec["escape_positions"], sec["escape_values"], cb_book)
        dev = m.EncodedStreams(
            n, int(sec["m"]), torch.from_numpy(np.frombuffer(sec["packed_codes"], np.uint8).copy()).cuda(),
            torch.from_numpy(np.frombuffer(sec["sign_mantissa"], np.uint8).copy()).cuda(),
            torch.from_numpy(sec["chunk_counts"].astype(np.uint32)).cuda(),
            torch.from_numpy(np.ascontiguousarray(sec["escape_positions"])).cuda(),
            torch.from_numpy(np.ascontiguousarray(sec["escape_values"])).cuda(), cb_book)
        for s_ in (streams, dev):
            if want is None:
                out = m.decode(s_, cfg, cb_book).words
                out = out.cpu().numpy() if isinstance(out, torch.Tensor) else out
                assert np.array_equal(out, O.decode(sec, p, book)), name
            else:
                with pytest.raises(m.CorruptionError) as exc:
                    m.decode(s_, cfg, cb_book)
                assert exc.value.chunk == want, name
        checked += want is not None
    assert checked >= 10


@pytest.mark.parametrize("fmt_id", [1, 2])
@pytest.mark.parametrize("voff,poff", [(0, 0), (1, 0), (0, 1), (3, 2), (9, 3), (15, 1)])
def test_packed_values_unaligned_buffers(fmt_id, voff, poff):
    """K6 (escape values -> 5 / 4-bit stream) with the raw-value and packed
    outputs at arbitrary byte offsets (the C ABI takes any pointers): its
    16-byte-load and word-store fast paths fall back to bytes and the
    stream is still the reference's _pack_values (codec.py:241-266); the
    cases' M are not multiples of 32, so the ragged last unit is covered."""
    m = sz()
    from paper_2605_01708_b200 import _native as N
    from paper_2605_01708_b200.codec import (EncodeBuffers, _config_params, launch_encode,
                                             packed_nbytes)
    n = 3 * 16384 + 77 + 131 * voff + 29 * poff
    words, book = dense_case(fmt_id, n, 0.0789, 4, 7 + voff + 16 * poff)
    fmt, cfg = config(fmt_id, 4, 1024, book)
    ref = O.encode(words, O.Params(fmt_id, 4, False, 1024, False), book)
    mm = int(ref["m"])
    assert mm % 32
    w = fmt.exp_bits
    bufs = EncodeBuffers(n, cfg, mm, torch.device("cuda"))
    vals_big = torch.zeros(mm + 64, dtype=torch.uint8, device="cuda")
    pack_big = torch.zeros(packed_nbytes(mm, w) + 64, dtype=torch.uint8, device="cuda")
    bufs.values = vals_big[voff:voff + mm]
    bufs.values_packed = pack_big[poff:poff + packed_nbytes(mm, w)]
    launch_encode(torch.from_numpy(words).cuda(), _config_params(cfg, cfg.codebook), bufs)
    torch.cuda.synchronize()
    assert int(bufs.m.item()) == mm
    assert np.array_equal(bufs.values.cpu().numpy(), ref["escape_values"])
    got = bufs.values_packed.cpu().numpy()
    assert got.tobytes() == O.pack_le(ref["escape_values"], w)
    # nothing written outside the packed section
    assert not pack_big[:poff].any() and not pack_big[poff + packed_nbytes(mm, w):].any()


@pytest.mark.parametrize("off", [0, 1, 5, 8, 15])
@pytest.mark.parametrize("fmt_id,cb", [(0, 3), (0, 4)])
def test_k3e_values_at_any_alignment(fmt_id, cb, off, dec_path):
    """The K3e stagers copy a tile's value run with 16-byte loads staged at
    the run's own address mod 16 (vshift); a values section at any byte
    offset (e.g. sliced out of a container in HBM) decodes bit-exactly on
    both decoder paths."""
    m = sz()
    from paper_2605_01708_b200.codec import EncodedStreams
    n = 5 * 8192 + 333
    words, book = dense_case(fmt_id, n, 0.0689, cb, 31 + off)
    fmt, cfg = config(fmt_id, cb, 1024, book)
    stream = m.RawTensorStream(fmt, torch.from_numpy(words).cuda())
    enc = m.encode(stream, cfg)
    big = torch.zeros(enc.n_escapes + 32, dtype=torch.uint8, device="cuda")
    big[off:off + enc.n_escapes] = enc.escape_values
    moved = EncodedStreams(enc.n_elements, enc.n_escapes, enc.packed_codes, enc.sign_mantissa,
                           enc.chunk_counts, enc.escape_positions,
                           big[off:off + enc.n_escapes], enc.codebook, enc.values_packed)
    dec = m.decode(moved, cfg, enc.codebook)
    assert torch.equal(dec.words, stream.words)
