"""GPU parity: the sm_100a kernels against the reference's golden vectors and
the CPU oracle, byte for byte (sections) and bit for bit (decoded words)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import sz_oracle as O
from sz_testutil import golden, golden_case_ids, oracle_params

pytestmark = pytest.mark.gpu

SECTIONS = ("chunk_counts", "packed_codes", "sign_mantissa", "escape_positions",
            "escape_values")


def sz():
    import paper_2605_01708_b200 as m
    return m


def make_config(case, pinned=True):
    m = sz()
    fmt = [m.ElementFormat.BF16, m.ElementFormat.FP8_E5M2, m.ElementFormat.FP8_E4M3][case["fmt"]]
    mode = m.CodebookMode.TOP15_SENTINEL if case["sentinel"] else m.CodebookMode.TOPK_EXPLICIT
    pos = m.PositionMode.ABSOLUTE_32 if case["abs32"] else m.PositionMode.CHUNK_RELATIVE
    book = (m.ExponentCodebook(fmt, tuple(case["book"]), case["code_bits"], mode)
            if pinned and case["pinned"] else None)
    return fmt, m.CodecConfig(fmt, case["code_bits"], mode, case["chunk"], pos, book)


@pytest.mark.parametrize("device_api", [False, True], ids=["host-api", "device-api"])
@pytest.mark.parametrize("cid", golden_case_ids())
def test_encode_decode_matches_reference(cid, device_api):
    m = sz()
    g = golden()
    case = g.case(cid)
    words = g.arr(cid, "words")
    fmt, cfg = make_config(case)
    src = torch.from_numpy(words.copy()).cuda() if device_api else words
    stream = m.RawTensorStream(fmt, src)
    enc = m.encode(stream, cfg)
    assert enc.n_escapes == case["m"]
    assert list(enc.codebook.entries) == case["book"]
    assert enc.on_device == device_api
    got = dict(enc.section_bytes())
    for name in SECTIONS:
        assert got[name] == g.arr(cid, name).tobytes(), name
    assert enc.payload_nbytes == case["payload_nbytes"]
    dec = m.decode(enc, cfg, enc.codebook)
    out = dec.words.cpu().numpy() if device_api else dec.words
    assert np.array_equal(out, words)
    quad = m.encode_quad(stream, cfg)
    assert dict(quad.section_bytes()) == got


@pytest.mark.parametrize("cid", golden_case_ids())
def test_decode_k3e_path_matches_reference(cid, monkeypatch):
    # every chunk-relative golden case (chunk >= 32) decoded through the
    # escape-dense pre-pass path (K3e bitmap + sentinel-style staging),
    # whatever its escape rate; other modes ignore the switch
    monkeypatch.setenv("SZ_DEC_MARKED", "1")
    m = sz()
    g = golden()
    case = g.case(cid)
    words = g.arr(cid, "words")
    fmt, cfg = make_config(case)
    enc = m.encode(m.RawTensorStream(fmt, torch.from_numpy(words.copy()).cuda()), cfg)
    dec = m.decode(enc, cfg, enc.codebook)
    assert np.array_equal(dec.words.cpu().numpy(), words)


@pytest.mark.parametrize("cid", golden_case_ids())
def test_histogram_matches_reference(cid):
    m = sz()
    g = golden()
    case = g.case(cid)
    fmt, _ = make_config(case)
    stats = m.build_histogram(m.RawTensorStream(fmt, g.arr(cid, "words")))
    assert np.array_equal(stats.counts, g.arr(cid, "hist"))
    assert m.entropy_bits(stats) == pytest.approx(case["entropy"], abs=1e-12)


@pytest.mark.parametrize("path", ["auto", "k3e"])
@pytest.mark.parametrize("verdict", golden().corruptions, ids=lambda v: v["id"])
def test_corruption_verdicts_match_reference(verdict, path, monkeypatch):
    if path == "k3e":
        monkeypatch.setenv("SZ_DEC_MARKED", "1")
    m = sz()
    g = golden()
    base, words = g.corruption_base(verdict)
    if base is None:
        fmt = m.ElementFormat.BF16
        book = m.select_codebook(m.build_histogram(m.RawTensorStream(fmt, words)), 4,
                                 m.CodebookMode.TOPK_EXPLICIT)
        cfg = m.CodecConfig(fmt, codebook=book)
    else:
        fmt = list(m.ElementFormat)[base["fmt"]]
        mode = m.CodebookMode.TOP15_SENTINEL if base["sentinel"] else m.CodebookMode.TOPK_EXPLICIT
        book = m.ExponentCodebook(fmt, tuple(base["book"]), base["code_bits"], mode)
        cfg = m.CodecConfig(fmt, base["code_bits"], mode, base["chunk"],
                            m.PositionMode.ABSOLUTE_32 if base["abs32"]
                            else m.PositionMode.CHUNK_RELATIVE, book)
    sec = g.corruption_sections(verdict)
    streams = m.EncodedStreams(
        sec["n"], sec["m"], sec["packed_codes"], sec["sign_mantissa"], sec["chunk_counts"],
        sec["escape_positions"], sec["escape_values"], book)
    if verdict["raised"] is None:
        assert np.array_equal(m.decode(streams, cfg, book).words, words)
        return
    with pytest.raises(m.CorruptionError) as exc:
        m.decode(streams, cfg, book)
    assert exc.value.chunk == verdict["chunk"]


@pytest.mark.parametrize("fmt_id", [0, 1, 2])
def test_split_reconstruct_exhaustive(fmt_id):
    m = sz()
    fmt = list(m.ElementFormat)[fmt_id]
    words = np.arange(1 << fmt.word_bits, dtype=fmt.word_dtype)
    e, a = m.split_fields(words, fmt)
    oe, oa = O.split(words, fmt_id)
    assert np.array_equal(e, oe) and np.array_equal(a, oa)
    assert np.array_equal(m.reconstruct(m.SplitFields(e, a), fmt), words)


@pytest.mark.parametrize("bits", [3, 4])
@pytest.mark.parametrize("n", [0, 1, 7, 8, 9, 1000, 4097])
def test_pack_unpack_codes(bits, n):
    m = sz()
    rng = np.random.default_rng(n * 10 + bits)
    codes = rng.integers(0, 1 << bits, size=n, dtype=np.uint8)
    packed = m.pack_codes(codes, bits)
    assert packed == O.pack_le(codes, bits)
    assert np.array_equal(m.unpack_codes(packed, n, bits), codes)
    with pytest.raises(m.CodeRangeError):
        m.pack_codes(np.array([1 << bits], dtype=np.uint8), bits)


def test_known_answers():
    m = sz()
    # test_formats.py / test_codec.py known answers
    assert m.pack_codes([1, 2], 4) == bytes([0x21])
    assert m.pack_codes([7] * 8, 3) == b"\xff\xff\xff"
    book = m.ExponentCodebook(m.ElementFormat.BF16, (0x7F,), 4, m.CodebookMode.TOPK_EXPLICIT)
    cfg = m.CodecConfig(m.ElementFormat.BF16, codebook=book)
    streams = m.EncodedStreams(2, 0, bytes([0]), bytes([0x00, 0x80]),
                               np.zeros(1, np.uint32), np.zeros(0, np.uint16),
                               np.zeros(0, np.uint8), book)
    assert m.decode(streams, cfg, book).words.tolist() == [0x3F80, 0xBF80]


def test_single_escape_location():
    # test_codec.py:84-101
    m = sz()
    words = O.exact_stream(0, 1024, 0.0, 6, O.BF16_BOOK, O.BF16_ESC)
    book_words = words.copy()
    words[700] = O.join(np.array([0x10]), np.array([0x55]), 0)[0]
    stream = m.RawTensorStream(m.ElementFormat.BF16, words)
    book = m.select_codebook(m.build_histogram(m.RawTensorStream(m.ElementFormat.BF16, book_words)),
                             4, m.CodebookMode.TOPK_EXPLICIT)
    cfg = m.CodecConfig(m.ElementFormat.BF16, codebook=book)
    enc = m.encode(stream, cfg)
    assert enc.n_escapes == 1 and enc.chunk_counts.tolist() == [1]
    assert enc.escape_positions.tolist() == [700] and enc.escape_values.tolist() == [0x10]
    assert enc.packed_codes[350] & 0x0F == 0
    assert np.array_equal(m.decode(enc, cfg, enc.codebook).words, words)
    chunks = list(enc.escape_chunks())
    assert chunks[0].count == 1 and chunks[0].index == 0


def test_zero_coverage_all_escape():
    m = sz()
    words = O.exact_stream(0, 4096, 0.0, 14, O.BF16_BOOK, O.BF16_ESC)
    book = m.ExponentCodebook(m.ElementFormat.BF16, (1, 2), 4, m.CodebookMode.TOPK_EXPLICIT)
    cfg = m.CodecConfig(m.ElementFormat.BF16, codebook=book)
    stream = m.RawTensorStream(m.ElementFormat.BF16, words)
    enc = m.encode(stream, cfg, capacity=16)  # forces the overflow-retry protocol
    assert enc.n_escapes == 4096
    assert np.array_equal(m.decode(enc, cfg, book).words, words)


def test_errors_and_empty():
    m = sz()
    with pytest.raises(m.EmptyInputError):
        m.encode(m.RawTensorStream(m.ElementFormat.BF16, np.zeros(0, np.uint16)),
                 m.CodecConfig(m.ElementFormat.BF16))
    with pytest.raises(m.ConfigError):
        m.encode(m.RawTensorStream(m.ElementFormat.FP8_E5M2, np.zeros(4, np.uint8)),
                 m.CodecConfig(m.ElementFormat.BF16))
    with pytest.raises(m.EmptyInputError):
        m.build_histogram(m.RawTensorStream(m.ElementFormat.BF16, np.zeros(0, np.uint16)))


@pytest.mark.parametrize("fmt_id,n,rate,chunk", [
    (0, 1 << 22, 0.0016, 1024), (0, (1 << 22) + 777, 0.0123, 256), (0, 3_000_001, 0.05, 4096),
    (1, 1 << 22, 0.0016, 1024), (1, (1 << 22) + 5, 0.0123, 65536), (2, 1 << 21, 0.05, 1024),
    # FP8 at realistic rates over several K2b groups (~52-62 records per
    # 32K-element tile: the two-records-per-lane gather, its >64 tail loop)
    (1, (1 << 24) + 12345, 0.0019, 1024), (2, (1 << 23) + 3, 0.0016, 4096),
])
def test_large_streams_match_oracle(fmt_id, n, rate, chunk):
    m = sz()
    bk, esc = {0: (O.BF16_BOOK, O.BF16_ESC), 1: (O.E5M2_BOOK, O.E5M2_ESC),
               2: (O.E4M3_BOOK, O.E4M3_ESC)}[fmt_id]
    words = O.exact_stream(fmt_id, n, rate, 42 + fmt_id, bk, esc)
    book = tuple(e for e, _ in bk)
    fmt = list(m.ElementFormat)[fmt_id]
    cb = 4 if len(book) == 16 else 3
    cfg = m.CodecConfig(fmt, cb, chunk_size=chunk,
                        codebook=m.ExponentCodebook(fmt, book, cb, m.CodebookMode.TOPK_EXPLICIT))
    stream = m.RawTensorStream(fmt, torch.from_numpy(words).cuda())
    enc = m.encode(stream, cfg)
    ref = O.encode(words, O.Params(fmt_id, cb, False, chunk, False), book)
    assert enc.n_escapes == ref["m"] == round(rate * n)
    assert dict(enc.section_bytes())["packed_codes"] == ref["packed_codes"]
    assert [b for _, b in enc.section_bytes()] == O.section_bytes(ref)
    dec = m.decode(enc, cfg, enc.codebook)
    assert m.compare_streams(stream, dec).ok


def test_compare_streams_reports_first_mismatch():
    m = sz()
    a = np.arange(100_000, dtype=np.uint16)
    b = a.copy()
    b[[777, 5000, 99_999]] ^= 1
    r = m.compare_streams(m.RawTensorStream(m.ElementFormat.BF16, a),
                          m.RawTensorStream(m.ElementFormat.BF16, b))
    assert (r.ok, r.mismatch_count, r.first_mismatch_index) == (False, 3, 777)
    r = m.compare_streams(m.RawTensorStream(m.ElementFormat.FP8_E5M2, a.view(np.uint8)),
                          m.RawTensorStream(m.ElementFormat.FP8_E5M2, b.view(np.uint8)))
    assert (r.mismatch_count, r.first_mismatch_index) == (3, 2 * 777)


def test_coverage_by_group():
    m = sz()
    clean = O.exact_stream(0, 10_000, 0.0, 4, O.BF16_BOOK, O.BF16_ESC)
    dirty = O.exact_stream(0, 10_000, 0.0123, 5, O.BF16_BOOK, O.BF16_ESC)
    stream = m.RawTensorStream(m.ElementFormat.BF16, np.concatenate([clean, dirty]))
    book = m.select_codebook(m.build_histogram(m.RawTensorStream(m.ElementFormat.BF16, clean)),
                             4, m.CodebookMode.TOPK_EXPLICIT)
    assert m.coverage_by_group(stream, 10_000, book).tolist() == [1.0, 0.9877]


@pytest.mark.parametrize("seed", range(40))
def test_random_lengths_roundtrip(seed):
    # hypothesis-style sweep of ragged lengths (test_codec.py:256-260)
    m = sz()
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 40_000))
    fmt_id = seed % 3
    words = O.random_words(fmt_id, n, seed)
    fmt = list(m.ElementFormat)[fmt_id]
    stream = m.RawTensorStream(fmt, words)
    for cfg in (m.CodecConfig(fmt), m.CodecConfig(fmt, 3, chunk_size=int(rng.integers(1, 3000))),
                m.CodecConfig(fmt, mode=m.CodebookMode.TOP15_SENTINEL),
                m.CodecConfig(fmt, position_mode=m.PositionMode.ABSOLUTE_32)):
        enc = m.encode(stream, cfg)
        p = O.Params(fmt_id, cfg.code_bits, cfg.sentinel, cfg.chunk_size, cfg.abs32)
        ref = O.encode(words, p, enc.codebook.entries)
        assert [b for _, b in enc.section_bytes()] == O.section_bytes(ref)
        assert m.verify_roundtrip(stream, cfg).ok


@pytest.mark.parametrize("host_kind", ["numpy", "pinned", "pageable"])
def test_host_pipeline_matches_oracle(host_kind, monkeypatch):
    """Host-resident streams go through the piecewise H2D/K2/D2H pipeline;
    force tiny pieces so a modest stream spans several of them."""
    m = sz()
    from paper_2605_01708_b200 import hostpipe
    monkeypatch.setattr(hostpipe, "PIECE_ELEMS", 1 << 16)
    n = (1 << 18) + 12345
    words = O.exact_stream(0, n, 0.0123, 77, O.BF16_BOOK, O.BF16_ESC)
    book = tuple(e for e, _ in O.BF16_BOOK)
    cfg = m.CodecConfig(m.ElementFormat.BF16, chunk_size=1024, codebook=m.ExponentCodebook(
        m.ElementFormat.BF16, book, 4, m.CodebookMode.TOPK_EXPLICIT))
    if host_kind == "numpy":
        src = words
    else:
        src = torch.from_numpy(words.copy())
        if host_kind == "pinned":
            src = src.pin_memory()
    stream = m.RawTensorStream(m.ElementFormat.BF16, src)
    assert hostpipe.pipelinable(cfg, n)
    enc = m.encode(stream, cfg)
    ref = O.encode(words, O.Params(0), book)
    assert [b for _, b in enc.section_bytes()] == O.section_bytes(ref)
    dec = m.decode(enc, cfg, enc.codebook)
    out = dec.words.numpy() if isinstance(dec.words, torch.Tensor) else dec.words
    assert np.array_equal(out, words)
    # a corrupted host stream still raises with the reference's verdict
    if host_kind == "numpy":
        pos = enc.escape_positions.copy()
        pos[3] = 1024
        bad = m.EncodedStreams(enc.n_elements, enc.n_escapes, enc.packed_codes,
                               enc.sign_mantissa, enc.chunk_counts, pos, enc.escape_values,
                               enc.codebook)
        with pytest.raises(m.CorruptionError) as exc:
            m.decode(bad, cfg, enc.codebook)
        sec = dict(ref, escape_positions=pos)
        with pytest.raises(O.OracleCorruption) as oexc:
            O.decode(sec, O.Params(0), book)
        assert exc.value.chunk == oexc.value.chunk


@pytest.mark.parametrize("fmt_id", [0, 1])
@pytest.mark.parametrize("rate", [0.0016, 0.0789, 0.5])
def test_gpu_piece_codec_loopback(rate, fmt_id):
    """The handoff's product binding (GpuPieceCodec) on one GPU: encode each
    piece into its frame (M on the device), copy the frame as the NCCL send
    would, decode it in place; pieces over the frame capacity go through the
    spill path exactly as HandoffSender/Receiver run it."""
    m = sz()
    from paper_2605_01708_b200.distributed import GpuPieceCodec
    n, piece = 300_000, 1 << 16
    bk, esc = (O.BF16_BOOK, O.BF16_ESC) if fmt_id == 0 else (O.E5M2_BOOK, O.E5M2_ESC)
    fmt = list(m.ElementFormat)[fmt_id]
    words = O.exact_stream(fmt_id, n, rate, 3, bk, esc)
    book = m.ExponentCodebook(fmt, tuple(e for e, _ in bk), 4, m.CodebookMode.TOPK_EXPLICIT)
    cfg = m.CodecConfig(fmt, codebook=book)
    tx, rx = GpuPieceCodec(cfg, book), GpuPieceCodec(cfg, book)
    src = torch.from_numpy(words).cuda()
    out = torch.empty_like(src)
    bounds = [(lo, min(n, lo + piece)) for lo in range(0, n, piece)]
    for k, (lo, hi) in enumerate(bounds):
        fr = tx.encode_frame(src[lo:hi], k % 2)
        dst = rx.recv_frame(hi - lo, k % 2)
        dst.copy_(fr)
        rx.decode_frame(dst, hi - lo, out[lo:hi], k % 2, k)
    spills = tx.overflowed()
    assert bool(spills) == (rate > 1 / 32)
    for k, mk in spills:
        lo, hi = bounds[k]
        fr = tx.spill_frame(src[lo:hi], mk)
        dst = rx.recv_frame(hi - lo, "spill", capacity=mk)
        dst.copy_(fr)
        rx.decode_frame(dst, hi - lo, out[lo:hi], "spill", k, capacity=mk)
    rx.finish({k for k, _ in spills})
    assert torch.equal(out, src)
