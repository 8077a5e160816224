"""SPLZ container framing (container.py) on the host: the oracle and the
package's host path against the reference's own container bytes, and the
reference's parse verdicts (exception class + section) on mutated files."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import sz_oracle as O
from sz_testutil import golden, golden_case_ids, oracle_params


def sz():
    import paper_2605_01708_b200 as m
    return m


def container_mod():
    from paper_2605_01708_b200 import container
    return container


def host_streams(cid):
    """EncodedStreams with reference-typed host sections from the golden files."""
    m = sz()
    g = golden()
    case = g.case(cid)
    fmt = [m.ElementFormat.BF16, m.ElementFormat.FP8_E5M2, m.ElementFormat.FP8_E4M3][case["fmt"]]
    mode = m.CodebookMode.TOP15_SENTINEL if case["sentinel"] else m.CodebookMode.TOPK_EXPLICIT
    pos = m.PositionMode.ABSOLUTE_32 if case["abs32"] else m.PositionMode.CHUNK_RELATIVE
    book = m.ExponentCodebook(fmt, tuple(case["book"]), case["code_bits"], mode)
    cfg = m.CodecConfig(fmt, case["code_bits"], mode, case["chunk"], pos, book)
    pos_dtype = np.dtype(case["pos_dtype"])
    enc = m.EncodedStreams(
        case["n"], case["m"], g.arr(cid, "packed_codes").tobytes(),
        g.arr(cid, "sign_mantissa").tobytes(),
        g.arr(cid, "chunk_counts").view("<u4"),
        g.arr(cid, "escape_positions").view(pos_dtype),
        g.arr(cid, "escape_values_raw"), book,
        g.arr(cid, "escape_values").tobytes())
    return enc, cfg, book


@pytest.mark.parametrize("cid", golden_case_ids())
def test_oracle_container_matches_reference(cid):
    g = golden()
    case = g.case(cid)
    p = oracle_params(case)
    sec = O.encode(g.arr(cid, "words"), p, tuple(case["book"]))
    assert O.container_bytes(sec, p, case["book"]) == g.arr(cid, "container").tobytes()


@pytest.mark.parametrize("cid", golden_case_ids())
def test_host_container_roundtrip_matches_reference(cid):
    C = container_mod()
    g = golden()
    enc, cfg, book = host_streams(cid)
    ref = g.arr(cid, "container").tobytes()
    assert C.container_to_bytes(enc, cfg, book) == ref
    streams, cfg2, book2 = C.container_from_bytes(ref)
    assert cfg2 == cfg and book2.entries == book.entries
    assert streams.n_elements == enc.n_elements and streams.n_escapes == enc.n_escapes
    assert streams.packed_codes == enc.packed_codes
    assert streams.sign_mantissa == enc.sign_mantissa
    assert np.array_equal(streams.chunk_counts, enc.chunk_counts)
    assert np.array_equal(streams.escape_positions, enc.escape_positions)
    assert np.array_equal(streams.escape_values, enc.escape_values)


def _verdicts():
    return golden().manifest["container_verdicts"]


@pytest.mark.parametrize("v", _verdicts(), ids=lambda v: v["id"])
def test_container_parse_verdicts_match_reference(v):
    m = sz()
    C = container_mod()
    data = golden()._npz[v["id"]].tobytes()
    if v["raised"] is None:
        C.container_from_bytes(data)
        return
    with pytest.raises(m.SplitZipError) as ei:
        C.container_from_bytes(data)
    assert type(ei.value).__name__ == v["raised"]
    assert getattr(ei.value, "section", None) == v["section"]


def test_codebook_and_raw_records_roundtrip(tmp_path):
    m = sz()
    C = container_mod()
    book = m.ExponentCodebook(m.ElementFormat.BF16, (0x7F, 0x80, 0x7E), 4,
                              m.CodebookMode.TOPK_EXPLICIT)
    rec = C.codebook_record_bytes(book)
    assert rec == b"SZCB" + bytes([1, 0, 4, 0, 3, 0x7F, 0x80, 0x7E])   # 9 + k bytes
    assert C.codebook_from_bytes(rec).entries == book.entries
    with pytest.raises(m.LengthMismatchError):
        C.codebook_from_bytes(rec + b"\x00")
    words = np.arange(1000, dtype=np.uint16)
    st = m.RawTensorStream(m.ElementFormat.BF16, words)
    path = tmp_path / "x.szrw"
    C.write_raw_tensor(st, path)
    back = C.read_raw_tensor(path)
    assert back.fmt is m.ElementFormat.BF16 and np.array_equal(back.words, words)
    with pytest.raises(m.BadMagicError):
        C.raw_tensor_from_bytes(b"XXXX" + path.read_bytes()[4:])
    with pytest.raises(m.TruncatedError):
        C.raw_tensor_from_bytes(path.read_bytes()[:-1])
