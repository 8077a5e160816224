"""Real-KV ingestion, CPU side: kv_extractor's dumps of
real attention K/V (offline random-gpt2, pkg/kv_extractor/src/kv_extractor/
extract.py:85-94,128-189) read through the package's ``read_raw_tensor``
and the oracle pinned to the reference's calibrate / verify --dynamic /
compress results on them (tests/golden/make_realkv.py).  The reference's
own acceptance figures for these dumps are 99.99% top-16 coverage and 2.55
bits/exponent (pkg/test_output.txt:345, test_extract.py:103-118)."""

from __future__ import annotations

import json

import numpy as np
import pytest

from oracle import sz_oracle as O
from sz_testutil import GOLDEN_DIR, realkv, sha256

FMTS = {"bf16": 0, "e5m2": 1}


def test_manifest_matches_extractor_contract():
    r = realkv()
    man = json.loads((r.dir / "manifest.json").read_text())
    assert man == r.ref["extract"]["manifest"]
    # random-gpt2: 4 layers x {K, V}, 4 heads x head_dim 32 per token
    assert len(man["files"]) == 8 and man["element_format"] == "bf16"
    for rec in man["files"]:
        assert rec["elements"] == man["token_count"] * 4 * 32


@pytest.mark.parametrize("fmt", FMTS)
def test_words_match_reference_digests(fmt):
    r = realkv()
    for f in r.files():
        assert sha256(r.words(fmt, f)) == r.dump(fmt, f)["words_sha256"], f


def test_read_raw_tensor_host_parse():
    import paper_2605_01708_b200 as sz
    r = realkv()
    for f in r.files():
        s = sz.read_raw_tensor(r.dir / f)
        assert s.fmt is sz.ElementFormat.BF16
        assert np.array_equal(np.asarray(s.words), r.words("bf16", f))


@pytest.mark.parametrize("fmt", FMTS)
def test_oracle_calibration_matches_reference(fmt):
    r = realkv()
    cal = r.calibrate(fmt)
    counts = sum(O.histogram(r.words(fmt, f), FMTS[fmt]) for f in r.files())
    assert counts.tolist() == cal["counts"]
    p = counts[counts > 0] / counts.sum()
    assert abs(float(-(p * np.log2(p)).sum()) - cal["entropy_bits"]) < 1e-12
    order = O.ranked(counts)
    assert abs(counts[order[:16]].sum() / counts.sum() - cal["top16_coverage"]) < 1e-15
    assert list(O.choose_book(counts, 4, False)) == cal["books"]["4_explicit"]
    assert list(O.choose_book(counts, 3, False)) == cal["books"]["3_explicit"]
    assert list(O.choose_book(counts, 4, True)) == cal["books"]["4_sentinel"]
    if fmt == "bf16":  # the reference's acceptance line (test_output.txt:345)
        assert cal["top16_coverage"] > 0.9999 and round(cal["entropy_bits"], 2) == 2.55


@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("cfg", list(realkv().CONFIGS))
def test_oracle_encode_matches_reference(fmt, cfg):
    r = realkv()
    code_bits, sentinel, chunk, abs32, key = r.CONFIGS[cfg]
    p = O.Params(FMTS[fmt], code_bits, sentinel, chunk, abs32)
    for f in r.files():
        words = r.words(fmt, f)
        want = r.dump(fmt, f)["configs"][cfg]
        book = (tuple(r.calibrate(fmt)["books"][key]) if key
                else O.choose_book(O.histogram(words, FMTS[fmt]), code_bits, sentinel))
        assert list(book) == want["book"]
        sec = O.encode(words, p, book)
        names = ["chunk_counts", "packed_codes", "sign_mantissa", "escape_positions",
                 "escape_values"]
        got = dict(zip(names, (sha256(b) for b in O.section_bytes(sec))))
        assert got == want["sections"], f
        assert sec["m"] == want["m"]
        assert O.payload_bytes(sec["n"], sec["m"], p) == want["payload_nbytes"]
        assert sha256(O.container_bytes(sec, p, book)) == want["container_sha256"]
        assert np.array_equal(O.decode(sec, p, book), words)
