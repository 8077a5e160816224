"""CPU-only checks: the C-ABI library loads and exports its header's symbols,
and the host-side logic (config validation, size formulas, codebook
selection, error classes) matches the reference's golden outputs."""

from __future__ import annotations

import re
from pathlib import Path

import numpy as np
import pytest

import paper_2605_01708_b200 as m
from paper_2605_01708_b200 import _native as N
from sz_testutil import ROOT, golden

HEADER = ROOT / "include" / "splitzip_b200.h"


def header_functions() -> set[str]:
    text = HEADER.read_text()
    return set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(sz_[a-z0-9_]+)\(", text, re.M))


def test_library_exports_every_header_symbol():
    lib = N.load_library(require_gpu=False)
    declared = header_functions()
    assert declared, "no declarations parsed"
    assert declared == set(N.EXPORTED_SYMBOLS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.sz_abi_version() == N.ABI_VERSION


def test_struct_layouts_match_header():
    import ctypes as C
    assert C.sizeof(N.SzParams) == 6 * 4 + 256 + 16
    assert C.sizeof(N.SzDecodeStatus) == 8 + 13 * 8 + 16
    assert C.sizeof(N.SzEncoded) == 9 * 8
    assert C.sizeof(N.SzEncodedIn) == 5 * 8 + 3 * 8 + 8


def test_workspace_queries_need_no_gpu():
    lib = N.load_library(require_gpu=False)
    cfg = m.CodecConfig(m.ElementFormat.BF16,
                        codebook=m.ExponentCodebook(m.ElementFormat.BF16, tuple(range(0x70, 0x80)),
                                                    4, m.CodebookMode.TOPK_EXPLICIT))
    from paper_2605_01708_b200.codec import _config_params
    p = _config_params(cfg, cfg.codebook)
    assert lib.sz_encode_workspace_bytes(1 << 31, p) >= (1 << 31) // 16384 * 8
    assert lib.sz_decode_workspace_bytes(1 << 31, 0, p) >= ((1 << 31) // 1024 + 1) * 8


def test_no_gpu_means_loud_failure(monkeypatch):
    import torch
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    with pytest.raises(m.NativeError):
        m.encode(m.RawTensorStream(m.ElementFormat.BF16, np.ones(8, np.uint16)),
                 m.CodecConfig(m.ElementFormat.BF16))


def test_kernel_params_marked_lut():
    from paper_2605_01708_b200.codec import kernel_params
    book = m.ExponentCodebook(m.ElementFormat.BF16, (0x7F, 0x80), 4, m.CodebookMode.TOPK_EXPLICIT)
    p = kernel_params(m.ElementFormat.BF16, 4, m.CodebookMode.TOPK_EXPLICIT, 1024, False, book)
    assert p.enc_lut[0x7F] == 0 and p.enc_lut[0x80] == 1 and p.enc_lut[0x10] == 0x10
    assert p.dec_lut[0] == 0x7F and p.dec_lut[1] == 0x80 and p.n_entries == 2
    sent = m.ExponentCodebook(m.ElementFormat.BF16, (0x7F,), 4, m.CodebookMode.TOP15_SENTINEL)
    p = kernel_params(m.ElementFormat.BF16, 4, m.CodebookMode.TOP15_SENTINEL, 1024, False, sent)
    assert p.enc_lut[0x10] == 0x1F and p.sentinel == 1


@pytest.mark.parametrize("case", golden().cases, ids=lambda c: c["id"])
def test_host_formulas_and_selection_match_reference(case):
    fmt = list(m.ElementFormat)[case["fmt"]]
    mode = m.CodebookMode.TOP15_SENTINEL if case["sentinel"] else m.CodebookMode.TOPK_EXPLICIT
    pos = m.PositionMode.ABSOLUTE_32 if case["abs32"] else m.PositionMode.CHUNK_RELATIVE
    cfg = m.CodecConfig(fmt, case["code_bits"], mode, case["chunk"], pos)
    n, mm = case["n"], case["m"]
    assert m.compressed_payload_bytes(n, mm, cfg) == case["formula_payload"]
    assert m.compression_ratio(n, mm, cfg) == pytest.approx(case["formula_ratio"], rel=1e-12)
    stats = m.CalibrationStats(fmt, golden().arr(case["id"], "hist"), n)
    if not case["pinned"]:
        assert list(m.select_codebook(stats, case["code_bits"], mode).entries) == case["book"]
    assert m.entropy_bits(stats) == pytest.approx(case["entropy"], abs=1e-12)
    assert m.top_k_coverage(stats, 8) == pytest.approx(case["top8"], abs=1e-15)


def test_config_validation_matches_reference():
    bf = m.ElementFormat.BF16
    with pytest.raises(m.ConfigError):
        m.CodecConfig(bf, code_bits=5)
    with pytest.raises(m.ConfigError):
        m.CodecConfig(bf, chunk_size=0)
    with pytest.raises(m.ConfigError):
        m.CodecConfig(bf, chunk_size=65537)
    with pytest.raises(m.ConfigError):
        m.CodecConfig(bf, position_mode="bogus")
    assert m.CodecConfig(bf, chunk_size=65537, position_mode=m.PositionMode.ABSOLUTE_32).position_nbytes == 4
    assert m.CodecConfig(bf, chunk_size=256).position_nbytes == 1
    assert m.CodecConfig(bf).position_nbytes == 2
    with pytest.raises(m.ConfigError):
        m.ExponentCodebook(bf, (1, 1), 4, m.CodebookMode.TOPK_EXPLICIT)
    with pytest.raises(m.ConfigError):
        m.ExponentCodebook(bf, tuple(range(16)), 4, m.CodebookMode.TOP15_SENTINEL)
    book = m.ExponentCodebook(m.ElementFormat.FP8_E5M2, (8,), 4, m.CodebookMode.TOPK_EXPLICIT)
    with pytest.raises(m.ConfigError):
        m.CodecConfig(bf, codebook=book)
    assert m.compressed_payload_bytes(1024, 0, m.CodecConfig(bf)) == 1540
    assert m.compression_ratio(1000, 0, m.CodecConfig(bf)) == pytest.approx(4 / 3)


def test_tie_break_and_merge():
    counts = np.zeros(256, np.int64)
    counts[[30, 10, 20]] = 5
    stats = m.CalibrationStats(m.ElementFormat.BF16, counts, 15)
    assert m.select_codebook(stats, 3, m.CodebookMode.TOPK_EXPLICIT).entries[:2] == (10, 20)
    merged = m.merge_stats(stats, stats)
    assert merged.total == 30 and merged.counts[10] == 10


def test_error_hierarchy():
    assert issubclass(m.CorruptionError, m.SplitZipError)
    assert issubclass(m.TruncatedError, m.ContainerError)
    e = m.CorruptionError("x", chunk=3)
    assert e.chunk == 3 and "chunk 3" in str(e)
