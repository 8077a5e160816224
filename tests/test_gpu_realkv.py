"""Real-KV ingestion on the GPU: ``read_raw_tensor`` of
kv_extractor's real attention K/V dumps -> K1 calibration (per-file
histograms, ``merge_stats``, entropy, coverage, ``select_codebook``,
``coverage_by_group``) -> K2 encode -> K3/K4 decode, each checked against
what the REAL reference computed on the same files
(tests/golden/make_realkv.py: the CLI's calibrate, cli.py:164-199, and
verify --dynamic / compress, cli.py:214-228): section SHA-256s, M, payload
size, container bytes and bit-exact round trips."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from sz_testutil import realkv, sha256

pytestmark = pytest.mark.gpu

FMTS = ("bf16", "e5m2")


def sz():
    import paper_2605_01708_b200 as m
    return m


def _fmt(name):
    m = sz()
    return {"bf16": m.ElementFormat.BF16, "e5m2": m.ElementFormat.FP8_E5M2}[name]


def _streams(fmt):
    m = sz()
    r = realkv()
    out = []
    for f in r.files():
        if fmt == "bf16":
            s = m.read_raw_tensor(r.dir / f)     # the .szrw layout, parsed on the host
            words = torch.from_numpy(np.asarray(s.words).copy()).cuda()
        else:
            words = torch.from_numpy(r.words(fmt, f)).cuda()
        out.append((f, m.RawTensorStream(_fmt(fmt), words)))
    return out


@pytest.mark.parametrize("fmt", FMTS)
def test_calibration_on_device_matches_reference(fmt):
    m = sz()
    cal = realkv().calibrate(fmt)
    streams = _streams(fmt)
    stats = m.merge_stats(*(m.build_histogram(s) for _, s in streams))
    assert stats.counts.tolist() == cal["counts"] and stats.total == cal["elements"]
    assert abs(m.entropy_bits(stats) - cal["entropy_bits"]) < 1e-12
    assert abs(m.top_k_coverage(stats, 8) - cal["top8_coverage"]) < 1e-15
    assert abs(m.top_k_coverage(stats, 16) - cal["top16_coverage"]) < 1e-15
    for key, (cb, mode) in {"4_explicit": (4, m.CodebookMode.TOPK_EXPLICIT),
                            "3_explicit": (3, m.CodebookMode.TOPK_EXPLICIT),
                            "4_sentinel": (4, m.CodebookMode.TOP15_SENTINEL)}.items():
        assert list(m.select_codebook(stats, cb, mode).entries) == cal["books"][key]
    book = m.select_codebook(stats, 4, m.CodebookMode.TOPK_EXPLICIT)
    for (_, s), want in zip(streams, cal["group_coverage_1024"]):
        got = m.coverage_by_group(s, 1024, book).cpu().numpy()
        assert got.tolist() == want


def _config(fmt, name):
    m = sz()
    r = realkv()
    code_bits, sentinel, chunk, abs32, key = r.CONFIGS[name]
    mode = m.CodebookMode.TOP15_SENTINEL if sentinel else m.CodebookMode.TOPK_EXPLICIT
    pos = m.PositionMode.ABSOLUTE_32 if abs32 else m.PositionMode.CHUNK_RELATIVE
    book = (m.ExponentCodebook(_fmt(fmt), tuple(r.calibrate(fmt)["books"][key]), code_bits,
                               mode) if key else None)
    return m.CodecConfig(_fmt(fmt), code_bits, mode, chunk, pos, book)


@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("name", list(realkv().CONFIGS))
def test_encode_decode_matches_reference(fmt, name):
    m = sz()
    from paper_2605_01708_b200 import container as C
    r = realkv()
    cfg = _config(fmt, name)
    for f, s in _streams(fmt):
        want = r.dump(fmt, f)["configs"][name]
        enc = m.encode(s, cfg)
        assert list(enc.codebook.entries) == want["book"]
        got = {k: sha256(v) for k, v in enc.section_bytes()}
        assert got == want["sections"], f
        assert enc.n_escapes == want["m"] and enc.payload_nbytes == want["payload_nbytes"]
        dec = m.decode(enc, cfg, enc.codebook)
        assert torch.equal(dec.words, s.words), f
        buf = C.encode_container(s, cfg)
        assert buf.numel() == want["container_nbytes"]
        assert sha256(buf.cpu().numpy()) == want["container_sha256"], f
        assert torch.equal(C.decode_container(buf).words, s.words)


@pytest.mark.parametrize("fmt", FMTS)
def test_host_stream_path_matches_reference(fmt):
    """Host-resident dumps (numpy words) through the pipelined H2D -> K2 -> D2H
    path, dynamic codebook, as ``splitzip verify --dynamic`` runs them."""
    m = sz()
    r = realkv()
    cfg = _config(fmt, "dyn4")
    for f in r.files():
        words = r.words(fmt, f)
        s = m.RawTensorStream(_fmt(fmt), words)
        enc = m.encode(s, cfg)
        want = r.dump(fmt, f)["configs"]["dyn4"]
        assert {k: sha256(v) for k, v in enc.section_bytes()} == want["sections"], f
        assert np.array_equal(np.asarray(m.decode(enc, cfg, enc.codebook).words), words)
