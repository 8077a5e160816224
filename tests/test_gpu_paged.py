"""Paged-KV encode/decode (sz_encode_segments / sz_decode_segments): sections
byte-identical to ``encode`` of the gathered words, and a bit-exact decode
straight into a receiver's own blocks."""

from __future__ import annotations

import pytest
import torch

pytestmark = pytest.mark.gpu

BF16_BOOK = tuple((0x70 + i, 0.72 ** i) for i in range(16))
BF16_ESC = tuple(range(0x10, 0x18))
E5_BOOK = tuple((8 + i, 0.72 ** i) for i in range(16))
E5_ESC = (0, 1, 2, 3, 28, 29, 30, 31)


def sz():
    import paper_2605_01708_b200 as m
    return m


def _sel(c, ids):
    """c[ids] for uint16/uint8 caches (index kernels lack UInt16)."""
    v = c.view(torch.int16) if c.dtype == torch.uint16 else c.view(torch.int8)
    return v[ids].view(c.dtype)


def make(fmt_name, block_shape, layers, num_blocks, rate, mode="explicit", chunk=1024,
         seed=3):
    m = sz()
    from paper_2605_01708_b200.engine import synth_kv
    fmt = m.ElementFormat.from_name(fmt_name)
    bw, esc = (BF16_BOOK, BF16_ESC) if fmt is m.ElementFormat.BF16 else (E5_BOOK, E5_ESC)
    per_block = 1
    for d in block_shape:
        per_block *= d
    caches = [synth_kv(num_blocks * per_block, fmt, seed + l, bw, esc, rate)
              .view(num_blocks, *block_shape) for l in range(layers)]
    cmode = m.CodebookMode.from_name(mode)
    entries = tuple(e for e, _ in bw)[: 15 if mode == "sentinel" else 16]
    book = m.ExponentCodebook(fmt, entries, 4, cmode)
    cfg = m.CodecConfig(fmt, 4, cmode, chunk, codebook=book)
    return m, fmt, caches, cfg


@pytest.mark.parametrize("fmt_name,block_shape,rate,mode,chunk", [
    ("bf16", (2, 16, 8, 128), 0.0016, "explicit", 1024),    # vLLM block, 64 KiB (> tile)
    ("bf16", (2, 16, 1, 64), 0.0123, "explicit", 256),      # 4 KiB blocks (< tile)
    ("e5m2", (2, 16, 8, 128), 0.0016, "explicit", 1024),    # 32 KiB = one FP8 tile
    ("e5m2", (2, 4, 2, 32), 0.05, "explicit", 3000),        # 1 KiB blocks, odd chunk
    ("bf16", (2, 16, 4, 64), 0.5, "explicit", 1024),        # escape-heavy: K2b re-derives
    ("bf16", (2, 16, 8, 128), 0.0027, "sentinel", 1024),    # sentinel decode kernel
])
def test_paged_sections_and_roundtrip(fmt_name, block_shape, rate, mode, chunk):
    from paper_2605_01708_b200 import paged
    m, fmt, caches, cfg = make(fmt_name, block_shape, 3, 40, rate, mode, chunk)
    g = torch.Generator().manual_seed(7)
    ids = torch.randperm(40, generator=g)[:23].cuda()
    gathered = torch.cat([_sel(c, ids).reshape(-1) for c in caches])
    ref = m.encode(m.RawTensorStream(fmt, gathered), cfg)
    enc = paged.encode_kv_blocks(caches, ids, cfg)
    assert enc.n_escapes == ref.n_escapes
    assert dict(enc.section_bytes()) == dict(ref.section_bytes())
    # and both equal the CPU oracle's encode of the gathered words
    from oracle import sz_oracle as O
    p = O.Params({"bf16": 0, "e5m2": 1}[fmt_name], 4, mode == "sentinel", chunk, False)
    osec = O.encode(gathered.cpu().numpy(), p, tuple(cfg.codebook.entries))
    assert [b for _, b in enc.section_bytes()] == O.section_bytes(osec)
    # decode into a different pool with a different block table
    dst = [torch.zeros_like(c) for c in caches]
    ids2 = torch.randperm(40, generator=g)[:23].cuda()
    paged.decode_kv_blocks(enc, cfg, enc.codebook, dst, ids2)
    back = torch.cat([_sel(c, ids2).reshape(-1) for c in dst])
    assert torch.equal(back, gathered)
    # untouched blocks stay untouched
    mask = torch.ones(40, dtype=torch.bool)
    mask[ids2.cpu()] = False
    for c in dst:
        assert not bool(_sel(c, mask.nonzero().reshape(-1).cuda()).view(torch.uint8).any())


@pytest.mark.parametrize("fmt_name,block_shape", [
    ("bf16", (2, 16, 8, 128)),   # 64 KiB blocks: one 256-row box per tile
    ("bf16", (2, 4, 1, 64)),     # 1 KiB blocks: 32 eight-row boxes per tile
    ("e5m2", (2, 16, 2, 128)),   # 8 KiB FP8 blocks
])
def test_paged_va_window_matches_bulk_copies(fmt_name, block_shape):
    """The tensor-map path over the caches' VA window and the per-segment
    1-D bulk copies produce the same sections."""
    from paper_2605_01708_b200 import paged
    m, fmt, caches, cfg = make(fmt_name, block_shape, 4, 64, 0.01)
    ids = torch.randperm(64, generator=torch.Generator().manual_seed(3))[:45].cuda()
    addrs, seg = paged.kv_block_table(caches, ids)
    win = paged.kv_va_window(caches)
    assert win is not None
    a = paged.encode_segments(addrs, seg, cfg, va_window=win)
    b = paged.encode_segments(addrs, seg, cfg)
    assert a.n_escapes == b.n_escapes
    assert dict(a.section_bytes()) == dict(b.section_bytes())


def test_paged_rejects_bad_blocks():
    from paper_2605_01708_b200 import paged
    m, fmt, caches, cfg = make("bf16", (3, 16, 8, 128), 1, 8, 0.0016)   # 96 KiB: not 2^k
    with pytest.raises(m.ConfigError):
        paged.encode_kv_blocks(caches, torch.arange(4, device="cuda"), cfg)
    m, fmt, caches, cfg = make("bf16", (2, 16, 8, 128), 1, 8, 0.0016)
    nobook = m.CodecConfig(fmt)
    with pytest.raises(m.ConfigError):
        paged.encode_kv_blocks(caches, torch.arange(4, device="cuda"), nobook)


def test_concurrent_encodes_on_two_streams_do_not_interfere():
    """No hidden global state in the C ABI: two engines with different
    codebooks encode/decode on two streams at once, both bit-exact and both
    equal to their serial results."""
    import paper_2605_01708_b200 as m
    from paper_2605_01708_b200.engine import DeviceCodec, synth_kv
    fmt = m.ElementFormat.BF16
    n = (1 << 23) + 1000
    w1 = synth_kv(n, fmt, 1, BF16_BOOK, BF16_ESC, 0.0016)
    w2 = synth_kv(n, fmt, 2, BF16_BOOK, BF16_ESC, 0.05)
    b1 = m.ExponentCodebook(fmt, tuple(e for e, _ in BF16_BOOK), 4, m.CodebookMode.TOPK_EXPLICIT)
    b2 = m.ExponentCodebook(fmt, tuple(e for e, _ in BF16_BOOK)[::-1], 4,
                            m.CodebookMode.TOPK_EXPLICIT)
    e1 = DeviceCodec(m.CodecConfig(fmt, codebook=b1), b1, n, capacity=n // 4)
    e2 = DeviceCodec(m.CodecConfig(fmt, codebook=b2), b2, n, capacity=n // 4)
    e1.encode(w1); e2.encode(w2)
    torch.cuda.synchronize()
    ref1 = dict(e1.streams().section_bytes())
    ref2 = dict(e2.streams().section_bytes())
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        e1.encode(w1, stream=s1)
        e2.encode(w2, stream=s2)
        e1.decode(stream=s1)
        e2.decode(stream=s2)
    torch.cuda.synchronize()
    assert dict(e1.streams().section_bytes()) == ref1
    assert dict(e2.streams().section_bytes()) == ref2
    assert torch.equal(e1.out, w1) and torch.equal(e2.out, w2)


def test_decode_segments_checks_section_lengths():
    """decode_segments raises CorruptionError like decode on sections that
    contradict the header, before any kernel writes into live blocks."""
    import dataclasses
    from paper_2605_01708_b200 import paged
    m, fmt, caches, cfg = make("bf16", (2, 16, 8, 128), 2, 16, 0.01)
    ids = torch.arange(8, device="cuda")
    enc = paged.encode_kv_blocks(caches, ids, cfg)
    dst = [torch.zeros_like(c) for c in caches]
    cases = {
        "codes": dataclasses.replace(enc, packed_codes=enc.packed_codes[:-1]),
        "sm": dataclasses.replace(enc, sign_mantissa=enc.sign_mantissa[:-1]),
        "values": dataclasses.replace(enc, escape_values=enc.escape_values[:-1]),
        "positions": dataclasses.replace(enc, escape_positions=enc.escape_positions[:-1]),
        "counts": dataclasses.replace(enc, chunk_counts=enc.chunk_counts[:-1]),
        "m_gt_n": dataclasses.replace(enc, n_escapes=enc.n_elements + 1),
    }
    for name, bad in cases.items():
        with pytest.raises(m.CorruptionError):
            paged.decode_kv_blocks(bad, cfg, enc.codebook, dst, ids)
        for c in dst:
            assert not bool(c.view(torch.uint8).any()), name


def test_engine_device_m_is_clamped_to_capacity():
    """DeviceCodec with a capacity below the input's escape count: the
    decoder (M read on the device) never reads past the escape buffers and
    check_status raises instead of returning wrong words."""
    import paper_2605_01708_b200 as m
    from paper_2605_01708_b200.engine import DeviceCodec, synth_kv
    fmt = m.ElementFormat.BF16
    n = 1 << 20
    book = m.ExponentCodebook(fmt, tuple(e for e, _ in BF16_BOOK), 4,
                              m.CodebookMode.TOPK_EXPLICIT)
    eng = DeviceCodec(m.CodecConfig(fmt, codebook=book), book, n, capacity=64)
    w = synth_kv(n, fmt, 4, BF16_BOOK, BF16_ESC, 0.05)
    eng.encode(w)
    eng.decode()
    assert eng.n_escapes() > 64
    with pytest.raises(m.NativeError, match="capacity"):
        eng.check_status()
    eng.ensure_capacity(w)
    eng.decode()
    eng.check_status()
    assert torch.equal(eng.out, w)
