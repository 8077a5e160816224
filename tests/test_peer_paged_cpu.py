"""Host-side logic of the peer-store handoff and the paged-KV API that needs
no GPU: the slot layout both processes carve identically, and the paged
API's input validation (it must refuse, not fall back)."""

from __future__ import annotations

import pytest
import torch


def sz():
    import paper_2605_01708_b200 as m
    return m


@pytest.mark.parametrize("fmt_name,mode,bits,chunk", [
    ("bf16", "explicit", 4, 1024), ("e5m2", "explicit", 4, 256), ("bf16", "sentinel", 4, 1024),
    ("e4m3", "explicit", 3, 3000)])
def test_slot_layout_is_aligned_disjoint_and_sized_for_all_escapes(fmt_name, mode, bits, chunk):
    m = sz()
    from paper_2605_01708_b200.peer import SlotLayout
    fmt = m.ElementFormat.from_name(fmt_name)
    cfg = m.CodecConfig(fmt, bits, m.CodebookMode.from_name(mode), chunk)
    piece = chunk * 777
    lay = SlotLayout(piece, cfg, 3)
    spans = []
    for d in lay.slot:
        sizes = {"codes": -(-piece * bits // 8), "sm": cfg.sm_nbytes(piece),
                 "counts": 4 * cfg.n_chunks(piece),
                 "positions": 0 if cfg.sentinel else piece * cfg.position_nbytes,
                 "values": piece, "m": 8}       # worst case: every element escapes
        for f, size in sizes.items():
            if size == 0:
                assert d[f] is None
                continue
            assert d[f] % 256 == 0
            spans.append((d[f], d[f] + size))
    spans.append((lay.ready, lay.ready + 8 * lay.slots))
    spans.sort()
    assert all(a[1] <= b[0] for a, b in zip(spans, spans[1:]))
    assert spans[-1][1] <= lay.total and lay.total % 256 == 0
    assert SlotLayout(piece, cfg, 3).slot == lay.slot     # deterministic on both sides


def test_paged_api_refuses_host_tensors():
    m = sz()
    from paper_2605_01708_b200 import paged
    caches = [torch.zeros(4, 2, 16, 8, 128, dtype=torch.uint16)]
    with pytest.raises(m.ConfigError):
        paged.kv_block_table(caches, torch.arange(2))
    with pytest.raises(m.ConfigError):
        paged.kv_block_table([], torch.arange(2))


def test_peer_requires_chunk_aligned_pieces():
    m = sz()
    from paper_2605_01708_b200 import peer
    fmt = m.ElementFormat.BF16
    book = m.ExponentCodebook(fmt, (0x7F, 0x80), 4, m.CodebookMode.TOPK_EXPLICIT)
    cfg = m.CodecConfig(fmt, codebook=book)
    with pytest.raises(ValueError):
        peer.connect_pair("send", 1, 1000, cfg, book, loopback=True)
