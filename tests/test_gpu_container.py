"""Device-side SPLZ framing (sz_frame_container) against the reference's own
container bytes, device-container parsing + decode, and the sync-free
engine path (encode -> frame with M read on the GPU)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from sz_testutil import golden, golden_case_ids

pytestmark = pytest.mark.gpu


def sz():
    import paper_2605_01708_b200 as m
    return m


def C():
    from paper_2605_01708_b200 import container
    return container


def make_config(case):
    m = sz()
    fmt = [m.ElementFormat.BF16, m.ElementFormat.FP8_E5M2, m.ElementFormat.FP8_E4M3][case["fmt"]]
    mode = m.CodebookMode.TOP15_SENTINEL if case["sentinel"] else m.CodebookMode.TOPK_EXPLICIT
    pos = m.PositionMode.ABSOLUTE_32 if case["abs32"] else m.PositionMode.CHUNK_RELATIVE
    book = m.ExponentCodebook(fmt, tuple(case["book"]), case["code_bits"], mode)
    return fmt, m.CodecConfig(fmt, case["code_bits"], mode, case["chunk"], pos, book)


@pytest.mark.parametrize("cid", golden_case_ids())
def test_device_container_matches_reference(cid):
    m = sz()
    g = golden()
    case = g.case(cid)
    fmt, cfg = make_config(case)
    words = torch.from_numpy(g.arr(cid, "words").copy()).cuda()
    ref = g.arr(cid, "container").tobytes()
    enc = m.encode(m.RawTensorStream(fmt, words), cfg)
    assert C().container_to_bytes(enc, cfg, enc.codebook) == ref
    buf = C().encode_container(m.RawTensorStream(fmt, words), cfg)
    assert buf.is_cuda and buf.cpu().numpy().tobytes() == ref
    dec = C().decode_container(buf)
    assert torch.equal(dec.words, words)
    # host bytes of a device-framed container decode through the host path too
    dec_h = C().decode_container(ref)
    assert np.array_equal(dec_h.words, g.arr(cid, "words"))


def _verdicts():
    return golden().manifest["container_verdicts"]


@pytest.mark.parametrize("v", _verdicts(), ids=lambda v: v["id"])
def test_device_container_parse_verdicts(v):
    m = sz()
    data = torch.from_numpy(golden()._npz[v["id"]].copy()).cuda()
    if v["raised"] is None:
        C().decode_container(data)
        return
    with pytest.raises(m.SplitZipError) as ei:
        C().container_from_bytes(data)
    assert type(ei.value).__name__ == v["raised"]
    assert getattr(ei.value, "section", None) == v["section"]


@pytest.mark.parametrize("fmt_name,rate", [("bf16", 0.0016), ("e5m2", 0.0016), ("bf16", 0.05)])
def test_engine_frame_is_sync_free_and_exact(fmt_name, rate):
    """DeviceCodec.encode -> frame enqueued back to back (M never leaves the
    GPU) equals the host-assembled reference container of the same sections."""
    m = sz()
    from paper_2605_01708_b200.engine import DeviceCodec, synth_kv
    fmt = m.ElementFormat.from_name(fmt_name)
    if fmt is m.ElementFormat.BF16:
        bw, esc = tuple((0x70 + i, 0.72 ** i) for i in range(16)), tuple(range(0x10, 0x18))
    else:
        bw, esc = tuple((8 + i, 0.72 ** i) for i in range(16)), (0, 1, 2, 3, 28, 29, 30, 31)
    n = (1 << 22) + 4097
    words = synth_kv(n, fmt, 5, bw, esc, rate)
    book = m.ExponentCodebook(fmt, tuple(e for e, _ in bw), 4, m.CodebookMode.TOPK_EXPLICIT)
    cfg = m.CodecConfig(fmt, codebook=book)
    eng = DeviceCodec(cfg, book, n, capacity=n // 8)
    out = torch.empty(eng.container_capacity(), dtype=torch.uint8, device="cuda")
    nb = torch.zeros(1, dtype=torch.int64, device="cuda")
    eng.encode(words)
    eng.frame(out, nb)
    total = int(nb.item())
    host = C().container_to_bytes(eng.streams().to_host(), cfg, book)
    assert total == len(host)
    assert out[:total].cpu().numpy().tobytes() == host
    dec = C().decode_container(out[:total])
    assert torch.equal(dec.words, words)
