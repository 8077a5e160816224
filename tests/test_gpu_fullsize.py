"""Parity at BASELINE.json's full sizes (configs 2 and 3: 2^31 KV words on one
GPU) through size-independent properties: the decode of the
encode is bit-exact, the chunk counts add up to M and never exceed a chunk,
the payload ratio sits at the reference's acceptance value, and the GPU's
global sections restricted to chunk-aligned slices at the start, middle and
end of the stream equal the oracle's encode of those slices."""
import numpy as np
import pytest
import torch

from sz_testutil import ROOT  # noqa: F401  (puts the repo on sys.path)

pytestmark = pytest.mark.gpu

N = 1 << 31
SLICE = 1 << 20


def _profile(fmt_name):
    if fmt_name == "bf16":
        return 0, tuple((0x70 + i, 0.72 ** i) for i in range(16)), tuple(range(0x10, 0x18))
    return 1, tuple((8 + i, 0.72 ** i) for i in range(16)), (0, 1, 2, 3, 28, 29, 30, 31)


@pytest.mark.parametrize("fmt_name,ratio", [("bf16", 1.3256), ("e5m2", 1.1324)])
def test_full_size_roundtrip_and_slice_parity(fmt_name, ratio):
    import paper_2605_01708_b200 as sz
    from oracle import sz_oracle as O
    from paper_2605_01708_b200.engine import DeviceCodec, synth_kv

    fmt_id, bw, esc = _profile(fmt_name)
    fmt = sz.ElementFormat.from_name(fmt_name)
    words = synth_kv(N, fmt, 11, bw, esc, 0.0016)
    book = sz.ExponentCodebook(fmt, tuple(e for e, _ in bw), 4, sz.CodebookMode.TOPK_EXPLICIT)
    cfg = sz.CodecConfig(fmt, codebook=book)
    eng = DeviceCodec(cfg, book, N)
    m = eng.ensure_capacity(words)
    eng.decode()
    eng.check_status()
    res = eng.compare(words, eng.out).cpu().numpy()
    assert int(res[0]) == 0, f"{int(res[0])} mismatches, first at {int(res[1])}"

    st = eng.streams(m)
    counts = st.chunk_counts.to(torch.int64)
    assert int(counts.sum().item()) == m
    assert int(counts.max().item()) <= cfg.chunk_size
    assert N * fmt.word_nbytes / eng.payload_nbytes(m) == pytest.approx(ratio, abs=2e-3)

    c = cfg.chunk_size
    sm_bits = {0: 8, 1: 3}[fmt_id]
    prefix = torch.cumsum(counts, 0)
    for a in (0, (N // 2 // c) * c + 7 * c, N - SLICE):
        b = a + SLICE
        ka, kb = a // c, b // c
        o0 = int(prefix[ka - 1].item()) if ka else 0
        o1 = int(prefix[kb - 1].item())
        ref = O.encode(words[a:b].cpu().numpy(), O.Params(fmt_id, 4, False, c, False),
                       book.entries)
        assert ref["packed_codes"] == st.packed_codes[a // 2:b // 2].cpu().numpy().tobytes()
        assert ref["sign_mantissa"] == \
            st.sign_mantissa[a * sm_bits // 8:b * sm_bits // 8].cpu().numpy().tobytes()
        assert np.array_equal(ref["chunk_counts"], counts[ka:kb].cpu().numpy())
        assert int(ref["m"]) == o1 - o0
        assert np.array_equal(ref["escape_positions"], st.escape_positions[o0:o1].cpu().numpy())
        assert np.array_equal(ref["escape_values"], st.escape_values[o0:o1].cpu().numpy())
    del eng, words
    torch.cuda.empty_cache()
