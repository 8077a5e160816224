"""Small encode/decode runs across formats/modes for compute-sanitizer."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_01708_b200 as sz  # noqa: E402
from oracle import sz_oracle as O  # noqa: E402

for fmt_id, fmt, bk, esc in ((0, sz.ElementFormat.BF16, O.BF16_BOOK, O.BF16_ESC),
                             (1, sz.ElementFormat.FP8_E5M2, O.E5M2_BOOK, O.E5M2_ESC)):
    for rate, chunk, mode, pos, bits in (
            (0.0016, 1024, "explicit", "chunk", 4), (0.3, 256, "explicit", "chunk", 4),
            (0.01, 3000, "explicit", "chunk", 4), (0.01, 1024, "explicit", "abs32", 4),
            (0.01, 1024, "sentinel", "chunk", 4), (0.07, 1024, "explicit", "chunk", 3),
            (0.3, 1024, "explicit", "abs32", 4),
            (0.01, 1, "explicit", "chunk", 4)):   # 300003 counts: multi-CTA reduce-then-scan
        n = 300_003 if chunk == 1 else 200_003
        words = O.exact_stream(fmt_id, n, rate, 5, bk, esc)
        m = sz.CodebookMode.from_name(mode)
        book = tuple(e for e, _ in bk)[: (15 if mode == "sentinel" else (1 << bits))]
        cfg = sz.CodecConfig(fmt, bits, m, chunk, pos, sz.ExponentCodebook(fmt, book, bits, m))
        st = sz.RawTensorStream(fmt, torch.from_numpy(words).cuda())
        enc = sz.encode(st, cfg)
        dec = sz.decode(enc, cfg, enc.codebook)
        assert sz.compare_streams(st, dec).ok
        sz.build_histogram(st)
torch.cuda.synchronize()
print("sanitize ok")

# paged KV (segments) and device container framing
from paper_2605_01708_b200 import container, paged  # noqa: E402
from paper_2605_01708_b200.engine import synth_kv  # noqa: E402
for fmt, bk, esc in ((sz.ElementFormat.BF16, O.BF16_BOOK, O.BF16_ESC),
                     (sz.ElementFormat.FP8_E5M2, O.E5M2_BOOK, O.E5M2_ESC)):
    book = sz.ExponentCodebook(fmt, tuple(e for e, _ in bk), 4, sz.CodebookMode.TOPK_EXPLICIT)
    cfg = sz.CodecConfig(fmt, codebook=book)
    caches = [synth_kv(24 * 2 * 16 * 2 * 64, fmt, 9 + l, bk, esc, 0.05).view(24, 2, 16, 2, 64)
              for l in range(2)]
    ids = torch.randperm(24)[:11].cuda()
    enc = paged.encode_kv_blocks(caches, ids, cfg)
    dst = [torch.zeros_like(c) for c in caches]
    paged.decode_kv_blocks(enc, cfg, book, dst, ids.flip(0))
    words = synth_kv(70_001, fmt, 3, bk, esc, 0.01)
    buf = container.encode_container(sz.RawTensorStream(fmt, words), cfg)
    assert torch.equal(container.decode_container(buf).words, words)
torch.cuda.synchronize()
print("sanitize paged+container ok")
