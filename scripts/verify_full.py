"""Full-size (2^31-word) bitwise round-trip verification through the timed
engine path, checked with K7 and by an independent torch.equal."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2605_01708_b200 as sz  # noqa: E402
from paper_2605_01708_b200.engine import DeviceCodec, synth_kv  # noqa: E402

for fmt_name, n in (("bf16", 1 << 31), ("e5m2", 1 << 31)):
    fmt = sz.ElementFormat.from_name(fmt_name)
    if fmt is sz.ElementFormat.BF16:
        bw, esc = tuple((0x70 + i, 0.72 ** i) for i in range(16)), tuple(range(0x10, 0x18))
    else:
        bw, esc = tuple((8 + i, 0.72 ** i) for i in range(16)), (0, 1, 2, 3, 28, 29, 30, 31)
    for rate in (0.0016, 0.05):
        words = synth_kv(n, fmt, 11, bw, esc, rate)
        book = sz.ExponentCodebook(fmt, tuple(e for e, _ in bw), 4, sz.CodebookMode.TOPK_EXPLICIT)
        eng = DeviceCodec(sz.CodecConfig(fmt, codebook=book), book, n)
        m = eng.ensure_capacity(words)
        for rep in range(3):
            eng.out.fill_(0)
            eng.encode(words)
            eng.decode()
            eng.check_status()
            same = torch.equal(eng.out, words)
            k7 = eng.compare(words, eng.out).cpu().tolist()
            print(fmt_name, rate, rep, "M", m, "torch.equal", same, "K7 mismatches", k7[0], flush=True)
            assert same and k7[0] == 0
        del words, eng
        torch.cuda.empty_cache()
print("verify_full ok")
