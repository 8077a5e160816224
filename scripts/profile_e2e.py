"""Time the phases of the host-pipelined decode (diagnostics only)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_01708_b200 as sz  # noqa: E402
from paper_2605_01708_b200 import hostpipe  # noqa: E402
from paper_2605_01708_b200.engine import synth_kv  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 31
fmt = sz.ElementFormat.from_name(sys.argv[2] if len(sys.argv) > 2 else "bf16")
if fmt is sz.ElementFormat.BF16:
    bw, esc = tuple((0x70 + i, 0.72 ** i) for i in range(16)), tuple(range(0x10, 0x18))
else:
    bw, esc = tuple((8 + i, 0.72 ** i) for i in range(16)), (0, 1, 2, 3, 28, 29, 30, 31)
words = synth_kv(n, fmt, 7, bw, esc, 0.0016)
host = torch.empty(n, dtype=fmt.torch_dtype, pin_memory=True)
host.copy_(words)
book = sz.ExponentCodebook(fmt, tuple(e for e, _ in bw), 4, sz.CodebookMode.TOPK_EXPLICIT)
cfg = sz.CodecConfig(fmt, codebook=book)


def T(label, fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    print(f"{label:40s} {1e3 * (time.perf_counter() - t):9.1f} ms", flush=True)
    return r


for rep in range(3):
    enc = T("encode (public API)", lambda: sz.encode(sz.RawTensorStream(fmt, host), cfg))
    counts_np = T("counts to numpy", lambda: sz.codec.to_numpy(enc.chunk_counts))
    T("pinned alloc 4 GiB", lambda: torch.empty(n, dtype=fmt.torch_dtype, pin_memory=True))
    out = T("decode_host", lambda: hostpipe.decode_host(enc, cfg, book, counts_np))
    dec = T("decode (public API)", lambda: sz.decode(enc, cfg, book))
    del dec, out, enc
