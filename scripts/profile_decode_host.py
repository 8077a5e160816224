"""Phase timing of the public-API host decode (diagnostics)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_01708_b200 as sz  # noqa: E402
from paper_2605_01708_b200 import codec, hostpipe  # noqa: E402
from paper_2605_01708_b200.engine import synth_kv  # noqa: E402

fmt = sz.ElementFormat.from_name(sys.argv[1] if len(sys.argv) > 1 else "e5m2")
n = 1 << 31
if fmt is sz.ElementFormat.BF16:
    bw, esc = tuple((0x70 + i, 0.72 ** i) for i in range(16)), tuple(range(0x10, 0x18))
else:
    bw, esc = tuple((8 + i, 0.72 ** i) for i in range(16)), (0, 1, 2, 3, 28, 29, 30, 31)
words = synth_kv(n, fmt, 7, bw, esc, 0.0016)
host = torch.empty(n, dtype=fmt.torch_dtype, pin_memory=True)
host.copy_(words)
book = sz.ExponentCodebook(fmt, tuple(e for e, _ in bw), 4, sz.CodebookMode.TOPK_EXPLICIT)
cfg = sz.CodecConfig(fmt, codebook=book)

orig = {}


def wrap(mod, name):
    f = getattr(mod, name)

    def g(*a, **k):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize()
        print(f"    {name:28s} {1e3 * (time.perf_counter() - t):8.1f} ms", flush=True)
        return r
    setattr(mod, name, g)


for nm in ("to_numpy",):
    wrap(codec, nm)
wrap(hostpipe, "decode_host")
wrap(hostpipe, "host_tensor")
_empty = torch.empty


for rep in range(4):
    enc = sz.encode(sz.RawTensorStream(fmt, host), cfg)
    torch.cuda.synchronize()
    t = time.perf_counter()
    dec = sz.decode(enc, cfg, book)
    torch.cuda.synchronize()
    print(f"rep {rep}: decode (public API) {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
    del dec, enc
