"""Where does the host-pipeline decode lose time on some calls? Times every
pinned allocation made inside decode_host, for several back-to-back
encode/decode calls (diagnostics only)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2605_01708_b200 as sz  # noqa: E402
from paper_2605_01708_b200 import hostpipe  # noqa: E402
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

_empty = torch.empty
log = []


def empty(*a, **k):
    t = time.perf_counter()
    r = _empty(*a, **k)
    if k.get("pin_memory"):
        log.append((r.numel() * r.element_size(), time.perf_counter() - t))
    return r


torch.empty = empty
for rep in range(6):
    t0 = time.perf_counter()
    enc = sz.encode(sz.RawTensorStream(fmt, host), cfg)
    t1 = time.perf_counter()
    log.clear()
    dec = sz.decode(enc, cfg, book)
    t2 = time.perf_counter()
    big = [(b >> 20, round(dt * 1e3, 2)) for b, dt in log if b > (1 << 20)]
    print(f"rep {rep}: encode {1e3 * (t1 - t0):.1f} ms decode {1e3 * (t2 - t1):.1f} ms "
          f"pinned allocs (MiB, ms) {big}", flush=True)
    del dec, enc
