"""Small driver for ncu: encode + decode a 2^28-word (512 MiB) synthetic KV
stream a few times (inputs 4x larger than L2).  Not a benchmark."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2605_01708_b200 as sz  # noqa: E402
from paper_2605_01708_b200.engine import DeviceCodec, synth_kv  # noqa: E402

fmt_name = sys.argv[1] if len(sys.argv) > 1 else "bf16"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 28
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
bits = int(sys.argv[4]) if len(sys.argv) > 4 else 4      # 3: top-8 book
chunk = int(sys.argv[5]) if len(sys.argv) > 5 else 1024
mode_name = sys.argv[6] if len(sys.argv) > 6 else "explicit"   # | sentinel | abs32
fmt = sz.ElementFormat.from_name(fmt_name)
if fmt is sz.ElementFormat.BF16:
    bw, esc = tuple((0x70 + i, 0.72 ** i) for i in range(16)), tuple(range(0x10, 0x18))
else:
    bw, esc = tuple((8 + i, 0.72 ** i) for i in range(16)), (0, 1, 2, 3, 28, 29, 30, 31)
words = synth_kv(n, fmt, 7, bw, esc, 0.0016)
mode = sz.CodebookMode.TOP15_SENTINEL if mode_name == "sentinel" else sz.CodebookMode.TOPK_EXPLICIT
k = (1 << bits) - (1 if mode_name == "sentinel" else 0)
book = sz.ExponentCodebook(fmt, tuple(e for e, _ in bw)[:k], bits, mode)
cfg = sz.CodecConfig(fmt, bits, mode, chunk,
                     sz.PositionMode.ABSOLUTE_32 if mode_name == "abs32" else
                     sz.PositionMode.CHUNK_RELATIVE, book)
eng = DeviceCodec(cfg, book, n)
eng.ensure_capacity(words)
for _ in range(reps):
    eng.encode(words)
    eng.decode()
from paper_2605_01708_b200.calibration import build_histogram_device  # noqa: E402
build_histogram_device(words, fmt)
torch.cuda.synchronize()
eng.check_status()
print("ok")
