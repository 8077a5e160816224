"""Read-only HBM bandwidth on this GPU (for K1's roofline, a read-only
stream): torch reductions over a 4 GiB buffer (no writes but the scalar),
device-timed, best of 10; and K1 itself on the same bytes for comparison."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_01708_b200.calibration import build_histogram_device  # noqa: E402
import paper_2605_01708_b200 as sz  # noqa: E402

n_bytes = 1 << 32
x = torch.randint(0, 1 << 15, (n_bytes // 2,), dtype=torch.int16, device="cuda")


def best(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


f32 = x.view(torch.float32)
out = {}
ms = best(lambda: torch.sum(f32))
out["torch_sum_f32_gbs"] = round(n_bytes / ms / 1e6, 1)
ms = best(lambda: torch.amax(x.view(torch.int32)))
out["torch_amax_i32_gbs"] = round(n_bytes / ms / 1e6, 1)
ms = best(lambda: build_histogram_device(x, sz.ElementFormat.BF16))
out["k1_hist_bf16_uniform_gbs"] = round(n_bytes / ms / 1e6, 1)
# K1 on KV-like words (the reference profile: 16 in-book exponents + escapes)
from paper_2605_01708_b200.engine import synth_kv  # noqa: E402
del x, f32
kv = synth_kv(n_bytes // 2, sz.ElementFormat.BF16, 7, tuple((0x70 + i, 0.72 ** i) for i in range(16)),
              tuple(range(0x10, 0x18)), 0.0016)
ms = best(lambda: build_histogram_device(kv, sz.ElementFormat.BF16))
out["k1_hist_bf16_kv_gbs"] = round(n_bytes / ms / 1e6, 1)
print(json.dumps(out))
