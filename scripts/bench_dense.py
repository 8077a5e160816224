"""Escape-rate sweep of the decoder's two chunk-relative paths on one B200:
the stagers' own walk over positions (SZ_DEC_MARKED=0) against the K3e
pre-pass (escape bitmap + per-tile counts, SZ_DEC_MARKED=1), plus the
automatic choice.  Sets the crossover `kDenseDiv` in sz_decode.cu.

Input: SZ_DENSE_N words (default 2^31) of synthetic KV (K8) with the
reference profile's top-16 book and uniform escapes at each rate, and the
top-8 3-bit books (the escape rate their profile implies).  Device time:
CUDA events over 5 decodes after 3 warm-ups, bitwise verified first.
One JSON line per (config, path).
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2605_01708_b200 as sz  # noqa: E402
from paper_2605_01708_b200.engine import DeviceCodec, synth_kv  # noqa: E402

N = int(os.environ.get("SZ_DENSE_N", 1 << 31))
RATES = [float(r) for r in os.environ.get(
    "SZ_DENSE_RATES", "0.0016,0.004,0.008,0.012,0.016,0.024,0.04,0.0789").split(",")]
FMTS = os.environ.get("SZ_DENSE_FMTS", "bf16,e5m2").split(",")
PATHS = os.environ.get("SZ_DENSE_PATHS", "0,1").split(",")


def profile(fmt):
    if fmt is sz.ElementFormat.BF16:
        return tuple((0x70 + i, 0.72 ** i) for i in range(16)), tuple(range(0x10, 0x18))
    return tuple((8 + i, 0.72 ** i) for i in range(16)), (0, 1, 2, 3, 28, 29, 30, 31)


def timed_decode(eng, words, reps=5):
    eng.decode()
    eng.check_status()
    assert int(eng.compare(words, eng.out)[0].item()) == 0
    for _ in range(3):
        eng.decode()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        eng.decode()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    for fname in FMTS:
        fmt = sz.ElementFormat.BF16 if fname == "bf16" else sz.ElementFormat.FP8_E5M2
        bw, esc = profile(fmt)
        cases = [(f"{fname} top16 4-bit eps={r}", bw, r, 4, 16) for r in RATES]
        cases.append((f"{fname} top8 3-bit", bw, 0.0016, 3, 8))
        for name, weights, rate, bits, k in cases:
            words = synth_kv(N, fmt, 7, weights, esc, rate)
            book = sz.ExponentCodebook(fmt, tuple(e for e, _ in weights)[:k], bits,
                                       sz.CodebookMode.TOPK_EXPLICIT)
            cfg = sz.CodecConfig(fmt, bits, sz.CodebookMode.TOPK_EXPLICIT, 1024,
                                 sz.PositionMode.CHUNK_RELATIVE, book)
            eng = DeviceCodec(cfg, book, N)
            m = eng.ensure_capacity(words)
            # workspace for either path (the automatic sizing only makes room
            # for K3e when M calls for it)
            eng.dec_ws = torch.empty(eng.lib.sz_decode_workspace_bytes(N, N, eng.params),
                                     dtype=torch.uint8, device=eng.device)
            for path in PATHS:
                os.environ["SZ_DEC_MARKED"] = path
                ms = timed_decode(eng, words)
                print(json.dumps({"config": name, "path": {"0": "stager", "1": "k3e"}[path],
                                  "escape_rate": round(m / N, 5), "decode_ms": round(ms, 4),
                                  "decode_gbs": round(N * fmt.word_nbytes / ms / 1e6, 1)}),
                      flush=True)
            os.environ.pop("SZ_DEC_MARKED", None)
            del eng, words
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
