"""Paged-KV codec throughput on one GPU.

Llama-3.1-8B KV in a vLLM-style pool: 32 layers x [num_blocks, 2, 16, 8, 128]
BF16 (64 KiB per block); a 32K-token request owns 2048 random blocks per
layer (4 GiB).  Compares, device-timed (CUDA events, 3 warm-up + 10 timed):
  paged encode   encode_kv_blocks (full tiles through a 128B-swizzled tensor
                 map over the caches' VA window, sz_encode_segments_va)
  paged encode (bulk copies)  one 1-D bulk copy per block (sz_encode_segments)
  gather+encode  torch gather into a contiguous buffer, then encode
  paged decode   decode straight into another pool's blocks
  decode+scatter decode contiguous, then torch scatter into the blocks
GB/s = BF16 bytes of the request / time.  One JSON line on stdout.
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2605_01708_b200 as sz  # noqa: E402
from paper_2605_01708_b200 import _native as N  # noqa: E402
from paper_2605_01708_b200 import paged  # noqa: E402
from paper_2605_01708_b200.codec import EncodeBuffers, _config_params, launch_encode  # noqa: E402
from paper_2605_01708_b200.engine import DeviceCodec, synth_kv  # noqa: E402

LAYERS, POOL, REQ = 32, 2304, 2048
BLOCK = (2, 16, 8, 128)
fmt = sz.ElementFormat.BF16
bw, esc = tuple((0x70 + i, 0.72 ** i) for i in range(16)), tuple(range(0x10, 0x18))
book = sz.ExponentCodebook(fmt, tuple(e for e, _ in bw), 4, sz.CodebookMode.TOPK_EXPLICIT)
cfg = sz.CodecConfig(fmt, codebook=book)
per_block = 2 * 16 * 8 * 128
caches = [synth_kv(POOL * per_block, fmt, 100 + l, bw, esc, 0.0016).view(POOL, *BLOCK)
          for l in range(LAYERS)]
g = torch.Generator().manual_seed(1)
ids = torch.randperm(POOL, generator=g)[:REQ].cuda()
ids2 = torch.randperm(POOL, generator=g)[:REQ].cuda()
dst = [torch.empty_like(c) for c in caches]
addrs, seg = paged.kv_block_table(caches, ids)
addrs2, _ = paged.kv_block_table(dst, ids2)
n = LAYERS * REQ * per_block
raw = n * 2
lib = N.load_library()
params = _config_params(cfg, book)
eng = DeviceCodec(cfg, book, n)
bufs = eng.bufs
gath = torch.empty(n, dtype=torch.int16, device="cuda")
i16 = [c.view(torch.int16) for c in caches]
d16 = [c.view(torch.int16) for c in dst]


def paged_encode_bulk():
    N.check(lib.sz_encode_segments(N.ptr(addrs), addrs.numel(), seg, params, bufs.struct(),
                                   N.ptr(eng.enc_ws), eng.enc_ws.numel(), N.stream_handle()),
            "enc")


win = paged.kv_va_window(caches)


def paged_encode():
    N.check(lib.sz_encode_segments_va(N.ptr(addrs), addrs.numel(), seg, win[0], win[1], params,
                                      bufs.struct(), N.ptr(eng.enc_ws), eng.enc_ws.numel(),
                                      N.stream_handle()), "enc")


def gather_encode():
    torch.cat([c[ids].reshape(-1) for c in i16], out=gath)
    launch_encode(gath.view(torch.uint16), params, bufs, eng.enc_ws)


def paged_decode():
    src = eng.decode_struct()
    N.check(lib.sz_decode_segments(src, params, N.ptr(addrs2), addrs2.numel(), seg,
                                   N.ptr(eng.status), N.ptr(eng.dec_ws), eng.dec_ws.numel(),
                                   N.stream_handle()), "dec")


def decode_scatter():
    out = eng.decode()
    o = out.view(torch.int16).view(LAYERS, REQ, *BLOCK)
    for l in range(LAYERS):
        d16[l].index_copy_(0, ids2, o[l])


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3


eng.ensure_capacity(torch.cat([c[ids].reshape(-1) for c in i16]).view(torch.uint16))
res = {}
for name, fn in (("paged_encode", paged_encode), ("paged_encode_bulk_copies", paged_encode_bulk),
                 ("gather_then_encode", gather_encode),
                 ("paged_decode", paged_decode), ("decode_then_scatter", decode_scatter)):
    t = timeit(fn)
    res[name + "_gbs"] = round(raw / t / 1e9, 1)
# correctness: paged round trip into dst equals the request's blocks
paged_encode()
paged_decode()
eng.check_status()
ok = all(torch.equal(d16[l][ids2], i16[l][ids]) for l in range(LAYERS))
res.update({"workload": f"Llama-3.1-8B KV, vLLM blocks {list(BLOCK)} BF16 (64 KiB), "
                        f"{LAYERS} layers x {REQ} of {POOL} blocks (32K tokens, 4 GiB)",
            "bitexact": ok, "bytes": raw})
print(json.dumps(res))
