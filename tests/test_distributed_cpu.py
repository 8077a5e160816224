"""World-size-2 gloo tests of the multi-GPU host logic (run on CPU here).

The handoff protocol and the sharded calibration are exercised end to end
with an oracle-backed ``PieceCodec`` stub standing in for the GPU kernels
(test-only injection; the product binding is GpuPieceCodec)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import sz_oracle as O


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class OraclePieceCodec:
    """CPU stand-in for GpuPieceCodec: same Sections on the wire."""

    device = torch.device("cpu")

    def __init__(self, config, book):
        from paper_2605_01708_b200.codec import CodecConfig  # noqa: F401
        self.config, self.book = config, tuple(book)
        self.p = O.Params(config.fmt.code, config.code_bits, config.sentinel,
                          config.chunk_size, config.abs32)

    def encode(self, words, slot):
        from paper_2605_01708_b200.distributed import Sections
        sec = O.encode(words.numpy(), self.p, self.book)
        t = lambda b: torch.from_numpy(np.frombuffer(bytes(b), dtype=np.uint8).copy())
        return Sections(sec["n"], sec["m"], t(sec["chunk_counts"].astype("<u4").tobytes()),
                        t(sec["packed_codes"]), t(sec["sign_mantissa"]),
                        t(np.ascontiguousarray(sec["escape_positions"]).tobytes()),
                        torch.from_numpy(sec["escape_values"].copy()))

    def empty_sections(self, n, m, slot):
        from paper_2605_01708_b200.distributed import Sections, section_sizes
        sizes = section_sizes(self.config, n, m)
        return Sections(n, m, *[torch.empty(s, dtype=torch.uint8) for s in sizes])

    def decode_into(self, sec, out, slot):
        pos_dt = self.config.position_np_dtype
        d = {"n": sec.n, "m": sec.m,
             "chunk_counts": sec.counts.numpy().view(np.uint32),
             "packed_codes": sec.codes.numpy().tobytes(),
             "sign_mantissa": sec.sm.numpy().tobytes(),
             "escape_positions": sec.positions.numpy().view(pos_dt),
             "escape_values": sec.values.numpy()}
        out.copy_(torch.from_numpy(O.decode(d, self.p, self.book).astype(np.int32)).to(out.dtype)
                  if out.dtype != torch.uint16 else
                  torch.from_numpy(O.decode(d, self.p, self.book)))

    def finish(self):
        pass


def _worker(rank, world, port, q, rate, piece):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2605_01708_b200 as sz
        from paper_2605_01708_b200.distributed import (HandoffReceiver, HandoffSender,
                                                       calibrate_sharded, shard_range)
        fmt = sz.ElementFormat.BF16
        n = 70_001
        words = O.exact_stream(0, n, rate, 5, O.BF16_BOOK, O.BF16_ESC)
        # sharded calibration == calibration of the whole stream
        lo, hi = shard_range(n, world, rank, 1024)
        local = torch.from_numpy(O.histogram(words[lo:hi], 0))
        book = calibrate_sharded(local, fmt, 4, sz.CodebookMode.TOPK_EXPLICIT)
        whole = O.choose_book(O.histogram(words, 0), 4, False)
        assert book.entries == whole, (book.entries, whole)
        cfg = sz.CodecConfig(fmt, codebook=book)
        codec = OraclePieceCodec(cfg, book.entries)
        if rank == 0:
            stats = HandoffSender(codec, 1, piece).send(torch.from_numpy(words.copy()))
            ref = O.encode(words, O.Params(0), book.entries)
            q.put(("sender", stats["escapes"] == ref["m"], stats["pieces"]))
        else:
            out = HandoffReceiver(codec, 0, torch.uint16).recv()
            q.put(("receiver", bool(np.array_equal(out.numpy(), words)), n))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("rate,piece", [(0.0016, 16384), (0.5, 8192), (0.0, 1 << 20)])
def test_handoff_protocol_gloo(rate, piece):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, rate, piece)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    res = {k: (ok, x) for k, ok, x in (q.get(timeout=5) for _ in range(2))}
    assert res["sender"][0] and res["receiver"][0]


def test_shard_ranges_cover_and_align():
    from paper_2605_01708_b200.distributed import kv_shard_shape, shard_range
    for n in (1, 1023, 1024, 10_000, 1 << 20):
        for world in (1, 2, 4, 8):
            spans = [shard_range(n, world, r, 1024) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert all(lo % 1024 == 0 or lo == n for lo, _ in spans)
    assert kv_shard_shape(80, 131072, 8, 128, 8) == (80, 2, 131072, 1, 128)
    assert kv_shard_shape(32, 32768, 8, 128, 4, by="layer") == (8, 2, 32768, 8, 128)
    with pytest.raises(ValueError):
        kv_shard_shape(80, 16, 8, 128, 3)


def test_sharded_sections_concatenate_to_global():
    """Chunk-relative mode: per-shard encodings concatenated section-wise equal
    the global encoding (the property that makes sharding collective-free)."""
    from paper_2605_01708_b200.distributed import shard_range
    n = 100_003
    words = O.exact_stream(0, n, 0.0123, 9, O.BF16_BOOK, O.BF16_ESC)
    book = tuple(e for e, _ in O.BF16_BOOK)
    p = O.Params(0)
    whole = O.encode(words, p, book)
    parts = [O.encode(words[lo:hi], p, book)
             for lo, hi in (shard_range(n, 4, r, 1024) for r in range(4))]
    for key in ("packed_codes", "sign_mantissa"):
        assert b"".join(x[key] for x in parts) == whole[key]
    for key in ("chunk_counts", "escape_positions", "escape_values"):
        assert np.array_equal(np.concatenate([x[key] for x in parts]), whole[key])
