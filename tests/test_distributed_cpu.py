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
    """CPU stand-in for GpuPieceCodec: the same FrameLayout buffers on the
    wire (header N, M + sections at their offsets), capacity and spill
    semantics included; sections from the oracle."""

    device = torch.device("cpu")

    def __init__(self, config, book, capacity=None):
        self.config, self.book, self.capacity = config, tuple(book), capacity
        self.p = O.Params(config.fmt.code, config.code_bits, config.sentinel,
                          config.chunk_size, config.abs32)
        self.log, self.over = [], []

    def _cap(self, n, capacity):
        from paper_2605_01708_b200.distributed import default_frame_capacity
        if capacity is not None:
            return max(1, min(n, capacity))
        return max(1, min(n, self.capacity)) if self.capacity else default_frame_capacity(n)

    def _frame(self, words, cap):
        from paper_2605_01708_b200.distributed import FrameLayout
        n = words.numel()
        sec = O.encode(words.numpy(), self.p, self.book)
        lay = FrameLayout(self.config, n, cap)
        fr = torch.zeros(lay.wire_bytes, dtype=torch.uint8)
        fr[:16].view(torch.int64)[:] = torch.tensor([n, sec["m"]])
        k = min(sec["m"], cap)
        put = lambda name, b: lay.view(fr, name)[:len(b)].copy_(
            torch.from_numpy(np.frombuffer(bytes(b), dtype=np.uint8).copy()))
        put("counts", sec["chunk_counts"].astype("<u4").tobytes())
        put("codes", sec["packed_codes"])
        put("sm", sec["sign_mantissa"])
        put("positions", np.ascontiguousarray(sec["escape_positions"][:k]).tobytes())
        put("values", sec["escape_values"][:k].tobytes())
        return fr, sec["m"]

    def encode_frame(self, words, slot):
        fr, m = self._frame(words, self._cap(words.numel(), None))
        self.log.append((words.numel(), m))
        return fr

    def overflowed(self):
        out = [(k, m) for k, (n, m) in enumerate(self.log) if m > self._cap(n, None)]
        self.log = []
        return out

    def spill_frame(self, words, m):
        return self._frame(words, max(1, m))[0]

    def recv_frame(self, n, slot, capacity=None):
        from paper_2605_01708_b200.distributed import FrameLayout
        return torch.empty(FrameLayout(self.config, n, self._cap(n, capacity)).wire_bytes,
                           dtype=torch.uint8)

    def decode_frame(self, frame, n, out, slot, piece, capacity=None):
        from paper_2605_01708_b200.distributed import FrameLayout
        cap = self._cap(n, capacity)
        lay = FrameLayout(self.config, n, cap)
        hn, m = (int(v) for v in frame[:16].view(torch.int64))
        assert hn == n
        if m > cap:
            self.over.append((piece, slot == "spill"))
            return
        pos_dt = self.config.position_np_dtype
        d = {"n": n, "m": m,
             "chunk_counts": lay.view(frame, "counts").numpy().view(np.uint32),
             "packed_codes": lay.view(frame, "codes").numpy().tobytes(),
             "sign_mantissa": lay.view(frame, "sm").numpy().tobytes(),
             "escape_positions": lay.view(frame, "positions").numpy().view(pos_dt)[:m],
             "escape_values": lay.view(frame, "values").numpy()[:m]}
        out.copy_(torch.from_numpy(O.decode(d, self.p, self.book)))

    def finish(self, redone=None):
        redone = redone or set()
        left = [k for k, spill in self.over if spill or k not in redone]
        assert not left, f"pieces {left} overflowed without a spill frame"
        self.over = []


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
            # pieces over the frame capacity (1/32 of the piece, >= 1024)
            # travel as spill frames
            from paper_2605_01708_b200.distributed import default_frame_capacity
            want = 0
            for lo in range(0, n, piece):
                w = words[lo:lo + piece]
                want += O.encode(w, O.Params(0), book.entries)["m"] > default_frame_capacity(w.size)
            q.put(("sender", stats["spilled"] == want, stats["pieces"]))
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


@pytest.mark.parametrize("fmt_name,cb,chunk,n,cap", [
    ("bf16", 4, 1024, 1 << 20, 1 << 15), ("bf16", 3, 256, 70_001, 4096),
    ("e5m2", 4, 1024, 1 << 20, 1 << 15), ("e4m3", 3, 64, 12_345, 12_345),
])
def test_frame_layout_offsets(fmt_name, cb, chunk, n, cap):
    """FrameLayout: a 16-byte header, then counts, codes, sign|mantissa,
    positions, values in serialization order (codec.py:176-184), each
    256-byte aligned (the decoder reads codes / sign|mantissa with 16-byte
    bulk copies), the wire ending after the values, FP8's packed-values
    scratch after the wire."""
    import paper_2605_01708_b200 as sz
    from paper_2605_01708_b200.distributed import FrameLayout
    from paper_2605_01708_b200.formats import packed_nbytes
    fmt = sz.ElementFormat.from_name(fmt_name)
    cfg = sz.CodecConfig(fmt, cb, chunk_size=chunk)
    lay = FrameLayout(cfg, n, cap)
    order = ["counts", "codes", "sm", "positions", "values"]
    assert [lay.off[k] for k in order] == sorted(lay.off[k] for k in order)
    assert lay.off["counts"] >= 16
    for k in order:
        assert lay.off[k] % 256 == 0
    assert lay.size["counts"] == 4 * cfg.n_chunks(n)
    assert lay.size["codes"] == packed_nbytes(n, cb)
    assert lay.size["sm"] == cfg.sm_nbytes(n)
    assert lay.size["positions"] == cap * cfg.position_nbytes
    assert lay.size["values"] == cap
    assert lay.wire_bytes >= lay.off["values"] + cap
    assert lay.packed_off >= lay.wire_bytes
    extra = packed_nbytes(cap, fmt.exp_bits) if fmt.exp_bits != 8 else 0
    assert lay.total >= lay.packed_off + extra
