"""Fused encode -> peer-store handoff (peer.py, sz_peer_signal/wait): the
sender's encoder writes into the receiver's slots, device flags order the
two sides.  One GPU: loopback in one process (two streams), and two
processes on the same GPU sharing the buffers as CUDA IPC handles."""

from __future__ import annotations

import os

import pytest
import torch

pytestmark = pytest.mark.gpu

BF16_BOOK = tuple((0x70 + i, 0.72 ** i) for i in range(16))
BF16_ESC = tuple(range(0x10, 0x18))
E5_BOOK = tuple((8 + i, 0.72 ** i) for i in range(16))
E5_ESC = (0, 1, 2, 3, 28, 29, 30, 31)


def setup(fmt_name, n, rate, seed=5):
    import paper_2605_01708_b200 as m
    from paper_2605_01708_b200.engine import synth_kv
    fmt = m.ElementFormat.from_name(fmt_name)
    bw, esc = (BF16_BOOK, BF16_ESC) if fmt is m.ElementFormat.BF16 else (E5_BOOK, E5_ESC)
    words = synth_kv(n, fmt, seed, bw, esc, rate)
    book = m.ExponentCodebook(fmt, tuple(e for e, _ in bw), 4, m.CodebookMode.TOPK_EXPLICIT)
    return m, fmt, words, book, m.CodecConfig(fmt, codebook=book)


@pytest.mark.parametrize("fmt_name,rate", [("bf16", 0.0016), ("e5m2", 0.0016), ("bf16", 0.6)])
def test_peer_loopback_roundtrip(fmt_name, rate):
    from paper_2605_01708_b200 import peer
    m, fmt, words, book, cfg = setup(fmt_name, 5 * (1 << 20) + 3 * 1024, rate)
    snd, rcv = peer.connect_pair("send", 0, 1 << 20, cfg, book, slots=2, loopback=True,
                                 timeout_s=10)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = torch.empty_like(words)
    torch.cuda.synchronize()
    for rep in range(2):   # generations keep counting across transfers
        out.zero_()
        torch.cuda.synchronize()
        rcv.recv(out, stream=s2)
        snd.send(words, stream=s1)
        torch.cuda.synchronize()
        snd.check()
        rcv.check()
        assert torch.equal(out, words)
    snd.close()
    rcv.close()
    snd.release()
    rcv.release()


def _ipc_worker(rank, world, port, fmt_name, q, cross=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank if cross else 0)
    try:
        from paper_2605_01708_b200 import peer
        m, fmt, words, book, cfg = setup(fmt_name, 3 * (1 << 20) + 2048, 0.0016)
        import gc
        if rank == 0:
            snd = peer.connect_pair("send", 1, 1 << 20, cfg, book, slots=2, timeout_s=20)
            dist.barrier()
            snd.send(words)
            torch.cuda.synchronize()
            snd.check()
            ok = True
            snd.close()
            dist.barrier()
            snd.release()
        else:
            rcv = peer.connect_pair("recv", 0, 1 << 20, cfg, book, slots=2, timeout_s=20)
            out = torch.empty_like(words)
            dist.barrier()
            rcv.recv(out)
            torch.cuda.synchronize()
            rcv.check()
            ok = bool(torch.equal(out, words))
            rcv.close()
            dist.barrier()
            rcv.release()
        gc.collect()
        torch.cuda.synchronize()
        dist.barrier()       # both sides released the peer's memory
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


two_gpus = pytest.mark.skipif(torch.cuda.device_count() < 2,
                              reason="needs two GPUs (cuda:0 -> cuda:1 over NVLink)")


@pytest.mark.parametrize("cross", [False, pytest.param(True, marks=two_gpus)],
                         ids=["same-gpu", "cuda0-to-cuda1"])
@pytest.mark.parametrize("fmt_name", ["bf16", "e5m2"])
def test_peer_two_processes_ipc(fmt_name, cross):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + (os.getpid() % 200) + (7 if cross else 0)
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, fmt_name, q, cross))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res == {0: True, 1: True}
    assert [p.exitcode for p in procs] == [0, 0]


def _nccl_frames_worker(rank, world, port, fmt_name, rate, q):
    """HandoffSender/Receiver over NCCL with GpuPieceCodec frames, rank r on
    cuda:r: one framed buffer per piece, spill frames for overflowing pieces."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    try:
        from paper_2605_01708_b200.distributed import (GpuPieceCodec, HandoffReceiver,
                                                       HandoffSender)
        m, fmt, words, book, cfg = setup(fmt_name, 3 * (1 << 20) + 4096, rate)
        codec = GpuPieceCodec(cfg, book)
        if rank == 0:
            st = HandoffSender(codec, 1, 1 << 20).send(words)
            ok = (st["spilled"] > 0) == (rate > 1 / 32)
        else:
            out = HandoffReceiver(codec, 0, words.dtype).recv()
            ok = bool(torch.equal(out, words))
        torch.cuda.synchronize()
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@two_gpus
@pytest.mark.parametrize("fmt_name,rate", [("bf16", 0.0016), ("bf16", 0.0789), ("e5m2", 0.0016)])
def test_nccl_frame_handoff_two_gpus(fmt_name, rate):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29900 + (os.getpid() % 90)
    procs = [ctx.Process(target=_nccl_frames_worker, args=(r, 2, port, fmt_name, rate, q))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res == {0: True, 1: True}
    assert [p.exitcode for p in procs] == [0, 0]
