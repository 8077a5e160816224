"""Prefill -> decode handoff throughput (BASELINE.json config 5).

torchrun --nproc-per-node 2 scripts/bench_handoff.py   (pairs 2i -> 2i+1, NVLink)
python scripts/bench_handoff.py --loopback               (one GPU: sender and
    receiver share the device; measures the pipelined encode -> slot -> decode
    path, not NVLink)

Per distribution (realistic eps = 0.16%, escape-heavy 7.89%): the raw NCCL
send of the BF16 words in the same pieces, and the fused codec handoff
(peer.py: the encoder stores straight into the receiver's HBM, device flags,
decode on arrival).  Effective GB/s = raw BF16 bytes / device time, max over
the pair's ranks.  One JSON line from rank 0.
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2605_01708_b200 as sz  # noqa: E402
from paper_2605_01708_b200 import peer  # noqa: E402
from paper_2605_01708_b200.engine import synth_kv  # noqa: E402

BOOK = tuple((0x70 + i, 0.72 ** i) for i in range(16))
ESC = tuple(range(0x10, 0x18))


def handoff_bench(n: int, piece: int, reps: int, loopback: bool, rank: int = 0, world: int = 1,
                  group=None, obj_group=None, timeout_s: float = 30.0,
                  raw_baseline: bool = True) -> dict:
    fmt = sz.ElementFormat.BF16
    book = sz.ExponentCodebook(fmt, tuple(e for e, _ in BOOK), 4, sz.CodebookMode.TOPK_EXPLICIT)
    cfg = sz.CodecConfig(fmt, codebook=book)
    raw = n * 2
    res = {"bytes": raw, "piece_elems": piece, "reps": reps}
    sender = (rank % 2 == 0)
    partner = rank + 1 if sender else rank - 1

    def agree(ok: bool) -> bool:
        """All ranks vote (CPU group, bounded by its timeout)."""
        if loopback or world == 1:
            return ok
        t = torch.tensor([int(ok)])
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=obj_group)
        return bool(t.item())

    def max_ms(ms):
        if loopback or world == 1:
            return ms
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        return float(t.item())

    def timed(fn):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if not loopback and world > 1:
            dist.barrier(group=group)
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(reps):
            fn()
        ev1.record()
        torch.cuda.synchronize()
        return max_ms(ev0.elapsed_time(ev1) / reps)

    for tag, rate in (("realistic_eps0.16", 0.0016), ("escape_heavy_eps7.89", 0.0789)):
        words = synth_kv(n, fmt, 11 + rank // 2, BOOK, ESC, rate)
        out = torch.empty_like(words)
        entry = {}
        if not loopback and raw_baseline:
            # raw baseline: NCCL P2P of the BF16 words in the same pieces
            def raw_send():
                ops = []
                for lo in range(0, n, piece):
                    t = words[lo:lo + piece] if sender else out[lo:lo + piece]
                    ops.append(dist.P2POp(dist.isend if sender else dist.irecv, t, partner,
                                          group=group))
                for r in dist.batch_isend_irecv(ops):
                    r.wait()
            raw_send()
            entry["raw_nccl_gbs"] = round(raw / (timed(raw_send) / 1e3) / 1e9, 1)
        if loopback:
            snd, rcv = peer.connect_pair("send", 0, piece, cfg, book, slots=2, loopback=True,
                                         timeout_s=timeout_s)
            s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

            def codec():
                rcv.recv(out, stream=s2)
                snd.send(words, stream=s1)
                torch.cuda.current_stream().wait_stream(s1)
                torch.cuda.current_stream().wait_stream(s2)
        else:
            link, err = None, None
            try:
                link = peer.connect_pair("send" if sender else "recv", partner, piece, cfg,
                                         book, slots=2, group=obj_group, timeout_s=timeout_s)
            except Exception as exc:  # noqa: BLE001 — every rank must reach the vote
                err = exc
            if not agree(err is None):
                raise RuntimeError(f"peer link setup failed on some rank: {err!r}")

            def codec():
                if sender:
                    link.send(words)
                else:
                    link.recv(out)
        codec()
        torch.cuda.synchronize()
        entry["codec_peer_gbs"] = round(raw / (timed(codec) / 1e3) / 1e9, 1)
        if loopback:
            snd.check()
            rcv.check()
            entry["bitexact"] = bool(torch.equal(out, words))
            snd.close(); rcv.close(); snd.release(); rcv.release()
        else:
            link.check()
            if not sender:
                entry["bitexact"] = bool(torch.equal(out, words))
            link.close()
            dist.barrier(group=group)
            link.release()
            ok = torch.tensor([int(entry.get("bitexact", True))], device="cuda")
            dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
            entry["bitexact"] = bool(ok.item())
        if not loopback and raw_baseline:
            # NCCL variant: one framed buffer per piece (distributed.FrameLayout),
            # M on the device, spill frames after the last piece
            from paper_2605_01708_b200.distributed import (GpuPieceCodec, HandoffReceiver,
                                                           HandoffSender)
            pc = GpuPieceCodec(cfg, book)
            got = {}

            def frames():
                if sender:
                    got["stats"] = HandoffSender(pc, partner, piece, group=group).send(words)
                else:
                    got["out"] = HandoffReceiver(pc, partner, words.dtype, group=group).recv()
            frames()
            torch.cuda.synchronize()
            entry["codec_nccl_frames_gbs"] = round(raw / (timed(frames) / 1e3) / 1e9, 1)
            ok = torch.tensor([int(sender or torch.equal(got["out"], words))], device="cuda")
            dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
            entry["nccl_frames_bitexact"] = bool(ok.item())
            if sender:
                entry["nccl_frames_wire_bytes"] = got["stats"]["wire_bytes"]
                entry["nccl_frames_spilled"] = got["stats"]["spilled"]
        m = int(sz.encode(sz.RawTensorStream(fmt, words[:1 << 24]), cfg).n_escapes)
        entry["escape_rate"] = round(m / (1 << 24), 5)
        res[tag] = entry
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--loopback", action="store_true")
    ap.add_argument("--elems", type=int, default=1 << 30)       # 2 GiB of BF16 per pair
    ap.add_argument("--piece", type=int, default=1 << 27)       # 256 MiB pieces
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: test the multi-process path with every rank on one GPU "
                         "(no raw NCCL baseline)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % torch.cuda.device_count())
    if args.loopback:
        res = handoff_bench(args.elems, args.piece, args.reps, True)
        res["mode"] = "loopback: sender and receiver on one GPU (no NVLink)"
    else:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
        if world % 2:
            raise SystemExit("needs an even number of ranks (pairs 2i -> 2i+1)")
        import datetime
        gloo = dist.new_group(backend="gloo", timeout=datetime.timedelta(seconds=120))
        res = handoff_bench(args.elems, args.piece, args.reps, False, rank, world,
                            obj_group=gloo, raw_baseline=args.backend == "nccl")
        res["mode"] = (f"{world // 2} concurrent pair(s) 2i -> 2i+1 over NVLink"
                       if args.backend == "nccl" else
                       "gloo test mode: every rank on one GPU (time-sliced; not a measurement)")
        res["pairs"] = world // 2
    if rank == 0:
        print(json.dumps(res), flush=True)
    if not args.loopback:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
