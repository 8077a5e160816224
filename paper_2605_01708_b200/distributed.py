"""Multi-GPU paths: sharded KV, sharded calibration, and the
pipelined prefill -> decode handoff.

* Sharding: KV caches split by KV head (tensor parallel) or by layer are
  independent units — chunk-relative escape addressing makes every shard
  self-contained, so each rank encodes/decodes its own shard with no
  data-path collective (weak scaling).
* Calibration: the only real exchange.  Each rank builds its exponent
  histogram on its shard (K1) and one all-reduce(sum) of the int64 bins
  equals ``merge_stats`` (calibration.py:88-96: histograms are additive);
  every rank then runs the same deterministic ``select_codebook``.
* Handoff: GPU i encodes chunk-aligned pieces and ships the compressed
  sections to GPU j with NCCL point-to-point (NVLink/NVSwitch); GPU j
  decodes each piece as it lands.  Encode of piece k+1, transfer of piece k
  and decode of piece k-1 overlap.  Per piece the wire carries a 2-word
  header (elements, escapes) then the sections in serialization order
  (codec.py:176-184): counts, codes, sign|mantissa, positions, values.

The codec itself is injected (``PieceCodec``) so the protocol is exercised by
CPU/gloo tests with the oracle; the product binding is ``GpuPieceCodec``.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Protocol

import numpy as np
import torch
import torch.distributed as dist

from .calibration import CalibrationStats, CodebookMode, ExponentCodebook, select_codebook
from .codec import CodecConfig, compressed_payload_bytes, packed_nbytes
from .formats import ElementFormat

__all__ = [
    "kv_shard_shape", "shard_range", "calibrate_sharded", "PieceCodec", "GpuPieceCodec",
    "Sections", "HandoffSender", "HandoffReceiver", "send_raw", "recv_raw",
]


# ----------------------------------------------------------------- sharding
def kv_shard_shape(layers: int, tokens: int, kv_heads: int, head_dim: int, world: int,
                   by: str = "head") -> tuple[int, ...]:
    """Shape of one rank's KV shard, layout [layer][K,V][token][head][dim]."""
    if by == "head":
        if kv_heads % world:
            raise ValueError(f"{kv_heads} KV heads do not split over {world} ranks")
        return (layers, 2, tokens, kv_heads // world, head_dim)
    if by == "layer":
        if layers % world:
            raise ValueError(f"{layers} layers do not split over {world} ranks")
        return (layers // world, 2, tokens, kv_heads, head_dim)
    raise ValueError(f"unknown shard axis {by!r}")


def shard_range(n: int, world: int, rank: int, align: int) -> tuple[int, int]:
    """Contiguous, ``align``-aligned [lo, hi) split of n elements (the last
    rank takes the remainder) — per-shard sections concatenate to the
    global encoding when ``align`` is a multiple of the chunk size."""
    units = -(-n // align)
    per = units // world
    extra = units % world
    lo_u = rank * per + min(rank, extra)
    hi_u = lo_u + per + (1 if rank < extra else 0)
    return min(n, lo_u * align), min(n, hi_u * align)


def calibrate_sharded(local_counts: torch.Tensor, fmt: ElementFormat, code_bits: int,
                      mode: CodebookMode, group=None) -> ExponentCodebook:
    """All-reduce(sum) the per-rank histograms, then select the codebook.

    ``local_counts`` is the rank's int64 histogram (K1 output on the GPU, or
    any tensor on the group's device type).  Deterministic on every rank.
    """
    counts = local_counts.to(torch.int64).clone()
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    c = counts.cpu().numpy()
    return select_codebook(CalibrationStats(fmt, c, int(c.sum())), code_bits, mode)


# ----------------------------------------------------------------- handoff
@dataclass
class Sections:
    """One piece's compressed sections as flat byte tensors + counts."""

    n: int
    m: int
    counts: torch.Tensor      # uint8 view of u32 counts
    codes: torch.Tensor
    sm: torch.Tensor
    positions: torch.Tensor   # uint8 view
    values: torch.Tensor      # raw exponent bytes

    def wire(self) -> list[torch.Tensor]:
        return [t for t in (self.counts, self.codes, self.sm, self.positions, self.values)
                if t.numel()]

    @property
    def nbytes(self) -> int:
        return sum(t.numel() for t in self.wire())


class PieceCodec(Protocol):
    """Codec seen by the handoff: ``slot`` (0/1) selects one of two buffer
    sets so piece k+1 can be encoded/received while piece k is in flight."""

    device: torch.device

    def encode(self, words: torch.Tensor, slot: int) -> Sections: ...

    def empty_sections(self, n: int, m: int, slot: int) -> Sections: ...

    def decode_into(self, sec: Sections, out: torch.Tensor, slot: int) -> None: ...

    def finish(self) -> None: ...


def section_sizes(config: CodecConfig, n: int, m: int) -> tuple[int, int, int, int, int]:
    return (4 * config.n_chunks(n), packed_nbytes(n, config.code_bits), config.sm_nbytes(n),
            m * config.position_nbytes if not config.sentinel else 0, m)


class GpuPieceCodec:
    """Product binding: the sm_100a kernels through the C ABI (DeviceCodec),
    two engines per piece length (ping-pong), decode verdicts checked once at
    the end so decode never stalls the receive loop."""

    def __init__(self, config: CodecConfig, codebook: ExponentCodebook,
                 capacity: int | None = None):
        self.config, self.codebook, self.capacity = config, codebook, capacity
        from . import _native as N
        self.device = N.device()
        self._eng: dict[tuple[int, int], object] = {}
        self._used: list = []

    def _engine(self, n: int, slot: int):
        from .engine import DeviceCodec
        key = (n, slot)
        if key not in self._eng:
            self._eng[key] = DeviceCodec(self.config, self.codebook, n, capacity=self.capacity,
                                         device=self.device)
        return self._eng[key]

    def encode(self, words: torch.Tensor, slot: int) -> Sections:
        eng = self._engine(words.numel(), slot)
        m = eng.ensure_capacity(words)   # host learns M (sizes the escape sends)
        b = eng.bufs
        pos = b.positions[:m].view(torch.uint8) if b.positions is not None else \
            torch.empty(0, dtype=torch.uint8, device=self.device)
        return Sections(words.numel(), m, b.counts.view(torch.uint8), b.codes, b.sm, pos,
                        b.values[:m])

    def empty_sections(self, n: int, m: int, slot: int) -> Sections:
        sizes = section_sizes(self.config, n, m)
        ts = [torch.empty(sz, dtype=torch.uint8, device=self.device) for sz in sizes]
        return Sections(n, m, *ts)

    def decode_into(self, sec: Sections, out: torch.Tensor, slot: int) -> None:
        eng = self._engine(sec.n, slot)
        cfg = self.config
        counts = sec.counts.view(torch.uint32) if sec.counts.numel() else None
        pos = sec.positions.view(cfg.position_torch_dtype) if sec.positions.numel() else None
        src = eng.decode_struct(codes=sec.codes, sm=sec.sm, counts=counts, positions=pos,
                                values=sec.values if sec.m else None, m=sec.m)
        # each decode gets its own status word so verdicts survive until finish()
        import torch as _t
        from . import _native as N
        status = _t.empty(N.STATUS_BYTES, dtype=_t.uint8, device=self.device)
        N.check(eng.lib.sz_decode(src, eng.params, N.ptr(out), N.ptr(status), N.ptr(eng.dec_ws),
                                  eng.dec_ws.numel(), N.stream_handle()), "decode")
        self._used.append((status, sec))

    def finish(self) -> None:
        from .codec import _raise_from_status, EncodedStreams
        for status, sec in self._used:
            raw = status.cpu().numpy()
            if raw[:8 + 8 * 13].any():
                es = EncodedStreams(sec.n, sec.m, sec.codes, sec.sm,
                                    sec.counts.view(torch.uint32), sec.positions, sec.values,
                                    self.codebook)
                _raise_from_status(raw, es, self.config, self.codebook, sec.values)
        self._used.clear()


class HandoffSender:
    """Sender rank: encode chunk-aligned pieces and ship them (NCCL P2P)."""

    def __init__(self, codec: PieceCodec, peer: int, piece: int, group=None):
        self.codec, self.peer, self.piece, self.group = codec, peer, piece, group

    def send(self, words: torch.Tensor) -> dict:
        n = words.numel()
        pieces = -(-n // self.piece)
        dev = self.codec.device
        dist.send(torch.tensor([n, pieces], dtype=torch.int64, device=dev), self.peer,
                  group=self.group)
        wire_bytes, escapes = 16, 0
        inflight: list[tuple[list, torch.Tensor | None]] = [([], None), ([], None)]
        for k in range(pieces):
            slot = k % 2
            for r in inflight[slot][0]:   # buffers of piece k-2 must have left
                r.wait()
            sec = self.codec.encode(words[k * self.piece:(k + 1) * self.piece], slot)
            h = torch.tensor([sec.n, sec.m], dtype=torch.int64, device=dev)
            reqs = [dist.isend(h, self.peer, group=self.group)]
            reqs += [dist.isend(t, self.peer, group=self.group) for t in sec.wire()]
            inflight[slot] = (reqs, h)   # h kept alive until its send completes
            wire_bytes += 16 + sec.nbytes
            escapes += sec.m
        for reqs, _ in inflight:
            for r in reqs:
                r.wait()
        return {"pieces": pieces, "wire_bytes": wire_bytes, "escapes": escapes}


class HandoffReceiver:
    """Receiver rank: receive each piece and decode it as soon as it lands."""

    def __init__(self, codec: PieceCodec, peer: int, dtype: torch.dtype, group=None):
        self.codec, self.peer, self.dtype, self.group = codec, peer, dtype, group

    def recv(self) -> torch.Tensor:
        dev = self.codec.device
        hdr = torch.empty(2, dtype=torch.int64, device=dev)
        dist.recv(hdr, self.peer, group=self.group)
        n, pieces = (int(v) for v in hdr.cpu().tolist())
        out = torch.empty(n, dtype=self.dtype, device=dev)
        lo = 0
        for k in range(pieces):
            h = torch.empty(2, dtype=torch.int64, device=dev)
            dist.recv(h, self.peer, group=self.group)
            pn, pm = (int(v) for v in h.cpu().tolist())
            sec = self.codec.empty_sections(pn, pm, k % 2)
            reqs = [dist.irecv(t, self.peer, group=self.group) for t in sec.wire()]
            for r in reqs:
                r.wait()
            self.codec.decode_into(sec, out[lo:lo + pn], k % 2)
            lo += pn
        self.codec.finish()
        return out


def send_raw(words: torch.Tensor, peer: int, piece: int, group=None) -> int:
    """Baseline: ship the raw words in the same piece sizes."""
    for k in range(0, words.numel(), piece):
        dist.send(words[k:k + piece].contiguous(), peer, group=group)
    return words.numel() * words.element_size()


def recv_raw(out: torch.Tensor, peer: int, piece: int, group=None) -> torch.Tensor:
    for k in range(0, out.numel(), piece):
        buf = out[k:k + piece]
        tmp = torch.empty_like(buf)
        dist.recv(tmp, peer, group=group)
        buf.copy_(tmp)
    return out
