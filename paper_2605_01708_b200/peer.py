"""Fused encode -> NVLink peer stores: the prefill -> decode handoff without
NCCL (config 5 of BASELINE.json).

``distributed.HandoffSender/Receiver`` encode into local buffers and ship the
sections with NCCL point-to-point: the compressed bytes are written to HBM,
read back by NCCL's copy kernels (which occupy SMs the codec wants) and
written again on the peer.  Here the sender's encoder writes its sections
*directly into the receiver's HBM* through peer-mapped pointers — each code,
sign-mantissa and escape byte crosses NVLink exactly once, straight from the
encode kernel's stores — and the two GPUs order themselves with device-side
flags (``sz_peer_signal`` / ``sz_peer_wait``): the host only enqueues.

Pipeline per piece k (slot = k mod S; S receive slots in the receiver's HBM,
each sized for the worst case of every element escaping, so the escape
stream can never overflow):

    sender   stream: wait free[slot] >= k//S -> encode(piece k -> peer slot)
                     -> signal ready[slot] = k//S + 1            (peer memory)
    receiver stream: wait ready[slot] >= k//S + 1 -> decode(slot -> out)
                     -> signal free[slot] = k//S + 1             (sender memory)

so piece k+1 is encoded (and travels) while piece k is decoded.  The
receiver's slots and the sender's free flags each live in one dedicated
device region (``sz_device_alloc``) whose 64-byte CUDA IPC handle is passed
once over the process group; both sides carve it with the same layout.  In
one process (``loopback=True``) the "peer" is the same GPU and the regions
are used directly — the single-GPU tests and ``scripts/bench_handoff.py
--loopback``.
"""

from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

from . import _native as N
from .calibration import ExponentCodebook
from .codec import CodecConfig, _config_params
from .errors import CorruptionError, NativeError
from .formats import packed_nbytes

__all__ = ["SlotLayout", "PeerSender", "PeerReceiver", "connect_pair"]

_ALIGN = 256


def _up(x: int) -> int:
    return (x + _ALIGN - 1) // _ALIGN * _ALIGN


class SlotLayout:
    """Byte offsets of S landing slots (codes, sm, counts, positions, values,
    M) + the ready flags in one region; identical on both sides."""

    FIELDS = ("codes", "sm", "counts", "positions", "values", "m")

    def __init__(self, piece: int, config: CodecConfig, slots: int):
        self.piece, self.slots = piece, slots
        sizes = {
            "codes": packed_nbytes(piece, config.code_bits),
            "sm": config.sm_nbytes(piece),
            "counts": 4 * config.n_chunks(piece),
            "positions": 0 if config.sentinel else piece * config.position_nbytes,
            "values": piece,
            "m": 8,
        }
        off = 0
        self.slot: list[dict[str, int | None]] = []
        for _ in range(slots):
            d = {}
            for f in self.FIELDS:
                d[f] = off if sizes[f] else None
                off = _up(off + sizes[f])
            self.slot.append(d)
        self.ready = off
        self.total = _up(off + 8 * slots)


class _Region:
    """A dedicated device allocation: owned (cudaMalloc), IPC-mapped from
    another process, or (loopback) a borrowed view of a local one."""

    def __init__(self, nbytes: int | None = None, handle: bytes | None = None,
                 view_of: "_Region | None" = None):
        self.lib = N.load_library()
        self.kind = "view" if view_of is not None else ("ipc" if handle is not None else "owned")
        if view_of is not None:
            self.base = view_of.base
            return
        p = C.c_void_p()
        if handle is None:
            N.check(self.lib.sz_device_alloc(nbytes, C.byref(p)), "device_alloc")
        else:
            buf = (C.c_uint8 * 64).from_buffer_copy(handle)
            N.check(self.lib.sz_ipc_import(buf, C.byref(p)), "ipc_import")
        self.base = p.value

    def handle(self) -> bytes:
        buf = (C.c_uint8 * 64)()
        N.check(self.lib.sz_ipc_export(self.base, buf), "ipc_export")
        return bytes(buf)

    def close(self) -> None:
        if self.base and self.kind == "owned":
            self.lib.sz_device_free(self.base)
        elif self.base and self.kind == "ipc":
            self.lib.sz_ipc_close(self.base)
        self.base = None


class PeerSender:
    """Sender end: encode each piece straight into the receiver's slot."""

    def __init__(self, config: CodecConfig, codebook: ExponentCodebook, layout: SlotLayout,
                 slots_region: _Region, device, timeout_s: float = 30.0):
        self.lib = N.load_library()
        self.config, self.codebook, self.lay = config, codebook, layout
        self.piece, self.slots = layout.piece, layout.slots
        self.params = _config_params(config, codebook)
        self.remote = slots_region                 # receiver's slots (peer-mapped)
        self.free = _Region(_up(8 * self.slots))   # written by the receiver
        self.timeout_ns = int(timeout_s * 1e9)
        self.timed_out = torch.zeros(1, dtype=torch.int32, device=device)
        self.ws = torch.empty(self.lib.sz_encode_workspace_bytes(self.piece, self.params),
                              dtype=torch.uint8, device=device)
        eb = config.fmt.exp_bits
        self.vp = (torch.empty(packed_nbytes(self.piece, eb), dtype=torch.uint8, device=device)
                   if eb != 8 else None)
        self.k = 0

    def send(self, words: torch.Tensor, stream=None) -> int:
        """Enqueue every piece of ``words``; returns the number of pieces."""
        n = words.numel()
        h = N.stream_handle(stream)
        pieces = -(-n // self.piece)
        base = self.remote.base
        for i in range(pieces):
            slot, gen = self.k % self.slots, self.k // self.slots
            lo, hi = i * self.piece, min(n, (i + 1) * self.piece)
            N.check(self.lib.sz_peer_wait(self.free.base + 8 * slot, gen, self.timeout_ns,
                                          N.ptr(self.timed_out), h), "peer_wait")
            o = self.lay.slot[slot]
            out = N.SzEncoded()
            out.d_codes, out.d_sm = base + o["codes"], base + o["sm"]
            out.d_counts = base + o["counts"] if o["counts"] is not None else None
            out.d_positions = base + o["positions"] if o["positions"] is not None else None
            out.d_values = base + o["values"]
            out.d_values_packed = N.ptr(self.vp)
            out.d_n_escapes = base + o["m"]
            out.escape_capacity = hi - lo
            out.d_escape_base = None
            N.check(self.lib.sz_encode(N.ptr(words) + lo * words.element_size(), hi - lo,
                                       self.params, out, N.ptr(self.ws), self.ws.numel(), h),
                    "encode(peer)")
            N.check(self.lib.sz_peer_signal(base + self.lay.ready + 8 * slot, gen + 1, h),
                    "peer_signal")
            self.k += 1
        return pieces

    def check(self) -> None:
        if int(self.timed_out.item()):
            raise NativeError("peer handoff: sender timed out waiting for a free slot")

    def close(self) -> None:
        """Unmap the peer's region (both ends close, then both release)."""
        torch.cuda.synchronize()
        self.remote.close()

    def release(self) -> None:
        """Free this end's own region (after the peer closed its mapping)."""
        self.free.close()


class PeerReceiver:
    """Receiver end: decode each landed piece, then free its slot."""

    def __init__(self, config: CodecConfig, codebook: ExponentCodebook, layout: SlotLayout,
                 device, timeout_s: float = 30.0):
        self.lib = N.load_library()
        self.config, self.codebook, self.lay = config, codebook, layout
        self.piece, self.slots = layout.piece, layout.slots
        self.params = _config_params(config, codebook)
        self.region = _Region(layout.total)        # the landing slots
        self.free_remote: _Region | None = None    # sender's free flags (peer-mapped)
        self.dec_ws = torch.empty(self.lib.sz_decode_workspace_bytes(self.piece, 0, self.params),
                                  dtype=torch.uint8, device=device)
        self.timeout_ns = int(timeout_s * 1e9)
        self.timed_out = torch.zeros(1, dtype=torch.int32, device=device)
        self.statuses: list[torch.Tensor] = []
        self.k = 0

    def recv(self, out: torch.Tensor, stream=None) -> torch.Tensor:
        """Enqueue the decode of every piece of ``out`` (the caller knows its
        size and shares the piece length with the sender)."""
        n = out.numel()
        h = N.stream_handle(stream)
        pieces = -(-n // self.piece)
        base = self.region.base
        for i in range(pieces):
            slot, gen = self.k % self.slots, self.k // self.slots
            lo, hi = i * self.piece, min(n, (i + 1) * self.piece)
            N.check(self.lib.sz_peer_wait(base + self.lay.ready + 8 * slot, gen + 1,
                                          self.timeout_ns, N.ptr(self.timed_out), h),
                    "peer_wait")
            o = self.lay.slot[slot]
            src = N.SzEncodedIn()
            src.d_codes, src.d_sm = base + o["codes"], base + o["sm"]
            k_chunks = self.config.n_chunks(hi - lo)
            src.d_counts = base + o["counts"] if k_chunks else None
            src.d_positions = base + o["positions"] if o["positions"] is not None else None
            src.d_values = base + o["values"]
            src.n_elements, src.n_escapes, src.n_counts = hi - lo, 0, k_chunks
            src.d_n_escapes = base + o["m"]
            st = torch.empty(N.STATUS_BYTES, dtype=torch.uint8, device=out.device)
            N.check(self.lib.sz_decode(src, self.params, N.ptr(out) + lo * out.element_size(),
                                       N.ptr(st), N.ptr(self.dec_ws), self.dec_ws.numel(), h),
                    "decode(peer)")
            self.statuses.append(st)
            N.check(self.lib.sz_peer_signal(self.free_remote.base + 8 * slot, gen + 1, h),
                    "peer_signal")
            self.k += 1
        return out

    def check(self) -> None:
        """Synchronise; raise on a timeout or a corrupt piece."""
        if int(self.timed_out.item()):
            raise NativeError("peer handoff: receiver timed out waiting for a piece")
        bad = [i for i, st in enumerate(self.statuses)
               if st.cpu().numpy()[:8 + 8 * N.NUM_CHECKS].any()]
        self.statuses.clear()
        if bad:
            raise CorruptionError(f"peer handoff: decode checks failed on piece(s) {bad}")

    def close(self) -> None:
        """Unmap the peer's region (both ends close, then both release)."""
        torch.cuda.synchronize()
        if self.free_remote is not None:
            self.free_remote.close()

    def release(self) -> None:
        """Free this end's own region (after the peer closed its mapping)."""
        self.region.close()


def _preload(config: CodecConfig, codebook: ExponentCodebook, dev) -> None:
    """Launch once every kernel the link uses (this encode/decode template
    instantiation, the signal and the poller).  With CUDA lazy loading a
    kernel's first launch loads its module, which cannot complete while a
    poller of this process spins on the GPU — the poller would wait for a
    signal that never launches (observed: every first-use wait timed out)."""
    from .engine import DeviceCodec
    lib = N.load_library()
    n = config.chunk_size * max(1, -(-(1 << 16) // config.chunk_size))
    eng = DeviceCodec(config, codebook, n, capacity=n, device=dev)
    words = torch.zeros(n, dtype=config.fmt.torch_dtype, device=dev)
    eng.encode(words)
    eng.decode()
    flag = torch.zeros(1, dtype=torch.int64, device=dev)
    N.check(lib.sz_peer_signal(N.ptr(flag), 1, N.stream_handle()), "peer_signal")
    N.check(lib.sz_peer_wait(N.ptr(flag), 1, int(1e9), None, N.stream_handle()), "peer_wait")
    torch.cuda.synchronize()


def connect_pair(role: str, peer: int, piece: int, config: CodecConfig,
                 codebook: ExponentCodebook, slots: int = 2, group=None,
                 loopback: bool = False, timeout_s: float = 30.0):
    """Set up one direction of a handoff.

    Multi-process: both ranks call it (``role`` "send" / "recv", ``peer`` the
    other rank); the two regions' IPC handles cross over ``group`` once.
    ``loopback=True`` (one process, one GPU) returns ``(sender, receiver)``.
    Teardown: ``close()`` on both ends (unmaps the peer's region), a
    barrier, then ``release()`` on both (frees the own region).
    """
    if piece % config.chunk_size and config.chunked:
        raise ValueError("piece must be a multiple of the chunk size")
    dev = N.device()
    _preload(config, codebook, dev)
    lay = SlotLayout(piece, config, slots)
    if loopback:
        rcv = PeerReceiver(config, codebook, lay, dev, timeout_s)
        snd = PeerSender(config, codebook, lay, _Region(view_of=rcv.region), dev, timeout_s)
        rcv.free_remote = _Region(view_of=snd.free)
        return snd, rcv
    if role == "recv":
        rcv = PeerReceiver(config, codebook, lay, dev, timeout_s)
        dist.send_object_list([rcv.region.handle()], dst=peer, group=group)
        box = [None]
        dist.recv_object_list(box, src=peer, group=group)
        rcv.free_remote = _Region(handle=box[0])
        return rcv
    box = [None]
    dist.recv_object_list(box, src=peer, group=group)
    snd = PeerSender(config, codebook, lay, _Region(handle=box[0]), dev, timeout_s)
    dist.send_object_list([snd.free.handle()], dst=peer, group=group)
    return snd
