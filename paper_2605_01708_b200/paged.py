"""Paged KV caches: encode a request's KV straight from its
cache blocks and decode straight into the receiver's blocks.

Serving engines keep KV in fixed-size blocks scattered over a pool (vLLM:
one tensor per layer, ``[num_blocks, 2, block_size, kv_heads, head_dim]``;
a request owns the blocks listed in its block table).  Compressing such a
request with the flat API first needs a gather copy — 2 bytes read + 2
written per BF16 element, more HBM traffic than the codec itself (3.5 B per
element).  Here the stream is *defined* as the concatenation of segments
(one per layer x block, in that order) and the kernels address the blocks
in place: the encoder's producer warp bulk-copies each tile from its block,
the decoder stores each 32-byte slot into its destination block
(``sz_encode_segments`` / ``sz_decode_segments``).  Sections are
byte-identical to ``encode`` of the gathered words, so containers, the
handoff and ``decode`` interoperate unchanged.

Segments must be the same power-of-two size (>= 32 bytes) and 32-byte
aligned; the codebook must be pinned (``CodecConfig.codebook`` — paged
serving uses an offline-calibrated codebook, §4).
"""

from __future__ import annotations

from typing import Sequence

import torch

from . import _native as N
from .calibration import ExponentCodebook
from .codec import (CodecConfig, EncodeBuffers, EncodedStreams, _config_params,
                    _raise_from_status, check_section_lengths, default_capacity)
from .errors import ConfigError
from .formats import packed_nbytes

__all__ = ["kv_block_table", "kv_va_window", "encode_segments", "decode_segments", "encode_kv_blocks",
           "decode_kv_blocks"]


def kv_block_table(kv_caches: Sequence[torch.Tensor] | torch.Tensor,
                   block_ids: torch.Tensor) -> tuple[torch.Tensor, int]:
    """Device address of every (layer, block) segment, layer-major, and the
    segment size in bytes.  Each ``kv_caches[l]`` is ``[num_blocks, ...]``
    with contiguous blocks (``stride(0)`` elements apart)."""
    caches = [kv_caches] if isinstance(kv_caches, torch.Tensor) else list(kv_caches)
    if not caches:
        raise ConfigError("no KV caches given")
    dev = caches[0].device
    ids = block_ids.to(device=dev, dtype=torch.int64).reshape(-1)
    seg_bytes = None
    rows = []
    for c in caches:
        if not c.is_cuda:
            raise ConfigError("KV caches must be CUDA tensors")
        blk = c[0]
        if not blk.is_contiguous():
            raise ConfigError("each KV-cache block must be contiguous")
        nbytes = blk.numel() * c.element_size()
        stride = c.stride(0) * c.element_size()
        if seg_bytes is None:
            seg_bytes = nbytes
        elif nbytes != seg_bytes:
            raise ConfigError("all layers must use the same block size")
        rows.append(c.data_ptr() + ids * stride)
    if seg_bytes < 32 or seg_bytes & (seg_bytes - 1):
        raise ConfigError(f"block size {seg_bytes} B is not a power of two >= 32")
    addrs = torch.cat(rows)
    if bool(((addrs & 31) != 0).any()):
        raise ConfigError("KV-cache blocks must be 32-byte aligned")
    return addrs.contiguous(), int(seg_bytes)


def _need_book(config: CodecConfig) -> ExponentCodebook:
    if config.codebook is None:
        raise ConfigError("paged encode needs a pinned codebook (CodecConfig.codebook)")
    return config.codebook


def kv_va_window(kv_caches: Sequence[torch.Tensor] | torch.Tensor) -> tuple[int, int] | None:
    """Virtual-address window [lo, hi) spanning the KV-cache tensors, or None
    when a block could sit off the 128-byte grid (then the encoder keeps its
    1-D bulk copies).  Host-side only: tensor base pointers and strides."""
    caches = [kv_caches] if isinstance(kv_caches, torch.Tensor) else list(kv_caches)
    if any(c.data_ptr() % 128 or (c.stride(0) * c.element_size()) % 128 for c in caches):
        return None
    lo = min(c.data_ptr() for c in caches)
    hi = max(c.data_ptr() + c.numel() * c.element_size() for c in caches)
    return lo, hi


def encode_segments(seg_addrs: torch.Tensor, seg_bytes: int, config: CodecConfig, *,
                    capacity: int | None = None,
                    va_window: tuple[int, int] | None = None) -> EncodedStreams:
    """Encode the stream formed by the segments (device sections; the
    reference ``encode`` of the gathered words, codec.py:299-321).
    ``va_window`` (see ``kv_va_window``) lets full tiles arrive through a
    swizzled tensor map over that window (``sz_encode_segments_va``)."""
    lib = N.load_library()
    book = _need_book(config)
    params = _config_params(config, book)
    n_segs = seg_addrs.numel()
    n = n_segs * seg_bytes // config.fmt.word_nbytes
    dev = seg_addrs.device
    cap = min(n, capacity if capacity is not None else default_capacity(n))
    ws = torch.empty(lib.sz_encode_workspace_bytes(n, params), dtype=torch.uint8, device=dev)

    def run(cap):
        bufs = EncodeBuffers(n, config, cap, dev)
        lo, hi = va_window if va_window is not None else (0, 0)
        N.check(lib.sz_encode_segments_va(N.ptr(seg_addrs), n_segs, seg_bytes, lo, hi, params,
                                          bufs.struct(), N.ptr(ws), ws.numel(),
                                          N.stream_handle()), "encode_segments")
        return bufs

    bufs = run(cap)
    m = int(bufs.m.cpu().numpy()[0])
    if m > cap:  # overflow protocol (as encode): re-run with the exact count
        bufs = run(m)
    pos = (bufs.positions[:m] if bufs.positions is not None
           else torch.empty(0, dtype=torch.uint8, device=dev))
    vp = (bufs.values_packed[:packed_nbytes(m, config.fmt.exp_bits)]
          if bufs.values_packed is not None else None)
    return EncodedStreams(n, m, bufs.codes, bufs.sm, bufs.counts, pos, bufs.values[:m], book, vp)


def decode_segments(streams: EncodedStreams, config: CodecConfig, codebook: ExponentCodebook,
                    seg_addrs: torch.Tensor, seg_bytes: int) -> None:
    """Decode device sections straight into the segments (codec.py:421-536
    semantics; CorruptionError as ``decode``)."""
    from .formats import to_device
    lib = N.load_library()
    n, m = int(streams.n_elements), int(streams.n_escapes)
    if n * config.fmt.word_nbytes != seg_addrs.numel() * seg_bytes:
        raise ConfigError(f"{seg_addrs.numel()} segments of {seg_bytes} B do not hold "
                          f"{n} elements")
    # the same length / pad / N / M checks decode performs before launching:
    # a section shorter than the header says must raise here, never be read
    # past by the kernel that writes into live KV blocks
    check_section_lengths(streams, config, codebook)
    params = _config_params(config, codebook)
    dev = seg_addrs.device
    codes = to_device(streams.packed_codes, torch.uint8, align=16)
    sm = to_device(streams.sign_mantissa, torch.uint8, align=16)
    counts = to_device(streams.chunk_counts, torch.uint32, align=16) if config.chunked else None
    pos = (to_device(streams.escape_positions, config.position_torch_dtype, align=16)
           if (not config.sentinel and m) else None)
    vals = to_device(streams.escape_values, torch.uint8, align=16) if m else None
    src = N.SzEncodedIn()
    src.d_codes, src.d_sm = N.ptr(codes), N.ptr(sm)
    src.d_counts = N.ptr(counts) if counts is not None and counts.numel() else None
    src.d_positions, src.d_values = N.ptr(pos), N.ptr(vals)
    src.n_elements, src.n_escapes = n, m
    src.n_counts = counts.numel() if counts is not None else 0
    src.d_n_escapes = None
    status = torch.empty(N.STATUS_BYTES, dtype=torch.uint8, device=dev)
    ws = torch.empty(lib.sz_decode_workspace_bytes(n, m, params), dtype=torch.uint8, device=dev)
    N.check(lib.sz_decode_segments(src, params, N.ptr(seg_addrs), seg_addrs.numel(), seg_bytes,
                                   N.ptr(status), N.ptr(ws), ws.numel(), N.stream_handle()),
            "decode_segments")
    _raise_from_status(status.cpu().numpy(), streams, config, codebook, vals)


def encode_kv_blocks(kv_caches, block_ids: torch.Tensor, config: CodecConfig, *,
                     capacity: int | None = None) -> EncodedStreams:
    """Encode a request's KV blocks (all layers, layer-major) in place."""
    addrs, seg = kv_block_table(kv_caches, block_ids)
    return encode_segments(addrs, seg, config, capacity=capacity,
                           va_window=kv_va_window(kv_caches))


def decode_kv_blocks(streams: EncodedStreams, config: CodecConfig, codebook: ExponentCodebook,
                     kv_caches, block_ids: torch.Tensor) -> None:
    """Decode into the receiver's own blocks (its block ids may differ)."""
    addrs, seg = kv_block_table(kv_caches, block_ids)
    decode_segments(streams, config, codebook, addrs, seg)
