"""Preallocated, synchronisation-free codec engine for fixed-size streams.

``DeviceCodec`` owns every device buffer one encode -> decode cycle needs
(sections, escape capacity, workspaces, decode status) for a fixed element
count, so a serving loop / the handoff pipeline / the benchmark can enqueue
K2 and K3+K4 back to back on a stream with no allocation and no host round
trip: the decoder reads the escape count M straight from the encoder's
device word (``sz_encoded_in.d_n_escapes``).  The public ``encode``/``decode``
functions in codec.py are the reference-shaped API on top of the same ABI.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .calibration import ExponentCodebook
from .codec import (CodecConfig, EncodeBuffers, EncodedStreams, _config_params,
                    _raise_from_status, default_capacity, launch_encode)
from .formats import packed_nbytes


class DeviceCodec:
    def __init__(self, config: CodecConfig, codebook: ExponentCodebook, n: int,
                 capacity: int | None = None, device: torch.device | None = None):
        self.lib = N.load_library()
        if codebook.fmt is not config.fmt:
            raise ValueError("codebook / config format mismatch")
        self.config, self.codebook, self.n = config, codebook, n
        self.device = device or N.device()
        self.params = _config_params(config, codebook)
        self.capacity = max(1, min(n, capacity if capacity is not None
                                       else default_capacity(n)))
        self.bufs = EncodeBuffers(n, config, self.capacity, self.device)
        self.enc_ws = torch.empty(self.lib.sz_encode_workspace_bytes(n, self.params),
                                  dtype=torch.uint8, device=self.device)
        self.dec_ws = torch.empty(self.lib.sz_decode_workspace_bytes(n, 0, self.params),
                                  dtype=torch.uint8, device=self.device)
        self.status = torch.empty(N.STATUS_BYTES, dtype=torch.uint8, device=self.device)
        self.out = torch.empty(n, dtype=config.fmt.torch_dtype, device=self.device)

    # ------------------------------------------------------------ encode
    def encode(self, words: torch.Tensor, stream=None) -> None:
        """Enqueue K2 (+K6) for ``words`` (aligned CUDA tensor of n words)."""
        if words.numel() != self.n:
            raise ValueError(f"engine sized for {self.n} elements, got {words.numel()}")
        launch_encode(words, self.params, self.bufs, self.enc_ws, stream)

    def n_escapes(self) -> int:
        """Synchronising read of M (8 bytes)."""
        return int(self.bufs.m.cpu().numpy()[0])

    def ensure_capacity(self, words: torch.Tensor) -> int:
        """Encode once and grow the escape buffers if M overflowed them."""
        self.encode(words)
        m = self.n_escapes()
        if m > self.capacity:
            self.capacity = m
            self.bufs = EncodeBuffers(self.n, self.config, m, self.device)
            self.encode(words)
        # an escape-dense stream: room for the decoder's K3e path (escape
        # bitmap + per-tile counts), which it then takes for this M
        need = self.lib.sz_decode_workspace_bytes(self.n, m, self.params)
        if need > self.dec_ws.numel():
            self.dec_ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        return m

    def streams(self, m: int | None = None) -> EncodedStreams:
        """Reference-shaped view of the current sections (device tensors)."""
        m = self.n_escapes() if m is None else m
        b = self.bufs
        pos = b.positions[:m] if b.positions is not None else \
            torch.empty(0, dtype=torch.uint8, device=self.device)
        vp = (b.values_packed[:packed_nbytes(m, self.config.fmt.exp_bits)]
              if b.values_packed is not None else None)
        return EncodedStreams(self.n, m, b.codes, b.sm, b.counts, pos, b.values[:m],
                              self.codebook, vp)

    def payload_nbytes(self, m: int) -> int:
        from .codec import compressed_payload_bytes
        return compressed_payload_bytes(self.n, m, self.config)

    # ------------------------------------------------------------ decode
    def decode_struct(self, codes=None, sm=None, counts=None, positions=None, values=None,
                      m_dev: torch.Tensor | None = None, m: int | None = None) -> N.SzEncodedIn:
        b = self.bufs
        codes = b.codes if codes is None else codes
        sm = b.sm if sm is None else sm
        counts = b.counts if counts is None else counts
        positions = b.positions if positions is None else positions
        values = b.values if values is None else values
        src = N.SzEncodedIn()
        src.d_codes, src.d_sm = N.ptr(codes), N.ptr(sm)
        src.d_counts = N.ptr(counts) if counts is not None and counts.numel() else None
        src.d_positions, src.d_values = N.ptr(positions), N.ptr(values)
        src.n_elements = self.n
        src.n_counts = counts.numel() if counts is not None else 0
        if m is None:
            # device-resident M, clamped to what the escape buffers hold; a
            # larger M (encoder overflow) raises in check_status
            src.n_escapes = min(self.capacity, values.numel())
            src.d_n_escapes = N.ptr(b.m if m_dev is None else m_dev)
        else:
            src.n_escapes = m
            src.d_n_escapes = None
        return src

    def decode(self, out: torch.Tensor | None = None, stream=None, src: N.SzEncodedIn | None = None
               ) -> torch.Tensor:
        """Enqueue K3 + K4 on the engine's own sections (M read on device)."""
        out = self.out if out is None else out
        src = self.decode_struct() if src is None else src
        N.check(self.lib.sz_decode(src, self.params, N.ptr(out), N.ptr(self.status),
                                   N.ptr(self.dec_ws), self.dec_ws.numel(),
                                   N.stream_handle(stream)), "decode")
        return out

    def check_status(self) -> None:
        """Synchronise and raise CorruptionError if the last decode failed."""
        raw = self.status.cpu().numpy()
        _raise_from_status(raw, self.streams(), self.config, self.codebook, self.bufs.values)

    # ------------------------------------------------------------ framing
    def container_capacity(self) -> int:
        """Bytes of an SPLZ container holding up to ``capacity`` escapes."""
        return int(self.lib.sz_container_bytes(self.n, self.capacity, self.params))

    def frame(self, out: torch.Tensor, nbytes_dev: torch.Tensor, stream=None) -> None:
        """Enqueue ``sz_frame_container`` on the current sections: the SPLZ
        file image in ``out``, its length in ``nbytes_dev`` — M is read on the
        device, so encode -> frame -> send needs no host round trip."""
        from .container import frame_device
        frame_device(self.params, self.n, self.bufs.struct(), out, nbytes_dev, stream)

    # ------------------------------------------------------------ compare
    def compare(self, a: torch.Tensor, b: torch.Tensor, stream=None) -> torch.Tensor:
        res = torch.empty(2, dtype=torch.int64, device=self.device)
        N.check(self.lib.sz_compare(N.ptr(a), N.ptr(b), a.numel(),
                                    self.config.fmt.word_nbytes, N.ptr(res),
                                    N.stream_handle(stream)), "compare")
        return res


def synth_kv(n: int, fmt, seed: int, book_weights, escapes, escape_rate: float,
             device: torch.device | None = None) -> torch.Tensor:
    """Synthetic KV words generated on the device (K8): exponent distribution
    of the reference's datagen profile (in-book weights + uniform escapes at
    ``escape_rate``), uniform sign|mantissa."""
    lib = N.load_library()
    dev = device or N.device()
    exps = [e for e, _ in book_weights] + list(escapes)
    w = np.array([w for _, w in book_weights], dtype=np.float64)
    probs = np.concatenate([(1 - escape_rate) * w / w.sum(),
                            np.full(len(escapes), escape_rate / max(len(escapes), 1))])
    cdf = np.minimum(np.round(np.cumsum(probs) * 2**32), 2**32 - 1).astype(np.uint32)
    cdf[-1] = 2**32 - 1
    words = torch.empty(n, dtype=fmt.torch_dtype, device=dev)
    exps_np = np.ascontiguousarray(exps, dtype=np.uint8)
    cdf_np = np.ascontiguousarray(cdf)
    N.check(lib.sz_synth_words(N.ptr(words), n, fmt.code, seed,
                               exps_np.ctypes.data, cdf_np.ctypes.data, len(exps),
                               N.stream_handle()), "synth")
    return words
