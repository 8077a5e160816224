"""Robustness golden verdicts, produced by running the REAL reference package.

Run in the build container (the only place ``/root/reference`` exists):

    python tests/golden/make_robustness.py

It ports the reference's own container-robustness harnesses and records,
for every mutated container, what the reference does with it:

* truncation at every offset (``pkg/tests/test_container.py:134-138``,
  ``pkg/tests/test_acceptance.py:295-309``);
* 1500 seeded single-bit flips (``test_container.py:146-165``, seed 2024);
* 1000 seeded single-byte XORs (``test_acceptance.py:311-337``, seed 1234);
* every nonzero pad bit the format leaves: code stream (``codec.py:441-442``),
  FP8 3-bit sign-mantissa stream (``codec.py:236-237``), FP8 5/4-bit escape
  values (``codec.py:255-256``);
* the same bit-flip / byte-XOR / truncation harness over further bases the
  reference's tests do not build (E5M2, E4M3, sentinel, abs32, 3-bit codes,
  u8 positions), with their own seeds, so every mode's parse + decode
  validation sees random damage.

For each mutation it stores the stage that failed (``parse`` =
``container_from_bytes``, ``decode`` = ``decode``), the exception class,
``section`` (TruncatedError) / ``chunk`` (CorruptionError) and message, or,
when the reference decodes the damaged bytes, a BLAKE2b digest of the
decoded words and their mismatch count against the original.  Mutations
are stored as (offset, xor) pairs or truncation lengths, so the files stay
small: ``tests/golden/robust.npz`` (base containers + original words) and
``tests/golden/robust.json.gz``.  Nothing on the GPU box reads
``/root/reference``.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import shutil
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def load_reference():
    scratch = Path(tempfile.mkdtemp(prefix="szref_"))
    shutil.copytree("/root/reference/pkg/src/splitzip", scratch / "splitzip")
    sys.path.insert(0, str(scratch))
    import splitzip  # noqa: E402
    return splitzip


def digest(words: np.ndarray) -> str:
    return hashlib.blake2b(np.ascontiguousarray(words).tobytes(), digest_size=16).hexdigest()


def main():
    sz = load_reference()
    from splitzip import container as C

    BF16, E5M2, E4M3 = (sz.ElementFormat.BF16, sz.ElementFormat.FP8_E5M2,
                        sz.ElementFormat.FP8_E4M3)
    EXPL, SENT = sz.CodebookMode.TOPK_EXPLICIT, sz.CodebookMode.TOP15_SENTINEL
    CHUNK, ABS = sz.PositionMode.CHUNK_RELATIVE, sz.PositionMode.ABSOLUTE_32

    def exact(fmt, n, rate, seed, book, esc):
        return sz.generate(sz.ExponentSpec(fmt, count=n, seed=seed, in_book=book,
                                           escape_values=esc, escape_rate=rate,
                                           exact_counts=True))

    def pinned(fmt, entries, code_bits=4, mode=EXPL, **kw):
        return sz.CodecConfig(fmt, code_bits, mode,
                              codebook=sz.ExponentCodebook(fmt, tuple(entries), code_bits,
                                                           mode), **kw)

    arrays: dict[str, np.ndarray] = {}
    bases: dict[str, dict] = {}
    verdicts: list[dict] = []

    def verdict(stream, data: bytes) -> dict:
        try:
            streams, config, codebook = C.container_from_bytes(data)
        except sz.SplitZipError as exc:
            return {"stage": "parse", "raised": type(exc).__name__,
                    "section": getattr(exc, "section", None),
                    "chunk": getattr(exc, "chunk", None), "msg": str(exc)}
        try:
            dec = sz.decode(streams, config, codebook)
        except sz.SplitZipError as exc:
            return {"stage": "decode", "raised": type(exc).__name__, "section": None,
                    "chunk": getattr(exc, "chunk", None), "msg": str(exc)}
        words = np.asarray(dec.words)
        same_n = words.size == stream.n_elements
        mism = int(np.count_nonzero(words != stream.words)) if same_n else -1
        return {"stage": "ok", "raised": None, "digest": digest(words), "n": int(words.size),
                "mismatches": mism}

    def add_base(bid, stream, config, *, flips=0, flip_seed=0, xors=0, xor_seed=0,
                 truncate=True, pads=()):
        enc = sz.encode(stream, config)
        data = C.container_to_bytes(enc, config, enc.codebook)
        arrays[f"{bid}/container"] = np.frombuffer(data, np.uint8)
        arrays[f"{bid}/words"] = np.asarray(stream.words)
        bases[bid] = {"n": enc.n_elements, "m": enc.n_escapes, "nbytes": len(data),
                      "fmt": stream.fmt.cli_name}
        assert verdict(stream, data)["mismatches"] == 0

        def run(kind, muts):
            for mut in muts:
                if kind == "truncate":
                    bad = data[:mut]
                else:
                    pos, x = mut
                    b = bytearray(data)
                    b[pos] ^= x
                    bad = bytes(b)
                v = verdict(stream, bad)
                if v["stage"] == "ok" and bid == "small_bf16":
                    # the reference's harness asserts no damage decodes silently
                    # (its container makes every byte load-bearing; the extra
                    # bases leave unused codebook entries, so a silent decode
                    # is recorded there, not asserted away)
                    assert v["mismatches"] != 0, (bid, kind, mut)
                verdicts.append({"base": bid, "kind": kind,
                                 "mut": mut if kind == "truncate" else list(mut), **v})

        if truncate:
            run("truncate", list(range(len(data))))
        if flips:
            # test_container.py:146-152 (the reference draws pos, then bit)
            rng = np.random.default_rng(flip_seed)
            muts = []
            for _ in range(flips):
                pos = int(rng.integers(0, len(data)))
                bit = int(rng.integers(0, 8))
                muts.append((pos, 1 << bit))
            run("bitflip", muts)
        if xors:
            # test_acceptance.py:315-320 (pos, then delta in [1, 256))
            rng = np.random.default_rng(xor_seed)
            muts = []
            for _ in range(xors):
                pos = int(rng.integers(0, len(data)))
                delta = int(rng.integers(1, 256))
                muts.append((pos, delta))
            run("bytexor", muts)
        # every pad bit of the requested sections, one at a time
        header = 28 + 9 + len(enc.codebook.entries)
        offs, off = {}, header
        for name, sec in enc.section_bytes():
            offs[name] = (off, len(sec))
            off += len(sec)
        fmt = config.fmt
        widths = {"packed_codes": (enc.n_elements, config.code_bits),
                  "sign_mantissa": (enc.n_elements, fmt.sm_bits),
                  "escape_values": (enc.n_escapes, fmt.exp_bits)}
        for name in pads:
            lo, ln = offs[name]
            cnt, w = widths[name]
            used = cnt * w
            muts = [(lo + b // 8, 1 << (b % 8)) for b in range(used, ln * 8)]
            assert muts, (bid, name)
            run("pad_" + name, muts)
        return enc

    B16 = tuple((0x70 + i, 1.0) for i in range(16))
    # 1. The reference's own small container (test_container.py:46-62 ==
    #    test_acceptance.py:287-294): BF16, 128 words, chunk 32, 8 escapes.
    s = exact(BF16, 128, 0.0625, 42, B16, (0x10, 0x20))
    add_base("small_bf16", s, pinned(BF16, [e for e, _ in B16], chunk_size=32),
             flips=1500, flip_seed=2024, xors=1000, xor_seed=1234)

    # 2. Further bases, every mode (seeds 3000+; the same harness).
    E16 = tuple((8 + i, 0.72 ** i) for i in range(16))
    EE = (0, 1, 2, 3, 28, 29, 30, 31)
    F8 = tuple((4 + i, 0.72 ** i) for i in range(8))
    FE = (0, 1, 2, 3, 12, 13, 14, 15)
    ent = lambda b: [e for e, _ in b]
    # E5M2: odd N (code pad nibble), 3N not a multiple of 8 (SM pad), 5M not a
    # multiple of 8 (values pad).
    s = exact(E5M2, 133, 7 / 133, 3001, E16, EE)
    enc = add_base("e5m2_c32", s, pinned(E5M2, ent(E16), chunk_size=32),
                   flips=400, flip_seed=3001, xors=300, xor_seed=3101,
                   pads=("packed_codes", "sign_mantissa", "escape_values"))
    assert (enc.n_escapes * 5) % 8 and (enc.n_elements * 3) % 8
    # BF16 odd N: the code stream's high pad nibble (codec.py:441-442)
    s = exact(BF16, 257, 0.03, 3002, B16, (0x10, 0x20, 0x30))
    add_base("bf16_odd", s, pinned(BF16, ent(B16), chunk_size=64),
             flips=300, flip_seed=3002, xors=200, xor_seed=3102, pads=("packed_codes",))
    # BF16 sentinel (TOP15) with u8 positions absent; marks in the code plane
    s = exact(BF16, 200, 0.05, 3003, B16[:15], (0x10, 0x20))
    add_base("bf16_sent", s, pinned(BF16, ent(B16[:15]), mode=SENT, chunk_size=64),
             flips=300, flip_seed=3003, xors=200, xor_seed=3103)
    # BF16 abs32 positions
    s = exact(BF16, 180, 0.05, 3004, B16, (0x10, 0x20))
    add_base("bf16_abs32", s, pinned(BF16, ent(B16), position_mode=ABS),
             flips=300, flip_seed=3004, xors=200, xor_seed=3104)
    # BF16 3-bit codes over a 6-entry book (codes 6, 7 out of range), odd 3N
    s = exact(BF16, 171, 0.05, 3005, B16[:6], (0x10, 0x20))
    add_base("bf16_tri", s, pinned(BF16, ent(B16[:6]), code_bits=3, chunk_size=48),
             flips=300, flip_seed=3005, xors=200, xor_seed=3105, pads=("packed_codes",))
    # E4M3 3-bit codes, 4-bit values (4M odd -> a pad nibble)
    s = exact(E4M3, 150, 7 / 150, 3006, F8, FE)
    enc = add_base("e4m3_tri", s, pinned(E4M3, ent(F8), code_bits=3, chunk_size=40),
                   flips=300, flip_seed=3006, xors=200, xor_seed=3106,
                   pads=("packed_codes", "escape_values"))
    # E5M2 sentinel
    s = exact(E5M2, 141, 0.05, 3007, E16[:15], EE)
    add_base("e5m2_sent", s, pinned(E5M2, ent(E16[:15]), mode=SENT, chunk_size=32),
             flips=300, flip_seed=3007, xors=200, xor_seed=3107,
             pads=("sign_mantissa", "escape_values"))
    # BF16 chunk 512 (u16 positions), a chunk larger than the stream
    s = exact(BF16, 300, 0.04, 3008, B16, (0x10, 0x20))
    add_base("bf16_c512", s, pinned(BF16, ent(B16), chunk_size=512),
             flips=300, flip_seed=3008, xors=200, xor_seed=3108)

    np.savez_compressed(HERE / "robust.npz", **arrays)
    blob = json.dumps({"generator": "tests/golden/make_robustness.py (reference splitzip 0.1.0)",
                       "bases": bases, "verdicts": verdicts}, separators=(",", ":"))
    with gzip.GzipFile(HERE / "robust.json.gz", "wb", mtime=0) as f:
        f.write(blob.encode())
    kinds: dict[str, int] = {}
    for v in verdicts:
        key = f"{v['stage']}:{v['raised']}"
        kinds[key] = kinds.get(key, 0) + 1
    print(f"{len(verdicts)} verdicts over {len(bases)} bases; {kinds}; "
          f"{(HERE / 'robust.npz').stat().st_size} + {(HERE / 'robust.json.gz').stat().st_size} B")


if __name__ == "__main__":
    main()
